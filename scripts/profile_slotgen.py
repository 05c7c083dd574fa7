"""Device time of the GPU slot generator at C2 (273 PRB, 2 UE, doubletdl):
float32 (device variates, complex64 outputs) and float64 (complex128
outputs) synthesis, and the bit-error counter.

  python scripts/profile_slotgen.py [--slots 32] [--reps 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2409_02912_b200.config import SlotConfig  # noqa: E402
from paper_2409_02912_b200.slotgen import GpuSlotSource, count_bit_errors  # noqa: E402


def timed(fn, reps):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(reps):
        fn(i)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slots", type=int, default=32)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    cfg = SlotConfig(num_subcarriers=3276, num_ues=2)
    B = args.slots
    src = GpuSlotSource(cfg)
    mods = torch.full((B * 2,), 4, dtype=torch.int32, device="cuda")
    n0 = torch.full((B,), 0.1, dtype=torch.float64, device="cuda")
    for name, kw in (("fp32 synthesis (c64 out)", {}), ("fp64 synthesis (c128 out)", dict(y_dtype=torch.complex128)),
                     ("fp32 + h_eff", dict(with_h_eff=True))):
        box = {}

        def gen(i, kw=kw, box=box):
            box["b"] = src.generate(B, mods, n0, seed=1, first_slot=i * B, out=box.get("b"), **kw)
        ms = timed(gen, args.reps)
        out_bytes = sum(t.numel() * t.element_size() for t in box["b"][:4] if t is not None)
        print(f"{name:28s} {ms * 1e3 / B:8.2f} us/slot  {B / ms * 1e3:10.0f} slots/s  "
              f"{out_bytes / ms / 1e6:8.1f} GB/s of outputs")
    b = box["b"]
    llr = torch.randn((B, 2, 3276, 14, 4), device="cuda")
    errs = torch.zeros(B * 2, dtype=torch.int64, device="cuda")
    ms = timed(lambda i: count_bit_errors(cfg, llr, b.labels, b.mod_order, out=errs), args.reps)
    rd = llr.numel() * 4 + b.labels.numel()
    print(f"{'count_bit_errors':28s} {ms * 1e3 / B:8.2f} us/slot  {rd / ms / 1e6:8.1f} GB/s read")


if __name__ == "__main__":
    main()
