"""Small workload that launches every receiver kernel, for compute-sanitizer.

  compute-sanitizer --tool memcheck  --error-exitcode 9 python scripts/sanitize.py
  compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/sanitize.py --quick
  compute-sanitizer --tool initcheck --error-exitcode 9 python scripts/sanitize.py
  compute-sanitizer --tool synccheck --error-exitcode 9 python scripts/sanitize.py

Runs every golden case (tests/golden, reference-generated) in the four
precision modes through the drop-in plus the slot generator, the LDPC decoder
and the classical receivers, and checks the outputs loosely against the
goldens so a kernel that silently misbehaves under the tool is noticed.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import golden_cases as gc  # noqa: E402
from paper_2409_02912_b200 import nrx as gnrx  # noqa: E402

GATE = {"fp32": 1e-5, "fp32_simt": 1e-5, "bf16": 3e-2, "fp16": 1e-2}


def receiver(precisions, cases):
    for name in cases:
        c = gc.load_case(name)
        y, books, n0 = c.call_args()
        for prec in precisions:
            llr, chest = gnrx.nrx_forward(y, books, c.cfg, c.mcs, c.weights, c.config, n0, precision=prec)
            torch.cuda.synchronize()
            scale = max(float(np.abs(r).max()) for r in c.llrs)
            err = max(float(np.abs(np.asarray(g) - r).max()) for g, r in zip(llr, c.llrs)) / scale
            status = "ok" if err <= GATE[prec] else "FAIL"
            print(f"{name:>24s} {prec:>9s}: rel LLR err {err:.2e} {status}", flush=True)
            if status != "ok":
                raise SystemExit(f"{name} {prec}: {err}")


def others():
    from paper_2409_02912_b200 import classical, ldpc, slotgen
    from paper_2409_02912_b200.config import SlotConfig, default_mcs_table
    from paper_2409_02912_b200.synth import synth_slots
    dev = torch.device("cuda", 0)
    cfg = SlotConfig(num_subcarriers=48, num_ues=2, comb_size=2)
    mcs = default_mcs_table()[14]
    batch = slotgen.GpuSlotSource(cfg, device=dev).generate(4, mcs.modulation_order, 0.1, seed=1)
    torch.cuda.synchronize()
    print("slotgen ok", tuple(batch.y.shape), flush=True)
    y, books, _ = synth_slots(cfg, [4, 4], 2, 0.1, seed=3)
    classical.ls_lmmse_llrs(y, books, cfg, [mcs] * 2, 0.1)
    torch.cuda.synchronize()
    print("classical ls_lmmse ok", flush=True)
    dec = ldpc.GpuLdpc(ldpc.ira_code(120), device=dev)
    dec.decode(torch.randn(8, dec.code.n, device=dev), iterations=3)
    torch.cuda.synchronize()
    print("ldpc ok", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="two cases, fp32 + fp16 only (racecheck is slow)")
    ap.add_argument("--receiver-only", action="store_true")
    args = ap.parse_args()
    names = gc.case_names()
    if args.quick:
        receiver(("fp32", "fp16"), names[:2])
    else:
        receiver(("fp32", "fp32_simt", "bf16", "fp16"), names)
    if not args.receiver_only:
        others()
    print("sanitize workload done", flush=True)


if __name__ == "__main__":
    main()
