"""Per-kernel device times (CUDA events from the library's profiling hook) of
one batched C2 forward, with algorithmic FLOP/s and bytes per kernel."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2409_02912_b200 import _lib
from paper_2409_02912_b200.engine import NrxEngine

ap = argparse.ArgumentParser()
ap.add_argument("--slots", type=int, default=32)
ap.add_argument("--precision", default="bf16")
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()

cfg, config, w, _ = bench.c2_setup()
dev = torch.device("cuda", 0)
eng = NrxEngine(config, w, precision=args.precision, device=dev)
B = args.slots
y, pil, nf, mods = bench.gpu_batch(cfg, B, dev)
U, S, T = cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols
llr = torch.empty((B, U, S, T, 4), dtype=torch.float32, device=dev)
chest = torch.empty((B, U, S, T, 4), dtype=torch.complex64, device=dev)
st = torch.cuda.current_stream()
for _ in range(3):
    eng.forward_device(cfg, y, pil, nf, mods, 2, llr, chest, stream=st)
torch.cuda.synchronize()
with _lib.KernelTimer(tuple(_lib.KERNEL_IDS), max_records=4096) as kt:
    for _ in range(args.reps):
        eng.forward_device(cfg, y, pil, nf, mods, 2, llr, chest, stream=st)
    torch.cuda.synchronize()
    rec = kt.collect()
d, h, k = 56, 56, 3
res = B * U * S * T
flops = {"ls_feat": 0, "conv_state_init0": 2 * 9 * 19 * d, "conv_state_init1": 2 * 9 * d * d,
         "msg_agg": 2 * 2 * d * h, "conv_update0": 2 * 9 * (2 * d + 2) * d, "conv_update1": 2 * 9 * d * d,
         "readout": 2 * (2 * d * h + h * 4 + h * 8)}
total = 0.0
out = {}
for name, ms in rec.items():
    per_launch = float(np.mean(ms))
    n_per_fwd = len(ms) / args.reps
    total += per_launch * n_per_fwd
    tf = flops[name] * res / (per_launch / 1e3) / 1e12
    out[name] = {"ms": round(per_launch, 4), "launches_per_fwd": n_per_fwd, "tflops": round(tf, 1)}
for name, ms in rec.items():  # kernels launched several times per forward: per position
    k = int(round(len(ms) / args.reps))
    if k > 1:
        print(f"{name:18s} per launch position: " + ", ".join(f"{float(np.mean(ms[i::k])):.4f}" for i in range(k)))
for name, v in out.items():
    v["share"] = round(v["ms"] * v["launches_per_fwd"] / total, 3)
    print(f"{name:18s} {v['ms']:8.4f} ms x{v['launches_per_fwd']:.0f}  {v['tflops']:7.1f} TFLOP/s  share {v['share']:.3f}")
print(f"sum {total:.3f} ms per forward of {B} slots -> {B / total * 1e3:.0f} slots/s")
print(json.dumps(out))
