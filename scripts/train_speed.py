"""Training steps/s on the GPU: hand-written kernels (kernels="nrx") vs
cuDNN / cuBLAS (kernels="torch"), same batches, desk and RT models.

  python scripts/train_speed.py [--steps 60]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights  # noqa: E402
from paper_2409_02912_b200.slotgen import GpuSlotSource  # noqa: E402
from paper_2409_02912_b200.training import Adam, GpuTrainConfig, TorchNrxGraph, train_gpu  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=60)
    args = ap.parse_args()
    table = default_mcs_table()
    out = {}
    for d, batch in ((16, 16), (56, 32)):
        cfg = SlotConfig(num_subcarriers=96, num_ues=2)
        config = NrxConfig.from_table(table, (14,), d_s=d, num_iterations=2)
        w = init_weights(config, 0)
        src = GpuSlotSource(cfg)
        for kernels in ("nrx", "nrx_tc", "torch"):
            tcfg = GpuTrainConfig(batch_size=batch, steps=args.steps, snr_lo_db=4.0, snr_hi_db=24.0,
                                  learning_rate=1e-3, seed=1)
            g = TorchNrxGraph(config, w, src.device, kernels=kernels)
            train_gpu(config, w, src, table, GpuTrainConfig(batch_size=batch, steps=5, seed=1), graph=g,
                      adam=Adam(lr=1e-3))  # warm-up
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, _, hist = train_gpu(config, w, src, table, tcfg, graph=g, adam=Adam(lr=1e-3), log_every=args.steps - 1)
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
            out[f"d{d}_b{batch}_{kernels}"] = {"steps_per_s": round(args.steps / el, 1),
                                               "last_loss": round(hist[-1][1]["total"], 4)}
            print(f"d_s={d} batch={batch} kernels={kernels}: {args.steps / el:.1f} steps/s", flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
