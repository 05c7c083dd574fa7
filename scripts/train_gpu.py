"""Train an NRX on the GPU (torch training step, GPU slot generator) and
save an NRXW checkpoint; reports steps/s (the reference trains the desk
model at ~6 steps/s on 6 CPU threads, tests/golden/train_desk_long.py).

  python scripts/train_gpu.py --d 16 --it 2 --S 96 --steps 2000 --out gpurun_out/desk_gpu.nrxw
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2409_02912_b200.config import (NrxConfig, SlotConfig, checkpoint_load, checkpoint_save,  # noqa: E402
                                          default_mcs_table, init_weights)
from paper_2409_02912_b200.engine import NrxEngine  # noqa: E402
from paper_2409_02912_b200.slotgen import GpuSlotSource, evaluate_uncoded  # noqa: E402
from paper_2409_02912_b200.training import GpuTrainConfig, train_gpu  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=16)
    ap.add_argument("--it", type=int, default=2)
    ap.add_argument("--S", type=int, default=96)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--lr", type=float, default=2e-3)
    ap.add_argument("--out", default="gpurun_out/nrx_gpu.nrxw")
    ap.add_argument("--init", default=None, help="continue from this NRXW checkpoint")
    ap.add_argument("--seed", type=int, default=0, help="slot-stream seed of the training batches")
    args = ap.parse_args()
    table = default_mcs_table()
    cfg = SlotConfig(num_subcarriers=args.S, num_ues=2)
    if args.init:
        config, w = checkpoint_load(args.init)
    else:
        config = NrxConfig.from_table(table, (14,), d_s=args.d, num_iterations=args.it)
        w = init_weights(config, 0)
    src = GpuSlotSource(cfg)
    tcfg = GpuTrainConfig(batch_size=args.batch, steps=args.steps, snr_lo_db=4.0, snr_hi_db=24.0, learning_rate=args.lr,
                          seed=args.seed)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    graph, _, hist = train_gpu(config, w, src, table, tcfg, log_every=max(1, args.steps // 10))
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    for s, l in hist:
        print(s, round(l["total"], 4), flush=True)
    trained = graph.numpy_weights()
    checkpoint_save(args.out, config, trained)
    eng = NrxEngine(config, trained, "fp16")
    rec = evaluate_uncoded(eng, src, (table[14], table[14]), [5, 10, 15, 20, 25], n_slots=64, batch=32, seed=5)
    print({"steps": args.steps, "wall_s": round(el, 1), "steps_per_s": round(args.steps / el, 1),
           "uncoded_ber": [(r.snr_db, round(r.ber, 4)) for r in rec]})


if __name__ == "__main__":
    main()
