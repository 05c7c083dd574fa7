"""Coded TBLER / BER sweeps on the GPU (the reference's evaluate_tbler,
evaluation.py:212-268, with every step on the device): the desk receiver
(reference-trained d_s=16 checkpoint) against the classical baselines on the
same slots, and the baselines at the full 273-PRB C2 size.

  python scripts/tbler_sweep.py [--out profiles/r1_tbler.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2409_02912_b200.classical import GpuKBest, GpuLmmseKBest, GpuLsLmmse, estimate_covariance  # noqa: E402
from paper_2409_02912_b200.config import McsEntry, SlotConfig, checkpoint_load, default_mcs_table  # noqa: E402
from paper_2409_02912_b200.engine import NrxEngine  # noqa: E402
from paper_2409_02912_b200.ldpc import evaluate_coded, slot_code  # noqa: E402
from paper_2409_02912_b200.slotgen import GpuSlotSource  # noqa: E402


def sweep(label, cfg, mcs, receivers, snrs, n_slots, batch):
    src = GpuSlotSource(cfg)
    built = {}                                   # UEs with the same MCS share one code (and one decode call)
    for m in mcs:
        if (m.modulation_order, m.code_rate) not in built:
            built[(m.modulation_order, m.code_rate)] = slot_code(cfg, m)
    codes = [built[(m.modulation_order, m.code_rate)] for m in mcs]
    out = {"config": label, "num_subcarriers": cfg.num_subcarriers, "ues": cfg.num_ues,
           "mcs": [(m.index, m.modulation_order, round(m.code_rate, 4)) for m in mcs],
           "codeword_bits": codes[0].num_tx_bits, "payload_bits": codes[0].k_eff, "slots_per_point": n_slots,
           "curves": {}}
    for name, make in receivers:
        rx = make(src)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        recs = evaluate_coded(rx, src, mcs, snrs, n_slots=n_slots, batch=batch, seed=1, receiver=name, codes=codes)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        out["curves"][name] = {"snr_db": [r.snr_db for r in recs], "tbler": [round(r.tbler, 4) for r in recs],
                               "ber": [round(r.ber, 5) for r in recs], "blocks": recs[0].blocks,
                               "wall_s": round(el, 2),
                               "slots_per_s": round(n_slots * len(snrs) / el, 1)}
        print(label, name, out["curves"][name], flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/tbler.json")
    ap.add_argument("--rt", default="", help="NRXW checkpoint of an RT model to add to the C2 sweep")
    ap.add_argument("--c2-slots", type=int, default=256, help="slots per SNR point at C2")
    args = ap.parse_args()
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    config, w = checkpoint_load(os.path.join(here, "tests", "golden", "desk_d16_it2_long.nrxw"))
    res = []
    # desk slot: the trained desk receiver vs the baselines (16-QAM, low rate for the weak desk model)
    cfg = SlotConfig(num_subcarriers=96, num_ues=2)
    mcs = (McsEntry(14, 4, 0.3), McsEntry(14, 4, 0.3))
    rxs = [("nrx", lambda s: NrxEngine(config, w, precision="fp16")),
           ("ls_lmmse", lambda s: GpuLsLmmse(4, 4)),
           ("lmmse_kbest", lambda s: GpuLmmseKBest(estimate_covariance(s, 200, seed=3), 4, 4, 16)),
           ("perfect_kbest", lambda s: GpuKBest(4, 4, 16))]
    res.append(sweep("desk 96 subcarriers", cfg, mcs, rxs, [0.0, 5.0, 10.0, 15.0, 20.0, 25.0], 256, 64))
    # 273 PRB C2 slots, MCS 14 (16-QAM, r = 553/1024): the baselines through the scalable IRA code
    cfg = SlotConfig(num_subcarriers=3276, num_ues=2)
    t = default_mcs_table()
    rxs = [("ls_lmmse", lambda s: GpuLsLmmse(4, 4)),
           ("lmmse_kbest", lambda s: GpuLmmseKBest(estimate_covariance(s, 200, seed=3), 4, 4, 16)),
           ("perfect_kbest", lambda s: GpuKBest(4, 4, 16))]
    if args.rt:
        rt_config, rt_w = checkpoint_load(args.rt)
        rxs.insert(0, ("nrx_rt_gpu_trained", lambda s: NrxEngine(rt_config, rt_w, precision="fp16")))
    res.append(sweep("C2 273 PRB", cfg, (t[14], t[14]), rxs, [4.0, 6.0, 8.0, 10.0, 12.0, 14.0, 16.0, 18.0, 20.0],
                     args.c2_slots, 16))
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
