import sys, time, numpy as np
sys.path.insert(0, '.')
import torch
from oracle import nrx_oracle as orc
from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights
from paper_2409_02912_b200.nrx import nrx_forward
from paper_2409_02912_b200.synth import synth_slots
t = default_mcs_table()
for S, U, d in ((96, 2, 56), (288, 1, 56), (96, 2, 16), (3276, 2, 56)):
    cfg = SlotConfig(num_subcarriers=S, num_ues=U, comb_size=2)
    config = NrxConfig.from_table(t, (14,), d_s=d, num_iterations=2)
    w = orc.perturb_biases(init_weights(config, 3))
    mcs = tuple(t[14] for _ in range(U))
    y, books, _ = synth_slots(cfg, [4]*U, 1, 0.1, seed=5)
    ref, rch = orc.nrx_forward(y, books, cfg, mcs, w, config, 0.1, dtype=np.float64)
    for prec in ("fp32", "fp32_simt", "fp16"):
        got, ch = nrx_forward(y, books, cfg, mcs, w, config, 0.1, precision=prec)
        torch.cuda.synchronize()
        scale = max(np.abs(r).max() for r in ref)
        err = max(float(np.abs(g - r).max()) for g, r in zip(got, ref)) / scale
        cerr = float(np.abs(ch - rch).max() / np.abs(rch).max())
        print(f"S={S} U={U} d={d} {prec}: max rel LLR err {err:.3g}  chest {cerr:.3g}", flush=True)
