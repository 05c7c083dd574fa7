"""Localise bf16-path errors: run one forward with n_it=1 and compare the
workspace intermediates (features, state after init, agg, conv0 output,
final state) against the float64 oracle."""
import sys

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import numpy as np
import torch

from golden_cases import load_case
from oracle import nrx_oracle as orc
from paper_2409_02912_b200 import _lib
from paper_2409_02912_b200.nrx import get_engine, noise_features, stack_pilots

name = sys.argv[1] if len(sys.argv) > 1 else "c1_small"
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
c = load_case(name)
n = c.y.shape[0]
cfg, config = c.cfg, c.config
U, S, T = cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols
eng = get_engine(c.weights, config, prec)
geo = _lib.buffer_geometry(config, cfg, prec)
print(name, prec, geo)
orders = np.array([m.modulation_order for m in c.mcs], dtype=np.int32)
width = max(config.llr_width(m) for m in orders)
llr, chest = eng.run_arrays(cfg, c.y, stack_pilots(c.books, n, cfg), noise_features(c.n0, n),
                            np.tile(orders, (n, 1)), 1, width)
torch.cuda.synchronize()
ws = eng._local().ws["ws"]
import ctypes
esz = 2 if prec == "bf16" else 4
cw = 16 // esz
rows = geo["rows_slab"]
NU = n * U
plane = NU * rows * esz


def take(off, C, dtype=torch.bfloat16 if prec == "bf16" else torch.float32, cwid=cw):
    b = ws[off:off + NU * rows * C * (torch.finfo(dtype).bits // 8)]
    t = b.view(dtype).reshape(NU, C // cwid, rows, cwid).float().cpu().numpy()
    t = t.transpose(0, 2, 1, 3).reshape(NU, rows, C)
    t = t[:, :S * geo["Tp"]].reshape(NU, S, geo["Tp"], C)[:, :, :T]
    return t


def align(off):
    return (off + 255) // 256 * 256


off_f = 0
off_h = align(off_f + plane * geo["Cf"])
off_s = align(off_h + plane * geo["Ch"])
off_a = align(off_s + plane * geo["Cs"])
off_32 = align(off_a + plane * geo["Ca"])
feats = take(off_f, geo["Cf"])
hbuf = take(off_h, geo["Ch"])
state = take(off_s, geo["Cs"])
agg = take(off_a, geo["Ca"])
d = config.d_s
ref_feats = c.features.reshape(NU, S, T, -1)
print("feats max err", np.abs(feats[..., :ref_feats.shape[-1]] - ref_feats).max(), "scale", np.abs(ref_feats).max())
w = {k: np.asarray(v, np.float64) for k, v in c.weights.items()}
x = ref_feats.astype(np.float64)
s0 = orc.conv_block(x, w, "state_init") if config.variant != "var_io" else None
pos = x[..., 4 * config.num_rx_ant:4 * config.num_rx_ant + 2]
msg = orc.mlp(s0, w, "iteration.msg")
ag = orc.sum_others(msg.reshape((n, U) + msg.shape[1:]), axis=1).reshape(msg.shape)
upd_in = np.concatenate([s0, ag, pos], axis=-1)
h0 = np.maximum(orc.conv2d_same(upd_in, w["iteration.update.conv0.w"]) + w["iteration.update.conv0.b"], 0)
s1 = s0 + orc.conv2d_same(h0, w["iteration.update.conv1.w"]) + w["iteration.update.conv1.b"]


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


print("agg (iter1) rel err", rel(agg[..., :d], ag))
print("h (update conv0) rel err", rel(hbuf[..., :d], h0))
print("state (after iter1) rel err", rel(state[..., :d], s1), "pos", rel(state[..., d:d + 2], pos))
if prec == "bf16":
    s32 = take(off_32, (d + 3) // 4 * 4, torch.float32, 4)
    print("state32 rel err", rel(s32[..., :d], s1))
ref_llr, ref_chest = orc.nrx_forward(*c.call_args()[:2], cfg, c.mcs, c.weights, config, c.call_args()[2],
                                     num_iterations=1, dtype=np.float64)
got = [llr[:, u, ..., :r.shape[-1]] for u, r in enumerate([l if l.ndim == 4 else l[None] for l in ref_llr])]
for u, r in enumerate(ref_llr):
    r = r if r.ndim == 4 else r[None]
    print("llr u", u, "rel err", rel(got[u], r))
