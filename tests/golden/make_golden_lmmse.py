"""Golden vectors for the covariance-based LMMSE channel estimator and the
lmmse_kbest receiver, made by the REFERENCE itself.

Run in the build container (where the read-only reference lives):

    PYTHONPATH=/root/reference/pkg/src python -B tests/golden/make_golden_lmmse.py

For the 2-UE slot-generator fixtures it estimates the sample covariances with
the reference (channel.estimate_covariance channel.py:239-268, 120 draws of
its TdlChannelSource), runs lmmse_estimate (classical.py:81-103) and the
"lmmse_kbest" receiver (evaluation.py:136-138, K = 16), and stores the
covariances, the channel estimates and the LLR grids as lm_<case>.npz.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = os.environ.get("NRX_REFERENCE_SRC", "/root/reference/pkg/src")
if REF not in sys.path:
    sys.path.insert(0, REF)

from nrxsim import channel as ch  # noqa: E402
from nrxsim import classical as cl  # noqa: E402
from nrxsim.constellation import build_constellation  # noqa: E402
from nrxsim.evaluation import _kbest_grids  # noqa: E402
from nrxsim.slot import PilotBook, SlotConfig  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
SAMPLES = 120
COV_SEED = 4


def main():
    with open(os.path.join(OUT, "slotgen_index.json")) as f:
        index = json.load(f)
    for meta in index:
        if meta["name"] not in ("sg_desk", "sg_mixed", "sg_b8_t7"):
            continue
        slot = dict(meta["slot"])
        if "pilot_symbols" in slot:
            slot["pilot_symbols"] = tuple(slot["pilot_symbols"])
        cfg = SlotConfig(**slot)
        profiles = [ch.PROFILES[p]().with_doppler(fd) for p, fd in zip(meta["profiles"], meta["doppler"])]
        cov = ch.estimate_covariance(ch.TdlChannelSource(profiles), cfg, SAMPLES, seed=COV_SEED)
        with np.load(os.path.join(OUT, f"{meta['name']}.npz")) as z:
            y, pil = z["y"], z["pilots"]
        est = []
        for i in range(y.shape[0]):
            vals = np.zeros((cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols), complex)
            for u in range(cfg.num_ues):
                sc = cfg.comb_subcarriers(u)
                vals[u][np.ix_(sc, list(cfg.pilot_symbols))] = pil[i, u, :sc.size]
            est.append(cl.lmmse_estimate(y[i], PilotBook(vals, cfg), cfg, cov, meta["n0"]).h_eff)
        est = np.stack(est)
        consts = [build_constellation(m) for m in meta["orders"]]
        grids = _kbest_grids(y, est, meta["n0"], consts, cfg, 16, 20.0)
        out = dict(r_f=cov.freq, r_t=cov.time, h_est=est)
        for u, g in enumerate(grids):
            out[f"llr_{u}"] = g
        np.savez_compressed(os.path.join(OUT, f"lm_{meta['name']}.npz"), **out)
        print(meta["name"], {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
