"""Golden vectors for the classical baseline receiver, made by the REFERENCE.

Run in the build container (where the read-only reference lives):

    PYTHONPATH=/root/reference/pkg/src python -B tests/golden/make_golden_classical.py

For every slot-generator fixture (tests/golden/sg_*.npz: received grids of the
reference's own generator), runs the reference's "ls_lmmse" receiver —
ls_estimate -> lmmse_equalize -> exact app_demap -> clip (classical.py:40-174,
evaluation.py:79-84,130-135) — and stores the per-UE LLR grids next to it as
cl_<case>.npz.
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

from nrxsim import classical as cl  # noqa: E402
from nrxsim.constellation import build_constellation  # noqa: E402
from nrxsim.slot import PilotBook, SlotConfig  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
CLIP = 20.0


def main():
    with open(os.path.join(OUT, "slotgen_index.json")) as f:
        index = json.load(f)
    for meta in index:
        slot = dict(meta["slot"])
        if "beams" in slot:
            slot["beams"] = tuple(tuple(complex(*v) if isinstance(v, list) else v for v in b) for b in slot["beams"])
        if "pilot_symbols" in slot:
            slot["pilot_symbols"] = tuple(slot["pilot_symbols"])
        cfg = SlotConfig(**slot)
        with np.load(os.path.join(OUT, f"{meta['name']}.npz")) as z:
            y, pil = z["y"], z["pilots"]
        n = y.shape[0]
        est = []
        for i in range(n):
            vals = np.zeros((cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols), complex)
            for u in range(cfg.num_ues):
                sc = cfg.comb_subcarriers(u)
                vals[u][np.ix_(sc, list(cfg.pilot_symbols))] = pil[i, u, :sc.size]
            est.append(cl.ls_estimate(y[i], PilotBook(vals, cfg), cfg).h_eff)
        zz, nvar = cl.lmmse_equalize(y, np.stack(est), meta["n0"])
        out = {}
        for u, m in enumerate(meta["orders"]):
            llr = cl.app_demap(zz[:, u], build_constellation(m), nvar[:, u], mode="exact")
            out[f"llr_{u}"] = np.clip(llr, -CLIP, CLIP)
        np.savez_compressed(os.path.join(OUT, f"cl_{meta['name']}.npz"), **out)
        print(meta["name"], {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
