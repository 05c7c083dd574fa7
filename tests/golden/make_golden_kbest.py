"""Golden vectors for the K-Best baseline, made by the REFERENCE itself.

Run in the build container (where the read-only reference lives):

    PYTHONPATH=/root/reference/pkg/src python -B tests/golden/make_golden_kbest.py

For every slot-generator fixture (tests/golden/sg_*.npz, received grids and
true effective channels of the reference's own generator) runs the
reference's "perfect_kbest" receiver — K-Best detection with max-log LLRs on
the true channel (classical.kbest_detect classical.py:195-261 through
evaluation._kbest_grids :87-111) — for K = 16 and K = 4, and stores the per-UE
LLR grids as kb_<case>.npz.
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

from nrxsim.constellation import build_constellation  # noqa: E402
from nrxsim.evaluation import _kbest_grids  # noqa: E402
from nrxsim.slot import SlotConfig  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


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
            y, h = z["y"], z["h_eff"]
        consts = [build_constellation(m) for m in meta["orders"]]
        out = {}
        for k in (16, 4):
            grids = _kbest_grids(y, h, meta["n0"], consts, cfg, k, 20.0)
            for u, g in enumerate(grids):
                out[f"k{k}_llr_{u}"] = g
        np.savez_compressed(os.path.join(OUT, f"kb_{meta['name']}.npz"), **out)
        print(meta["name"], {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
