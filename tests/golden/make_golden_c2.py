"""Golden outputs of the REFERENCE at full C2 size (273 PRB / 2 UE / 4 RX,
RT model d_s=56 N_it=2, bias-perturbed random-init weights).

Run in the build container (where the read-only reference lives):

    PYTHONPATH=/root/reference/pkg/src python -B tests/golden/make_golden_c2.py

The input slot is regenerable without the reference: ``synth_slots`` of this
package (numpy, seeded) rounded to complex64, pilots from ``generate_pilots``
(bit-identical to the reference's), weights ``init_weights(config, 0)`` +
``perturb_biases`` (bit-identical).  The reference's own ``nrx_forward`` (its
own SlotConfig / PilotBook / McsEntry / NrxConfig types, ``ad.Tensor``
weights) computes the outputs; the fixture keeps every 8th subcarrier of the
LLR and channel-estimate grids (and the full-grid max |LLR|), which keeps it
small while covering the whole band.
"""

from __future__ import annotations

import dataclasses
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.environ.get("NRX_REFERENCE_SRC", "/root/reference/pkg/src")
for p in (REF, ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

from nrxsim import autodiff as ad  # noqa: E402
from nrxsim import nrx as rnrx  # noqa: E402
from nrxsim import slot as rslot  # noqa: E402

from golden_cases import C2_REF273_SEED, c2_ref273_case  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
STRIDE = 8


def main():
    cfg, config, w, mcs, y, books = c2_ref273_case()
    rcfg = rslot.SlotConfig(**{f.name: getattr(cfg, f.name) for f in dataclasses.fields(rslot.SlotConfig)})
    rconfig = rnrx.NrxConfig(**{f.name: getattr(config, f.name) for f in dataclasses.fields(rnrx.NrxConfig)})
    rmcs = tuple(rslot.McsEntry(m.index, m.modulation_order, m.code_rate) for m in mcs)
    rbook = rslot.PilotBook(values=books[0].values, config=rcfg)
    rw = {k: ad.Tensor(v, requires_grad=True) for k, v in w.items()}
    llrs, chest = rnrx.nrx_forward(y[0], rbook, rcfg, rmcs, rw, rconfig, 0.1)
    llr = np.stack(llrs).astype(np.float32)              # (U, S, T, 4)
    chest = np.asarray(chest, dtype=np.complex64)        # (U, S, T, B)
    np.savez_compressed(os.path.join(OUT, "c2_ref273.npz"), seed=C2_REF273_SEED, stride=STRIDE,
                        llr=llr[:, ::STRIDE], chest=chest[:, ::STRIDE],
                        llr_absmax=np.float64(np.abs(llr).max()), chest_absmax=np.float64(np.abs(chest).max()))
    print("wrote c2_ref273.npz", llr.shape, float(np.abs(llr).max()))


if __name__ == "__main__":
    main()
