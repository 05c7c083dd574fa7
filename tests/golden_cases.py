"""Load the reference-generated golden fixtures (tests/golden/*.npz)."""

from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

from paper_2409_02912_b200.config import McsEntry, NrxConfig, PilotBook, SlotConfig

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def case_names():
    with open(os.path.join(GOLDEN, "index.json")) as fh:
        return json.load(fh)


@dataclass
class GoldenCase:
    name: str
    cfg: SlotConfig
    config: NrxConfig
    mcs: tuple
    y: np.ndarray            # (N, S, T, B) complex128
    books: list              # per-slot PilotBook
    n0: np.ndarray           # (N,)
    n0_arg: object           # what the reference was called with
    squeeze: bool
    weights: dict
    features: np.ndarray
    llrs: list
    chest: np.ndarray
    bits: list

    def call_args(self):
        """(y, books, n0) exactly as passed to the reference nrx_forward."""
        if self.squeeze:
            return self.y[0], self.books[0], self.n0_arg
        return self.y, self.books, self.n0_arg


def load_case(name: str) -> GoldenCase:
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    s = meta["slot"]
    s["pilot_symbols"] = tuple(s["pilot_symbols"])
    cfg = SlotConfig(**s)
    c = meta["nrx"]
    for k in ("supported_mcs", "io_modulations"):
        c[k] = tuple(c[k])
    config = NrxConfig(**c)
    mcs = tuple(McsEntry(i, m, r) for i, m, r in meta["mcs"])
    pilots = z["pilots"]
    books = [PilotBook(values=pilots[i], config=cfg) for i in range(pilots.shape[0])]
    n0 = z["n0"]
    n0_arg = float(n0[0]) if meta["n0_scalar"] else n0
    weights = {k[2:]: z[k] for k in z.files if k.startswith("w:")}
    llrs = [z[f"llr{u}"] for u in range(cfg.num_ues)]
    bits = [z[f"bits{u}"] for u in range(cfg.num_ues)]
    return GoldenCase(name, cfg, config, mcs, z["y"], books, n0, n0_arg, meta["squeeze"],
                      weights, z["features"], llrs, z["chest"], bits)


C2_REF273_SEED = 2409


def c2_ref273_case():
    """The full-size C2 case of tests/golden/c2_ref273.npz (regenerable without
    the reference): (cfg, config, weights, mcs, y (1,S,T,B), books)."""
    from oracle.nrx_oracle import perturb_biases
    from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights
    from paper_2409_02912_b200.synth import synth_slots
    table = default_mcs_table()
    cfg = SlotConfig(num_subcarriers=3276, num_ues=2, comb_size=2)
    config = NrxConfig.from_table(table, (14,), d_s=56, num_iterations=2)
    w = perturb_biases(init_weights(config, seed=0))
    y, books, _ = synth_slots(cfg, [4, 4], 1, 0.1, seed=C2_REF273_SEED)
    y = y.astype(np.complex64).astype(np.complex128)
    return cfg, config, w, (table[14], table[14]), y, books


def load_c2_ref273():
    """c2_ref273_case() + the reference's outputs on it (every 8th subcarrier)."""
    with np.load(os.path.join(GOLDEN, "c2_ref273.npz")) as z:
        gold = {k: z[k] for k in z.files}
    return c2_ref273_case() + (gold,)
