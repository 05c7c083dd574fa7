"""Loader of the slot-generator golden fixtures (tests/golden/make_golden_slotgen.py)."""

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _index():
    with open(os.path.join(GOLDEN, "slotgen_index.json")) as f:
        return json.load(f)


def case_names():
    return [c["name"] for c in _index()]


class SlotCase:
    def __init__(self, meta, arrays):
        from paper_2409_02912_b200.config import SlotConfig
        from paper_2409_02912_b200 import slotgen
        self.meta = meta
        self.a = arrays
        slot = dict(meta["slot"])
        if "beams" in slot:
            slot["beams"] = tuple(tuple(complex(*v) if isinstance(v, list) else v for v in b) for b in slot["beams"])
        if "pilot_symbols" in slot:
            slot["pilot_symbols"] = tuple(slot["pilot_symbols"])
        self.cfg = SlotConfig(**slot)
        self.profiles = [slotgen.PROFILES[p]().with_doppler(fd) for p, fd in zip(meta["profiles"], meta["doppler"])]
        self.orders = tuple(meta["orders"])
        self.n0 = meta["n0"]
        self.n = meta["n_slots"]
        self.seed = meta["seed"]

    def variates(self):
        return {k: self.a[k] for k in ("angles", "phases", "labels", "noise", "pilots")}


def load_case(name) -> SlotCase:
    meta = next(c for c in _index() if c["name"] == name)
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        arrays = {k: z[k] for k in z.files}
    return SlotCase(meta, arrays)
