"""CPU checks of the classical baseline: the oracle against the reference's
own ls_lmmse outputs (tests/golden/cl_sg_*.npz)."""

import os

import numpy as np
import pytest

from oracle import classical_oracle as co
from oracle import slotgen_oracle as so
from slotgen_cases import case_names, load_case

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_cl(name):
    with np.load(os.path.join(GOLDEN, f"cl_{name}.npz")) as z:
        return [z[f"llr_{u}"] for u in range(len(z.files))]


@pytest.mark.parametrize("name", case_names())
def test_oracle_matches_reference_ls_lmmse(name):
    c = load_case(name)
    ref = load_cl(name)
    got = co.ls_lmmse_llrs(c.cfg, c.a["y"], c.a["pilots"], c.n0, c.orders, so.gray_points)
    for g, r in zip(got, ref):
        np.testing.assert_allclose(g, r, rtol=1e-9, atol=1e-9)
