"""Pin the CPU oracle (oracle/nrx_oracle.py) against the reference's own
outputs (tests/golden/*.npz, written by tests/golden/make_golden.py)."""

import numpy as np
import pytest

from golden_cases import case_names, load_case
from oracle import nrx_oracle as orc
from paper_2409_02912_b200 import config as pcfg

CASES = case_names()


@pytest.mark.parametrize("name", CASES)
def test_features_bit_exact(name):
    c = load_case(name)
    n = c.y.shape[0]
    ls = np.stack([orc.ls_estimate(c.y[i], c.books[i].values, c.cfg) for i in range(n)])
    feats = orc.assemble_features(c.y, ls, c.n0, c.cfg, c.config)
    np.testing.assert_array_equal(feats, c.features)


@pytest.mark.parametrize("name", CASES)
def test_forward_matches_reference(name):
    c = load_case(name)
    y, books, n0 = c.call_args()
    llrs, chest = orc.nrx_forward(y, books, c.cfg, c.mcs, c.weights, c.config, n0)
    assert len(llrs) == len(c.llrs)
    scale = max(np.abs(l).max() for l in c.llrs)
    for got, ref in zip(llrs, c.llrs):
        assert got.shape == ref.shape and got.dtype == np.float32
        # same fp32 GEMM shapes as the reference: agreement to fp32 rounding
        np.testing.assert_allclose(got, ref, rtol=0, atol=2e-6 * scale)
    assert chest.shape == c.chest.shape and chest.dtype == np.complex64
    np.testing.assert_allclose(chest, c.chest, rtol=0, atol=2e-6 * np.abs(c.chest).max())


@pytest.mark.parametrize("name", CASES)
def test_fp64_replay_close_to_reference(name):
    """The float64 replay is the calibration reference: the reference's fp32
    output sits within ~1e-5 relative of it."""
    c = load_case(name)
    y, books, n0 = c.call_args()
    llrs, _ = orc.nrx_forward(y, books, c.cfg, c.mcs, c.weights, c.config, n0, dtype=np.float64)
    scale = max(np.abs(l).max() for l in c.llrs)
    for got, ref in zip(llrs, c.llrs):
        assert np.abs(got - ref).max() <= 1e-5 * scale


@pytest.mark.parametrize("name", CASES)
def test_product_init_weights_match_reference(name):
    c = load_case(name)
    w = pcfg.init_weights(c.config, seed=7)
    assert set(w) == set(c.weights)
    w_bias = orc.perturb_biases(w, seed=99)
    for k in w:
        ref = c.weights[k]
        if k.endswith(".b") and np.any(ref != 0):
            np.testing.assert_array_equal(w_bias[k], ref)
        else:
            np.testing.assert_array_equal(w[k], ref)


@pytest.mark.parametrize("name", CASES)
def test_product_pilots_match_reference(name):
    # golden books were generated with slot_seed = case_id * 1000 + i
    c = load_case(name)
    idx = CASES.index(name) + 1
    for i, book in enumerate(c.books):
        got = pcfg.generate_pilots(c.cfg, slot_seed=idx * 1000 + i)
        np.testing.assert_array_equal(got.values, book.values)


def test_sum_others_definition():
    x = np.random.default_rng(6).normal(size=(2, 3, 4)).astype(np.float32)
    ref = (x.astype(np.float64).sum(axis=1, keepdims=True) - x).astype(np.float32)
    np.testing.assert_array_equal(orc.sum_others(x, axis=1), ref)
    np.testing.assert_array_equal(orc.sum_others(x[:, :1], axis=1), 0.0)


def test_conv_matches_naive_loops():
    rng = np.random.default_rng(2)
    x = rng.normal(size=(1, 4, 5, 2))
    w = rng.normal(size=(3, 3, 2, 4))
    out = orc.conv2d_same(x, w)
    xp = np.pad(x, ((0, 0), (1, 1), (1, 1), (0, 0)))
    ref = np.zeros((1, 4, 5, 4))
    for i in range(4):
        for j in range(5):
            ref[0, i, j] = np.einsum("abc,abco->o", xp[0, i:i + 3, j:j + 3], w)
    np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-12)


def test_positional_encoding_hand_value():
    cfg = pcfg.SlotConfig(num_subcarriers=24, num_symbols=14, pilot_symbols=(2, 11))
    pe = orc.positional_encoding(cfg, ue=0)
    assert abs(pe[0, 7, 0] - 4 / 14) < 1e-7
    for s in cfg.comb_subcarriers(0):
        for t in cfg.pilot_symbols:
            assert pe[s, t, 0] == 0 and pe[s, t, 1] == 0


def test_oracle_matches_reference_at_273prb():
    """The oracle against the reference's own C2 outputs (273 PRB, RT model):
    every 8th subcarrier of the LLR / chest grids, fp32 rounding level."""
    from golden_cases import load_c2_ref273
    cfg, config, w, mcs, y, books, gold = load_c2_ref273()
    llrs, chest = orc.nrx_forward(y[0], books[0], cfg, mcs, w, config, 0.1)
    st = int(gold["stride"])
    got = np.stack(llrs)[:, ::st]
    scale = float(gold["llr_absmax"])
    assert got.shape == gold["llr"].shape
    assert np.abs(got - gold["llr"]).max() <= 2e-6 * scale
    assert np.abs(chest[:, ::st] - gold["chest"]).max() <= 2e-6 * float(gold["chest_absmax"])
