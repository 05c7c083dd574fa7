"""CPU checks of the LDPC layer: the oracle decoder against the reference's
own decoder outputs (golden fixtures from tests/golden/make_golden_ldpc.py),
the scalable IRA construction (structure, encoder parity, rate matching at
the 273-PRB codeword size), and C-ABI validation without a GPU."""

import ctypes
import json
import os
import time

import numpy as np
import pytest

from oracle import ldpc_oracle as lo
from paper_2409_02912_b200 import _lib
from paper_2409_02912_b200.ldpc import LdpcCode, ira_code, rate_matched_ira_code

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_names():
    with open(os.path.join(GOLDEN, "ldpc_index.json")) as f:
        return [c["name"] for c in json.load(f)]


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        a = {k: z[k] for k in z.files}
    code = LdpcCode(int(a["n"]), int(a["k"]), a["row_cols"], a["col_rows"], a["col_slots"], a["info_positions"],
                    a["punctured"], a["shortened"])
    return code, a


@pytest.mark.parametrize("name", golden_names())
def test_oracle_decoder_bit_exact_vs_reference(name):
    code, a = load_golden(name)
    np.testing.assert_array_equal(code.tx_positions, a["tx_positions"])
    for it, dk, ok in ((20, "dec20", "ok20"), (3, "dec3", "ok3")):
        dec, done = lo.decode(code, a["llr"], it)
        np.testing.assert_array_equal(done, a[ok])
        np.testing.assert_array_equal(dec, a[dk])


def test_ira_structure():
    code = ira_code(500, seed=3)
    n, m, k = code.n, code.num_checks, code.k
    assert (n, m, k) == (1000, 500, 500)
    deg = (code.col_rows >= 0).sum(axis=1)
    assert (deg[:k] == 3).all()
    chain, z = code.chain_cols, code.chain_step
    assert z == 32                                              # ceil(500 / 16)
    assert sorted(chain.tolist()) == list(range(k, n))
    assert (deg[chain[: m - z]] == 2).all() and (deg[chain[m - z:]] == 1).all()
    # every check: exactly three information columns, chain positions i-Z and i
    rc = code.row_cols
    info_deg = ((rc >= 0) & (rc < k)).sum(axis=1)
    assert (info_deg == 3).all()
    for i in (0, 1, 31, 32, 250, m - 1):
        par = sorted(c for c in rc[i] if c >= k)
        want = sorted([chain[i]] + ([chain[i - z]] if i >= z else []))
        assert par == want
    # column lists consistent with the row lists, no repeated check in a column
    for j in range(n):
        rows = [r for r in code.col_rows[j] if r >= 0]
        assert len(set(rows)) == len(rows)
        for r, s in zip(code.col_rows[j], code.col_slots[j]):
            if r >= 0:
                assert rc[r, s] == j
    assert np.array_equal(ira_code(500, seed=3).row_cols, rc)          # deterministic
    assert not np.array_equal(ira_code(500, seed=4).row_cols, rc)


def test_ira_codewords_satisfy_parity_and_decode():
    code = rate_matched_ira_code(1152, 553 / 1024)
    rng = np.random.default_rng(0)
    info = (rng.random((6, code.k_eff)) < 0.5).astype(np.uint8)
    cw = lo.staircase_codeword(code, info)
    assert lo.check_parity(code.row_cols, cw).all()
    tx = cw[:, code.tx_positions].astype(np.float64)
    dec, ok = lo.decode(code, 20.0 * (2 * tx - 1), 20)
    assert ok.all()
    np.testing.assert_array_equal(dec, info)
    # BPSK over AWGN at a comfortable SNR, clipped like evaluation.py:200-201
    sigma = 0.6
    rx = (2 * tx - 1) + sigma * rng.normal(size=tx.shape)
    dec, ok = lo.decode(code, np.clip(2 * rx / sigma ** 2, -20, 20), 20)
    assert ok.mean() > 0.8 and (dec[ok] == info[ok]).all()


@pytest.mark.parametrize("e,rate", [(1152, 553 / 1024), (900, 0.33), (576, 679 / 1024), (900, 0.75)])
def test_ira_rate_matching_like_reference(e, rate):
    code = rate_matched_ira_code(e, rate)
    k_eff = int(round(rate * e))
    assert code.num_tx_bits == e and code.k_eff == k_eff
    assert code.n == 2 * max(k_eff, e - k_eff)
    assert np.array_equal(code.shortened, code.info_positions[: code.k - k_eff])
    # punctured = trailing parity columns = chain positions spread along the accumulator
    if code.punctured.size > 1:
        pos = np.sort(np.flatnonzero(np.isin(code.chain_cols, code.punctured)))
        assert np.diff(pos).max() <= 4 * code.num_checks / code.punctured.size + 2


def test_ira_scales_to_273_prb_codeword():
    e = 3276 * 12 * 4                      # C2 16-QAM stream: 157,248 coded bits
    t0 = time.perf_counter()
    code = rate_matched_ira_code(e, 553 / 1024)
    assert time.perf_counter() - t0 < 20.0
    assert code.num_tx_bits == e and code.n == 2 * int(round(553 / 1024 * e)) == 169840
    rng = np.random.default_rng(1)
    info = (rng.random((1, code.k_eff)) < 0.5).astype(np.uint8)
    assert lo.check_parity(code.row_cols, lo.staircase_codeword(code, info)).all()


def test_ldpc_create_validation_without_gpu():
    lib = _lib.load()
    d = _lib.LdpcDesc()
    h = ctypes.c_void_p()
    assert lib.nrx_ldpc_create(ctypes.byref(d), ctypes.byref(h)) == 1          # n = 0
    code = ira_code(8)
    rc = np.ascontiguousarray(code.row_cols, dtype=np.int32)
    cr = np.ascontiguousarray(code.col_rows, dtype=np.int32)
    cs = np.ascontiguousarray(code.col_slots, dtype=np.int32)
    info = np.ascontiguousarray(code.info_positions, dtype=np.int32)
    d.n, d.m, d.k, d.dmax, d.cdeg = code.n, code.num_checks, code.k, rc.shape[1], 3
    d.row_cols, d.col_rows, d.col_slots, d.info_positions = rc.ctypes.data, cr.ctypes.data, cs.ctypes.data, info.ctypes.data
    d.cdeg = 4
    assert lib.nrx_ldpc_create(ctypes.byref(d), ctypes.byref(h)) == 2          # column degree > 3
    d.cdeg = 3
    bad = rc.copy()
    bad[0, 0] = code.n
    d.row_cols = bad.ctypes.data
    assert lib.nrx_ldpc_create(ctypes.byref(d), ctypes.byref(h)) == 1          # column index out of range
    assert lib.nrx_ldpc_decode(None, 1, None, 20, None, None, None, 0, None) == 1
