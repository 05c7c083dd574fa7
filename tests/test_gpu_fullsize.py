"""Parity at the benchmark's full size (273 PRB = 3276 subcarriers, 2 UE,
4 RX, d_s = 56), for every precision mode with its gate (test_gpu_parity):

* C2 against the REFERENCE's own outputs (tests/golden/c2_ref273.npz, every
  8th subcarrier of the LLR / chest grids; tests/golden/make_golden_c2.py);
* C3 masking (QPSK + 64-QAM), C3 var_io, the 256-QAM masked-readout
  extension and C4 (N_it = 8 at depths 8 and 3) against the float64 oracle
  (nrx.py:237-249, 270-289 paths at full size);
* a paired uncoded BER / BLER comparison at C2 with the GPU-trained RT
  checkpoint (checkpoints/rt_d56_it2_gpu.nrxw): 64 slots x 3 SNR points, GPU
  vs the oracle on the same slots.
"""

import os

import numpy as np
import pytest

from oracle import nrx_oracle as orc
from test_gpu_parity import GATES, check_chest, check_llrs

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PRECISIONS = ["fp32", "fp32_simt", "bf16", "fp16"]
S_FULL = 3276


@pytest.mark.parametrize("precision", PRECISIONS)
def test_c2_273prb_vs_reference_golden(precision):
    from golden_cases import load_c2_ref273
    from paper_2409_02912_b200.nrx import nrx_forward
    cfg, config, w, mcs, y, books, gold = load_c2_ref273()
    llrs, chest = nrx_forward(y[0], books[0], cfg, mcs, w, config, 0.1, precision=precision)
    st = int(gold["stride"])
    got = np.stack(llrs)[:, ::st]
    ref = gold["llr"].astype(np.float64)
    scale = float(gold["llr_absmax"])
    gate = GATES[precision]
    err = np.abs(got - ref)
    assert err.max() <= gate["max"] * scale, err.max() / scale
    assert np.percentile(err, 99) <= gate["p99"] * scale
    sure = np.abs(ref) > gate["max"] * scale
    np.testing.assert_array_equal(got[sure] > 0, ref[sure] > 0)
    assert np.abs(chest[:, ::st] - gold["chest"]).max() <= gate["max"] * float(gold["chest_absmax"])


def _full(variant, supported, orders, n_it=2, m_ext=False, seed=0, n0=0.1):
    from paper_2409_02912_b200.config import (NrxConfig, SlotConfig, default_mcs_table, extended_mcs_table,
                                              init_weights)
    from paper_2409_02912_b200.synth import synth_slots
    t = extended_mcs_table() if m_ext else default_mcs_table()
    cfg = SlotConfig(num_subcarriers=S_FULL, num_ues=2, comb_size=2)
    config = NrxConfig.from_table(t, supported, variant=variant, d_s=56, num_iterations=n_it)
    w = init_weights(config, seed)
    if n_it <= 2:
        w = orc.perturb_biases(w)
    by_order = {t[i].modulation_order: t[i] for i in supported}
    mcs = tuple(by_order[m] for m in orders)
    y, books, _ = synth_slots(cfg, list(orders), 1, n0, seed=seed + 11)
    return cfg, config, w, mcs, y, books


_ORACLE = {}


def _oracle(key, cfg, config, w, mcs, y, books, n0=0.1, depth=None):
    if key not in _ORACLE:
        _ORACLE[key] = orc.nrx_forward(y, books, cfg, mcs, w, config, n0, num_iterations=depth, dtype=np.float64)
    return _ORACLE[key]


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("case", ["c3_masking_qpsk_64qam", "c3_var_io", "qam256_extension"])
def test_c3_full_size(case, precision):
    from paper_2409_02912_b200.nrx import nrx_forward
    if case == "c3_masking_qpsk_64qam":
        args = _full("masking", (9, 14, 19), (2, 6), seed=1)
    elif case == "c3_var_io":
        args = _full("var_io", (9, 14, 19), (6, 2), seed=2)
    else:
        args = _full("masking", (9, 14, 19, 27), (8, 2), m_ext=True, seed=3)
    cfg, config, w, mcs, y, books = args
    n0 = 0.01 if case == "qam256_extension" else 0.1
    ref, ref_chest = _oracle(case, cfg, config, w, mcs, y, books, n0)
    got, chest = nrx_forward(y, books, cfg, mcs, w, config, n0, precision=precision)
    widths = [m.modulation_order for m in mcs]
    assert [g.shape[-1] for g in got] == widths
    check_llrs(got, ref, precision, case)
    check_chest(chest, ref_chest, precision)


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("depth", [8, 3])
def test_c4_full_size(depth, precision):
    from paper_2409_02912_b200.nrx import nrx_forward
    cfg, config, w, mcs, y, books = _full("single", (14,), (4, 4), n_it=8, seed=4)
    ref, _ = _oracle(("c4", depth), cfg, config, w, mcs, y, books, depth=depth)
    got, _ = nrx_forward(y, books, cfg, mcs, w, config, 0.1, num_iterations=depth, precision=precision)
    check_llrs(got, ref, precision, f"C4 depth {depth}", depth=depth)


def test_c2_paired_ber_bler_trained_checkpoint():
    """Uncoded BER / BLER of the GPU receiver (every precision) and of the
    oracle on the same 64 C2 slots at 8 / 12 / 16 dB, with the GPU-trained
    RT checkpoint.  fp32 modes: every flipped hard decision lies inside the
    1e-5 band and per-(slot, UE) block errors are identical; bf16 / fp16:
    BER statistically indistinguishable (<= 3 sigma) and <= 1 % of blocks
    disagree.  A block is one UE's data bits of one slot."""
    from paper_2409_02912_b200.config import SlotConfig, checkpoint_load, default_mcs_table
    from paper_2409_02912_b200.nrx import nrx_forward
    from paper_2409_02912_b200.synth import synth_slots
    config, w = checkpoint_load(os.path.join(ROOT, "checkpoints", "rt_d56_it2_gpu.nrxw"))
    table = default_mcs_table()
    mcs = (table[14], table[14])
    cfg = SlotConfig(num_subcarriers=S_FULL, num_ues=2, comb_size=2)
    s_idx, t_idx = np.nonzero(cfg.data_mask)
    n_slots, chunk = 64, 4
    band = {"fp32": 1e-5, "fp32_simt": 1e-5, "bf16": 2e-2, "fp16": 5e-3}
    for snr_db in (8.0, 12.0, 16.0):
        n0 = 10 ** (-snr_db / 10)
        y, books, bits = synth_slots(cfg, [4, 4], n_slots, n0, seed=int(snr_db) * 31)
        ref = [np.concatenate(x) for x in zip(*[
            orc.nrx_forward(y[i:i + chunk], books[i:i + chunk], cfg, mcs, w, config, n0)[0]
            for i in range(0, n_slots, chunk)])]
        ref_err = [((r[:, s_idx, t_idx] > 0) != b) for r, b in zip(ref, bits)]
        n_bits = sum(e.size for e in ref_err)
        ber_ref = sum(int(e.sum()) for e in ref_err) / n_bits
        blk_ref = np.stack([e.reshape(n_slots, -1).any(axis=1) for e in ref_err])
        assert 1e-4 < ber_ref < 0.3, ber_ref
        scale = max(float(np.abs(r).max()) for r in ref)
        for precision in PRECISIONS:
            got, _ = nrx_forward(y, books, cfg, mcs, w, config, n0, precision=precision)
            err = [((g[:, s_idx, t_idx] > 0) != b) for g, b in zip(got, bits)]
            ber = sum(int(e.sum()) for e in err) / n_bits
            blk = np.stack([e.reshape(n_slots, -1).any(axis=1) for e in err])
            for r, g in zip(ref, got):
                rr, gg = r[:, s_idx, t_idx], g[:, s_idx, t_idx]
                flip = (rr > 0) != (gg > 0)
                assert np.all(np.abs(rr[flip]) <= band[precision] * scale), (precision, snr_db)
            sigma = np.sqrt(ber_ref * (1 - ber_ref) / n_bits)
            assert abs(ber - ber_ref) <= 3 * sigma, (precision, snr_db, ber, ber_ref)
            if precision.startswith("fp32"):
                np.testing.assert_array_equal(blk, blk_ref)
            else:
                assert np.mean(blk != blk_ref) <= 0.01, (precision, snr_db)
