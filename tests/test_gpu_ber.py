"""Uncoded BER / BLER of the GPU receiver vs the CPU reference path on the
same Monte-Carlo batch (north_star: "statistically indistinguishable").

Uses a briefly trained desk model (tests/golden/desk_d16_it2.nrxw, made by
the reference's own trainer, tests/golden/train_desk_ckpt.py) so the BER is
far from the trivial 0.5 of random weights.  Paired test on identical
inputs: every hard-decision disagreement must lie where the reference LLR is
within the precision's error band, and the BER difference is bounded by the
disagreement rate (and must sit inside the binomial 3-sigma band of the
reference BER)."""

import os

import numpy as np
import pytest

from oracle import nrx_oracle as orc

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
CKPT = os.path.join(HERE, "golden", "desk_d16_it2.nrxw")
BAND = {"fp32": 1e-5, "fp32_simt": 1e-5, "bf16": 2e-2, "fp16": 5e-3}


def _batch(n_slots=24, S=96, snr_db=10.0, seed=21):
    from paper_2409_02912_b200.config import SlotConfig
    from paper_2409_02912_b200.synth import synth_slots
    cfg = SlotConfig(num_subcarriers=S, num_ues=2, comb_size=2)
    n0 = 10 ** (-snr_db / 10)
    y, books, bits = synth_slots(cfg, [4, 4], n_slots, n0, seed=seed)
    return cfg, y, books, bits, n0


def _errors(llrs, bits, cfg):
    s_idx, t_idx = np.nonzero(cfg.data_mask)
    bit_err = [((l[:, s_idx, t_idx] > 0) != b) for l, b in zip(llrs, bits)]     # (N, n_data, m) per UE
    ber = float(np.mean([e.mean() for e in bit_err]))
    block = np.stack([e.reshape(e.shape[0], -1).any(axis=1) for e in bit_err])  # (U, N)
    return ber, block, bit_err


@pytest.mark.parametrize("precision", ["fp32", "fp32_simt", "bf16", "fp16"])
def test_uncoded_ber_matches_reference(precision):
    from paper_2409_02912_b200.config import checkpoint_load, default_mcs_table
    from paper_2409_02912_b200.nrx import nrx_forward
    config, w = checkpoint_load(CKPT)
    table = default_mcs_table()
    mcs = (table[14], table[14])
    cfg, y, books, bits, n0 = _batch()
    ref, _ = orc.nrx_forward(y, books, cfg, mcs, w, config, n0)
    got, _ = nrx_forward(y, books, cfg, mcs, w, config, n0, precision=precision)
    ber_ref, blk_ref, e_ref = _errors(ref, bits, cfg)
    ber_got, blk_got, e_got = _errors(got, bits, cfg)
    assert 0.01 < ber_ref < 0.45, ber_ref                       # a trained, non-trivial receiver
    scale = max(np.abs(r).max() for r in ref)
    s_idx, t_idx = np.nonzero(cfg.data_mask)
    n_bits = sum(e.size for e in e_ref)
    disagree = 0
    for r, gl in zip(ref, got):
        rr, gg = r[:, s_idx, t_idx], gl[:, s_idx, t_idx]
        diff = (rr > 0) != (gg > 0)
        disagree += int(diff.sum())
        # every flipped hard decision sits inside the precision's error band
        assert np.all(np.abs(rr[diff]) <= BAND[precision] * scale)
    assert abs(ber_got - ber_ref) <= disagree / n_bits + 1e-12
    sigma = np.sqrt(ber_ref * (1 - ber_ref) / n_bits)
    assert abs(ber_got - ber_ref) <= 3 * sigma
    if precision.startswith("fp32"):
        np.testing.assert_array_equal(blk_got, blk_ref)          # block errors identical
    else:
        assert np.mean(blk_got != blk_ref) <= 0.05
