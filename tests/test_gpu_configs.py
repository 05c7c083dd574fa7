"""GPU parity on the BASELINE.json configurations other than the benchmark's
C2 slot (which tests/test_gpu_parity.py covers):

  C1  1 UE, 24 PRB, 16-QAM, RT model (d_s=56, N_it=2)
  C3  mixed modulation orders through the masked readout (QPSK/64-QAM), the
      var_io variant, and the 256-QAM extension (m_max = 8)
  C4  the large non-real-time variant (d_s=56, N_it=8) plus depth control
All against the float64 CPU oracle with the per-precision gates of
tests/test_gpu_parity.py."""

import warnings

import numpy as np
import pytest

from oracle import nrx_oracle as orc
from test_gpu_parity import check_chest, check_llrs

pytestmark = pytest.mark.gpu

PRECISIONS = ["fp32", "fp32_simt", "bf16", "fp16"]


def _run(cfg, config, w, mcs, n_slots, seed, precision, num_iterations=None, n0=0.1):
    from paper_2409_02912_b200.nrx import nrx_forward
    from paper_2409_02912_b200.synth import synth_slots
    y, books, _ = synth_slots(cfg, [m.modulation_order for m in mcs], n_slots, n0, seed=seed)
    ref, ref_chest = orc.nrx_forward(y, books, cfg, mcs, w, config, n0, num_iterations=num_iterations,
                                     dtype=np.float64)
    got, chest = nrx_forward(y, books, cfg, mcs, w, config, n0, num_iterations=num_iterations,
                             precision=precision)
    return got, ref, chest, ref_chest


@pytest.mark.parametrize("precision", PRECISIONS)
def test_c1_single_ue_24prb(precision):
    from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights
    t = default_mcs_table()
    cfg = SlotConfig(num_subcarriers=288, num_ues=1, comb_size=2)
    config = NrxConfig.from_table(t, (14,), d_s=56, num_iterations=2)
    w = orc.perturb_biases(init_weights(config, 3))
    got, ref, chest, ref_chest = _run(cfg, config, w, (t[14],), 2, 5, precision)
    check_llrs(got, ref, precision, "C1")
    check_chest(chest, ref_chest, precision)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_c3_mixed_mcs_masking(precision):
    from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights
    t = default_mcs_table()
    cfg = SlotConfig(num_subcarriers=480, num_ues=2, comb_size=2)
    config = NrxConfig.from_table(t, (9, 14, 19), variant="masking", d_s=56, num_iterations=2)
    w = orc.perturb_biases(init_weights(config, 4))
    got, ref, chest, ref_chest = _run(cfg, config, w, (t[9], t[19]), 2, 6, precision)
    assert got[0].shape[-1] == 2 and got[1].shape[-1] == 6      # label-prefix masking per UE
    check_llrs(got, ref, precision, "C3 masking")
    check_chest(chest, ref_chest, precision)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_c3_var_io(precision):
    from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights
    t = default_mcs_table()
    cfg = SlotConfig(num_subcarriers=240, num_ues=2, comb_size=2)
    config = NrxConfig.from_table(t, (9, 14, 19), variant="var_io", d_s=56, num_iterations=2)
    w = orc.perturb_biases(init_weights(config, 5))
    got, ref, chest, ref_chest = _run(cfg, config, w, (t[19], t[9]), 2, 7, precision)
    assert got[0].shape[-1] == 6 and got[1].shape[-1] == 2
    check_llrs(got, ref, precision, "C3 var_io")
    check_chest(chest, ref_chest, precision)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_256qam_extension_shares_the_masked_readout(precision):
    """EXTENSION (not in the reference): m_max = 8; QPSK and 256-QAM UEs in
    one call through the same masked readout.  The oracle's network is
    order-agnostic (nrx.py:316-319 accepts any order <= m_max)."""
    from paper_2409_02912_b200.config import NrxConfig, SlotConfig, extended_mcs_table, init_weights
    t = extended_mcs_table()
    cfg = SlotConfig(num_subcarriers=240, num_ues=2, comb_size=2)
    config = NrxConfig.from_table(t, (9, 14, 19, 27), variant="masking", d_s=56, num_iterations=2)
    assert config.m_max == 8
    w = orc.perturb_biases(init_weights(config, 6))
    got, ref, chest, ref_chest = _run(cfg, config, w, (t[27], t[9]), 2, 8, precision, n0=0.01)
    assert got[0].shape[-1] == 8 and got[1].shape[-1] == 2
    check_llrs(got, ref, precision, "256-QAM")


@pytest.mark.parametrize("precision", PRECISIONS)
def test_c4_large_model_and_depth_control(precision):
    from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights
    t = default_mcs_table()
    cfg = SlotConfig(num_subcarriers=240, num_ues=2, comb_size=2)
    config = NrxConfig.from_table(t, (14,), d_s=56, num_iterations=8)
    w = init_weights(config, 7)  # zero biases: the SURVEY §8c calibration for N_it = 8
    for depth in (8, 3):
        got, ref, chest, ref_chest = _run(cfg, config, w, (t[14], t[14]), 1, 9, precision, num_iterations=depth)
        check_llrs(got, ref, precision, f"C4 depth {depth}", depth=depth)


@pytest.mark.parametrize("d,comb,S,U,T,pilots,freq", [
    (56, 4, 24, 3, 14, (2, 11), True),   # comb 4, three UE offsets, few interior rows
    (16, 2, 10, 2, 14, (2, 11), True),
    (16, 4, 8, 2, 7, (3,), True),        # no interior row at all, T = 7, one pilot symbol
    (56, 1, 12, 1, 14, (2, 11), True),   # comb 1
    (56, 2, 48, 2, 14, (0, 13), False),  # no frequency encoding, pilots on the edge symbols
])
def test_fp32x3_positional_fold_edges(d, comb, S, U, T, pilots, freq):
    """update.conv0 of the fp32 mode takes the positional channels out of the
    GEMM (upd0_posf): a per-(comb residue, symbol) table for interior rows and
    the 18-term sum at the band edges and pad rows.  Against the float64
    oracle at the fp32 gate over comb sizes, UE comb offsets, tiny grids and
    the frequency-encoding flag."""
    from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights
    t = default_mcs_table()
    cfg = SlotConfig(num_subcarriers=S, num_symbols=T, pilot_symbols=pilots, num_ues=U, comb_size=comb)
    config = NrxConfig.from_table(t, (14,), d_s=d, num_iterations=2, include_freq_encoding=freq)
    w = orc.perturb_biases(init_weights(config, 9))
    got, ref, chest, ref_chest = _run(cfg, config, w, tuple(t[14] for _ in range(U)), 2, 11, "fp32")
    check_llrs(got, ref, "fp32", f"posf d={d} comb={comb} S={S}")
    check_chest(chest, ref_chest, "fp32")


HIDDEN_LIMIT = {"fp32": 96, "fp32_simt": 256, "bf16": 64, "fp16": 64}  # nrx_host.cpp hidden_limit


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("d,h,U,comb,k,T,pilots,S", [
    (64, 64, 2, 2, 3, 14, (2, 11), 48),       # largest state depth
    (64, 96, 2, 2, 3, 14, (2, 11), 48),       # largest hidden width of the fp32 mode
    (56, 128, 2, 2, 3, 14, (2, 11), 48),      # beyond the tensor-core modes' hidden width: fp32_simt only
    (48, 48, 4, 4, 3, 14, (2, 11), 40),       # four UEs (direct sums over the others), N = 2 x 48 pair MMAs
    (24, 24, 2, 2, 1, 14, (2, 11), 60),       # 1x1 kernels
    (32, 32, 2, 2, 3, 32, (0, 9, 18, 27), 24),  # 32 symbols (the longest slot), four pilot symbols
])
def test_limit_configs_vs_oracle(precision, d, h, U, comb, k, T, pilots, S):
    """Model / slot shapes at the limits include/nrx_b200.h documents, run
    through the generic (not unrolled) kernel instances, against the float64
    oracle with the per-precision gates."""
    from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights
    t = default_mcs_table()
    cfg = SlotConfig(num_subcarriers=S, num_symbols=T, pilot_symbols=pilots, num_ues=U, comb_size=comb)
    config = NrxConfig.from_table(t, (14,), d_s=d, hidden_width=h, kernel_size=k, num_iterations=2)
    w = orc.perturb_biases(init_weights(config, 5))
    if -(-h // 16) * 16 > HIDDEN_LIMIT[precision]:
        # rejected up front (not at a kernel launch); the drop-in computes the call on the
        # fp32 SIMT kernels with a RuntimeWarning, the reference accepting any shape
        with pytest.warns(RuntimeWarning, match="does not support"):
            got, ref, chest, ref_chest = _run(cfg, config, w, tuple(t[14] for _ in range(U)), 2, 13, precision)
        precision = "fp32_simt"
    else:
        got, ref, chest, ref_chest = _run(cfg, config, w, tuple(t[14] for _ in range(U)), 2, 13, precision)
    check_llrs(got, ref, precision, f"limits d={d} h={h} U={U} k={k} T={T}")
    check_chest(chest, ref_chest, precision)


def tc_supported(precision, d, h, U, k):
    """Mirror of the tensor-core modes' shape limits (nrx_host.cpp make_geom)."""
    r16 = lambda v: -(-v // 16) * 16  # noqa: E731
    if precision == "fp32_simt":
        return True
    np_ = (56 if -(-d // 8) * 8 == 56 else r16(d)) if precision == "fp32" else r16(d)
    if k * k * (r16(d + 2) + r16(d)) * np_ * 2 > 170 * 1024:   # update.conv0 weights resident
        return False
    if r16(h) > (96 if precision == "fp32" else 64):            # hidden_limit
        return False
    if (precision == "fp32" or U != 2) and 2 * r16(h) + 2 * U * r16(d) > 512:   # message kernel TMEM
        return False
    return True


def _random_config(seed):
    rng = np.random.default_rng(seed)
    d = int(rng.choice([8, 12, 16, 24, 32, 40, 48, 56, 64]))
    h = int(min(96, rng.choice([d, d, 16, 24, 40, 72])))
    U = int(rng.integers(1, 4))
    comb = int(max(U, rng.choice([1, 2, 4])))
    k = int(rng.choice([1, 3, 3, 5]))
    T = int(rng.choice([7, 14, 14, 20]))
    pilots = tuple(sorted(rng.choice(T, size=int(rng.integers(1, 3)), replace=False).tolist()))
    S = int(rng.integers(4, 30)) * comb
    variant = str(rng.choice(["single", "masking", "var_io"]))
    noise, freq = bool(rng.integers(0, 2)), bool(rng.integers(0, 2))
    return d, h, U, comb, k, T, pilots, S, variant, noise, freq


@pytest.mark.parametrize("precision", ["fp32", "fp16"])
@pytest.mark.parametrize("seed", range(16))
def test_random_configs_vs_oracle(seed, precision):
    """Seeded random model / slot shapes (depth, hidden width, UEs, comb,
    kernel size, symbols, pilot symbols, variant, flags) through whichever
    kernel instances they select, against the float64 oracle."""
    from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights
    d, h, U, comb, k, T, pilots, S, variant, noise, freq = _random_config(seed)
    if precision == "fp16" and h > 64:
        h = 64
    t = default_mcs_table()
    cfg = SlotConfig(num_subcarriers=S, num_symbols=T, pilot_symbols=pilots, num_ues=U, comb_size=comb)
    supported = {"single": (14,), "masking": (9, 14, 19), "var_io": (9, 14, 19)}[variant]
    config = NrxConfig.from_table(t, supported, variant=variant, d_s=d, hidden_width=h, kernel_size=k,
                                  num_iterations=2, include_noise_plane=noise, include_freq_encoding=freq)
    w = orc.perturb_biases(init_weights(config, seed))
    rng = np.random.default_rng(100 + seed)
    mcs = tuple(t[int(rng.choice(supported))] for _ in range(U))
    if not tc_supported(precision, d, h, U, k):
        # beyond the tensor-core mode's limits (nrx_host.cpp make_geom): rejected up front,
        # and the drop-in computes the call on the fp32 SIMT kernels with a RuntimeWarning
        with pytest.warns(RuntimeWarning, match="does not support"):
            got, ref, chest, ref_chest = _run(cfg, config, w, mcs, 2, 20 + seed, precision)
        precision = "fp32_simt"
    else:  # inside the limits: the tensor-core path itself must take it (no silent fallback)
        with warnings.catch_warnings(record=True) as caught:
            warnings.simplefilter("always")
            got, ref, chest, ref_chest = _run(cfg, config, w, mcs, 2, 20 + seed, precision)
        fallbacks = [str(c.message) for c in caught if "does not support" in str(c.message)]
        assert not fallbacks, fallbacks
    check_llrs(got, ref, precision, f"random config {seed}: {_random_config(seed)}")
    check_chest(chest, ref_chest, precision)
