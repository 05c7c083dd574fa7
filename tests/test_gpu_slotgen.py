"""GPU slot generator and bit-error counter.

Reference-stream mode: fed the variates the reference drew, the GPU slot
equals the reference generator's output (golden fixtures) and the float64
oracle (C2 size) to 1e-12 of the grid's max magnitude (float64 summation
order is the only difference).  Device (Philox) mode: the statistical
properties the reference's own channel tests check (test_channel.py:34-98,
152-165), batch/rank invariance, and the end-to-end uncoded BER pipeline.
"""

import numpy as np
import pytest

from oracle import nrx_oracle as orc
from oracle import slotgen_oracle as so
from slotgen_cases import case_names, load_case

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def _tiny(**kw):
    from paper_2409_02912_b200.config import SlotConfig
    d = dict(num_subcarriers=4, num_symbols=4, pilot_symbols=(1,), num_ues=1, comb_size=1, bs_antennas=1,
             ue_antennas=1)
    d.update(kw)
    return SlotConfig(**d)


@pytest.mark.parametrize("name", case_names())
def test_reference_stream_matches_reference_generator(name):
    torch = _torch()
    from paper_2409_02912_b200.slotgen import GpuSlotSource
    c = load_case(name)
    src = GpuSlotSource(c.cfg, c.profiles)
    b = src.generate(c.n, c.orders, c.n0, variates=c.variates(), y_dtype=torch.complex128,
                     pilots_dtype=torch.complex128, with_h_eff=True, h_dtype=torch.complex128)
    torch.cuda.synchronize()
    y, h = b.y.cpu().numpy(), b.h_eff.cpu().numpy()
    np.testing.assert_allclose(y, c.a["y"], rtol=0, atol=1e-12 * np.abs(c.a["y"]).max())
    np.testing.assert_allclose(h, c.a["h_eff"], rtol=0, atol=1e-12 * np.abs(c.a["h_eff"]).max())
    np.testing.assert_array_equal(b.labels.cpu().numpy(), c.a["labels"])
    np.testing.assert_array_equal(b.pilots.cpu().numpy(), c.a["pilots"])
    # complex64 outputs are the float32 rounding of the same values
    b32 = src.generate(c.n, c.orders, c.n0, variates=c.variates())
    np.testing.assert_allclose(b32.y.cpu().numpy(), y.astype(np.complex64), rtol=0,
                               atol=1e-6 * np.abs(y).max())


def test_c2_reference_stream_vs_oracle():
    torch = _torch()
    from paper_2409_02912_b200.config import SlotConfig
    from paper_2409_02912_b200.slotgen import GpuSlotSource, doubletdl, reference_variates
    cfg = SlotConfig(num_subcarriers=3276, num_ues=2)
    prof = doubletdl()
    v = reference_variates(cfg, prof, (4, 4), [0], seed=0)
    b = GpuSlotSource(cfg, prof).generate(1, (4, 4), 0.1, variates=v, y_dtype=torch.complex128,
                                          with_h_eff=True, h_dtype=torch.complex128)
    y, h = so.synth_slot(cfg, prof, (4, 4), 0.1, v["angles"][0], v["phases"][0], v["labels"][0], v["noise"][0],
                         v["pilots"][0])
    np.testing.assert_allclose(b.y.cpu().numpy()[0], y, rtol=0, atol=1e-12 * np.abs(y).max())
    np.testing.assert_allclose(b.h_eff.cpu().numpy()[0], h, rtol=0, atol=1e-12 * np.abs(h).max())


def test_device_stream_deterministic_and_batch_invariant():
    torch = _torch()
    from paper_2409_02912_b200.config import SlotConfig
    from paper_2409_02912_b200.slotgen import GpuSlotSource
    cfg = SlotConfig(num_subcarriers=96, num_ues=2)
    src = GpuSlotSource(cfg)
    a = src.generate(8, (4, 6), 0.1, seed=5)
    ya, la, pa = a.y.clone(), a.labels.clone(), a.pilots.clone()
    b = src.generate(4, (4, 6), 0.1, seed=5, first_slot=4)
    assert torch.equal(ya[4:], b.y) and torch.equal(la[4:], b.labels) and torch.equal(pa[4:], b.pilots)
    c = src.generate(8, (4, 6), 0.1, seed=5)
    assert torch.equal(ya, c.y)
    d = src.generate(8, (4, 6), 0.1, seed=6)
    assert not torch.equal(ya, d.y)
    assert not torch.equal(ya[0], ya[1])
    # labels only on data REs, within the order; pilots QPSK unit modulus on the comb
    lab = la.cpu().numpy()
    assert not lab[:, :, :, list(cfg.pilot_symbols)].any()
    assert lab[:, 0].max() < 16 and lab[:, 1].max() < 64
    p = pa.cpu().numpy()
    np.testing.assert_allclose(np.abs(p), 1.0, rtol=1e-6)
    # complex64 outputs take the float32 synthesis; complex128 the float64 one,
    # on the same Philox variates
    e = src.generate(8, (4, 6), 0.1, seed=5, y_dtype=torch.complex128)
    y64 = e.y.cpu().numpy()
    assert torch.equal(e.labels, la)
    np.testing.assert_allclose(ya.cpu().numpy(), y64, rtol=0, atol=2e-4 * np.abs(y64).max())


def test_zero_doppler_is_time_constant():
    torch = _torch()
    from paper_2409_02912_b200.slotgen import GpuSlotSource, tdl_b
    cfg = _tiny(num_symbols=14)
    b = GpuSlotSource(cfg, [tdl_b(doppler_hz=0.0)]).generate(4, (4,), 0.0, with_h_eff=True,
                                                              h_dtype=torch.complex128)
    h = b.h_eff.cpu().numpy()
    assert np.max(np.abs(h - h[:, :, :, :1])) < 1e-12


def test_per_tap_power_monte_carlo():
    """Tap amplitudes recovered by least squares from the frequency response
    have the profile's powers (test_channel.py:47-62)."""
    torch = _torch()
    from paper_2409_02912_b200.slotgen import GpuSlotSource, tdl_b
    cfg = _tiny(num_subcarriers=24, num_symbols=1, pilot_symbols=(0,))
    prof = tdl_b(doppler_hz=0.0)
    b = GpuSlotSource(cfg, [prof]).generate(10_000, (2,), 0.0, seed=1, with_h_eff=True,
                                            h_dtype=torch.complex128)
    h = b.h_eff.cpu().numpy()[:, 0, :, 0, 0]                       # (draws, S)
    phase = np.exp(-2j * np.pi * cfg.subcarrier_spacing_hz * np.outer(prof.delays_s, np.arange(24)))
    amps = h @ np.linalg.pinv(phase)
    np.testing.assert_allclose(np.mean(np.abs(amps) ** 2, axis=0), prof.powers, rtol=0.05)


def test_doppler_autocorrelation_matches_bessel():
    torch = _torch()
    from scipy.special import j0
    from paper_2409_02912_b200.slotgen import GpuSlotSource, TdlProfile
    cfg = _tiny(num_subcarriers=1, num_symbols=14, pilot_symbols=(0,))
    fd = 400.0
    flat = TdlProfile("flat", np.array([0.0]), np.array([1.0]), fd, 0.0)
    b = GpuSlotSource(cfg, [flat]).generate(10_000, (2,), 0.0, seed=2, with_h_eff=True, h_dtype=torch.complex128)
    g = b.h_eff.cpu().numpy()[:, 0, 0, :, 0]                       # (draws, T)
    T = cfg.num_symbols
    acc = np.array([np.mean(np.mean(g[:, : T - lag].conj() * g[:, lag:], axis=1)) for lag in range(T)])
    tsym = (1.0 + cfg.cp_fraction) / cfg.subcarrier_spacing_hz
    expected = j0(2 * np.pi * fd * np.arange(T) * tsym)
    assert np.max(np.abs(acc.real - expected)) <= 0.05
    assert np.max(np.abs(acc.imag)) <= 0.05


@pytest.mark.parametrize("name", ["tdl_a", "tdl_b", "tdl_c", "tdl_d"])
def test_energy_normalization_all_profiles(name):
    torch = _torch()
    from paper_2409_02912_b200.slotgen import PROFILES, GpuSlotSource
    cfg = _tiny(num_subcarriers=4, num_symbols=2, pilot_symbols=(0,))
    b = GpuSlotSource(cfg, [PROFILES[name]()]).generate(10_000, (2,), 0.0, seed=3, with_h_eff=True,
                                                        h_dtype=torch.complex128)
    assert abs(float(np.mean(np.abs(b.h_eff.cpu().numpy()) ** 2)) - 1.0) < 0.05


def test_noise_power_and_transmit_symbols():
    """y - sum_u h_eff_u x_u is the noise: zero mean, power n0 split evenly
    between re and im (test_channel.py:152-165); x rebuilt on the host from
    the labels and pilots the generator reports."""
    torch = _torch()
    from paper_2409_02912_b200.config import SlotConfig
    from paper_2409_02912_b200.slotgen import GpuSlotSource
    cfg = SlotConfig(num_subcarriers=240, num_ues=2)
    n0 = 0.37
    b = GpuSlotSource(cfg).generate(8, (4, 6), n0, seed=7, y_dtype=torch.complex128, with_h_eff=True,
                                    h_dtype=torch.complex128, pilots_dtype=torch.complex128)
    y, h = b.y.cpu().numpy(), b.h_eff.cpu().numpy()
    lab, pil = b.labels.cpu().numpy(), b.pilots.cpu().numpy()
    x = np.stack([np.stack([so.transmit_grid(cfg, u, m, lab[i, u], pil[i, u]) for u, m in enumerate((4, 6))])
                  for i in range(8)])                                # (N, U, S, T)
    z = y - np.einsum("nustb,nust->nstb", h, x)
    assert abs(np.mean(np.abs(z) ** 2) - n0) / n0 < 0.03
    assert abs(np.mean(z.real ** 2) - n0 / 2) / n0 < 0.03
    assert abs(np.mean(z)) < 0.01
    # average data-symbol energy is 1 (test_slot.py:104-111)
    data = x[:, :, cfg.data_mask]
    assert abs(np.mean(np.abs(data) ** 2) - 1.0) < 0.02
    # a noiseless batch has zero residual
    b0 = GpuSlotSource(cfg).generate(2, (4, 6), 0.0, seed=7, y_dtype=torch.complex128, with_h_eff=True,
                                     h_dtype=torch.complex128)
    x0 = np.stack([np.stack([so.transmit_grid(cfg, u, m, b0.labels.cpu().numpy()[i, u], b0.pilots.cpu().numpy()[i, u])
                             for u, m in enumerate((4, 6))]) for i in range(2)])
    z0 = b0.y.cpu().numpy() - np.einsum("nustb,nust->nstb", b0.h_eff.cpu().numpy(), x0)
    assert np.abs(z0).max() < 1e-5                 # pilots were stored complex64 -> float32 rounding


def test_count_bit_errors_matches_numpy():
    torch = _torch()
    from paper_2409_02912_b200.config import SlotConfig
    from paper_2409_02912_b200.slotgen import count_bit_errors
    cfg = SlotConfig(num_subcarriers=120, num_ues=2)
    rng = np.random.default_rng(0)
    N, U, S, T, W = 5, 2, 120, 14, 6
    orders = np.array([[2, 6], [4, 4], [6, 2], [2, 2], [6, 6]], dtype=np.int32)
    llr = rng.standard_normal((N, U, S, T, W)).astype(np.float32)
    llr[0, 0] = np.abs(llr[0, 0])                  # one stream with every hard bit = 1
    lab = np.zeros((N, U, S, T), np.uint8)
    for n in range(N):
        for u in range(U):
            lab[n, u][cfg.data_mask] = rng.integers(0, 2 ** orders[n, u], size=cfg.num_data_res)
    want = np.zeros((N, U), np.int64)
    for n in range(N):
        for u in range(U):
            m = orders[n, u]
            bits = (lab[n, u][cfg.data_mask][:, None].astype(np.int64) >> np.arange(m - 1, -1, -1)) & 1
            want[n, u] = np.sum((llr[n, u][cfg.data_mask][:, :m] > 0) != bits)
    d = lambda a: torch.from_numpy(a).cuda()
    got = count_bit_errors(cfg, d(llr), d(lab), d(orders.reshape(-1)))
    np.testing.assert_array_equal(got.cpu().numpy().reshape(N, U), want)
    got2 = count_bit_errors(cfg, d(llr), d(lab), d(orders.reshape(-1)), out=got)   # accumulates
    np.testing.assert_array_equal(got2.cpu().numpy().reshape(N, U), 2 * want)


def _desk():
    import os
    from paper_2409_02912_b200.config import checkpoint_load, default_mcs_table
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "desk_d16_it2.nrxw")
    config, w = checkpoint_load(path)
    return config, w, default_mcs_table()


def test_gpu_pipeline_counts_equal_host_count_on_reference_stream():
    """Reference-stream slots -> GPU receiver -> GPU counter equals the host
    count of the same LLRs against the reference recipe's bits, and the
    oracle receiver on the same slots has the same BER within its band."""
    torch = _torch()
    from paper_2409_02912_b200.config import SlotConfig
    from paper_2409_02912_b200.engine import NrxEngine
    from paper_2409_02912_b200.nrx import noise_features
    from paper_2409_02912_b200.slotgen import GpuSlotSource, count_bit_errors, doubletdl, labels_to_bits, \
        reference_variates
    config, w, table = _desk()
    cfg = SlotConfig(num_subcarriers=96, num_ues=2)
    n, n0 = 16, 0.1
    v = reference_variates(cfg, doubletdl(), (4, 4), range(n), seed=21)
    b = GpuSlotSource(cfg).generate(n, (4, 4), n0, variates=v, y_dtype=torch.complex128,
                                    pilots_dtype=torch.complex128)
    eng = NrxEngine(config, w, precision="fp32")
    llr = torch.empty((n, 2, 96, 14, config.m_max), dtype=torch.float32, device="cuda")
    chest = torch.empty((n, 2, 96, 14, 4), dtype=torch.complex64, device="cuda")
    eng.forward_device(cfg, b.y, b.pilots, torch.from_numpy(noise_features(n0, n)).cuda(), b.mod_order,
                       config.num_iterations, llr, chest)
    errs = count_bit_errors(cfg, llr, b.labels, b.mod_order).cpu().numpy().reshape(n, 2)
    l = llr.cpu().numpy()
    s_idx, t_idx = np.nonzero(cfg.data_mask)
    bits = labels_to_bits(v["labels"], cfg, (4, 4))
    for u in range(2):
        host = ((l[:, u, s_idx, t_idx, :4] > 0) != bits[u]).reshape(n, -1).sum(axis=1)
        np.testing.assert_array_equal(errs[:, u], host)
    ber = errs.sum() / (n * 2 * cfg.num_data_res * 4)
    assert 0.01 < ber < 0.45
    # oracle receiver on the very same (reference) grids
    from paper_2409_02912_b200.config import PilotBook
    y = b.y.cpu().numpy()
    books = []
    for i in range(n):
        vals = np.zeros((2, 96, 14), complex)
        for u in range(2):
            sc = np.arange(u % 2, 96, 2)
            vals[u][np.ix_(sc, list(cfg.pilot_symbols))] = v["pilots"][i, u, :sc.size]
        books.append(PilotBook(vals, cfg))
    ref, _ = orc.nrx_forward(y, books, cfg, (table[14], table[14]), w, config, n0)
    ref_err = sum(((ref[u][:, s_idx, t_idx] > 0) != bits[u]).sum() for u in range(2))
    assert abs(int(ref_err) - int(errs.sum())) <= max(3, 0.002 * errs.sum())


def test_evaluate_uncoded_is_world_size_invariant():
    from paper_2409_02912_b200.config import SlotConfig
    from paper_2409_02912_b200.engine import NrxEngine
    from paper_2409_02912_b200.slotgen import GpuSlotSource, evaluate_uncoded
    config, w, table = _desk()
    cfg = SlotConfig(num_subcarriers=96, num_ues=2)
    src = GpuSlotSource(cfg)
    eng = NrxEngine(config, w, precision="fp16")
    mcs = (table[14], table[14])
    full = evaluate_uncoded(eng, src, mcs, [5.0, 15.0], n_slots=40, batch=16, seed=3)
    # two "ranks" of a world of 2, combined by summing their counters
    parts = [evaluate_uncoded(eng, src, mcs, [5.0, 15.0], n_slots=40, batch=7, seed=3, rank=r, world=2)
             for r in range(2)]
    for k in range(2):
        a, b0, b1 = full[k], parts[0][k], parts[1][k]
        assert (a.blocks, a.block_errors, a.bit_errors, a.bits) == (
            b0.blocks + b1.blocks, b0.block_errors + b1.block_errors, b0.bit_errors + b1.bit_errors,
            b0.bits + b1.bits)
    assert full[0].blocks == 80 and full[0].bits == 40 * cfg.num_data_res * 8
    assert full[0].ber > full[1].ber > 0.0          # higher SNR, fewer errors
