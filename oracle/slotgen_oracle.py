"""CPU oracle of the synthetic-slot generator (test infrastructure only).

Restates, in float64 numpy, what the reference's transmitter + channel do to
one uncoded slot once the random variates are fixed, so the GPU generator
(csrc/k_slotgen.cu) can be checked on identical variates.  Only tests/ may
import this module.  Pinned against the reference itself by
tests/golden/make_golden_slotgen.py (fixtures slotgen_*.npz) in
tests/test_slotgen_cpu.py.

Reference (file:line under /root/reference/pkg/src/nrxsim):
  jakes_gains      sample_tdl channel.py:139-145 (sum of sinusoids per tap)
  freq_response    cir_to_freq channel.py:113-124 and the axis move of
                   sample_tdl channel.py:146-148
  transmit_grid    generate_pilots slot.py:130-139 (values given), map_bits
                   constellation.py:44-50 on the data REs slot.py:106-109
  received_grid    beamform slot.py:231-233 + apply_channel channel.py:153-167
  effective        ChannelRealization.effective channel.py:101-104
"""

from __future__ import annotations

import numpy as np


def gray_points(order: int) -> np.ndarray:
    """Unit-energy Gray square QAM, point i labelled by the big-endian bits
    of i; even label positions steer the real axis (constellation.py:58-82)."""
    i = np.arange(2 ** order)
    lab = (i[:, None] >> np.arange(order - 1, -1, -1)) & 1

    def amp(bits):
        n = bits.shape[1]
        a = 1.0 - 2.0 * bits[:, n - 1].astype(np.float64)
        for lev in range(1, n):
            a = (1.0 - 2.0 * bits[:, n - 1 - lev].astype(np.float64)) * (2.0 ** lev - a)
        return a

    pts = amp(lab[:, 0::2]) + 1j * amp(lab[:, 1::2])
    return pts / np.sqrt(np.mean(np.abs(pts) ** 2))


def jakes_gains(angles, phases, powers, doppler_hz, num_symbols, symbol_duration_s):
    """angles/phases (B, Nu, L, NS) -> tap gains (B, Nu, L, T): for each tap
    sum_k exp(j (2 pi fD cos(angle_k) t Tsym + phase_k)) / sqrt(NS) * sqrt(p)."""
    ns = angles.shape[-1]
    t_sym = np.arange(num_symbols) * symbol_duration_s
    omega = 2.0 * np.pi * doppler_hz * np.cos(angles)
    arg = omega[..., None] * t_sym + phases[..., None]            # (B, Nu, L, NS, T)
    g = np.exp(1j * arg).sum(axis=3) / np.sqrt(ns)
    return g * np.sqrt(powers)[:, None]


def freq_response(gains, delays_s, scs_hz, num_subcarriers):
    """(B, Nu, L, T) tap gains -> (S, T, B, Nu) per-RE MIMO coefficients,
    H[s] = sum_l g_l exp(-j 2 pi s df tau_l)."""
    s = np.arange(num_subcarriers)
    ph = np.exp(-2j * np.pi * scs_hz * np.outer(delays_s, s))     # (L, S)
    h = np.einsum("bnlt,ls->bnts", gains, ph)                     # (B, Nu, T, S)
    return np.transpose(h, (3, 2, 0, 1))


def transmit_grid(cfg, ue, order, labels_ue, pilot_values_ue):
    """Stream symbols (S, T) of one UE: pilots on its comb at the pilot
    symbols, QAM points of the label indices on the data REs, zero elsewhere.
    labels_ue (S, T) label index; pilot_values_ue (F, K) comb pilot values."""
    S, T = cfg.num_subcarriers, cfg.num_symbols
    x = np.zeros((S, T), dtype=np.complex128)
    sc = np.arange(ue % cfg.comb_size, S, cfg.comb_size)
    x[np.ix_(sc, list(cfg.pilot_symbols))] = pilot_values_ue[: sc.size]
    data = np.ones((S, T), dtype=bool)
    data[:, list(cfg.pilot_symbols)] = False
    x[data] = gray_points(order)[labels_ue[data].astype(np.int64)]
    return x


def received_grid(h, x, beams, n0, noise_pairs):
    """h (U, S, T, B, Nu), x (U, S, T) stream symbols, beams (U, Nu),
    noise_pairs (S, T, B) complex unit normals -> y (S, T, B)."""
    tx = x[..., None] * beams[:, None, None, :]                   # (U, S, T, Nu)
    y = np.einsum("ustbn,ustn->stb", h, tx)
    if n0 > 0:
        y = y + np.sqrt(n0 / 2.0) * noise_pairs
    return y


def effective(h, beams):
    return np.einsum("ustbn,un->ustb", h, beams)


def synth_slot(cfg, profiles, orders, n0, angles, phases, labels, noise, pilots):
    """One slot from its variates (layouts of nrx_slot_variates without the
    slot axis) -> (y (S,T,B), h_eff (U,S,T,B))."""
    U, S, T = cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols
    tsym = (1.0 + cfg.cp_fraction) / cfg.subcarrier_spacing_hz
    beams = np.asarray(cfg.beam_matrix)
    h = np.zeros((U, S, T, cfg.bs_antennas, cfg.ue_antennas), dtype=np.complex128)
    x = np.zeros((U, S, T), dtype=np.complex128)
    for u in range(U):
        p = profiles[u]
        nt = p.delays_s.size
        g = jakes_gains(angles[u, :, :, :nt], phases[u, :, :, :nt], p.powers, p.doppler_hz, T, tsym)
        h[u] = freq_response(g, p.delays_s, cfg.subcarrier_spacing_hz, S)
        x[u] = transmit_grid(cfg, u, orders[u], labels[u], pilots[u])
    return received_grid(h, x, beams, n0, noise), effective(h, beams)
