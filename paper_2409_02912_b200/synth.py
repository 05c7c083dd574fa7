"""Synthetic uplink slots for benchmarks and tests (host, numpy).

Not the reference's TDL/LDPC transmitter (SURVEY.md finding 5: LDPC does
not scale to 273 PRB and is transparent to the receiver): random coded bits
are Gray-QAM mapped onto the data REs, the reference's seeded QPSK pilots
sit on each UE's comb, and each UE sees an effective (post-beamforming)
frequency-selective Rayleigh channel with a per-tap Doppler rotation,
plus complex white noise of power n0 (SNR = 1/n0, channel.py:10-11).
"""

from __future__ import annotations

import numpy as np

from .config import PilotBook, generate_pilots


def gray_qam(order: int) -> np.ndarray:
    """Unit-energy square QAM whose point i carries the big-endian label of
    i: even label positions steer the real axis, odd the imaginary one,
    each axis amplitude built by the quadrant recursion with bit 0 on the
    positive half-axis (constellation.py:1-11,58-82).  Orders 2/4/6 match
    the reference; 8 (256-QAM) is the labelled extension."""
    if order not in (2, 4, 6, 8):
        raise ValueError(f"unsupported modulation order {order}")
    idx = np.arange(2 ** order)
    labels = (idx[:, None] >> np.arange(order - 1, -1, -1)) & 1

    def axis(bits):
        amp = 1.0 - 2.0 * bits[:, -1]
        for level in range(1, bits.shape[1]):
            amp = (1.0 - 2.0 * bits[:, bits.shape[1] - 1 - level]) * (2.0 ** level - amp)
        return amp

    pts = axis(labels[:, 0::2]) + 1j * axis(labels[:, 1::2])
    return pts / np.sqrt(np.mean(np.abs(pts) ** 2))


def map_bits(bits: np.ndarray, order: int) -> np.ndarray:
    w = 1 << np.arange(order - 1, -1, -1)
    return gray_qam(order)[bits.astype(np.int64) @ w]


def rayleigh_channel(cfg, rng, num_taps: int = 6, delay_spread_s: float = 300e-9,
                     doppler_hz: float = 100.0) -> np.ndarray:
    """(U, S, T, B) effective channel, unit average gain."""
    U, S, T, B = cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, cfg.bs_antennas
    scs = getattr(cfg, "subcarrier_spacing_hz", 30e3)
    cp = getattr(cfg, "cp_fraction", 0.07)
    t_sym = (1.0 + cp) / scs
    delays = np.sort(rng.uniform(0.0, min(4 * delay_spread_s, 0.9 * cp / scs), size=(U, num_taps)), axis=1)
    delays[:, 0] = 0.0
    pw = np.exp(-delays / delay_spread_s)
    pw /= pw.sum(axis=1, keepdims=True)
    g0 = (rng.standard_normal((U, B, num_taps)) + 1j * rng.standard_normal((U, B, num_taps))) / np.sqrt(2)
    g0 *= np.sqrt(pw)[:, None, :]
    fd = doppler_hz * np.cos(rng.uniform(0, 2 * np.pi, size=(U, B, num_taps)))
    rot = np.exp(2j * np.pi * fd[..., None] * (np.arange(T) * t_sym))           # (U,B,L,T)
    phase = np.exp(-2j * np.pi * scs * delays[:, :, None] * np.arange(S))       # (U,L,S)
    return np.einsum("ublt,uls->ustb", g0[..., None] * rot, phase)


def synth_slots(cfg, orders, n_slots: int, n0: float, seed: int = 0, shared_book: bool = False):
    """Returns (y (N,S,T,B) complex128, books list, bits list per UE of
    (N, n_data, m_u) uint8)."""
    s_idx, t_idx = np.nonzero(cfg.data_mask) if hasattr(cfg, "data_mask") else None
    ys, books = [], []
    bits = [[] for _ in orders]
    for i in range(n_slots):
        rng = np.random.default_rng((seed, i, 0x5EED))
        book = generate_pilots(cfg, slot_seed=0 if shared_book else seed * 100003 + i)
        h = rayleigh_channel(cfg, rng)
        y = np.zeros((cfg.num_subcarriers, cfg.num_symbols, cfg.bs_antennas), dtype=np.complex128)
        for u, m in enumerate(orders):
            b = (rng.random((s_idx.size, m)) < 0.5).astype(np.uint8)
            x = np.array(book.values[u])
            x[s_idx, t_idx] = map_bits(b, m)
            y += h[u] * x[..., None]
            bits[u].append(b)
        y += np.sqrt(n0 / 2) * (rng.standard_normal(y.shape) + 1j * rng.standard_normal(y.shape))
        ys.append(y)
        books.append(book if not shared_book else books[0] if books else book)
    return np.stack(ys), books, [np.stack(b) for b in bits]


def random_grid(cfg, n_slots: int, seed: int = 0):
    """Unstructured random received grids + per-slot books (for parity tests)."""
    rng = np.random.default_rng(seed)
    y = rng.standard_normal((n_slots, cfg.num_subcarriers, cfg.num_symbols, cfg.bs_antennas)) \
        + 1j * rng.standard_normal((n_slots, cfg.num_subcarriers, cfg.num_symbols, cfg.bs_antennas))
    books = [generate_pilots(cfg, slot_seed=seed * 7919 + i) for i in range(n_slots)]
    return y, books


__all__ = ["gray_qam", "map_bits", "rayleigh_channel", "synth_slots", "random_grid", "PilotBook"]
