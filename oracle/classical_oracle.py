"""CPU oracle of the classical "ls_lmmse" baseline (test infrastructure only).

numpy restatement of the reference's ls_estimate (classical.py:40-78),
lmmse_equalize (:113-143) and exact app_demap (:150-174) plus the clip of
evaluation.py:79-84, vectorised over slots.  Only tests/ may import this
module.  Pinned to the reference's own outputs by
tests/golden/make_golden_classical.py -> tests/golden/cl_sg_*.npz
(tests/test_classical_cpu.py).
"""

from __future__ import annotations

import numpy as np

VAR_FLOOR = 1e-12


def ls_estimate(cfg, y, pilots):
    """y (N,S,T,B), pilots (N,U,F,K) comb values -> h (N,U,S,T,B)."""
    n, S, T, B = y.shape
    ps = np.asarray(cfg.pilot_symbols)
    t = np.arange(T)
    nearest = np.argmin(np.abs(t[:, None] - ps[None, :]), axis=1)
    out = np.empty((n, cfg.num_ues, S, T, B), dtype=np.complex128)
    for u in range(cfg.num_ues):
        sc = np.arange(u % cfg.comb_size, S, cfg.comb_size)
        p = pilots[:, u, :sc.size]                                     # (N, F, K)
        raw = y[:, sc][:, :, ps] * (p.conj() / np.abs(p) ** 2)[..., None]   # (N, F, K, B)
        s = np.arange(S)
        if sc.size == 1:
            freq = np.broadcast_to(raw[:, :1], (n, S) + raw.shape[2:])
        else:
            step = sc[1] - sc[0]
            j = np.clip((s - sc[0]) // step, 0, sc.size - 2)
            frac = ((s - sc[j]) / step)[None, :, None, None]
            freq = raw[:, j] + frac * (raw[:, j + 1] - raw[:, j])
        out[:, u] = freq[:, :, nearest, :]
    return out


def lmmse_equalize(y, h, n0):
    """y (N,S,T,B), h (N,U,S,T,B) -> z, nvar (N,U,S,T)."""
    hh = np.moveaxis(h, 1, -1)                                        # (N,S,T,B,U)
    u = hh.shape[-1]
    a = np.einsum("...bu,...bv->...uv", hh.conj(), hh) + max(float(n0), 0.0) * np.eye(u)
    rhs = np.einsum("...bu,...b->...u", hh.conj(), y)
    x = np.linalg.solve(a, rhs[..., None])[..., 0]
    a_inv = np.linalg.inv(a)
    mu = np.clip(1.0 - float(n0) * np.einsum("...uu->...u", a_inv).real, VAR_FLOOR, None)
    z = x / mu
    nvar = np.clip((1.0 - mu) / mu, VAR_FLOOR, None)
    return np.moveaxis(z, -1, 1), np.moveaxis(nvar, -1, 1)


def app_demap_exact(z, points, nvar):
    """(...) complex, (2^m,) points, (...) variances -> (..., m) logit LLRs."""
    m = int(np.log2(points.size))
    metric = -np.abs(z[..., None] - points) ** 2 / nvar[..., None]
    labels = (np.arange(points.size)[:, None] >> np.arange(m - 1, -1, -1)) & 1
    out = np.empty(z.shape + (m,))
    for k in range(m):
        one = labels[:, k] == 1

        def lse(v):
            top = v.max(axis=-1, keepdims=True)
            return (top + np.log(np.exp(v - top).sum(axis=-1, keepdims=True)))[..., 0]

        out[..., k] = lse(metric[..., one]) - lse(metric[..., ~one])
    return out


def ls_lmmse_llrs(cfg, y, pilots, n0, orders, points_of, clip=20.0):
    """Per-UE clipped LLR grids (N,S,T,m_u) of the ls_lmmse receiver."""
    z, nvar = lmmse_equalize(y, ls_estimate(cfg, y, pilots), n0)
    return [np.clip(app_demap_exact(z[:, u], points_of(m), nvar[:, u]), -clip, clip) for u, m in enumerate(orders)]
