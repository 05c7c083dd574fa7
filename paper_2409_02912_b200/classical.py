"""Classical baseline receivers on the GPU: the
reference's "ls_lmmse" ReceiverBank entry — comb LS estimate, per-RE LMMSE
equalisation, exact APP demapping, clipping — and its "perfect_kbest"
entry — K-Best detection with max-log LLRs on the true channel — as one
kernel each (``nrx_ls_lmmse``, ``nrx_kbest``, include/nrx_classical.h).

Reference interfaces mirrored (file:line under /root/reference/pkg/src/nrxsim):
  ls_estimate / lmmse_equalize / app_demap     classical.py:40-174
  kbest_detect                                 classical.py:195-261
  ReceiverBank.run("ls_lmmse" / "perfect_kbest")  evaluation.py:79-111, 130-140

``GpuLsLmmse`` has the ``forward_device`` signature of ``NrxEngine``, so the
GPU Monte-Carlo loops (slotgen.evaluate_uncoded, ldpc.evaluate_coded) run it
as the comparison receiver on exactly the same slots.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .slotgen import qam_table

LLR_CLIP = 20.0   # classical.py:24 / evaluation.py:27


@dataclass(frozen=True)
class _RxConfig:
    """The fields the GPU Monte-Carlo loops read from a receiver's config."""
    m_max: int
    num_iterations: int = 1
    variant: str = "single"


class GpuLsLmmse:
    """LS + LMMSE + exact APP demap on the device (float64 arithmetic)."""

    needs_n0 = True

    def __init__(self, bs_antennas: int = 4, m_max: int = 8, clip: float = LLR_CLIP, device=None):
        from .engine import _require_cuda
        torch = _require_cuda()
        self.lib = _lib.load()
        self.bs_antennas = int(bs_antennas)
        self.clip = float(clip)
        self.config = _RxConfig(m_max=int(m_max))
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._qam = np.ascontiguousarray(qam_table())

    def forward_device(self, cfg, y, pilots, noise_feat, mod_order, num_iterations, llr, chest=None,
                       workspace=None, stream=None, n0=None):
        """y (N,S,T,B), pilots (P,U,F,K), mod_order (N*U,) int32, n0 (N,)
        float64 device tensors -> llr (N,U,S,T,W) float32 (chest untouched)."""
        import torch
        if n0 is None:
            raise ValueError("the LMMSE receiver needs the linear noise power n0 per slot")
        n = y.shape[0]
        n0 = n0.to(device=self.device, dtype=torch.float64).reshape(-1).contiguous()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        s = _lib.slot_desc(cfg)
        rc = self.lib.nrx_ls_lmmse(ctypes.byref(s), self.bs_antennas, n, y.data_ptr(),
                                   int(y.dtype == torch.complex128), pilots.data_ptr(),
                                   int(pilots.dtype == torch.complex128), pilots.shape[0], n0.data_ptr(),
                                   mod_order.data_ptr(), self._qam.ctypes.data, self.clip, llr.data_ptr(),
                                   llr.shape[-1], st.cuda_stream)
        _lib.check(rc, "nrx_ls_lmmse")


class GpuKBest:
    """K-Best detection with max-log LLRs on the true effective channel
    (the reference's "perfect_kbest", evaluation.py:139-140); float64."""

    needs_n0 = True
    needs_h_eff = True

    def __init__(self, bs_antennas: int = 4, m_max: int = 8, k: int = 16, clip: float = LLR_CLIP, device=None,
                 reference_pairing: bool = True):
        """reference_pairing=True reproduces the reference bit for bit, whose
        interference term pairs R[level, level+1:] with the decided symbols in
        decision (descending-stream) order (classical.py:220-221) — correct
        for U <= 2 only; False uses the true R[level, j] x_j for any U."""
        from .engine import _require_cuda
        torch = _require_cuda()
        self.lib = _lib.load()
        self.bs_antennas, self.k, self.clip = int(bs_antennas), int(k), float(clip)
        self.reference_pairing = bool(reference_pairing)
        self.config = _RxConfig(m_max=int(m_max))
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._qam = np.ascontiguousarray(qam_table())

    def forward_device(self, cfg, y, pilots, noise_feat, mod_order, num_iterations, llr, chest=None,
                       workspace=None, stream=None, n0=None, h_eff=None):
        """y (N,S,T,B), h_eff (N,U,S,T,B), n0 (N,) float64, mod_order (N*U,)
        device tensors -> llr (N,U,S,T,W) float32 on the data REs (zeros elsewhere)."""
        import torch
        if n0 is None or h_eff is None:
            raise ValueError("K-Best needs the noise power n0 and the channel h_eff per slot")
        n0 = n0.to(device=self.device, dtype=torch.float64).reshape(-1).contiguous()
        h_eff = h_eff.contiguous()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        s = _lib.slot_desc(cfg)
        rc = self.lib.nrx_kbest(ctypes.byref(s), self.bs_antennas, y.shape[0], y.data_ptr(),
                                int(y.dtype == torch.complex128), h_eff.data_ptr(),
                                int(h_eff.dtype == torch.complex128), n0.data_ptr(), mod_order.data_ptr(),
                                self._qam.ctypes.data, self.k, int(self.reference_pairing), self.clip,
                                llr.data_ptr(), llr.shape[-1],
                                st.cuda_stream)
        _lib.check(rc, "nrx_kbest")


def kbest_llrs(y, h_eff, cfg, mcs_per_ue, n0, k: int = 16, clip: float = LLR_CLIP, device=None,
               reference_pairing: bool = True):
    """numpy drop-in for ReceiverBank.run("perfect_kbest"): y (N,S,T,B),
    true h_eff (N,U,S,T,B) -> list per UE of (N,S,T,m_u) float32 grids."""
    import torch
    y = np.asarray(y)
    n = y.shape[0]
    orders = [m.modulation_order for m in mcs_per_ue]
    rx = GpuKBest(cfg.bs_antennas, max(orders), k, clip, device, reference_pairing)
    dev = rx.device
    yt = torch.from_numpy(np.ascontiguousarray(y.astype(np.complex128))).to(dev)
    ht = torch.from_numpy(np.ascontiguousarray(np.asarray(h_eff).astype(np.complex128))).to(dev)
    n0_t = torch.from_numpy(np.broadcast_to(np.asarray(n0, dtype=np.float64).reshape(-1), (n,)).copy()).to(dev)
    mods = torch.tensor(orders * n, dtype=torch.int32, device=dev)
    llr = torch.empty((n, cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, max(orders)), dtype=torch.float32,
                      device=dev)
    rx.forward_device(cfg, yt, None, None, mods, 1, llr, n0=n0_t, h_eff=ht)
    out = llr.cpu().numpy()
    return [out[:, u, ..., :m] for u, m in enumerate(orders)]


def ls_lmmse_llrs(y, books, cfg, mcs_per_ue, n0, clip: float = LLR_CLIP, device=None):
    """numpy in/out drop-in for ReceiverBank.run("ls_lmmse") (evaluation.py:130-135):
    y (N,S,T,B), per-slot books (or one book), scalar or (N,) n0 -> list per UE
    of (N,S,T,m_u) float32 LLR grids clipped to +-clip."""
    import torch
    from .nrx import stack_pilots
    y = np.asarray(y)
    n = y.shape[0]
    orders = [m.modulation_order for m in mcs_per_ue]
    rx = GpuLsLmmse(cfg.bs_antennas, max(orders), clip, device)
    dev = rx.device
    pil = torch.from_numpy(np.ascontiguousarray(stack_pilots(books, n, cfg))).to(dev)
    yt = torch.from_numpy(np.ascontiguousarray(y.astype(np.complex128))).to(dev)
    n0_t = torch.from_numpy(np.broadcast_to(np.asarray(n0, dtype=np.float64).reshape(-1), (n,)).copy()).to(dev)
    mods = torch.tensor(orders * n, dtype=torch.int32, device=dev)
    llr = torch.empty((n, cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, max(orders)), dtype=torch.float32,
                      device=dev)
    rx.forward_device(cfg, yt, pil.to(torch.complex128), None, mods, 1, llr, n0=n0_t)
    out = llr.cpu().numpy()
    return [out[:, u, ..., :m] for u, m in enumerate(orders)]


__all__ = ["GpuLsLmmse", "GpuKBest", "ls_lmmse_llrs", "kbest_llrs", "LLR_CLIP"]


# ---------------------------------------------------------------------------
# covariance-based LMMSE channel estimation + K-Best ("lmmse_kbest")
# ---------------------------------------------------------------------------

VAR_FLOOR = 1e-12   # classical.py:25


@dataclass(frozen=True)
class CovarianceModel:
    """Sample frequency / time covariance of the effective per-stream channel
    (channel.CovarianceModel, channel.py:223-236), as device tensors."""
    freq: object     # (S, S) complex128
    time: object     # (T, T) complex128
    num_samples: int


def covariance_variates(cfg, profiles, num_samples: int, seed: int = 0, num_sinusoids: int = 32) -> dict:
    """The reference's draws for estimate_covariance (channel.py:239-268):
    sample i of UE u uses default_rng((seed, 0xC0F, i, u)) for the
    angles-then-phases of TdlChannelSource.sample.  Fed to the GPU slot
    generator they reproduce the reference's channel draws."""
    U, B, Nu = cfg.num_ues, cfg.bs_antennas, cfg.ue_antennas
    L = max(p.delays_s.size for p in profiles[:U])
    ang = np.zeros((num_samples, U, B, Nu, L, num_sinusoids))
    ph = np.zeros_like(ang)
    for i in range(num_samples):
        for u in range(U):
            r = np.random.default_rng((seed, 0xC0F, i, u))
            nt = profiles[u].delays_s.size
            ang[i, u, :, :, :nt] = r.uniform(0.0, 2.0 * np.pi, size=(B, Nu, nt, num_sinusoids))
            ph[i, u, :, :, :nt] = r.uniform(0.0, 2.0 * np.pi, size=(B, Nu, nt, num_sinusoids))
    return dict(angles=ang, phases=ph)


def estimate_covariance(source, num_samples: int, seed: int = 0, reference_stream: bool = False,
                        batch: int = 64) -> CovarianceModel:
    """GPU estimate_covariance: channels from the GPU slot generator (device
    Philox draws, or the reference's own draws with reference_stream=True),
    then R_f = sum h h^H over (draw, UE, symbol, antenna) and R_t likewise,
    Hermitian-symmetrised (channel.py:239-268)."""
    import torch
    if num_samples < 100:
        raise ValueError(f"need at least 100 samples for covariance estimation, got {num_samples}")
    cfg, dev = source.cfg, source.device
    U, S, T, B = cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, cfg.bs_antennas
    r_f = torch.zeros((S, S), dtype=torch.complex128, device=dev)
    r_t = torch.zeros((T, T), dtype=torch.complex128, device=dev)
    variates = covariance_variates(cfg, source.profiles, num_samples, seed, source.num_sinusoids) \
        if reference_stream else None
    for start in range(0, num_samples, batch):
        nb = min(batch, num_samples - start)
        v = None if variates is None else {k: a[start:start + nb] for k, a in variates.items()}
        sb = source.generate(nb, [2] * U, 0.0, seed=(int(seed) << 8) ^ 0xC0F, first_slot=start, variates=v,
                             with_h_eff=True, h_dtype=torch.complex128, y_dtype=torch.complex128)
        h = sb.h_eff                                                  # (n, U, S, T, B)
        hf = h.permute(2, 0, 1, 3, 4).reshape(S, -1)
        ht = h.permute(3, 0, 1, 2, 4).reshape(T, -1)
        r_f += hf @ hf.conj().T
        r_t += ht @ ht.conj().T
    r_f /= num_samples * U * T * B
    r_t /= num_samples * U * S * B
    return CovarianceModel(0.5 * (r_f + r_f.conj().T), 0.5 * (r_t + r_t.conj().T), num_samples)


def lmmse_weights(cfg, cov: CovarianceModel, n0: float):
    """Wiener filters of lmmse_estimate (classical.py:81-103): per UE the
    frequency filter W_f (S, F_u) from its comb and the time filter W_t (T, K)."""
    import torch
    n0e = max(float(n0), VAR_FLOOR)
    ps = torch.tensor(list(cfg.pilot_symbols), device=cov.time.device)
    eye = lambda k: torch.eye(k, dtype=torch.complex128, device=cov.time.device)
    r_t = cov.time
    w_t = torch.linalg.solve(r_t[ps][:, ps] + n0e * eye(ps.numel()), r_t[:, ps].conj().T).conj().T
    w_f = []
    for u in range(cfg.num_ues):
        sc = torch.arange(u % cfg.comb_size, cfg.num_subcarriers, cfg.comb_size, device=cov.freq.device)
        r_f = cov.freq
        w_f.append(torch.linalg.solve(r_f[sc][:, sc] + n0e * eye(sc.numel()), r_f[:, sc].conj().T).conj().T)
    return w_f, w_t


def lmmse_estimate(cfg, y, pilots, weights):
    """Device lmmse_estimate: comb LS values, then W_f along frequency and
    W_t along time.  y (N,S,T,B), pilots (P,U,F,K) comb values -> h (N,U,S,T,B)."""
    import torch
    w_f, w_t = weights
    y = y.to(torch.complex128)
    pil = pilots.to(torch.complex128)
    n = y.shape[0]
    ps = list(cfg.pilot_symbols)
    out = torch.empty((n, cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, cfg.bs_antennas),
                      dtype=torch.complex128, device=y.device)
    for u in range(cfg.num_ues):
        sc = torch.arange(u % cfg.comb_size, cfg.num_subcarriers, cfg.comb_size, device=y.device)
        p = pil[:, u, :sc.numel()].expand(n, -1, -1)                         # (N, F, K)
        raw = y[:, sc][:, :, ps] * (p.conj() / p.abs() ** 2)[..., None]      # (N, F, K, B)
        est_f = torch.einsum("sf,nfkb->nskb", w_f[u], raw)
        out[:, u] = torch.einsum("tk,nskb->nstb", w_t, est_f)
    return out


class GpuLmmseKBest:
    """The reference's "lmmse_kbest" receiver (evaluation.py:136-138): LMMSE
    channel estimate from sample covariances, then K-Best on the estimate."""

    needs_n0 = True

    def __init__(self, cov: CovarianceModel, bs_antennas: int = 4, m_max: int = 8, k: int = 16,
                 clip: float = LLR_CLIP, device=None, reference_pairing: bool = True):
        self.cov = cov
        self.kb = GpuKBest(bs_antennas, m_max, k, clip, device, reference_pairing)
        self.config = self.kb.config
        self.device = self.kb.device
        self._w = {}

    def forward_device(self, cfg, y, pilots, noise_feat, mod_order, num_iterations, llr, chest=None,
                       workspace=None, stream=None, n0=None):
        if n0 is None:
            raise ValueError("the LMMSE estimator needs the noise power n0")
        n0s = n0.reshape(-1).cpu().numpy()
        if not np.all(n0s == n0s[0]):
            raise ValueError("one n0 per call (the Wiener filters depend on it)")
        key = float(n0s[0])
        if key not in self._w:
            self._w = {key: lmmse_weights(cfg, self.cov, key)}
        h = lmmse_estimate(cfg, y, pilots, self._w[key])
        self.kb.forward_device(cfg, y, pilots, noise_feat, mod_order, num_iterations, llr, chest, workspace, stream,
                               n0=n0, h_eff=h)


__all__ += ["CovarianceModel", "covariance_variates", "estimate_covariance", "lmmse_weights", "lmmse_estimate",
            "GpuLmmseKBest"]
