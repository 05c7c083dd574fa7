"""GPU synthetic uplink slots and uncoded bit-error counting (SURVEY.md §8(f)
row 1: the step immediately upstream of the receiver, and its BER read-out).

The reference builds every Monte-Carlo slot on the host (48.6 ms per 273-PRB
slot), which caps any receiver throughput run.  Here a slot
batch is made on the device by ``libnrx_b200.so``'s ``nrx_synth_slots``
(include/nrx_slotgen.h) straight into the layouts ``nrx_forward`` reads, and
the hard decisions are scored by ``nrx_count_bit_errors`` — no host round
trip between generation, reception and counting.

Reference interfaces mirrored (file:line under /root/reference/pkg/src/nrxsim):
  TdlProfile, tdl_a..tdl_d, PROFILES  channel.py:29-95
  TdlChannelSource / doubletdl        channel.py:170-190, 226-228
  sample_tdl, cir_to_freq             channel.py:113-150
  apply_channel, effective            channel.py:101-104, 153-167
  generate_pilots, map_bits           slot.py:130-139, constellation.py:44-50
  MetricsRecord (ber / tbler)         evaluation.py:44-72

Two sources of randomness:
  * device (default): Philox4x32-10 keyed by (seed, global slot index), so a
    slot is the same whichever batch or rank generates it;
  * reference stream: ``reference_variates`` draws the variates on the host
    with numpy exactly as the reference's generators do, and the GPU slot then
    equals the reference's to float64 rounding (tests/test_gpu_slotgen.py).
LDPC is bypassed (labels are iid; SURVEY.md finding 5), so the counters are
uncoded BER and per-(slot, UE) "block" errors.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _lib
from .config import generate_pilots
from .synth import gray_qam

NUM_SINUSOIDS = 32


@dataclass(frozen=True)
class TdlProfile:
    """Tapped-delay-line power-delay profile with a Doppler spread."""

    name: str
    delays_s: np.ndarray
    powers: np.ndarray
    doppler_hz: float
    delay_spread_s: float

    def __post_init__(self):
        d = np.asarray(self.delays_s, dtype=np.float64)
        p = np.asarray(self.powers, dtype=np.float64)
        object.__setattr__(self, "delays_s", d)
        object.__setattr__(self, "powers", p)
        if d.ndim != 1 or p.shape != d.shape:
            raise ValueError("delays and powers must be 1-D and matched")
        if (d < 0).any() or (np.diff(d) < 0).any():
            raise ValueError("tap delays must be non-negative and ascending")
        if abs(p.sum() - 1.0) > 1e-9:
            raise ValueError(f"tap powers must sum to 1, got {p.sum()}")

    def with_doppler(self, doppler_hz: float) -> "TdlProfile":
        return TdlProfile(self.name, self.delays_s, self.powers, doppler_hz, self.delay_spread_s)


def _make_profile(name, delays_norm, powers_db, delay_spread_s, doppler_hz) -> TdlProfile:
    lin = 10.0 ** (np.asarray(powers_db, dtype=np.float64) / 10.0)
    lin /= lin.sum()
    return TdlProfile(name, np.asarray(delays_norm, dtype=np.float64) * delay_spread_s, lin,
                      doppler_hz, delay_spread_s)


# The reference's declared 5-tap desk profiles (channel.py:67-90).
def tdl_a(delay_spread_s=30e-9, doppler_hz=50.0) -> TdlProfile:
    return _make_profile("tdl_a", [0.0, 0.7, 1.5, 2.4, 3.6], [0.0, -3.0, -6.5, -10.0, -14.0],
                         delay_spread_s, doppler_hz)


def tdl_b(delay_spread_s=100e-9, doppler_hz=400.0) -> TdlProfile:
    return _make_profile("tdl_b", [0.0, 0.35, 0.9, 1.7, 3.0], [0.0, -1.5, -3.3, -5.7, -9.0],
                         delay_spread_s, doppler_hz)


def tdl_c(delay_spread_s=300e-9, doppler_hz=100.0) -> TdlProfile:
    return _make_profile("tdl_c", [0.0, 0.7, 1.4, 2.6, 4.4], [-1.0, 0.0, -2.4, -4.8, -8.2],
                         delay_spread_s, doppler_hz)


def tdl_d(delay_spread_s=60e-9, doppler_hz=20.0) -> TdlProfile:
    return _make_profile("tdl_d", [0.0, 0.5, 1.2, 2.0, 3.2], [0.0, -9.0, -12.0, -15.0, -18.0],
                         delay_spread_s, doppler_hz)


PROFILES = {"tdl_a": tdl_a, "tdl_b": tdl_b, "tdl_c": tdl_c, "tdl_d": tdl_d}


def doubletdl(profile_a=None, profile_b=None):
    """The two-UE evaluation channel: UE1 on TDL-B, UE2 on TDL-C (channel.py:226-228)."""
    return [profile_a or tdl_b(), profile_b or tdl_c()]


def qam_table() -> np.ndarray:
    """(340,) complex128: the Gray QAM points of orders 2, 4, 6, 8 in the
    order nrx_synth_slots indexes them (bit-identical to the reference's
    build_constellation(m).points for m in 2, 4, 6)."""
    return np.concatenate([gray_qam(m) for m in (2, 4, 6, 8)]).astype(np.complex128)


def channel_desc(cfg, profiles, num_sinusoids: int = NUM_SINUSOIDS) -> _lib.ChannelDesc:
    """SlotConfig antennas/numerology/beams + one TdlProfile per UE -> nrx_channel_desc."""
    U = cfg.num_ues
    if len(profiles) < U:
        raise ValueError(f"source has {len(profiles)} profiles for {U} UEs")
    if U > _lib.NRX_SG_MAX_UES or cfg.ue_antennas > _lib.NRX_SG_MAX_UE_ANT:
        raise ValueError(f"the GPU slot generator supports at most {_lib.NRX_SG_MAX_UES} UEs and "
                         f"{_lib.NRX_SG_MAX_UE_ANT} UE antennas")
    c = _lib.ChannelDesc()
    c.bs_antennas = cfg.bs_antennas
    c.ue_antennas = cfg.ue_antennas
    c.num_sinusoids = int(num_sinusoids)
    c.subcarrier_spacing_hz = float(cfg.subcarrier_spacing_hz)
    c.cp_fraction = float(cfg.cp_fraction)
    beams = cfg.beam_matrix
    for u in range(U):
        for a in range(cfg.ue_antennas):
            c.beams[u][a][0] = float(beams[u, a].real)
            c.beams[u][a][1] = float(beams[u, a].imag)
        p = profiles[u]
        if p.delays_s.size > _lib.NRX_SG_MAX_TAPS:
            raise ValueError(f"at most {_lib.NRX_SG_MAX_TAPS} taps are supported")
        c.profiles[u].num_taps = p.delays_s.size
        for l in range(p.delays_s.size):
            c.profiles[u].delays_s[l] = float(p.delays_s[l])
            c.profiles[u].powers[l] = float(p.powers[l])
        c.profiles[u].doppler_hz = float(p.doppler_hz)
    return c


def reference_variates(cfg, profiles, orders, slots, seed: int = 0, num_sinusoids: int = NUM_SINUSOIDS,
                       pilot_seed=None) -> dict:
    """Host-drawn variates of the reference's uncoded slot recipe, one entry
    per slot index i in ``slots`` (the recipe of tests/golden/make_golden.py,
    SURVEY.md §8d):
      pilots   generate_pilots(cfg, pilot_seed(i)), default seed*1000 + i
      bits     rng = default_rng((seed, i)); per UE rng.random((n_data, m)) < 0.5
      channel  TdlChannelSource.sample(cfg, (seed, i)): per UE
               default_rng((seed, i, u)).uniform(0, 2 pi) angles then phases
      noise    apply_channel(..., rng): rng.standard_normal twice (re, im)
    Returned arrays are in the nrx_slot_variates layouts."""
    slots = list(slots)
    N, U, S, T, B, Nu = len(slots), cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, cfg.bs_antennas, \
        cfg.ue_antennas
    L = max(p.delays_s.size for p in profiles[:U])
    comb, K = cfg.comb_size, len(cfg.pilot_symbols)
    F = -(-S // comb)
    s_idx, t_idx = np.nonzero(cfg.data_mask)
    ps = np.asarray(cfg.pilot_symbols)
    angles = np.zeros((N, U, B, Nu, L, num_sinusoids))
    phases = np.zeros_like(angles)
    labels = np.zeros((N, U, S, T), dtype=np.uint8)
    noise = np.zeros((N, S, T, B), dtype=np.complex128)
    pilots = np.zeros((N, U, F, K), dtype=np.complex128)
    pseed = pilot_seed or (lambda i: seed * 1000 + i)
    for j, i in enumerate(slots):
        book = generate_pilots(cfg, pseed(i))
        for u in range(U):
            sc = np.arange(u % comb, S, comb)
            pilots[j, u, :sc.size] = book.values[u][np.ix_(sc, ps)]
        rng = np.random.default_rng((seed, i))
        for u, m in enumerate(orders):
            bits = (rng.random((s_idx.size, m)) < 0.5).astype(np.int64)
            labels[j, u, s_idx, t_idx] = bits @ (1 << np.arange(m - 1, -1, -1))
        for u in range(U):
            r = np.random.default_rng((seed, i, u))
            nt = profiles[u].delays_s.size
            angles[j, u, :, :, :nt] = r.uniform(0.0, 2.0 * np.pi, size=(B, Nu, nt, num_sinusoids))
            phases[j, u, :, :, :nt] = r.uniform(0.0, 2.0 * np.pi, size=(B, Nu, nt, num_sinusoids))
        re = rng.standard_normal((S, T, B))
        noise[j] = re + 1j * rng.standard_normal((S, T, B))
    return dict(angles=angles, phases=phases, labels=labels, noise=noise, pilots=pilots)


def labels_to_bits(labels: np.ndarray, cfg, orders) -> list:
    """(N, U, S, T) label indices -> per UE (N, n_data, m) bits in the
    subcarrier-major data-RE order (slot.py:106-109)."""
    s_idx, t_idx = np.nonzero(cfg.data_mask)
    out = []
    for u, m in enumerate(orders):
        lab = labels[:, u, s_idx, t_idx].astype(np.int64)
        out.append(((lab[..., None] >> np.arange(m - 1, -1, -1)) & 1).astype(np.uint8))
    return out


class SlotBatch(NamedTuple):
    """One generated batch, all on the device, in nrx_forward's layouts."""
    y: object           # (N, S, T, B) complex64 / complex128
    pilots: object      # (N, U, F, K) complex
    labels: object      # (N, U, S, T) uint8 label index (0 off the data REs)
    h_eff: object       # (N, U, S, T, B) complex or None
    n0: object          # (N,) float64
    mod_order: object   # (N*U,) int32
    first_slot: int


class GpuSlotSource:
    """TdlChannelSource + transmitter + apply_channel on the GPU.

    ``profiles[u]`` is UE u's TdlProfile (default: doubletdl for two UEs).
    Thread-compatible: one source per thread (it owns its workspace)."""

    def __init__(self, cfg, profiles=None, device=None, num_sinusoids: int = NUM_SINUSOIDS, qam=None):
        from .engine import _require_cuda
        torch = _require_cuda()
        self.lib = _lib.load()
        self.cfg = cfg
        self.profiles = list(profiles if profiles is not None else (doubletdl() * 2)[: cfg.num_ues])
        self.num_sinusoids = int(num_sinusoids)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._s = _lib.slot_desc(cfg)
        self._c = channel_desc(cfg, self.profiles, num_sinusoids)
        code = self.lib.nrx_synth_validate(ctypes.byref(self._s), ctypes.byref(self._c))
        if code == 1:
            raise ValueError("invalid slot/channel description (e.g. a tap delay beyond the cyclic prefix bound, "
                             "channel.py:135-138)")
        _lib.check(code, "nrx_synth_validate")
        self._qam = np.ascontiguousarray((qam if qam is not None else qam_table()).astype(np.complex128))
        self._ws = None
        self.F = -(-cfg.num_subcarriers // cfg.comb_size)
        self.L = max(p.delays_s.size for p in self.profiles[: cfg.num_ues])

    def describe(self) -> str:
        return "gpu:" + "+".join(f"{p.name}({p.doppler_hz:g}Hz,{p.delay_spread_s * 1e9:g}ns)"
                                 for p in self.profiles[: self.cfg.num_ues])

    def _workspace(self, n):
        import torch
        nbytes = self.lib.nrx_synth_workspace_bytes(ctypes.byref(self._s), ctypes.byref(self._c), n)
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        return self._ws

    def generate(self, n_slots: int, mod_order, n0, seed: int = 0, first_slot: int = 0, variates=None,
                 y_dtype=None, pilots_dtype=None, with_h_eff: bool = False, h_dtype=None, out=None,
                 stream=None) -> SlotBatch:
        """Enqueue one batch of n_slots slots (global indices first_slot..).

        mod_order: (N, U) / (U,) ints or a device int32 tensor (N*U,);
        n0: scalar, (N,) array or device float64 tensor; variates: None
        (device Philox) or the dict of ``reference_variates`` (numpy or
        device tensors).  ``out`` reuses a previous SlotBatch's buffers."""
        import torch
        cfg, dev = self.cfg, self.device
        N, U, S, T, B = n_slots, cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, cfg.bs_antennas
        y_dtype = y_dtype or torch.complex64
        pilots_dtype = pilots_dtype or torch.complex64
        h_dtype = h_dtype or torch.complex64
        mods = self._dev(mod_order, torch.int32, (N * U,), broadcast_from=(U,))
        n0_t = self._dev(n0, torch.float64, (N,))
        if out is not None and out.y.shape[0] == N:
            y, pil, lab, heff = out.y, out.pilots, out.labels, out.h_eff
            if with_h_eff and heff is None:
                heff = torch.empty((N, U, S, T, B), dtype=h_dtype, device=dev)
        else:
            y = torch.empty((N, S, T, B), dtype=y_dtype, device=dev)
            pil = torch.empty((N, U, self.F, len(cfg.pilot_symbols)), dtype=pilots_dtype, device=dev)
            lab = torch.empty((N, U, S, T), dtype=torch.uint8, device=dev)
            heff = torch.empty((N, U, S, T, B), dtype=h_dtype, device=dev) if with_h_eff else None
        keep = []
        host_src = False
        var_s = None
        if variates is not None:
            var_s = _lib.SlotVariates()
            for name, dt in (("angles", torch.float64), ("phases", torch.float64), ("labels", torch.uint8),
                             ("noise", torch.complex128), ("pilots", torch.complex128)):
                v = variates.get(name)
                if v is None:
                    continue
                if not (isinstance(v, torch.Tensor) and v.device == dev):
                    host_src = True
                t = v if isinstance(v, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(v))
                t = t.to(device=dev, dtype=dt).contiguous()
                keep.append(t)
                setattr(var_s, name, t.data_ptr())
        ws = self._workspace(N)
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        code = self.lib.nrx_synth_slots(
            ctypes.byref(self._s), ctypes.byref(self._c), N, int(seed) & (2 ** 64 - 1), int(first_slot),
            mods.data_ptr(), n0_t.data_ptr(), ctypes.byref(var_s) if var_s is not None else None,
            self._qam.ctypes.data, y.data_ptr(), int(y.dtype == torch.complex128),
            pil.data_ptr(), int(pil.dtype == torch.complex128), lab.data_ptr(),
            heff.data_ptr() if heff is not None else None, int(heff is not None and heff.dtype == torch.complex128),
            ws.data_ptr(), ws.numel(), st.cuda_stream)
        _lib.check(code, "nrx_synth_slots")
        if host_src:
            st.synchronize()            # staged host variates must outlive the kernels
        return SlotBatch(y, pil, lab, heff, n0_t, mods, int(first_slot))

    def _dev(self, v, dtype, shape, broadcast_from=None):
        import torch
        if isinstance(v, torch.Tensor):
            t = v.to(device=self.device, dtype=dtype).reshape(-1)
            if t.numel() == 1:
                t = t.expand(int(np.prod(shape)))
            elif broadcast_from is not None and t.numel() == int(np.prod(broadcast_from)):
                t = t.repeat(int(np.prod(shape)) // t.numel())
            return t.contiguous()
        a = np.asarray(v)
        if a.size == 1:
            a = np.full(shape, a.reshape(-1)[0])
        elif broadcast_from is not None and a.size == int(np.prod(broadcast_from)):
            a = np.broadcast_to(a.reshape(1, -1), (int(np.prod(shape)) // a.size, a.size))
        a = np.array(a.reshape(shape), copy=True)
        return torch.from_numpy(a).to(device=self.device, dtype=dtype)


def count_bit_errors(cfg, llr, labels, mod_order, out=None, stream=None):
    """Adds the uncoded bit errors of every (slot, UE) to ``out`` (a device
    int64 tensor (N*U,), allocated zeroed when None) and returns it.
    llr: nrx_forward's (N, U, S, T, W) float32; labels (N, U, S, T) uint8;
    mod_order (N*U,) int32 — all on one device."""
    import torch
    lib = _lib.load()
    N, U = labels.shape[0], labels.shape[1]
    if out is None:
        out = torch.zeros(N * U, dtype=torch.int64, device=labels.device)
    for t in (llr, labels, mod_order, out):
        if not t.is_contiguous():
            raise ValueError("count_bit_errors expects contiguous tensors")
    st = stream if stream is not None else torch.cuda.current_stream(labels.device)
    s = _lib.slot_desc(cfg)
    code = lib.nrx_count_bit_errors(ctypes.byref(s), N, llr.data_ptr(), llr.shape[-1], labels.data_ptr(),
                                    mod_order.data_ptr(), out.data_ptr(), st.cuda_stream)
    _lib.check(code, "nrx_count_bit_errors")
    return out


@dataclass(frozen=True)
class UncodedRecord:
    """Counters of one (receiver, SNR) point, named like MetricsRecord
    (evaluation.py:44-72); a "block" is one (slot, UE) stream."""

    receiver: str
    snr_db: float
    blocks: int
    block_errors: int
    bit_errors: int
    bits: int

    @property
    def bler(self) -> float:
        return self.block_errors / self.blocks if self.blocks else float("nan")

    @property
    def ber(self) -> float:
        return self.bit_errors / self.bits if self.bits else float("nan")


def evaluate_uncoded(engine, source: GpuSlotSource, mcs_per_ue, snr_db_grid, n_slots: int, batch: int = 32,
                     seed: int = 0, num_iterations=None, receiver: str = "nrx", rank: int = 0, world: int = 1,
                     reduce=None) -> list:
    """Monte-Carlo uncoded BER/BLER of the GPU receiver on GPU-generated
    slots: generate -> nrx_forward -> count, batch by batch, all on the
    device.  Slot i of SNR point k is Philox slot (k, i) whatever the batch
    size, and rank r of ``world`` takes the contiguous slot shard
    shard_slots(n_slots, r, world); ``reduce`` (e.g. an all-reduce SUM over
    ranks) combines the four counters, so results are identical for any
    world size (the num_workers determinism of evaluation.py:212-268)."""
    import torch
    from .nrx import noise_features
    from .shard import shard_slots
    cfg = source.cfg
    U = cfg.num_ues
    orders = [m.modulation_order for m in mcs_per_ue]
    n_it = num_iterations or engine.config.num_iterations
    width = engine.config.m_max if engine.config.variant != "var_io" else max(orders)
    bits_per_slot = cfg.num_data_res * sum(orders)
    mine = shard_slots(n_slots, rank, world)
    dev = source.device
    cap = max(1, min(batch, len(mine)))
    mods = torch.tensor(orders * cap, dtype=torch.int32, device=dev)
    llr = torch.empty((cap, U, cfg.num_subcarriers, cfg.num_symbols, width), dtype=torch.float32, device=dev)
    chest = torch.empty((cap, U, cfg.num_subcarriers, cfg.num_symbols, cfg.bs_antennas), dtype=torch.complex64,
                        device=dev)
    errs = torch.zeros(cap * U, dtype=torch.int64, device=dev)
    records = []
    for k, snr_db in enumerate(snr_db_grid):
        n0 = 10.0 ** (-float(snr_db) / 10.0)
        n0_t = torch.full((cap,), n0, dtype=torch.float64, device=dev)
        nf = torch.from_numpy(noise_features(n0, cap)).to(dev)
        tot = torch.zeros(2, dtype=torch.int64, device=dev)       # block errors, bit errors
        out = None
        for start in range(mine.start, mine.stop, cap):
            nb = min(cap, mine.stop - start)
            sb = source.generate(nb, mods[: nb * U], n0_t[:nb], seed=(int(seed) << 16) + k, first_slot=start,
                                 out=out if out is not None and out.y.shape[0] == nb else None,
                                 with_h_eff=getattr(engine, "needs_h_eff", False))
            out = sb
            extra = {"n0": sb.n0} if getattr(engine, "needs_n0", False) else {}
            if getattr(engine, "needs_h_eff", False):
                extra["h_eff"] = sb.h_eff
            engine.forward_device(cfg, sb.y, sb.pilots, nf[:nb], sb.mod_order, n_it, llr[:nb], chest[:nb], **extra)
            e = errs[: nb * U].zero_()
            count_bit_errors(cfg, llr[:nb], sb.labels, sb.mod_order, out=e)
            tot += torch.stack([(e > 0).sum(), e.sum()])
        c = torch.tensor([len(mine) * U, 0, 0, len(mine) * bits_per_slot], dtype=torch.int64).to(dev)
        c[1:3] = tot
        if reduce is not None:
            c = reduce(c)
        c = [int(x) for x in c.cpu()]
        records.append(UncodedRecord(receiver, float(snr_db), c[0], c[1], c[2], c[3]))
    return records


__all__ = ["TdlProfile", "tdl_a", "tdl_b", "tdl_c", "tdl_d", "PROFILES", "doubletdl", "qam_table", "channel_desc",
           "reference_variates", "labels_to_bits", "SlotBatch", "GpuSlotSource", "count_bit_errors",
           "UncodedRecord", "evaluate_uncoded", "NUM_SINUSOIDS"]
