"""LDPC layer downstream of the receiver on the GPU:
min-sum decoding of the NRX LLRs, scalable codes with a linear-time encoder,
and the coded TBLER Monte-Carlo loop (generate -> receive -> decode -> count)
entirely on the device.

Reference interfaces mirrored (file:line under /root/reference/pkg/src/nrxsim):
  LdpcCode (fields, k_eff, tx_positions, num_tx_bits, rate)   ldpc.py:28-75
  LdpcCode.decode / check_parity                             ldpc.py:91-178
  rate_matched_code (shorten info, puncture trailing parity)  ldpc.py:303-330
  _evaluate_chunk / MetricsRecord / LLR_CLIP                  evaluation.py:27-72,165-209

Scalable mother codes.  The reference's column-weight-3 greedy construction
re-ranks every check for every edge (O(n m log m)) and encodes with a dense
k x m GF(2) matrix; a 273-PRB 16-QAM codeword (n0 = 169,838) is out of reach
for both.  ``ira_code`` builds a rate-1/2 irregular-repeat-accumulate code
instead: information columns of weight 3 spread over the checks by a seeded
socket permutation (every check gets exactly three), plus a staircase
(accumulator) parity part, so encoding is a handful of XOR chain walks.  The chain
order of the parity columns is a stride permutation, so the reference's
rate-matching rule (puncture the trailing parity positions) removes parity
bits spread evenly along the accumulator.  The same min-sum decoder runs the
reference's own codes bit-identically (tests/test_gpu_ldpc.py).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib

LLR_CLIP = 20.0           # evaluation.py:27
DECODER_ITERATIONS = 20   # EvalConfig.decoder_iterations, evaluation.py:45


@dataclass(frozen=True)
class LdpcCode:
    """Parity-check structure + rate matching (same fields as the reference;
    chain_cols is set for staircase codes and enables encoding)."""

    n: int
    k: int
    row_cols: np.ndarray        # (M, dmax) int32, -1 padded
    col_rows: np.ndarray        # (n, <=3) int32, -1 padded
    col_slots: np.ndarray       # (n, <=3) int32
    info_positions: np.ndarray  # (k,) ascending
    punctured: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    shortened: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    chain_cols: np.ndarray | None = None   # (M,) parity column of chain position i
    chain_step: int = 1                    # check i holds chain positions i - chain_step and i

    @property
    def num_checks(self) -> int:
        return self.row_cols.shape[0]

    @property
    def k_eff(self) -> int:
        return self.k - self.shortened.size

    @property
    def tx_positions(self) -> np.ndarray:
        skip = np.zeros(self.n, dtype=bool)
        skip[self.punctured] = True
        skip[self.shortened] = True
        return np.flatnonzero(~skip)

    @property
    def num_tx_bits(self) -> int:
        return self.n - self.punctured.size - self.shortened.size

    @property
    def rate(self) -> float:
        return self.k_eff / self.num_tx_bits

    @classmethod
    def from_reference(cls, code) -> "LdpcCode":
        """Wrap a reference ``nrxsim.ldpc.LdpcCode`` (decode-only on the GPU)."""
        return cls(int(code.n), int(code.k), np.asarray(code.row_cols), np.asarray(code.col_rows),
                   np.asarray(code.col_slots), np.asarray(code.info_positions),
                   np.asarray(code.punctured, dtype=np.int64), np.asarray(code.shortened, dtype=np.int64))


def _coprime_stride(m: int) -> int:
    g = max(1, int(round(m * (math.sqrt(5.0) - 1.0) / 2.0)))
    while math.gcd(g, m) != 1:
        g += 1
    return g % m if m > 1 else 0


def ira_code(k0: int, seed: int = 0) -> LdpcCode:
    """Rate-1/2 IRA mother code with k0 information bits (n = 2 k0, M = k0).

    Information column j sits in three distinct checks: 3 k0 sockets are
    dealt to the checks by a seeded permutation (three per check), and
    repeated checks inside a column are swapped away.  The parity part is a
    block staircase: check i holds accumulator positions i - Z and i, i.e. Z
    interleaved accumulator chains of length <= 16 (Z = ceil(k0 / 16)), the
    dual-diagonal structure of quasi-cyclic LDPC parity parts, so belief
    propagation crosses the accumulator in ~16 steps instead of k0.  Chain
    position i is parity column k0 + (i * g mod k0), g a stride near the
    golden ratio coprime to k0, which spreads the punctured tail columns."""
    if k0 < 3:
        raise ValueError(f"IRA code needs k0 >= 3, got {k0}")
    m, n = k0, 2 * k0
    rng = np.random.default_rng((0x1DA, k0, seed))
    rows = (rng.permutation(3 * k0) // 3).reshape(k0, 3)
    for _ in range(1000):
        dup = (rows[:, 0] == rows[:, 1]) | (rows[:, 0] == rows[:, 2]) | (rows[:, 1] == rows[:, 2])
        idx = np.flatnonzero(dup)
        if idx.size == 0:
            break
        other = rng.integers(0, k0, size=idx.size)
        slot = rng.integers(0, 3, size=idx.size)
        for a, b, s in zip(idx, other, slot):       # socket swap keeps every check at three
            mine = 1 if rows[a, 1] == rows[a, 2] else 0  # one socket of the repeated pair
            rows[a, mine], rows[b, s] = rows[b, s], rows[a, mine]
    else:  # pragma: no cover
        raise RuntimeError("could not place the information edges")
    rows.sort(axis=1)
    g = _coprime_stride(m)
    z = max(1, -(-m // 16))
    chain_cols = k0 + (np.arange(m, dtype=np.int64) * g) % m
    # edge list (column, row)
    e_col = [np.repeat(np.arange(k0), 3), chain_cols, chain_cols[: m - z]]
    e_row = [rows.reshape(-1), np.arange(m), np.arange(z, m)]
    col = np.concatenate(e_col)
    row = np.concatenate(e_row)
    order = np.lexsort((col, row))
    col, row = col[order], row[order]
    row_deg = np.bincount(row, minlength=m)
    dmax = int(row_deg.max())
    start = np.concatenate([[0], np.cumsum(row_deg)[:-1]])
    slot = np.arange(col.size) - start[row]
    row_cols = np.full((m, dmax), -1, dtype=np.int32)
    row_cols[row, slot] = col
    # per column: its checks ascending, with the slot each occupies in the row
    corder = np.lexsort((row, col))
    ccol, crow, cslot = col[corder], row[corder], slot[corder]
    col_deg = np.bincount(ccol, minlength=n)
    cstart = np.concatenate([[0], np.cumsum(col_deg)[:-1]])
    cpos = np.arange(ccol.size) - cstart[ccol]
    col_rows = np.full((n, 3), -1, dtype=np.int32)
    col_slots = np.full((n, 3), -1, dtype=np.int32)
    col_rows[ccol, cpos] = crow
    col_slots[ccol, cpos] = cslot
    return LdpcCode(n, k0, row_cols, col_rows, col_slots, np.arange(k0, dtype=np.int64),
                    chain_cols=chain_cols.astype(np.int64), chain_step=z)


def rate_matched_ira_code(num_tx_bits: int, rate: float, seed: int = 0) -> LdpcCode:
    """The reference's rate-matching rule (ldpc.py:303-330) on an IRA mother
    code: k_eff = round(rate E), k0 = max(k_eff, E - k_eff), shorten the first
    k0 - k_eff information positions, puncture the trailing parity positions."""
    if not 0.0 < rate < 1.0:
        raise ValueError(f"code rate must be in (0,1), got {rate}")
    k_eff = int(round(rate * num_tx_bits))
    if k_eff < 1 or k_eff >= num_tx_bits:
        raise ValueError(f"degenerate rate matching: E={num_tx_bits}, rate={rate}")
    k0 = max(k_eff, num_tx_bits - k_eff)
    base = ira_code(k0, seed)
    shortened = base.info_positions[: k0 - k_eff]
    parity_positions = np.setdiff1d(np.arange(base.n), base.info_positions)
    punctured = parity_positions[num_tx_bits - k_eff:]
    code = LdpcCode(base.n, base.k, base.row_cols, base.col_rows, base.col_slots, base.info_positions,
                    np.asarray(punctured, dtype=np.int64), np.asarray(shortened, dtype=np.int64), base.chain_cols,
                    base.chain_step)
    assert code.num_tx_bits == num_tx_bits and code.k_eff == k_eff
    return code


def slot_code(cfg, mcs, seed: int = 0) -> LdpcCode:
    """The code filling one UE stream's data REs (slot.py:170-172), IRA family."""
    return rate_matched_ira_code(cfg.num_data_res * mcs.modulation_order, mcs.code_rate, seed)


class GpuLdpc:
    """One code resident on the device: decode (any code) / encode (staircase codes)."""

    def __init__(self, code: LdpcCode, device=None):
        from .engine import _require_cuda
        torch = _require_cuda()
        self.lib = _lib.load()
        self.code = code
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        arr = {k: np.ascontiguousarray(np.asarray(v), dtype=np.int32) for k, v in
               dict(row_cols=code.row_cols, col_rows=code.col_rows, col_slots=code.col_slots,
                    info=code.info_positions, punct=code.punctured, short=code.shortened).items()}
        chain = None if code.chain_cols is None else np.ascontiguousarray(code.chain_cols, dtype=np.int32)
        d = _lib.LdpcDesc()
        d.n, d.m, d.k = code.n, code.num_checks, code.k
        d.dmax, d.cdeg = arr["row_cols"].shape[1], arr["col_rows"].shape[1]
        d.row_cols, d.col_rows, d.col_slots = (arr[k].ctypes.data for k in ("row_cols", "col_rows", "col_slots"))
        d.info_positions = arr["info"].ctypes.data
        d.n_punctured, d.punctured = arr["punct"].size, arr["punct"].ctypes.data if arr["punct"].size else None
        d.n_shortened, d.shortened = arr["short"].size, arr["short"].ctypes.data if arr["short"].size else None
        d.chain_cols = chain.ctypes.data if chain is not None else None
        d.chain_step = int(code.chain_step)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            code_rc = self.lib.nrx_ldpc_create(ctypes.byref(d), ctypes.byref(h))
        _lib.check(code_rc, "nrx_ldpc_create")
        self._h = h
        dims = (ctypes.c_int32 * 4)()
        self.lib.nrx_ldpc_dims(h, dims)
        self.n, self.k_eff, self.num_tx_bits, self.m = (int(x) for x in dims)
        self._ws = None

    def close(self):
        if getattr(self, "_h", None):
            self.lib.nrx_ldpc_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass

    def _workspace(self, n_cw):
        import torch
        nb = self.lib.nrx_ldpc_workspace_bytes(self._h, n_cw)
        if self._ws is None or self._ws.numel() < nb:
            self._ws = torch.empty(nb, dtype=torch.uint8, device=self.device)
        return self._ws

    def decode(self, llr, iterations: int = DECODER_ITERATIONS, stream=None):
        """llr (B, num_tx_bits) float32 device tensor (logit convention) ->
        (info (B, k_eff) uint8, success (B,) bool) device tensors."""
        import torch
        if llr.dim() != 2 or llr.shape[1] != self.num_tx_bits:
            raise ValueError(f"expected {self.num_tx_bits} LLRs, got {tuple(llr.shape)}")
        llr = llr.to(device=self.device, dtype=torch.float32).contiguous()
        b = llr.shape[0]
        info = torch.empty((b, self.k_eff), dtype=torch.uint8, device=self.device)
        ok = torch.empty(b, dtype=torch.uint8, device=self.device)
        ws = self._workspace(b)
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = self.lib.nrx_ldpc_decode(self._h, b, llr.data_ptr(), int(iterations), info.data_ptr(), ok.data_ptr(),
                                      ws.data_ptr(), ws.numel(), st.cuda_stream)
        _lib.check(rc, "nrx_ldpc_decode")
        return info, ok.bool()

    def encode(self, info, stream=None):
        """info (B, k_eff) uint8 device tensor -> transmitted bits (B, num_tx_bits) uint8."""
        import torch
        if info.dim() != 2 or info.shape[1] != self.k_eff:
            raise ValueError(f"expected {self.k_eff} info bits, got {tuple(info.shape)}")
        info = info.to(device=self.device, dtype=torch.uint8).contiguous()
        b = info.shape[0]
        tx = torch.empty((b, self.num_tx_bits), dtype=torch.uint8, device=self.device)
        ws = self._workspace(b)
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = self.lib.nrx_ldpc_encode(self._h, b, info.data_ptr(), tx.data_ptr(), ws.data_ptr(), ws.numel(),
                                      st.cuda_stream)
        _lib.check(rc, "nrx_ldpc_encode")
        return tx


@dataclass(frozen=True)
class MetricsRecord:
    """Error counts of one receiver at one SNR point (evaluation.py:56-72)."""

    receiver: str
    snr_db: float
    blocks: int
    block_errors: int
    bit_errors: int
    bits: int

    @property
    def tbler(self) -> float:
        return self.block_errors / self.blocks if self.blocks else float("nan")

    @property
    def ber(self) -> float:
        return self.bit_errors / self.bits if self.bits else float("nan")


def evaluate_coded(engine, source, mcs_per_ue, snr_db_grid, n_slots: int, batch: int = 32, seed: int = 0,
                   num_iterations=None, llr_clip: float = LLR_CLIP, decoder_iterations: int = DECODER_ITERATIONS,
                   receiver: str = "nrx", rank: int = 0, world: int = 1, reduce=None, codes=None) -> list:
    """Coded Monte-Carlo TBLER/BER of the GPU receiver (the path of
    evaluation._evaluate_chunk, evaluation.py:165-209) with every step on the
    device: payload bits -> IRA encode -> Gray labels on the data REs -> GPU
    slot generator -> nrx_forward -> data-RE LLRs clipped to +-llr_clip ->
    min-sum decode -> payload comparison.  One block = one UE codeword; bits =
    payload bits.  Slot i of SNR point k is the same whatever the batch size or
    rank (Philox keys); ``reduce`` combines the counters across ranks."""
    import torch
    from .nrx import noise_features
    from .shard import shard_slots
    cfg = source.cfg
    U, S, T = cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols
    lib = _lib.load()
    sdesc = _lib.slot_desc(cfg)
    orders = [m.modulation_order for m in mcs_per_ue]
    if not codes:
        built = {}                                # one code per distinct MCS
        for m in mcs_per_ue:
            if (m.modulation_order, m.code_rate) not in built:
                built[(m.modulation_order, m.code_rate)] = slot_code(cfg, m)
        codes = [built[(m.modulation_order, m.code_rate)] for m in mcs_per_ue]
    groups, dec_of = [], {}                       # UEs sharing a code object share a decoder
    for u, c in enumerate(codes):
        if id(c) in dec_of:
            groups[dec_of[id(c)]].append(u)
        else:
            dec_of[id(c)] = len(groups)
            groups.append([u])
    shared = [GpuLdpc(codes[g[0]], source.device) for g in groups]
    dec = [shared[dec_of[id(c)]] for c in codes]
    n_it = num_iterations or engine.config.num_iterations
    width = engine.config.m_max if engine.config.variant != "var_io" else max(orders)
    mine = shard_slots(n_slots, rank, world)
    dev = source.device
    cap = max(1, min(batch, len(mine)))
    mods = torch.tensor(orders * cap, dtype=torch.int32, device=dev)
    labels = torch.zeros((cap, U, S, T), dtype=torch.uint8, device=dev)
    llr = torch.empty((cap, U, S, T, width), dtype=torch.float32, device=dev)
    chest = torch.empty((cap, U, S, T, cfg.bs_antennas), dtype=torch.complex64, device=dev)
    st = torch.cuda.current_stream(dev)
    records = []
    for k, snr_db in enumerate(snr_db_grid):
        n0 = 10.0 ** (-float(snr_db) / 10.0)
        n0_t = torch.full((cap,), n0, dtype=torch.float64, device=dev)
        nf = torch.from_numpy(noise_features(n0, cap)).to(dev)
        errs = torch.zeros((U, cap), dtype=torch.int64, device=dev)
        tot = torch.zeros(2, dtype=torch.int64, device=dev)      # block errors, bit errors
        key = (int(seed) << 20) + (k << 4)
        for start in range(mine.start, mine.stop, cap):
            nb = min(cap, mine.stop - start)
            payload = [None] * U
            for users in groups:                  # one encode call per shared code
                d = dec[users[0]]
                info = torch.empty((len(users), nb, d.k_eff), dtype=torch.uint8, device=dev)
                for i, u in enumerate(users):     # payload bits keyed per UE
                    _lib.check(lib.nrx_random_bits(key + u, start, nb, d.k_eff, info[i].data_ptr(),
                                                   st.cuda_stream), "nrx_random_bits")
                    payload[u] = info[i]
                tx = d.encode(info.view(len(users) * nb, d.k_eff))
                for i, u in enumerate(users):
                    _lib.check(lib.nrx_bits_to_labels(ctypes.byref(sdesc), nb, u, orders[u],
                                                      tx[i * nb:(i + 1) * nb].data_ptr(), labels.data_ptr(),
                                                      st.cuda_stream), "nrx_bits_to_labels")
            sb = source.generate(nb, mods[: nb * U], n0_t[:nb], seed=key + 15, first_slot=start,
                                 variates={"labels": labels[:nb]}, with_h_eff=getattr(engine, "needs_h_eff", False))
            extra = {"n0": sb.n0} if getattr(engine, "needs_n0", False) else {}
            if getattr(engine, "needs_h_eff", False):
                extra["h_eff"] = sb.h_eff
            engine.forward_device(cfg, sb.y, sb.pilots, nf[:nb], sb.mod_order, n_it, llr[:nb], chest[:nb], **extra)
            errs.zero_()
            # UEs that share a code are decoded in one call (their 32-codeword
            # groups run concurrently); results are per codeword either way.
            for users in groups:
                d = dec[users[0]]
                cw_llr = torch.empty((len(users), nb, d.num_tx_bits), dtype=torch.float32, device=dev)
                for i, u in enumerate(users):
                    _lib.check(lib.nrx_extract_llrs(ctypes.byref(sdesc), nb, u, orders[u], llr.data_ptr(), width,
                                                    float(llr_clip), cw_llr[i].data_ptr(), st.cuda_stream),
                               "nrx_extract_llrs")
                info_hat, _ = d.decode(cw_llr.view(len(users) * nb, d.num_tx_bits), decoder_iterations)
                for i, u in enumerate(users):
                    _lib.check(lib.nrx_count_mismatches(nb, d.k_eff, info_hat[i * nb:(i + 1) * nb].data_ptr(),
                                                        payload[u].data_ptr(), errs[u].data_ptr(), st.cuda_stream),
                               "nrx_count_mismatches")
            e = errs[:, :nb]
            tot += torch.stack([(e > 0).sum(), e.sum()])
        blocks = len(mine) * U
        bits = len(mine) * sum(d.k_eff for d in dec)
        c = torch.tensor([blocks, 0, 0, bits], dtype=torch.int64).to(dev)
        c[1:3] = tot
        if reduce is not None:
            c = reduce(c)
        c = [int(x) for x in c.cpu()]
        records.append(MetricsRecord(receiver, float(snr_db), c[0], c[1], c[2], c[3]))
    for d in shared:
        d.close()
    return records


__all__ = ["LdpcCode", "ira_code", "rate_matched_ira_code", "slot_code", "GpuLdpc", "MetricsRecord",
           "evaluate_coded", "LLR_CLIP", "DECODER_ITERATIONS"]
