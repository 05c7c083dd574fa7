"""NrxEngine: one receiver model resident on one B200.

Owns the packed device weights, per-thread CUDA streams, workspaces and
pinned staging buffers, and calls the C-ABI entry point ``nrx_forward``
(include/nrx_b200.h).  Two ways in:

* ``forward_device``  device-resident tensors in and out (the paper's
  "inline acceleration" latency setting), no host copies;
* ``run``             numpy in, numpy out, with the semantics of the
  reference ``nrxsim.nrx.nrx_forward`` (nrx.py:345-385); host<->device
  copies are part of the call.

PyTorch is used for device memory, pinned memory and streams only; all
arithmetic happens in the CUDA kernels of libnrx_b200.so.
"""

from __future__ import annotations

import ctypes
import sys
import threading

import numpy as np

from . import _lib
from .config import weight_array


_TORCH = None


def _stage(torch, dst, arr):
    """Write a numpy array into a pinned staging tensor, converting the dtype
    (complex128 -> complex64, round to nearest as numpy).  torch's copy runs
    on all host threads (C2 y: 0.02 ms instead of 0.2 ms for np.copyto);
    arrays torch cannot wrap (read-only, negative strides) go through numpy."""
    if arr.flags.writeable and all(st >= 0 for st in arr.strides):
        try:
            dst.copy_(torch.from_numpy(arr))
            return
        except (TypeError, ValueError, RuntimeError):
            pass
    np.copyto(dst.numpy(), arr, casting="same_kind")


def _require_cuda():
    global _TORCH
    if _TORCH is None:
        import torch
        if not torch.cuda.is_available():
            raise _lib.NrxLibraryError("no CUDA device: the NRX B200 path has no CPU fallback")
        _TORCH = torch
    return _TORCH


def pack_weights(config, weights, precision: str = "fp32") -> np.ndarray:
    """Host-side repack of a weight dict (reference ``ad.Tensor`` values or
    arrays) into the kernels' layout via ``nrx_pack_weights`` (no GPU)."""
    lib = _lib.load()
    m = _lib.model_desc(config)
    prec = _lib.PRECISIONS[precision]
    _lib.check(lib.nrx_validate(ctypes.byref(m), None), "nrx_validate")
    names = _lib.weight_names(config)
    if set(names) != set(weights):
        raise ValueError(f"weights do not match the configuration: {sorted(set(names) ^ set(weights))}")
    arrays = []
    for i, name in enumerate(names):
        a = np.ascontiguousarray(weight_array(weights[name]), dtype=np.float32)
        if a.size != lib.nrx_weight_numel(ctypes.byref(m), i):
            raise ValueError(f"tensor '{name}' has {a.size} elements, expected {lib.nrx_weight_numel(ctypes.byref(m), i)}")
        arrays.append(a)
    ptrs = (ctypes.c_void_p * len(arrays))(*[a.ctypes.data for a in arrays])
    nbytes = lib.nrx_packed_weight_bytes(ctypes.byref(m), prec)
    if nbytes == 0:
        raise _lib.NrxLibraryError("nrx_packed_weight_bytes returned 0 (unsupported model)")
    out = np.zeros(nbytes, dtype=np.uint8)
    _lib.check(lib.nrx_pack_weights(ctypes.byref(m), prec, ptrs, len(arrays), out.ctypes.data),
               "nrx_pack_weights")
    return out


def pilot_comb_values(book_values: np.ndarray, cfg) -> np.ndarray:
    """(..., U, S, T) PilotBook values -> (..., U, F, K) values at each UE's
    comb subcarriers (u % comb + f*comb) and pilot symbols (slot.py:92-93,
    classical.py:43-44).  Entries past a UE's last comb subcarrier repeat a
    valid RE and are ignored by the kernel."""
    S, comb, U = cfg.num_subcarriers, cfg.comb_size, cfg.num_ues
    F = -(-S // comb)
    ps = list(cfg.pilot_symbols)
    book_values = np.asarray(book_values)
    out = np.empty(book_values.shape[:-3] + (U, F, len(ps)), dtype=book_values.dtype)
    for u in range(U):  # strided slices: no fancy-index gather over the grid
        o = u % comb
        sub = book_values[..., u, o::comb, :]            # (..., n_u, T)
        n_u = sub.shape[-2]
        for k, t in enumerate(ps):
            out[..., u, :n_u, k] = sub[..., t]
        if n_u < F:
            out[..., u, n_u:, :] = out[..., u, n_u - 1:n_u, :]
    return out


class NrxEngine:
    """Packed weights of one model on one device; thread-safe ``run``."""

    def __init__(self, config, weights, precision: str = "fp32", device=None):
        torch = _require_cuda()
        self.lib = _lib.load()
        self.config = config
        self.precision = precision
        self.prec_id = _lib.PRECISIONS[precision]
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._m = _lib.model_desc(config)
        packed = pack_weights(config, weights, precision)
        self.weights_dev = torch.from_numpy(packed).to(self.device)
        self._tls = threading.local()

    # -- per-thread resources --------------------------------------------------

    def _local(self):
        tls = self._tls
        if not hasattr(tls, "stream"):
            torch = _require_cuda()
            tls.stream = torch.cuda.Stream(device=self.device)
            tls.ws = {}
            tls.bufs = {}
        return tls

    def workspace(self, cfg, n_slots: int):
        torch = _require_cuda()
        s = _lib.slot_desc(cfg)
        nbytes = self.lib.nrx_workspace_bytes(ctypes.byref(self._m), ctypes.byref(s), n_slots, self.prec_id)
        if nbytes == 0:  # the model / slot is invalid, or outside this precision mode's limits
            code = self.lib.nrx_validate(ctypes.byref(self._m), ctypes.byref(s))
            _lib.check(code or 2, f"nrx_workspace_bytes ({self.precision})")
        tls = self._local()
        ws = tls.ws.get("ws")
        if ws is None or ws.numel() < nbytes:
            ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            tls.ws["ws"] = ws
        return ws

    def launch_count(self, cfg, num_iterations: int) -> int:
        s = _lib.slot_desc(cfg)
        return self.lib.nrx_forward_launch_count(ctypes.byref(self._m), ctypes.byref(s), self.prec_id,
                                                 int(num_iterations))

    # -- device-resident entry ---------------------------------------------------

    def forward_device(self, cfg, y, pilots, noise_feat, mod_order, num_iterations, llr, chest,
                       workspace=None, stream=None):
        """Enqueue one batched forward on device tensors.

        y (N,S,T,B) complex64/complex128; pilots (P,U,F,K) complex with P in
        {1, N}; noise_feat (N,) float32; mod_order (N*U,) int32; llr
        (N,U,S,T,W) float32 and chest (N,U,S,T,B) complex64 are written.
        """
        torch = _require_cuda()
        n = y.shape[0]
        s = _lib.slot_desc(cfg)
        ws = workspace if workspace is not None else self.workspace(cfg, n)
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._check_device_args(cfg, y, pilots, noise_feat, mod_order, llr, chest, ws)
        code = self.lib.nrx_forward(
            ctypes.byref(self._m), ctypes.byref(s), n, self.prec_id, int(num_iterations),
            y.data_ptr(), int(y.dtype == torch.complex128),
            pilots.data_ptr(), int(pilots.dtype == torch.complex128), pilots.shape[0],
            noise_feat.data_ptr(), mod_order.data_ptr(), self.weights_dev.data_ptr(),
            llr.data_ptr(), llr.shape[-1], chest.data_ptr(), ws.data_ptr(), ws.numel(), st.cuda_stream)
        if code == 5:
            raise ValueError(f"inference depth {num_iterations} outside [1, {self.config.num_iterations}]")
        _lib.check(code, "nrx_forward")

    def _check_device_args(self, cfg, y, pilots, noise_feat, mod_order, llr, chest, ws):
        """The C ABI reads raw pointers: check every tensor's device, layout,
        dtype and shape against the call's geometry before handing them over
        (a wrong dtype or a short buffer would otherwise be misread or
        overrun on the device)."""
        torch = _require_cuda()
        for name, t in (("y", y), ("pilots", pilots), ("noise_feat", noise_feat), ("mod_order", mod_order),
                        ("llr", llr), ("chest", chest), ("workspace", ws)):
            if not isinstance(t, torch.Tensor) or not t.is_contiguous() or t.device != self.device:
                raise ValueError(f"forward_device: {name} must be a contiguous tensor on {self.device}")
        U, S, T, B = cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, self.config.num_rx_ant
        F, K = -(-S // cfg.comb_size), len(cfg.pilot_symbols)
        n = y.shape[0] if y.dim() == 4 else -1
        cplx = (torch.complex64, torch.complex128)
        checks = (
            ("y", y.dtype in cplx and tuple(y.shape) == (n, S, T, B), f"complex (N,{S},{T},{B})"),
            ("pilots", pilots.dtype in cplx and pilots.dim() == 4 and pilots.shape[0] in (1, n)
             and tuple(pilots.shape[1:]) == (U, F, K), f"complex (1 or N,{U},{F},{K})"),
            ("noise_feat", noise_feat.dtype == torch.float32 and tuple(noise_feat.shape) == (n,), "float32 (N,)"),
            ("mod_order", mod_order.dtype == torch.int32 and tuple(mod_order.shape) == (n * U,), "int32 (N*U,)"),
            ("llr", llr.dtype == torch.float32 and llr.dim() == 5 and tuple(llr.shape[:4]) == (n, U, S, T)
             and 1 <= llr.shape[4] <= 8, f"float32 (N,{U},{S},{T},W<=8)"),
            ("chest", chest.dtype == torch.complex64 and tuple(chest.shape) == (n, U, S, T, B),
             f"complex64 (N,{U},{S},{T},{B})"))
        for name, ok, want in checks:
            if not ok:
                raise ValueError(f"forward_device: {name} must be {want}")
        s = _lib.slot_desc(cfg)
        need = self.lib.nrx_workspace_bytes(ctypes.byref(self._m), ctypes.byref(s), n, self.prec_id)
        if ws.dtype != torch.uint8 or ws.numel() < need:
            raise ValueError(f"forward_device: workspace must be a uint8 tensor of >= {need} bytes")

    # -- pipelined host-resident stream ------------------------------------------

    def run_stream(self, cfg, inputs, outputs, num_iterations: int):
        """Throughput entry for host-resident batches (a serving loop).

        inputs[i] = (y, pilots, noise_feat, mod_order) pinned CPU tensors of
        batch i, outputs[i] = (llr, chest) pinned CPU tensors it is written
        to.  H2D of batch i+1 and D2H of batch i-1 run on their own streams
        and overlap the forward of batch i (triple-buffered device inputs and
        outputs, so the copy engines never wait on a forward that is itself
        waiting for a buffer); returns after every output has landed in host
        memory.
        """
        torch = _require_cuda()
        if not inputs:
            return
        dev = self.device
        nbuf = 3
        s_in, s_cmp, s_out = (torch.cuda.Stream(device=dev) for _ in range(3))
        d_in = [tuple(torch.empty_like(t, device=dev) for t in inputs[0]) for _ in range(nbuf)]
        d_out = [tuple(torch.empty_like(t, device=dev) for t in outputs[0]) for _ in range(nbuf)]
        ws = self.workspace(cfg, inputs[0][0].shape[0])
        ev = {k: [torch.cuda.Event() for _ in range(nbuf)] for k in ("in", "cmp", "out")}
        started = [False] * nbuf
        for i, (src, dst) in enumerate(zip(inputs, outputs)):
            b = i % nbuf
            with torch.cuda.stream(s_in):
                if started[b]:
                    s_in.wait_event(ev["cmp"][b])          # forward i-nbuf done reading d_in[b]
                for d, h in zip(d_in[b], src):
                    d.copy_(h, non_blocking=True)
                ev["in"][b].record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev["in"][b])
                if started[b]:
                    s_cmp.wait_event(ev["out"][b])         # D2H i-nbuf done reading d_out[b]
                y, pil, nf, mods = d_in[b]
                self.forward_device(cfg, y, pil, nf, mods, num_iterations, d_out[b][0], d_out[b][1],
                                    workspace=ws, stream=s_cmp)
                ev["cmp"][b].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev["cmp"][b])
                for h, d in zip(dst, d_out[b]):
                    h.copy_(d, non_blocking=True)
                ev["out"][b].record(s_out)
            started[b] = True
        s_out.synchronize()

    # -- numpy entry with the reference's semantics ------------------------------

    def _staging(self, key, shape, dtype, pinned):
        torch = _require_cuda()
        tls = self._local()
        k = (key, tuple(shape), dtype, pinned)
        buf = tls.bufs.get(k)
        if buf is None:
            if pinned:
                buf = torch.empty(shape, dtype=dtype, pin_memory=True)
            else:
                buf = torch.empty(shape, dtype=dtype, device=self.device)
            tls.bufs[k] = buf
        return buf

    def _pinned_outputs(self, llr_shape, chest_shape):
        """Pinned host buffers the results are copied into and returned from
        (numpy views, no extra host copy).  A pool entry is reused only once
        the caller holds no reference to the arrays it returned (refcount of
        the owning ndarray back at its baseline); when all POOL entries are
        still referenced, fresh pageable arrays are returned instead."""
        torch = _require_cuda()
        tls = self._local()
        pool = tls.bufs.setdefault(("out_pool", tuple(llr_shape), tuple(chest_shape)), [])
        for ent in pool:
            if sys.getrefcount(ent[2]) <= 2 and sys.getrefcount(ent[3]) <= 2:  # the pool tuple + the argument
                return ent
        if len(pool) < self.POOL:
            h_llr = torch.empty(llr_shape, dtype=torch.float32, pin_memory=True)
            h_chest = torch.empty(chest_shape, dtype=torch.complex64, pin_memory=True)
            ent = (h_llr, h_chest, h_llr.numpy(), h_chest.numpy())
            pool.append(ent)
            return ent
        a, b = np.empty(llr_shape, np.float32), np.empty(chest_shape, np.complex64)
        return (torch.from_numpy(a), torch.from_numpy(b), a, b)

    POOL = 4

    def run_arrays(self, cfg, y: np.ndarray, pilot_vals: np.ndarray, noise_feat: np.ndarray,
                   mod_order: np.ndarray, num_iterations: int, llr_width: int, exact_inputs: bool = False):
        """numpy -> device -> numpy; returns (llr (N,U,S,T,W) f32, chest (N,U,S,T,B) c64).

        y (N,S,T,B) and pilot_vals (P,U,F,K) are shipped as complex64 unless
        ``exact_inputs`` (then complex128, so the float64 LS sees the same
        inputs as the reference).  Inputs are converted while being written
        into pinned staging (one pass); the results are pinned-memory arrays
        (see _pinned_outputs)."""
        return self.finish(self.enqueue_arrays(cfg, y, pilot_vals, noise_feat, mod_order, num_iterations,
                                               llr_width, exact_inputs))[:2]

    def enqueue_arrays(self, cfg, y, pilot_vals, noise_feat, mod_order, num_iterations, llr_width,
                       exact_inputs=False):
        """First half of run_arrays: stage the inputs, enqueue H2D, the forward
        and the D2H on this thread's stream; returns a handle for finish()."""
        torch = _require_cuda()
        cdt = torch.complex128 if exact_inputs else torch.complex64
        n = y.shape[0]
        U, S, T, B = cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, self.config.num_rx_ant
        tls = self._local()
        with torch.cuda.stream(tls.stream):
            h_y = self._staging("y", y.shape, cdt, True)
            _stage(torch, h_y, y)
            h_p = self._staging("p", pilot_vals.shape, cdt, True)
            _stage(torch, h_p, pilot_vals)
            h_n = self._staging("n", (n,), torch.float32, True)
            h_n.numpy()[...] = noise_feat
            h_m = self._staging("m", (n * U,), torch.int32, True)
            h_m.numpy()[...] = mod_order.reshape(-1)
            d_y = self._staging("y", y.shape, cdt, False)
            d_p = self._staging("p", pilot_vals.shape, cdt, False)
            d_n = self._staging("n", (n,), torch.float32, False)
            d_m = self._staging("m", (n * U,), torch.int32, False)
            for d, h in ((d_y, h_y), (d_p, h_p), (d_n, h_n), (d_m, h_m)):
                d.copy_(h, non_blocking=True)
            d_llr = self._staging("llr", (n, U, S, T, llr_width), torch.float32, False)
            d_chest = self._staging("chest", (n, U, S, T, B), torch.complex64, False)
            ws = self.workspace(cfg, n)
            self.forward_device(cfg, d_y, d_p, d_n, d_m, num_iterations, d_llr, d_chest, workspace=ws,
                                stream=tls.stream)
            h_llr, h_chest, llr_np, chest_np = self._pinned_outputs(d_llr.shape, d_chest.shape)
            h_llr.copy_(d_llr, non_blocking=True)
            h_chest.copy_(d_chest, non_blocking=True)
            h_flag = self._staging("flag", (4,), torch.uint8, True)
            h_flag.copy_(ws[:4], non_blocking=True)  # NRX_WS_FLAG_OFFSET: non-finite readout output
        return tls.stream, llr_np, chest_np, h_flag

    @staticmethod
    def finish(handle):
        """Wait for enqueue_arrays' work; returns (llr, chest, nonfinite) where
        nonfinite is the range-guard word of a tensor-core mode."""
        stream, llr_np, chest_np, h_flag = handle
        stream.synchronize()
        return llr_np, chest_np, bool(h_flag.numpy().any())

    def nonfinite_flag(self, workspace):
        """Device view of the range-guard word (NRX_WS_FLAG_OFFSET) of a
        workspace after forward_device: nonzero when a tensor-core readout
        wrote a non-finite output (fp16 operand overflow)."""
        return workspace[:4].view(_require_cuda().int32)
