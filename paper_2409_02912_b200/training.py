"""Training of the NRX on the GPU.

The reference trains with its own numpy autodiff on the CPU (multi-loss
BCE over the readouts of every iteration + gamma * MSE on the channel
readout, Adam; training.py:180-234, autodiff.py:358-525).  Here one training
step is the same graph in PyTorch autograd on the device: convolutions and
dense layers, forward and backward, run on hand-written kernels (by default
the tcgen05 fp32x3 GEMMs of csrc/k_train_tc.cu; the fp32 SIMT kernels of
csrc/k_train.cu or cuDNN / cuBLAS on request), torch autograd sequences them
and does the elementwise glue, the inputs come from the GPU slot generator
and the LS/feature kernel, and the Adam update (csrc/k_train.cu) follows the
reference's formula exactly.

Parity (tests/test_training_cpu.py, against tests/golden/train_*.npz made by
the reference's own train_step): loss, every gradient and the weights after
one Adam step, for the masking and var_io variants with inactive UEs.

Reference interfaces mirrored (file:line under /root/reference/pkg/src/nrxsim):
  nrx_forward_graph(training=True), _mlp, _conv_block,
  _grouped_state_init, cgnn_iteration, readout_llrs / readout_chest  nrx.py:221-342
  bce_with_logits (masked mean), mse (masked mean)                   autodiff.py:358-420
  train_step (per-iteration group weighting, gamma)                  training.py:180-234
  AdamState / adam_step                                              autodiff.py:485-525
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def _torch():
    import torch
    return torch


def fp32_math():
    """Context for the reference's fp32 arithmetic on the device: cuDNN
    convolutions default to TF32 on tensor cores (torch.backends.cudnn.
    allow_tf32), which would silently change the training graph's numerics;
    this turns TF32 off for convolutions and matmuls (forward and backward
    run inside it in train_step)."""
    import contextlib
    torch = _torch()

    @contextlib.contextmanager
    def ctx():
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        try:
            with torch.backends.cudnn.flags(enabled=True, allow_tf32=False):
                yield
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev
    return ctx()


def _nrx_lib():
    from . import _lib
    return _lib.load()


_CONV_FN = None
_CONV_TC_FN = None
_TC_WS = {}


def _tc_workspace(torch, device, nbytes):
    """One growing device workspace per device for the tensor-core training
    GEMMs (every op of a step runs on the same stream, so they can share it)."""
    ws = _TC_WS.get(device)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        _TC_WS[device] = ws
    return ws


def _nrx_conv_tc_fn():
    """torch.autograd.Function over the tcgen05 fp32x3 GEMMs of
    csrc/k_train_tc.cu (include/nrx_train.h nrx_train_conv_tc_*): the same
    three operators as _nrx_conv_fn at fp32 accuracy on the tensor cores."""
    global _CONV_TC_FN
    if _CONV_TC_FN is not None:
        return _CONV_TC_FN
    torch = _torch()

    def _stream(t):
        return torch.cuda.current_stream(t.device).cuda_stream

    def _ws(lib, x_shape, cin, cout, k, device):
        n, S, T = x_shape[0], x_shape[1], x_shape[2]
        need = lib.nrx_train_tc_workspace(n, S, T, cin, cout, k)
        if need == 0:
            raise RuntimeError(f"nrx_train_tc: unsupported shape {tuple(x_shape)} x ({k},{k},{cin},{cout})")
        return _tc_workspace(torch, device, need), need

    class NrxConvTc(torch.autograd.Function):
        @staticmethod
        def forward(ctx, x, w):
            x = x.contiguous()
            w = w.contiguous()
            n, S, T, cin = x.shape
            k, cout = w.shape[0], w.shape[3]
            lib = _nrx_lib()
            ws, nb = _ws(lib, x.shape, cin, cout, k, x.device)
            y = torch.empty((n, S, T, cout), dtype=torch.float32, device=x.device)
            code = lib.nrx_train_conv_tc_fwd(n, S, T, cin, cout, k, x.data_ptr(), w.data_ptr(), y.data_ptr(),
                                             ws.data_ptr(), nb, _stream(x))
            if code:
                raise RuntimeError(f"nrx_train_conv_tc_fwd failed ({code})")
            ctx.save_for_backward(x, w)
            return y

        @staticmethod
        def backward(ctx, dy):
            x, w = ctx.saved_tensors
            dy = dy.contiguous()
            n, S, T, cin = x.shape
            k, cout = w.shape[0], w.shape[3]
            lib = _nrx_lib()
            ws, nb = _ws(lib, x.shape, cin, cout, k, x.device)
            dx = dw = None
            if ctx.needs_input_grad[0]:
                dx = torch.empty_like(x)
                code = lib.nrx_train_conv_tc_dgrad(n, S, T, cin, cout, k, dy.data_ptr(), w.data_ptr(),
                                                   dx.data_ptr(), ws.data_ptr(), nb, _stream(dy))
                if code:
                    raise RuntimeError(f"nrx_train_conv_tc_dgrad failed ({code})")
            if ctx.needs_input_grad[1]:
                dw = torch.empty_like(w)
                code = lib.nrx_train_conv_tc_wgrad(n, S, T, cin, cout, k, x.data_ptr(), dy.data_ptr(),
                                                   dw.data_ptr(), ws.data_ptr(), nb, _stream(dy))
                if code:
                    raise RuntimeError(f"nrx_train_conv_tc_wgrad failed ({code})")
            return dx, dw

    _CONV_TC_FN = NrxConvTc
    return NrxConvTc


def _nrx_conv_fn():
    """torch.autograd.Function over the hand-written fp32 kernels of
    csrc/k_train.cu (include/nrx_train.h): 'same' convolution / dense layer
    forward, input gradient and kernel gradient (autodiff.py:302-350 and the
    matmul VJPs)."""
    global _CONV_FN
    if _CONV_FN is not None:
        return _CONV_FN
    torch = _torch()

    def _stream(t):
        return torch.cuda.current_stream(t.device).cuda_stream

    class NrxConv(torch.autograd.Function):
        @staticmethod
        def forward(ctx, x, w):
            # x (n, S, T, cin) NHWC, w (k, k, cin, cout)
            x = x.contiguous()
            w = w.contiguous()
            n, S, T, cin = x.shape
            k, cout = w.shape[0], w.shape[3]
            y = torch.empty((n, S, T, cout), dtype=torch.float32, device=x.device)
            code = _nrx_lib().nrx_train_conv_fwd(n, S, T, cin, cout, k, x.data_ptr(), w.data_ptr(), None,
                                                 y.data_ptr(), _stream(x))
            if code:
                raise RuntimeError(f"nrx_train_conv_fwd failed ({code})")
            ctx.save_for_backward(x, w)
            return y

        @staticmethod
        def backward(ctx, dy):
            x, w = ctx.saved_tensors
            dy = dy.contiguous()
            n, S, T, cin = x.shape
            k, cout = w.shape[0], w.shape[3]
            lib = _nrx_lib()
            dx = dw = None
            if ctx.needs_input_grad[0]:
                dx = torch.empty_like(x)
                code = lib.nrx_train_conv_dgrad(n, S, T, cin, cout, k, dy.data_ptr(), w.data_ptr(), dx.data_ptr(),
                                                _stream(dy))
                if code:
                    raise RuntimeError(f"nrx_train_conv_dgrad failed ({code})")
            if ctx.needs_input_grad[1]:
                dw = torch.empty_like(w)
                code = lib.nrx_train_conv_wgrad(n, S, T, cin, cout, k, x.data_ptr(), dy.data_ptr(), dw.data_ptr(),
                                                None, _stream(dy))
                if code:
                    raise RuntimeError(f"nrx_train_conv_wgrad failed ({code})")
            return dx, dw

    _CONV_FN = NrxConv
    return NrxConv


class TorchNrxGraph:
    """The NRX graph on torch tensors.  ``params`` maps the reference's weight
    names to leaf tensors (float32, requires_grad).

    kernels="nrx_tc" (default on CUDA devices) runs every convolution and
    dense layer, forward and backward, on the tcgen05 fp32x3 GEMMs of
    csrc/k_train_tc.cu; kernels="nrx" on the hand-written fp32 SIMT kernels of
    csrc/k_train.cu; torch autograd only sequences them and does the
    elementwise glue (bias, ReLU, residual, concat, sum of others, losses).
    kernels="torch" uses cuDNN / cuBLAS (with TF32 off, see fp32_math)."""

    def __init__(self, config, weights: dict, device="cpu", kernels=None):
        torch = _torch()
        self.config = config
        self.device = torch.device(device)
        self.kernels = kernels or ("nrx_tc" if self.device.type == "cuda" else "torch")
        if self.kernels not in ("nrx", "nrx_tc", "torch"):
            raise ValueError(f"unknown kernels {self.kernels!r}")
        if self.kernels != "torch" and self.device.type != "cuda":
            raise ValueError(f"kernels={self.kernels!r} needs a CUDA device")
        self.params = {k: torch.tensor(np.asarray(getattr(v, "data", v), dtype=np.float32), device=self.device,
                                       requires_grad=True) for k, v in weights.items()}

    def _conv_fn(self):
        return _nrx_conv_tc_fn() if self.kernels == "nrx_tc" else _nrx_conv_fn()

    def numpy_weights(self) -> dict:
        return {k: v.detach().cpu().numpy().copy() for k, v in self.params.items()}

    # -- blocks -------------------------------------------------------------
    def _conv(self, x, name):
        """'same' k x k convolution of NHWC x (H = subcarrier, W = symbol)
        with a (k, k, Cin, Cout) kernel (autodiff.py:324-350)."""
        w = self.params[name]
        if self.kernels != "torch":
            return self._conv_fn().apply(x, w)
        F = _torch().nn.functional
        k = w.shape[0]
        y = F.conv2d(x.permute(0, 3, 1, 2), w.permute(3, 2, 0, 1), padding=k // 2)
        return y.permute(0, 2, 3, 1)

    def _dense(self, x, name):
        """x (..., cin) @ W (cin, cout): a 1x1 convolution of the flattened rows."""
        w = self.params[name]
        if self.kernels == "torch":
            return x @ w
        lead = x.shape[:-1]
        rows = x.reshape(-1, 1, 1, x.shape[-1])
        y = self._conv_fn().apply(rows, w.reshape(1, 1, w.shape[0], w.shape[1]))
        return y.reshape(lead + (w.shape[1],))

    def _conv_block(self, x, prefix):
        torch = _torch()
        h = torch.relu(self._conv(x, f"{prefix}.conv0.w") + self.params[f"{prefix}.conv0.b"])
        return self._conv(h, f"{prefix}.conv1.w") + self.params[f"{prefix}.conv1.b"]

    def _mlp(self, x, prefix):
        torch = _torch()
        p = self.params
        h = torch.relu(self._dense(x, f"{prefix}.fc0.w") + p[f"{prefix}.fc0.b"])
        return self._dense(h, f"{prefix}.fc1.w") + p[f"{prefix}.fc1.b"]

    def _groups(self, mods):
        c = self.config
        if c.variant != "var_io":
            return [(None, np.arange(mods.size))]
        return [(m, np.flatnonzero(mods == m)) for m in c.io_modulations if np.any(mods == m)]

    # -- graph --------------------------------------------------------------
    def forward(self, feats, mods, active, num_iterations=None, training=True, collect_chest=True):
        """feats (N, U, S, T, Cin) float32 tensor, mods (N, U) ints, active
        (N, U) -> (llr_groups per iteration: [(tensor, slab idx)], chest per
        iteration) as nrx_forward_graph (nrx.py:302-342)."""
        torch = _torch()
        c = self.config
        n, u = feats.shape[0], feats.shape[1]
        n_it = c.num_iterations if num_iterations is None else int(num_iterations)
        x = feats.reshape((n * u,) + tuple(feats.shape[2:]))
        pos = x[..., 4 * c.num_rx_ant:4 * c.num_rx_ant + 2]
        mods = np.asarray(mods).reshape(-1)
        act = torch.as_tensor(np.asarray(active, dtype=np.float32), device=feats.device).reshape(n, u, 1, 1, 1)
        if c.variant != "var_io":
            state = self._conv_block(x, "state_init")
        else:
            parts, order = [], []
            for m, idx in self._groups(mods):
                it = torch.as_tensor(idx, device=feats.device)
                parts.append(self._conv_block(x[it], f"state_init.m{m}"))
                order.append(idx)
            inv = torch.as_tensor(np.argsort(np.concatenate(order)), device=feats.device)
            state = torch.cat(parts)[inv]
        llrs, chests = [], []

        def readouts(st):
            groups = []
            for m, idx in self._groups(mods):
                it = torch.as_tensor(idx, device=feats.device)
                prefix = "readout_llr" if m is None else f"readout_llr.m{m}"
                groups.append((self._mlp(st if m is None else st[it], prefix), idx))
            return groups

        for _ in range(n_it):
            msg = self._mlp(state, "iteration.msg")
            shaped = (msg.reshape((n, u) + tuple(msg.shape[1:])) * act).double()
            agg = (shaped.sum(dim=1, keepdim=True) - shaped).float()      # sum_others in float64
            upd_in = torch.cat([state, agg.reshape(state.shape), pos], dim=-1)
            state = state + self._conv_block(upd_in, "iteration.update")
            if training:
                llrs.append(readouts(state))
                if collect_chest:
                    chests.append(self._mlp(state, "readout_chest"))
        if not training:
            llrs = [readouts(state)]
            chests = [self._mlp(state, "readout_chest")]
        return llrs, chests


def _bce_masked_sum(logits, bits, mask):
    """sum(mask * ln(1 + exp(-(2b - 1) z))) (autodiff.py:358-394, overflow-free split)."""
    torch = _torch()
    a = -(2.0 * bits - 1.0) * logits
    per = torch.clamp(a, min=0) + torch.log1p(torch.exp(-a.abs()))
    return (per * mask).sum()


def training_loss(graph: TorchNrxGraph, feats, labels, label_mask, chest_target, active, mods, gamma: float):
    """The multi-loss of train_step (training.py:189-222): per iteration the
    masked-mean BCE over all LLR groups, plus gamma times the masked MSE of
    the channel readout; returns (total, bce, mse) tensors."""
    torch = _torch()
    n, u = labels.shape[0], labels.shape[1]
    flat_lab = labels.reshape((n * u,) + tuple(labels.shape[2:]))
    flat_mask = label_mask.reshape((n * u,) + tuple(label_mask.shape[2:]))
    flat_tgt = chest_target.reshape((n * u,) + tuple(chest_target.shape[2:]))
    cmask = torch.as_tensor(np.asarray(active, dtype=np.float32), device=labels.device).reshape(n * u, 1, 1, 1)
    cmask = cmask.expand_as(flat_tgt)
    llr_groups, chests = graph.forward(feats, mods, active, training=True, collect_chest=gamma > 0)
    bce, mse = [], []
    for it, groups in enumerate(llr_groups):
        num, den = 0.0, 0.0
        for t, idx in groups:
            ii = torch.as_tensor(idx, device=labels.device)
            w = t.shape[-1]
            mk = flat_mask[ii][..., :w]
            share = mk.sum()
            if float(share) == 0.0:
                continue   # a group of inactive slabs stays out of the graph (training.py:205-207)
            den = den + share
            num = num + _bce_masked_sum(t, flat_lab[ii][..., :w], mk)
        bce.append(num / den)
        if gamma > 0:
            mse.append((((chests[it] - flat_tgt) ** 2) * cmask).sum() / cmask.sum())
    bce_t = torch.stack(bce).sum()
    mse_t = torch.stack(mse).sum() if mse else torch.zeros((), device=labels.device)
    total = bce_t + gamma * mse_t if mse else bce_t
    return total, bce_t, mse_t


@dataclass
class Adam:
    """Bias-corrected Adam with the reference's update (autodiff.py:485-525):
    p -= (lr / (1 - b1^t)) * m / (sqrt(v / (1 - b2^t)) + eps)."""

    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    epsilon: float = 1e-8
    t: int = 0
    m: dict = field(default_factory=dict)
    v: dict = field(default_factory=dict)

    def step(self, params: dict, names) -> None:
        torch = _torch()
        self.t += 1
        c1 = 1.0 - self.beta1 ** self.t
        c2 = 1.0 - self.beta2 ** self.t
        with torch.no_grad():
            names = list(names)
            # the reference checks each gradient just before its update and raises at the
            # first bad one (earlier parameters already updated, autodiff.py:509-515); the
            # finiteness of all gradients is read back in one device sync instead of one per tensor
            bad, why = len(names), None
            for i, k in enumerate(names):
                if params[k].grad is None:
                    bad, why = i, f"missing gradient for parameter '{k}'"
                    break
            checked = [params[k].grad for k in names[:bad]]
            if checked:
                ok = torch.stack([torch.isfinite(g).all() for g in checked]).cpu().tolist()
                if not all(ok):
                    bad = ok.index(False)
                    why = f"non-finite gradient for parameter '{names[bad]}'"
            for i, k in enumerate(names):
                if i == bad:
                    raise ValueError(why)
                p = params[k]
                g = p.grad
                if k not in self.m:
                    self.m[k] = torch.zeros_like(p)
                    self.v[k] = torch.zeros_like(p)
                m, v = self.m[k], self.v[k]
                if p.is_cuda:  # hand-written update kernel (csrc/k_train.cu)
                    code = _nrx_lib().nrx_train_adam(p.numel(), p.data_ptr(), g.contiguous().data_ptr(),
                                                     m.data_ptr(), v.data_ptr(), self.lr, self.beta1, self.beta2,
                                                     self.epsilon, self.t, torch.cuda.current_stream(p.device).cuda_stream)
                    if code:
                        raise RuntimeError(f"nrx_train_adam failed ({code})")
                    continue
                m.mul_(self.beta1).add_((1.0 - self.beta1) * g)
                v.mul_(self.beta2).add_((1.0 - self.beta2) * g * g)
                p.sub_((self.lr / c1) * m / (torch.sqrt(v / c2) + self.epsilon))


def train_step(graph: TorchNrxGraph, adam: Adam, feats, labels, label_mask, chest_target, active, mods,
               gamma: float) -> dict:
    """One multi-loss gradient step (training.py:180-234): only parameters
    the loss touched are updated (the chest head sits out at gamma = 0, a
    var_io group may sit out a batch)."""
    torch = _torch()
    for p in graph.params.values():
        p.grad = None
    with fp32_math():
        total, bce, mse = training_loss(graph, feats, labels, label_mask, chest_target, active, mods, gamma)
        if not torch.isfinite(total):
            raise RuntimeError(f"non-finite training loss {float(total)}")
        total.backward()
    touched = [k for k, p in graph.params.items() if p.grad is not None]
    adam.step(graph.params, touched)
    for p in graph.params.values():
        p.grad = None
    return {"total": float(total.detach()), "bce": float(bce.detach()), "mse": float(mse.detach())}


__all__ = ["TorchNrxGraph", "training_loss", "train_step", "Adam", "fp32_math"]


# ---------------------------------------------------------------------------
# GPU training loop: batches from the GPU slot generator
# ---------------------------------------------------------------------------

def gpu_features(config, cfg, batch, n0):
    """(N, U, S, T, Cin) float32 features of a generated batch by the LS /
    feature kernel (nrx_ls_features, float32 chunk-planar) — the reference's
    assemble_features(y, ls_features(...)) (nrx.py:184-213)."""
    import ctypes
    torch = _torch()
    from . import _lib
    from .nrx import noise_features
    lib = _lib.load()
    n, U, S, T = batch.y.shape[0], cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols
    geo = _lib.buffer_geometry(config, cfg, "fp32_simt")
    out = torch.zeros(n * U, geo["Cf"] // 4, geo["rows_slab"], 4, device=batch.y.device)
    nf = torch.as_tensor(noise_features(np.asarray(n0, dtype=np.float64), n), device=batch.y.device)
    st = torch.cuda.current_stream(batch.y.device).cuda_stream
    code = lib.nrx_ls_features(ctypes.byref(_lib.model_desc(config)), ctypes.byref(_lib.slot_desc(cfg)), n, 0,
                               batch.y.data_ptr(), int(batch.y.dtype == torch.complex128), batch.pilots.data_ptr(),
                               int(batch.pilots.dtype == torch.complex128), batch.pilots.shape[0], nf.data_ptr(),
                               out.data_ptr(), st)
    _lib.check(code, "nrx_ls_features")
    f = out.permute(0, 2, 1, 3).reshape(n * U, geo["rows_slab"], geo["Cf"])
    f = f[:, :S * geo["Tp"]].reshape(n, U, S, geo["Tp"], geo["Cf"])
    cin = 4 * config.num_rx_ant + 2 + int(bool(config.include_noise_plane))
    return f[:, :, :, :T, :cin].contiguous()


@dataclass
class GpuTrainConfig:
    """The knobs of the reference's TrainConfig (training.py:38-79) that the
    GPU loop uses; labels are iid bits (the LDPC code does not change the
    bit statistics the receiver sees)."""
    batch_size: int = 16
    steps: int = 1000
    snr_lo_db: float = -4.0
    snr_hi_db: float = 4.0
    gamma: float = 0.1
    learning_rate: float = 1e-3
    supported_mcs: tuple = (14,)
    seed: int = 0


def gpu_training_batch(source, config, table, tcfg: GpuTrainConfig, step: int):
    """One batch on the device: per slot an SNR uniform in [lo, hi] dB and a
    supported MCS per UE, slots from the GPU slot generator with the true
    effective channel as the chest target (re/im interleaved per antenna,
    the reference's layout, training.py:154-156), labels and label masks on
    the data REs."""
    torch = _torch()
    cfg, dev = source.cfg, source.device
    n, U, S, T, B = tcfg.batch_size, cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, cfg.bs_antennas
    rng = np.random.default_rng((tcfg.seed, 0x7A, step))
    snr = rng.uniform(tcfg.snr_lo_db, tcfg.snr_hi_db, size=n)
    n0 = 10.0 ** (-snr / 10.0)
    picks = rng.choice(np.asarray(tcfg.supported_mcs), size=(n, U))
    mods = np.vectorize(lambda i: table[int(i)].modulation_order)(picks).astype(np.int32)
    sb = source.generate(n, torch.as_tensor(mods.reshape(-1), device=dev), torch.as_tensor(n0, device=dev),
                         seed=(tcfg.seed << 20) ^ 0x7A17, first_slot=step * n, with_h_eff=True)
    width = config.m_max
    data = torch.as_tensor(np.asarray(cfg.data_mask), device=dev)                       # (S, T)
    m_t = torch.as_tensor(mods, device=dev).reshape(n, U, 1, 1, 1)
    j = torch.arange(width, device=dev).reshape(1, 1, 1, 1, width)
    lab = sb.labels.to(torch.int64).unsqueeze(-1)
    bits = ((lab >> (m_t - 1 - j).clamp(min=0)) & 1).to(torch.float32)
    mask = ((j < m_t) & data.reshape(1, 1, S, T, 1)).to(torch.float32)
    h = sb.h_eff
    tgt = torch.stack([h.real, h.imag], dim=-1).reshape(n, U, S, T, 2 * B).to(torch.float32)
    return sb, n0, mods, bits * mask, mask, tgt


def train_gpu(config, weights, source, table, tcfg: GpuTrainConfig, graph=None, adam=None, log_every: int = 0,
              progress=None):
    """The reference's train() loop (training.py:254-284) on the device.
    Returns (graph, adam, history of (step, losses))."""
    dev = source.device
    graph = graph or TorchNrxGraph(config, weights, dev)
    adam = adam or Adam(lr=tcfg.learning_rate)
    active = np.ones((tcfg.batch_size, source.cfg.num_ues), dtype=np.float32)
    hist = []
    for step in range(tcfg.steps):
        sb, n0, mods, labels, mask, tgt = gpu_training_batch(source, config, table, tcfg, step)
        feats = gpu_features(config, source.cfg, sb, n0)
        losses = train_step(graph, adam, feats, labels, mask, tgt, active, mods, tcfg.gamma)
        if log_every and step % log_every == 0:
            hist.append((step, losses))
        if progress is not None:
            progress(step, losses)
    return graph, adam, hist


__all__ += ["gpu_features", "GpuTrainConfig", "gpu_training_batch", "train_gpu"]
