"""CPU oracle for the NRX inference forward pass — TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference receiver path
``nrxsim.nrx.nrx_forward`` (/root/reference/pkg/src/nrxsim/nrx.py:345-385)
and everything it calls.  It exists to *check* the CUDA implementation in
``paper_2409_02912_b200``; the product never imports it.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may use it.

Pinning: the restatement is validated against golden vectors produced by the
reference itself (``tests/golden/make_golden.py`` imports the reference read
only and records inputs, weights, features and outputs), see
``tests/test_oracle_golden.py``.  Feature assembly is bit-exact against the
reference; network outputs agree to fp32 rounding (the GEMM accumulation
order is BLAS-internal in the reference).

Every function cites the reference file:line it restates.  All functions are
duck-typed on the config objects: anything with the attribute names of the
reference ``SlotConfig`` / ``NrxConfig`` / ``McsEntry`` / ``PilotBook`` works.

``dtype`` selects the arithmetic: float32 reproduces the reference's
precision, float64 gives a high-precision replay used to calibrate the
tolerance of both the reference and the GPU path.
"""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# slot geometry                                            (slot.py:92-116)
# ---------------------------------------------------------------------------


def comb_subcarriers(num_subcarriers: int, comb_size: int, ue: int) -> np.ndarray:
    """UE ``ue``'s pilot comb: every comb_size-th subcarrier from ue % comb
    (slot.py:92-93)."""
    return np.arange(ue % comb_size, num_subcarriers, comb_size)


def data_mask(cfg) -> np.ndarray:
    """(S, T) data-RE mask: every RE outside the pilot symbols (slot.py:102-107)."""
    m = np.ones((cfg.num_subcarriers, cfg.num_symbols), dtype=bool)
    m[:, list(cfg.pilot_symbols)] = False
    return m


# ---------------------------------------------------------------------------
# LS channel estimate                                   (classical.py:40-78)
# ---------------------------------------------------------------------------


def ls_estimate(y: np.ndarray, pilot_values: np.ndarray, cfg) -> np.ndarray:
    """LS channel estimate on the full grid, (U, S, T, B) complex128.

    y: (S, T, B) complex; pilot_values: (U, S, T) complex (``PilotBook.values``).
    Per UE: raw LS at the comb x pilot-symbol REs (classical.py:40-46),
    linear interpolation over subcarriers with linear extrapolation at the
    comb edges (classical.py:49-61), nearest-pilot-symbol hold over time with
    ties resolved to the earlier symbol (classical.py:71,77).
    """
    S, T, B = cfg.num_subcarriers, cfg.num_symbols, cfg.bs_antennas
    ps = np.asarray(cfg.pilot_symbols)
    if ps.size == 0:
        raise ValueError("LS estimation needs a non-empty pilot set")
    # nearest pilot symbol per t: argmin keeps the first minimum -> earlier symbol
    nearest = np.argmin(np.abs(np.arange(T)[:, None] - ps[None, :]), axis=1)
    out = np.empty((cfg.num_ues, S, T, B), dtype=np.complex128)
    y = np.asarray(y)
    for u in range(cfg.num_ues):
        sc = comb_subcarriers(S, cfg.comb_size, u)
        p = np.asarray(pilot_values)[u][np.ix_(sc, ps)]            # (F, K)
        scale = p.conj() / np.abs(p) ** 2                          # conj(p)/|p|^2
        raw = y[np.ix_(sc, ps)] * scale[..., None]                 # (F, K, B)
        if sc.size == 1:
            freq = np.broadcast_to(raw[0], (S,) + raw.shape[1:])
        else:
            step = sc[1] - sc[0]
            s = np.arange(S)
            j = np.clip((s - sc[0]) // step, 0, sc.size - 2)
            frac = ((s - sc[j]) / step).reshape(-1, 1, 1)
            freq = raw[j] + frac * (raw[j + 1] - raw[j])           # (S, K, B)
        out[u] = freq[:, nearest, :]
    return out


# ---------------------------------------------------------------------------
# features                                                (nrx.py:159-213)
# ---------------------------------------------------------------------------


def positional_encoding(cfg, ue: int, include_freq: bool = True) -> np.ndarray:
    """(S, T, 2) float32: [distance to nearest pilot symbol / T, distance to
    nearest comb subcarrier of the UE / S] (nrx.py:159-173)."""
    S, T = cfg.num_subcarriers, cfg.num_symbols
    ps = np.asarray(cfg.pilot_symbols)
    dt = np.abs(np.arange(T)[:, None] - ps[None, :]).min(axis=1) / T
    sc = comb_subcarriers(S, cfg.comb_size, ue)
    df = np.abs(np.arange(S)[:, None] - sc[None, :]).min(axis=1) / S
    if not include_freq:
        df = np.zeros_like(df)
    pe = np.empty((S, T, 2), dtype=np.float32)
    pe[..., 0] = dt[None, :]
    pe[..., 1] = df[:, None]
    return pe


def interleave_re_im(x: np.ndarray) -> np.ndarray:
    """Complex (..., B) -> float32 (..., 2B) as re0, im0, re1, im1, ...
    (nrx.py:176-181)."""
    out = np.empty(x.shape + (2,), dtype=np.float32)
    out[..., 0] = x.real
    out[..., 1] = x.imag
    return out.reshape(x.shape[:-1] + (2 * x.shape[-1],))


def noise_feature(n0) -> np.ndarray:
    """log10 of the float32 noise power floored at 1e-30, float32 (nrx.py:199-201)."""
    return np.log10(np.maximum(np.asarray(n0, dtype=np.float32), np.float32(1e-30)))


def input_channels(config) -> int:
    """4B + 2 (+1 with the noise plane) (nrx.py:84-86)."""
    return 4 * config.num_rx_ant + 2 + (1 if config.include_noise_plane else 0)


def assemble_features(y, ls, n0, cfg, config) -> np.ndarray:
    """(N, U, S, T, C_in) float32 network input (nrx.py:184-202).

    Channels: [y re/im interleaved (2B)] [LS re/im interleaved (2B)]
    [dt, df] [log10 N0 plane (optional)].
    """
    n, u = ls.shape[0], ls.shape[1]
    S, T = cfg.num_subcarriers, cfg.num_symbols
    b2 = 2 * cfg.bs_antennas
    f = np.empty((n, u, S, T, input_channels(config)), dtype=np.float32)
    f[..., :b2] = interleave_re_im(y)[:, None]
    f[..., b2:2 * b2] = interleave_re_im(ls)
    for ue in range(u):
        f[:, ue, ..., 2 * b2:2 * b2 + 2] = positional_encoding(cfg, ue, config.include_freq_encoding)
    if config.include_noise_plane:
        f[..., -1] = noise_feature(n0).reshape(-1, 1, 1, 1)
    return f


def pilot_book_values(books, n: int):
    """Yield the (U, S, T) pilot array of sample i for a PilotBook or a
    per-sample list of books (nrx.py:210-212)."""
    for i in range(n):
        book = books[i] if isinstance(books, (list, tuple)) else books
        yield np.asarray(book.values)


# ---------------------------------------------------------------------------
# network                                     (nrx.py:221-342, autodiff.py)
# ---------------------------------------------------------------------------


def conv2d_same(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Stride-1 zero-'same'-padded NHWC convolution (autodiff.py:302-350).

    out[n,h,v,o] = sum_{a,b,i} xpad[n, h+a, v+b, i] * w[a, b, i, o]; the
    contraction is one GEMM over columns ordered (a, b, channel), the order
    the reference's im2col uses.
    """
    n, h, wd, c = x.shape
    kh, kw, ci, co = w.shape
    if ci != c:
        raise ValueError(f"conv2d channel mismatch: input {x.shape} vs kernel {w.shape}")
    ph, pw = kh // 2, kw // 2
    xp = np.zeros((n, h + 2 * ph, wd + 2 * pw, c), dtype=x.dtype)
    xp[:, ph:ph + h, pw:pw + wd] = x
    taps = [xp[:, a:a + h, b:b + wd, :] for a in range(kh) for b in range(kw)]
    cols = np.stack(taps, axis=3).reshape(n * h * wd, kh * kw * c)
    return (cols @ w.reshape(kh * kw * ci, co)).reshape(n, h, wd, co)


def mlp(x: np.ndarray, w: dict, prefix: str) -> np.ndarray:
    """relu(x W0 + b0) W1 + b1 on the last axis, no output activation (nrx.py:221-229)."""
    lead = x.shape[:-1]
    flat = x.reshape(-1, x.shape[-1])
    hid = np.maximum(flat @ w[f"{prefix}.fc0.w"] + w[f"{prefix}.fc0.b"], 0)
    out = hid @ w[f"{prefix}.fc1.w"] + w[f"{prefix}.fc1.b"]
    return out.reshape(lead + (out.shape[-1],))


def conv_block(x: np.ndarray, w: dict, prefix: str) -> np.ndarray:
    """conv(relu(conv(x) + b0)) + b1 (nrx.py:232-234)."""
    hid = np.maximum(conv2d_same(x, w[f"{prefix}.conv0.w"]) + w[f"{prefix}.conv0.b"], 0)
    return conv2d_same(hid, w[f"{prefix}.conv1.w"]) + w[f"{prefix}.conv1.b"]


def sum_others(x: np.ndarray, axis: int) -> np.ndarray:
    """For every slice u along ``axis``: sum of the other slices, reduced in
    float64 then cast back (autodiff.py:276-294).  A single slice gives 0."""
    acc = x.astype(np.float64)
    return (acc.sum(axis=axis, keepdims=True) - acc).astype(x.dtype)


def _as_array_dict(w: dict, dtype) -> dict:
    return {k: np.asarray(getattr(v, "data", v), dtype=dtype) for k, v in w.items()}


def forward_graph(features: np.ndarray, w: dict, config, mods: np.ndarray,
                  num_iterations: int | None = None, dtype=np.float32,
                  return_state: bool = False):
    """Inference-mode network on assembled features (nrx.py:302-342).

    features: (N, U, S, T, C_in); mods: (N, U) modulation order per slab.
    Returns (llr_slabs, chest_slabs) where llr_slabs is a list of
    (slab_indices, (n_slabs, S, T, width)) groups — one group for the
    single/masking variants, one per present IO order for var_io — and
    chest_slabs is (N*U, S, T, 2B).
    """
    n_it = config.num_iterations if num_iterations is None else int(num_iterations)
    if not 1 <= n_it <= config.num_iterations:
        raise ValueError(f"inference depth {n_it} outside [1, {config.num_iterations}]")
    allowed = set(config.io_modulations) if config.variant == "var_io" else set(range(1, config.m_max + 1))
    bad = set(int(m) for m in np.unique(mods)) - allowed
    if bad:
        raise ValueError(f"modulation orders {sorted(bad)} not supported by this model")
    wd = _as_array_dict(w, dtype)
    n, u = features.shape[:2]
    x = np.asarray(features, dtype=dtype).reshape((n * u,) + features.shape[2:])
    b4 = 4 * config.num_rx_ant
    pos = x[..., b4:b4 + 2]
    mod_slab = np.asarray(mods).reshape(-1)

    # state init, per-modulation weights for var_io           (nrx.py:237-249)
    if config.variant == "var_io":
        state = np.empty(x.shape[:3] + (config.d_s,), dtype=dtype)
        for m in config.io_modulations:
            idx = np.flatnonzero(mod_slab == m)
            if idx.size:
                state[idx] = conv_block(x[idx], wd, f"state_init.m{m}")
    else:
        state = conv_block(x, wd, "state_init")
    init_state = state

    # shared iteration block, all UEs read pre-update states  (nrx.py:252-263)
    for _ in range(n_it):
        msg = mlp(state, wd, "iteration.msg")
        agg = sum_others(msg.reshape((n, u) + msg.shape[1:]), axis=1).reshape(msg.shape)
        upd_in = np.concatenate([state, agg, pos], axis=-1)
        state = state + conv_block(upd_in, wd, "iteration.update")

    # readouts after the last iteration only                  (nrx.py:266-281,338-340)
    if config.variant == "var_io":
        groups = []
        for m in config.io_modulations:
            idx = np.flatnonzero(mod_slab == m)
            if idx.size:
                groups.append((idx, mlp(state[idx], wd, f"readout_llr.m{m}")))
    else:
        groups = [(np.arange(n * u), mlp(state, wd, "readout_llr"))]
    chest = mlp(state, wd, "readout_chest")
    if return_state:
        return groups, chest, init_state, state
    return groups, chest


def llr_width(config, modulation_order: int) -> int:
    """nrx.py:88-89."""
    return modulation_order if config.variant == "var_io" else config.m_max


def nrx_forward(y, books, cfg, mcs_per_ue, w, config, n0, num_iterations=None,
                apply_mask=True, dtype=np.float32, return_features=False):
    """Full receiver pass (nrx.py:345-385): validation, LS, features, network,
    per-UE LLR packing with label-prefix masking, planar chest decode."""
    unsupported = [m.index for m in mcs_per_ue if m.index not in config.supported_mcs]
    if unsupported:
        raise ValueError(f"MCS indices {unsupported} not in the model's supported set {config.supported_mcs}")
    y = np.asarray(y)
    single = y.ndim == 3
    if single:
        y = y[None]
    n = y.shape[0]
    n0_arr = np.full(n, n0, dtype=np.float64) if np.isscalar(n0) else np.asarray(n0)
    ls = np.stack([ls_estimate(y[i], vals, cfg) for i, vals in enumerate(pilot_book_values(books, n))])
    feats = assemble_features(y, ls, n0_arr, cfg, config)
    mods = np.tile([m.modulation_order for m in mcs_per_ue], (n, 1))
    groups, chest_slabs = forward_graph(feats, w, config, mods, num_iterations, dtype=dtype)

    U, S, T, B = cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, cfg.bs_antennas
    width = [llr_width(config, mcs_per_ue[ue].modulation_order) for ue in range(U)]
    full = np.zeros((n, U, S, T, max(width)), dtype=np.float32)
    for idx, vals in groups:
        full[idx // U, idx % U, ..., :vals.shape[-1]] = vals
    llrs = []
    for ue in range(U):
        m = mcs_per_ue[ue].modulation_order
        grid = full[:, ue, ..., :width[ue]]
        if apply_mask and config.variant != "var_io":
            if m > config.m_max:
                raise ValueError(f"cannot mask to order {m} from width {config.m_max}")
            grid = grid[..., :m]                                   # nrx.py:284-289
        llrs.append(grid[0] if single else grid)
    # planar decode: first B channels real, last B imaginary   (nrx.py:382-384)
    ch = chest_slabs.reshape(n, U, S, T, 2, B)
    chest = (ch[..., 0, :] + 1j * ch[..., 1, :]).astype(np.complex64)
    chest = chest[0] if single else chest
    if return_features:
        return llrs, chest, feats
    return llrs, chest


# ---------------------------------------------------------------------------
# weights                                      (nrx.py:92-133, autodiff.py:528-542)
# ---------------------------------------------------------------------------


def expected_shapes(config) -> dict:
    """name -> shape of every weight tensor (nrx.py:92-120)."""
    k, ds, hid = config.kernel_size, config.d_s, config.hidden_width or config.d_s
    cin = input_channels(config)
    shapes = {}

    def block(prefix, c0):
        shapes.update({f"{prefix}.conv0.w": (k, k, c0, ds), f"{prefix}.conv0.b": (ds,),
                       f"{prefix}.conv1.w": (k, k, ds, ds), f"{prefix}.conv1.b": (ds,)})

    def dense2(prefix, out):
        shapes.update({f"{prefix}.fc0.w": (ds, hid), f"{prefix}.fc0.b": (hid,),
                       f"{prefix}.fc1.w": (hid, out), f"{prefix}.fc1.b": (out,)})

    if config.variant == "var_io":
        for m in config.io_modulations:
            block(f"state_init.m{m}", cin)
            dense2(f"readout_llr.m{m}", m)
    else:
        block("state_init", cin)
        dense2("readout_llr", config.m_max)
    dense2("iteration.msg", ds)
    block("iteration.update", 2 * ds + 2)
    dense2("readout_chest", 2 * config.num_rx_ant)
    return shapes


def init_weights(config, seed: int) -> dict:
    """Glorot-uniform kernels, zero biases, float32, drawn in sorted-name
    order from default_rng((seed, 0x17EC)) (nrx.py:123-133, autodiff.py:528-542)."""
    rng = np.random.default_rng((seed, 0x17EC))
    out = {}
    for name, shape in sorted(expected_shapes(config).items()):
        if name.endswith(".b"):
            out[name] = np.zeros(shape, dtype=np.float32)
            continue
        if len(shape) == 4:
            fan_in, fan_out = shape[0] * shape[1] * shape[2], shape[0] * shape[1] * shape[3]
        else:
            fan_in, fan_out = shape
        lim = np.sqrt(6.0 / (fan_in + fan_out))
        out[name] = rng.uniform(-lim, lim, size=shape).astype(np.float32)
    return out


def perturb_biases(w: dict, seed: int = 99, scale: float = 0.1) -> dict:
    """Bias-exercising variant of a weight set: every bias
    drawn from N(0, scale^2); kernels unchanged."""
    rng = np.random.default_rng(seed)
    out = {}
    for name in sorted(w):
        arr = np.asarray(getattr(w[name], "data", w[name]), dtype=np.float32)
        out[name] = (rng.normal(0.0, scale, size=arr.shape).astype(np.float32)
                     if name.endswith(".b") else arr.copy())
    return out
