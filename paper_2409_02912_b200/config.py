"""Host-side mirror of the reference receiver's configuration types.

The drop-in ``nrx_forward`` accepts the reference's own objects
(``nrxsim.slot.SlotConfig``/``PilotBook``/``McsEntry``, ``nrxsim.nrx.NrxConfig``
and its ``dict[str, ad.Tensor]`` weights) by duck typing.  This module gives
the same types to users (and to the GPU box, where the reference package is
not installed): same field names, same validation and error texts, same
weight naming and seeded initialisation, same NRXW checkpoint format.

Reference interfaces mirrored (file:line under /root/reference/pkg/src/nrxsim):
  McsEntry            slot.py:23-35      default_mcs_table  slot.py:38-44
  SlotConfig          slot.py:47-116     PilotBook          slot.py:119-127
  generate_pilots     slot.py:130-139    NrxConfig          nrx.py:37-89
  expected_shapes     nrx.py:92-120      init_weights       nrx.py:123-133
  checkpoint_save     nrx.py:395-417     checkpoint_load    nrx.py:420-471

Extension (labelled, not in the reference): modulation order 8 (256-QAM) is
accepted by ``McsEntry(..., allow_extension=True)`` and by the 256-QAM table
row ``extended_mcs_table()``; the network handles it as m_max=8 through the
same masked readout.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

REFERENCE_ORDERS = (2, 4, 6)
EXTENDED_ORDERS = (2, 4, 6, 8)
VARIANTS = ("single", "masking", "var_io")
CKPT_MAGIC = b"NRXW"
CKPT_VERSION = 1


@dataclass(frozen=True)
class McsEntry:
    """MCS table row: index, bits per symbol, code rate."""

    index: int
    modulation_order: int
    code_rate: float
    allow_extension: bool = field(default=False, compare=False, repr=False)

    def __post_init__(self):
        orders = EXTENDED_ORDERS if self.allow_extension else REFERENCE_ORDERS
        if self.modulation_order not in orders:
            raise ValueError(f"MCS {self.index}: unsupported modulation order {self.modulation_order}")
        if not 0.0 < self.code_rate < 1.0:
            raise ValueError(f"MCS {self.index}: code rate {self.code_rate} outside (0,1)")


def default_mcs_table() -> dict:
    """The reference's shipped rows (1024-denominator rates)."""
    return {9: McsEntry(9, 2, 679 / 1024), 14: McsEntry(14, 4, 553 / 1024),
            19: McsEntry(19, 6, 517 / 1024)}


def extended_mcs_table() -> dict:
    """Reference rows plus a 256-QAM row (EXTENSION: MCS 27, m=8, r=948/1024)."""
    table = default_mcs_table()
    table[27] = McsEntry(27, 8, 948 / 1024, allow_extension=True)
    return table


@dataclass(frozen=True)
class SlotConfig:
    """Slot geometry and antenna setup (same fields/validation as the reference)."""

    num_subcarriers: int = 24
    num_symbols: int = 14
    pilot_symbols: tuple = (2, 11)
    comb_size: int = 2
    num_ues: int = 2
    bs_antennas: int = 4
    ue_antennas: int = 2
    beams: tuple = None
    subcarrier_spacing_hz: float = 30e3
    cp_fraction: float = 0.07

    def __post_init__(self):
        if any(t < 0 or t >= self.num_symbols for t in self.pilot_symbols):
            raise ValueError(f"pilot symbols {self.pilot_symbols} outside [0,{self.num_symbols})")
        if not self.pilot_symbols:
            raise ValueError("at least one pilot symbol is required")
        if self.num_ues > self.comb_size:
            raise ValueError(f"{self.num_ues} UEs cannot share a comb of size {self.comb_size}")
        if self.beams is None:
            v = tuple(np.ones(self.ue_antennas) / np.sqrt(self.ue_antennas))
            object.__setattr__(self, "beams", tuple(v for _ in range(self.num_ues)))
        elif len(self.beams) > self.num_ues:
            object.__setattr__(self, "beams", tuple(self.beams[: self.num_ues]))
        norms = np.linalg.norm(self.beam_matrix, axis=1)
        if not np.allclose(norms, 1.0, atol=1e-9):
            raise ValueError(f"beam vectors must have unit norm, got {norms}")

    @property
    def beam_matrix(self) -> np.ndarray:
        return np.asarray(self.beams, dtype=np.complex128).reshape(self.num_ues, self.ue_antennas)

    def comb_subcarriers(self, ue: int) -> np.ndarray:
        return np.arange(ue % self.comb_size, self.num_subcarriers, self.comb_size)

    @property
    def data_mask(self) -> np.ndarray:
        m = np.ones((self.num_subcarriers, self.num_symbols), dtype=bool)
        m[:, list(self.pilot_symbols)] = False
        return m

    @property
    def num_data_res(self) -> int:
        return int(self.data_mask.sum())

    def data_re_indices(self):
        return np.nonzero(self.data_mask)


@dataclass(frozen=True)
class PilotBook:
    """Known pilot values per UE, (U, S, T) complex, zero off the UE's pilot REs."""

    values: np.ndarray
    config: SlotConfig


def qpsk_points() -> np.ndarray:
    """Gray QPSK with bit=0 on the positive half-axis, label index = 2*b0 + b1
    (constellation.py:58-82 at order 2)."""
    b0 = np.array([0, 0, 1, 1])
    b1 = np.array([0, 1, 0, 1])
    return ((1 - 2 * b0) + 1j * (1 - 2 * b1)) / np.sqrt(2.0)


def generate_pilots(cfg, slot_seed: int) -> PilotBook:
    """Unit-modulus QPSK pilots on each UE's comb at the pilot symbols, drawn
    from default_rng((slot_seed, ue, 0xD5)) (slot.py:130-139)."""
    pts = qpsk_points()
    vals = np.zeros((cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols), dtype=np.complex128)
    ps = list(cfg.pilot_symbols)
    for u in range(cfg.num_ues):
        rng = np.random.default_rng((int(slot_seed), u, 0xD5))
        sc = np.arange(u % cfg.comb_size, cfg.num_subcarriers, cfg.comb_size)
        vals[u][np.ix_(sc, ps)] = pts[rng.integers(0, 4, size=(sc.size, len(ps)))]
    return PilotBook(values=vals, config=cfg)


@dataclass(frozen=True)
class NrxConfig:
    """Receiver architecture (same fields, defaults and validation as the reference)."""

    d_s: int = 16
    num_iterations: int = 4
    kernel_size: int = 3
    hidden_width: int = None
    variant: str = "single"
    supported_mcs: tuple = (14,)
    m_max: int = 4
    io_modulations: tuple = ()
    num_rx_ant: int = 4
    include_noise_plane: bool = True
    include_freq_encoding: bool = True

    def __post_init__(self):
        if self.d_s < 4:
            raise ValueError(f"state depth d_s must be >= 4, got {self.d_s}")
        if self.num_iterations < 1:
            raise ValueError("need at least one iteration")
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown variant '{self.variant}'")
        if self.kernel_size % 2 == 0:
            raise ValueError("kernel size must be odd")
        if self.variant == "var_io" and not self.io_modulations:
            raise ValueError("var_io needs io_modulations")
        if any(i < 0 or i > 31 for i in self.supported_mcs):
            raise ValueError("MCS indices must fit the checkpoint bitmap (0..31)")
        if self.hidden_width is None:
            object.__setattr__(self, "hidden_width", self.d_s)

    @classmethod
    def from_table(cls, mcs_table, supported_mcs, variant="single", **kw):
        orders = tuple(mcs_table[i].modulation_order for i in supported_mcs)
        if variant == "single" and len(set(orders)) != 1:
            raise ValueError("single variant expects one modulation order")
        io = tuple(sorted(set(orders))) if variant == "var_io" else ()
        return cls(variant=variant, supported_mcs=tuple(supported_mcs), m_max=max(orders),
                   io_modulations=io, **kw)

    @property
    def hidden(self) -> int:
        return self.hidden_width or self.d_s

    @property
    def input_channels(self) -> int:
        return 4 * self.num_rx_ant + 2 + (1 if self.include_noise_plane else 0)

    def llr_width(self, modulation_order: int) -> int:
        return modulation_order if self.variant == "var_io" else self.m_max


def expected_shapes(config) -> dict:
    """Weight name -> shape; conv kernels (k, k, Cin, Cout), dense (in, out)."""
    k, d = config.kernel_size, config.d_s
    h = config.hidden_width or d
    cin = 4 * config.num_rx_ant + 2 + (1 if config.include_noise_plane else 0)
    out = {}

    def add_conv_block(prefix, c_in):
        for i, (ci, co) in enumerate(((c_in, d), (d, d))):
            out[f"{prefix}.conv{i}.w"] = (k, k, ci, co)
            out[f"{prefix}.conv{i}.b"] = (co,)

    def add_mlp(prefix, width):
        for i, (ci, co) in enumerate(((d, h), (h, width))):
            out[f"{prefix}.fc{i}.w"] = (ci, co)
            out[f"{prefix}.fc{i}.b"] = (co,)

    io_sets = [f".m{m}" for m in config.io_modulations] if config.variant == "var_io" else [""]
    for tag in io_sets:
        add_conv_block(f"state_init{tag}", cin)
        add_mlp(f"readout_llr{tag}", int(tag[2:]) if tag else config.m_max)
    add_mlp("iteration.msg", d)
    add_conv_block("iteration.update", 2 * d + 2)
    add_mlp("readout_chest", 2 * config.num_rx_ant)
    return out


def _glorot_limit(shape) -> float:
    if len(shape) == 4:
        rf = shape[0] * shape[1]
        fan_in, fan_out = rf * shape[2], rf * shape[3]
    elif len(shape) == 2:
        fan_in, fan_out = shape
    else:
        fan_in = fan_out = int(np.prod(shape))
    return float(np.sqrt(6.0 / (fan_in + fan_out)))


def init_weights(config, seed: int) -> dict:
    """Seeded Glorot-uniform kernels and zero biases (float32 numpy arrays).

    Same draw order as the reference (sorted names, one
    ``default_rng((seed, 0x17EC))`` stream), so for the same config and seed
    the arrays are bit-identical to ``nrxsim.nrx.init_weights(...)[k].data``.
    """
    rng = np.random.default_rng((seed, 0x17EC))
    weights = {}
    for name, shape in sorted(expected_shapes(config).items()):
        if name.endswith(".b"):
            weights[name] = np.zeros(shape, dtype=np.float32)
        else:
            lim = _glorot_limit(shape)
            weights[name] = rng.uniform(-lim, lim, size=shape).astype(np.float32)
    return weights


def weight_array(w) -> np.ndarray:
    """Accept a reference ``ad.Tensor`` (``.data``) or an array."""
    return np.asarray(getattr(w, "data", w))


def checkpoint_save(path, config, weights) -> None:
    """NRXW v1: magic, <7I config block, <I count, then per tensor
    <H name length, name, <B rank, <rank*I dims, f32 LE payload."""
    shapes = expected_shapes(config)
    if set(shapes) != set(weights):
        raise ValueError(f"weights do not match the configuration: {sorted(set(shapes) ^ set(weights))}")
    flags = int(bool(config.include_noise_plane)) | (2 * int(bool(config.include_freq_encoding)))
    bitmap = sum(1 << i for i in set(config.supported_mcs))
    parts = [CKPT_MAGIC, struct.pack("<7I", CKPT_VERSION, config.d_s, config.num_iterations,
                                     VARIANTS.index(config.variant), config.m_max, flags, bitmap),
             struct.pack("<I", len(weights))]
    for name in sorted(weights):
        arr = np.ascontiguousarray(weight_array(weights[name]), dtype="<f4")
        raw = name.encode()
        parts += [struct.pack("<H", len(raw)), raw, struct.pack("<B", arr.ndim),
                  struct.pack(f"<{arr.ndim}I", *arr.shape), arr.tobytes()]
    with open(path, "wb") as fh:
        fh.write(b"".join(parts))


def checkpoint_load(path):
    """Parse an NRXW file into (NrxConfig, dict of float32 arrays), validating
    names and shapes against the configuration it implies."""
    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[:4] != CKPT_MAGIC:
        raise ValueError(f"{path}: bad magic {blob[:4]!r}, expected {CKPT_MAGIC!r}")
    version, d_s, n_it, variant_id, m_max, flags, bitmap = struct.unpack_from("<7I", blob, 4)
    if version != CKPT_VERSION:
        raise ValueError(f"{path}: unsupported checkpoint version {version}")
    (count,) = struct.unpack_from("<I", blob, 32)
    off, tensors = 36, {}
    for _ in range(count):
        (nlen,) = struct.unpack_from("<H", blob, off)
        name = blob[off + 2:off + 2 + nlen].decode()
        off += 2 + nlen
        (rank,) = struct.unpack_from("<B", blob, off)
        dims = struct.unpack_from(f"<{rank}I", blob, off + 1)
        off += 1 + 4 * rank
        size = int(np.prod(dims)) if rank else 1
        tensors[name] = np.frombuffer(blob, dtype="<f4", count=size, offset=off).reshape(dims).copy()
        off += 4 * size
    if off != len(blob):
        raise ValueError(f"{path}: {len(blob) - off} trailing bytes")
    io_mods = tuple(sorted({int(n.split(".m", 1)[1].split(".", 1)[0])
                            for n in tensors if n.startswith("state_init.m")}))
    if "readout_chest.fc1.b" not in tensors:
        raise ValueError(f"{path}: checkpoint lacks readout_chest.fc1.b")
    first_conv = next(n for n in sorted(tensors) if n.startswith("state_init") and n.endswith("conv0.w"))
    config = NrxConfig(
        d_s=d_s, num_iterations=n_it, kernel_size=tensors[first_conv].shape[0],
        hidden_width=tensors["iteration.msg.fc0.w"].shape[1], variant=VARIANTS[variant_id],
        supported_mcs=tuple(i for i in range(32) if bitmap >> i & 1), m_max=m_max,
        io_modulations=io_mods, num_rx_ant=tensors["readout_chest.fc1.b"].size // 2,
        include_noise_plane=bool(flags & 1), include_freq_encoding=bool(flags & 2))
    cin = tensors[first_conv].shape[2]
    if cin != config.input_channels:
        raise ValueError(f"{path}: {first_conv} has {cin} input channels, config implies {config.input_channels}")
    shapes = expected_shapes(config)
    if set(shapes) != set(tensors):
        raise ValueError(f"{path}: tensor names do not match config: {sorted(set(shapes) ^ set(tensors))}")
    for name, shape in shapes.items():
        if tensors[name].shape != shape:
            raise ValueError(f"{path}: tensor '{name}' has shape {tensors[name].shape}, expected {shape}")
    return config, tensors
