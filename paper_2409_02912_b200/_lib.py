"""ctypes binding of the C ABI in include/nrx_b200.h (libnrx_b200.so).

The shared library is built in-tree (``make`` / ``__graft_entry__.build()``)
next to this file.  There is no fallback: if the library or a CUDA device is
missing, the GPU entry points raise instead of silently computing on the CPU.
"""

from __future__ import annotations

import ctypes
import os

NRX_MAX_PILOT_SYMBOLS = 16
NRX_MAX_IO = 4
NRX_FP32, NRX_BF16, NRX_FP16, NRX_FP32X3 = 0, 1, 2, 3
# "fp32": the reference's fp32 accuracy on the tensor cores (fp16 hi/lo operand
# split, three MMAs per product); "fp32_simt": the same gate on fp32 FFMA.
PRECISIONS = {"fp32": NRX_FP32X3, "fp32_simt": NRX_FP32, "bf16": NRX_BF16, "fp16": NRX_FP16}
VARIANT_IDS = {"single": 0, "masking": 1, "var_io": 2}

LIB_PATH = os.environ.get("NRX_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                           "libnrx_b200.so")

# every symbol include/nrx_b200.h and include/nrx_slotgen.h declare
EXPORTED = ("nrx_abi_version", "nrx_status_string", "nrx_validate", "nrx_weight_count",
            "nrx_weight_name", "nrx_weight_numel", "nrx_packed_weight_bytes", "nrx_pack_weights",
            "nrx_workspace_bytes", "nrx_forward", "nrx_buffer_geometry", "nrx_ls_features",
            "nrx_forward_launch_count", "nrx_profile_enable", "nrx_profile_collect",
            "nrx_profile_disable", "nrx_kernel_name",
            # include/nrx_slotgen.h
            "nrx_synth_validate", "nrx_synth_workspace_bytes", "nrx_synth_slots",
            "nrx_count_bit_errors", "nrx_philox4x32_10",
            # include/nrx_ldpc.h
            "nrx_ldpc_create", "nrx_ldpc_destroy", "nrx_ldpc_dims", "nrx_ldpc_workspace_bytes",
            "nrx_ldpc_decode", "nrx_ldpc_encode", "nrx_random_bits", "nrx_bits_to_labels",
            "nrx_extract_llrs", "nrx_count_mismatches",
            # include/nrx_classical.h
            "nrx_ls_lmmse", "nrx_kbest",
            # include/nrx_train.h
            "nrx_train_conv_fwd", "nrx_train_conv_dgrad", "nrx_train_conv_wgrad", "nrx_train_adam",
            "nrx_train_tc_workspace", "nrx_train_conv_tc_fwd", "nrx_train_conv_tc_dgrad", "nrx_train_conv_tc_wgrad")
KERNEL_IDS = {"ls_feat": 0, "conv_state_init0": 1, "conv_state_init1": 2, "msg_agg": 3,
              "conv_update0": 4, "conv_update1": 5, "readout": 6}


class ModelDesc(ctypes.Structure):
    _fields_ = [("d_s", ctypes.c_int32), ("hidden", ctypes.c_int32), ("num_iterations", ctypes.c_int32),
                ("kernel_size", ctypes.c_int32), ("variant", ctypes.c_int32), ("m_max", ctypes.c_int32),
                ("n_io", ctypes.c_int32), ("io_orders", ctypes.c_int32 * NRX_MAX_IO),
                ("num_rx_ant", ctypes.c_int32), ("include_noise_plane", ctypes.c_int32),
                ("include_freq_encoding", ctypes.c_int32)]


class SlotDesc(ctypes.Structure):
    _fields_ = [("num_subcarriers", ctypes.c_int32), ("num_symbols", ctypes.c_int32),
                ("num_ues", ctypes.c_int32), ("comb_size", ctypes.c_int32),
                ("num_pilot_symbols", ctypes.c_int32),
                ("pilot_symbols", ctypes.c_int32 * NRX_MAX_PILOT_SYMBOLS)]


NRX_SG_MAX_UES, NRX_SG_MAX_TAPS, NRX_SG_MAX_UE_ANT = 4, 24, 4
NRX_SG_QAM_POINTS = 4 + 16 + 64 + 256


class TdlProfileDesc(ctypes.Structure):
    _fields_ = [("num_taps", ctypes.c_int32), ("delays_s", ctypes.c_double * NRX_SG_MAX_TAPS),
                ("powers", ctypes.c_double * NRX_SG_MAX_TAPS), ("doppler_hz", ctypes.c_double)]


class ChannelDesc(ctypes.Structure):
    _fields_ = [("bs_antennas", ctypes.c_int32), ("ue_antennas", ctypes.c_int32),
                ("num_sinusoids", ctypes.c_int32), ("subcarrier_spacing_hz", ctypes.c_double),
                ("cp_fraction", ctypes.c_double),
                ("beams", ((ctypes.c_double * 2) * NRX_SG_MAX_UE_ANT) * NRX_SG_MAX_UES),
                ("profiles", TdlProfileDesc * NRX_SG_MAX_UES)]


class SlotVariates(ctypes.Structure):
    _fields_ = [("angles", ctypes.c_void_p), ("phases", ctypes.c_void_p), ("labels", ctypes.c_void_p),
                ("noise", ctypes.c_void_p), ("pilots", ctypes.c_void_p)]


class LdpcDesc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("m", ctypes.c_int32), ("k", ctypes.c_int32), ("dmax", ctypes.c_int32),
                ("cdeg", ctypes.c_int32), ("row_cols", ctypes.c_void_p), ("col_rows", ctypes.c_void_p),
                ("col_slots", ctypes.c_void_p), ("info_positions", ctypes.c_void_p),
                ("n_punctured", ctypes.c_int32), ("punctured", ctypes.c_void_p),
                ("n_shortened", ctypes.c_int32), ("shortened", ctypes.c_void_p), ("chain_cols", ctypes.c_void_p),
                ("chain_step", ctypes.c_int32)]


class NrxLibraryError(RuntimeError):
    """A failed library call; ``status`` is the nrx_status code (0 if none)."""

    def __init__(self, msg, status: int = 0):
        super().__init__(msg)
        self.status = status


_LIB = None


def load() -> ctypes.CDLL:
    """Load libnrx_b200.so once; raise loudly if it was not built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise NrxLibraryError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build())")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, Z, V = ctypes.POINTER, ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p
    lib.nrx_abi_version.restype = I
    lib.nrx_status_string.restype = ctypes.c_char_p
    lib.nrx_status_string.argtypes = [I]
    lib.nrx_validate.argtypes = [P(ModelDesc), P(SlotDesc)]
    lib.nrx_weight_count.argtypes = [P(ModelDesc)]
    lib.nrx_weight_name.argtypes = [P(ModelDesc), I, ctypes.c_char_p, Z]
    lib.nrx_weight_numel.argtypes = [P(ModelDesc), I]
    lib.nrx_weight_numel.restype = ctypes.c_int64
    lib.nrx_packed_weight_bytes.argtypes = [P(ModelDesc), I]
    lib.nrx_packed_weight_bytes.restype = Z
    lib.nrx_pack_weights.argtypes = [P(ModelDesc), I, P(ctypes.c_void_p), I, V]
    lib.nrx_workspace_bytes.argtypes = [P(ModelDesc), P(SlotDesc), I, I]
    lib.nrx_workspace_bytes.restype = Z
    lib.nrx_forward.argtypes = [P(ModelDesc), P(SlotDesc), I, I, I, V, I, V, I, I, V, V, V, V, I, V, V, Z, V]
    lib.nrx_forward_launch_count.argtypes = [P(ModelDesc), P(SlotDesc), I, I]
    lib.nrx_buffer_geometry.argtypes = [P(ModelDesc), P(SlotDesc), I, P(ctypes.c_int32)]
    lib.nrx_ls_features.argtypes = [P(ModelDesc), P(SlotDesc), I, I, V, I, V, I, I, V, V, V]
    lib.nrx_profile_enable.argtypes = [ctypes.c_uint32, I]
    lib.nrx_profile_collect.argtypes = [P(ctypes.c_int32), P(ctypes.c_float), I]
    lib.nrx_profile_disable.restype = None
    lib.nrx_kernel_name.argtypes = [I]
    lib.nrx_kernel_name.restype = ctypes.c_char_p
    lib.nrx_synth_validate.argtypes = [P(SlotDesc), P(ChannelDesc)]
    lib.nrx_synth_workspace_bytes.argtypes = [P(SlotDesc), P(ChannelDesc), I]
    lib.nrx_synth_workspace_bytes.restype = Z
    lib.nrx_synth_slots.argtypes = [P(SlotDesc), P(ChannelDesc), I, ctypes.c_uint64, ctypes.c_uint64, V, V,
                                    P(SlotVariates), V, V, I, V, I, V, V, I, V, Z, V]
    lib.nrx_count_bit_errors.argtypes = [P(SlotDesc), I, V, I, V, V, V, V]
    lib.nrx_philox4x32_10.argtypes = [P(ctypes.c_uint32), P(ctypes.c_uint32), P(ctypes.c_uint32)]
    lib.nrx_philox4x32_10.restype = None
    lib.nrx_ldpc_create.argtypes = [P(LdpcDesc), P(ctypes.c_void_p)]
    lib.nrx_ldpc_destroy.argtypes = [V]
    lib.nrx_ldpc_destroy.restype = None
    lib.nrx_ldpc_dims.argtypes = [V, P(ctypes.c_int32)]
    lib.nrx_ldpc_workspace_bytes.argtypes = [V, I]
    lib.nrx_ldpc_workspace_bytes.restype = Z
    lib.nrx_ldpc_decode.argtypes = [V, I, V, I, V, V, V, Z, V]
    lib.nrx_ldpc_encode.argtypes = [V, I, V, V, V, Z, V]
    lib.nrx_random_bits.argtypes = [ctypes.c_uint64, ctypes.c_uint64, I, I, V, V]
    lib.nrx_bits_to_labels.argtypes = [P(SlotDesc), I, I, I, V, V, V]
    lib.nrx_extract_llrs.argtypes = [P(SlotDesc), I, I, I, V, I, ctypes.c_float, V, V]
    lib.nrx_count_mismatches.argtypes = [I, I, V, V, V, V]
    lib.nrx_ls_lmmse.argtypes = [P(SlotDesc), I, I, V, I, V, I, I, V, V, V, ctypes.c_float, V, I, V]
    lib.nrx_kbest.argtypes = [P(SlotDesc), I, I, V, I, V, I, V, V, V, I, I, ctypes.c_float, V, I, V]
    F32 = ctypes.c_float
    lib.nrx_train_conv_fwd.argtypes = [I, I, I, I, I, I, V, V, V, V, V]
    lib.nrx_train_conv_dgrad.argtypes = [I, I, I, I, I, I, V, V, V, V]
    lib.nrx_train_conv_wgrad.argtypes = [I, I, I, I, I, I, V, V, V, V, V]
    lib.nrx_train_adam.argtypes = [I, V, V, V, V, F32, F32, F32, F32, I, V]
    lib.nrx_train_tc_workspace.argtypes = [I, I, I, I, I, I]
    lib.nrx_train_tc_workspace.restype = ctypes.c_size_t
    for fn in (lib.nrx_train_conv_tc_fwd, lib.nrx_train_conv_tc_dgrad):
        fn.argtypes = [I, I, I, I, I, I, V, V, V, V, ctypes.c_size_t, V]
    lib.nrx_train_conv_tc_wgrad.argtypes = [I, I, I, I, I, I, V, V, V, V, ctypes.c_size_t, V]
    if lib.nrx_abi_version() != 1:
        raise NrxLibraryError("libnrx_b200.so ABI version mismatch")
    _LIB = lib
    return lib


def status_text(code: int) -> str:
    return load().nrx_status_string(int(code)).decode()


def check(code: int, what: str) -> None:
    if code != 0:
        raise NrxLibraryError(f"{what} failed: {status_text(code)} (status {code})", code)


def model_desc(config) -> ModelDesc:
    """NrxConfig (reference or mirror) -> nrx_model_desc."""
    m = ModelDesc()
    m.d_s = config.d_s
    m.hidden = config.hidden_width or config.d_s
    m.num_iterations = config.num_iterations
    m.kernel_size = config.kernel_size
    m.variant = VARIANT_IDS[config.variant]
    m.m_max = config.m_max
    orders = tuple(config.io_modulations) if config.variant == "var_io" else (config.m_max,)
    if len(orders) > NRX_MAX_IO:
        raise NrxLibraryError(f"at most {NRX_MAX_IO} IO sets are supported, got {len(orders)}")
    m.n_io = len(orders)
    for i, o in enumerate(orders):
        m.io_orders[i] = int(o)
    m.num_rx_ant = config.num_rx_ant
    m.include_noise_plane = int(bool(config.include_noise_plane))
    m.include_freq_encoding = int(bool(config.include_freq_encoding))
    return m


def slot_desc(cfg) -> SlotDesc:
    """SlotConfig (reference or mirror) -> nrx_slot_desc."""
    s = SlotDesc()
    s.num_subcarriers = cfg.num_subcarriers
    s.num_symbols = cfg.num_symbols
    s.num_ues = cfg.num_ues
    s.comb_size = cfg.comb_size
    ps = tuple(cfg.pilot_symbols)
    if len(ps) > NRX_MAX_PILOT_SYMBOLS:
        raise NrxLibraryError(f"at most {NRX_MAX_PILOT_SYMBOLS} pilot symbols are supported")
    s.num_pilot_symbols = len(ps)
    for i, p in enumerate(ps):
        s.pilot_symbols[i] = int(p)
    return s


def weight_names(config) -> list:
    lib = load()
    m = model_desc(config)
    n = lib.nrx_weight_count(ctypes.byref(m))
    buf = ctypes.create_string_buffer(256)
    out = []
    for i in range(n):
        lib.nrx_weight_name(ctypes.byref(m), i, buf, 256)
        out.append(buf.value.decode())
    return out


def buffer_geometry(config, cfg, precision: str) -> dict:
    lib = load()
    out = (ctypes.c_int32 * 8)()
    check(lib.nrx_buffer_geometry(ctypes.byref(model_desc(config)), ctypes.byref(slot_desc(cfg)),
                                  PRECISIONS[precision], out), "nrx_buffer_geometry")
    return dict(zip(("rows_slab", "Tp", "Cf", "Cs", "Ch", "Ca", "cw", "tiles"), list(out)))


class KernelTimer:
    """Collect per-launch device times of selected kernels (CUDA events
    recorded by the library around each launch, on the launch stream)."""

    def __init__(self, kernels=("conv_update0",), max_records: int = 4096):
        self.lib = load()
        self.mask = 0
        for k in kernels:
            self.mask |= 1 << KERNEL_IDS[k]
        self.max_records = max_records

    def __enter__(self):
        check(self.lib.nrx_profile_enable(self.mask, self.max_records), "nrx_profile_enable")
        return self

    def collect(self) -> dict:
        ids = (ctypes.c_int32 * self.max_records)()
        ms = (ctypes.c_float * self.max_records)()
        n = self.lib.nrx_profile_collect(ids, ms, self.max_records)
        if n < 0:
            raise NrxLibraryError("nrx_profile_collect failed")
        out = {}
        for i in range(n):
            out.setdefault(self.lib.nrx_kernel_name(ids[i]).decode(), []).append(ms[i])
        return out

    def __exit__(self, *exc):
        self.lib.nrx_profile_disable()
        return False
