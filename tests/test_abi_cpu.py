"""CPU-only checks of the C ABI: the library loads, exports every symbol the
header declares, names/validates/packs weights without a GPU."""

import ctypes
import glob
import os
import re

import numpy as np
import pytest

from paper_2409_02912_b200 import _lib
from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, expected_shapes, init_weights
from paper_2409_02912_b200.engine import pack_weights, pilot_comb_values

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = sorted(glob.glob(os.path.join(ROOT, "include", "*.h")))


def declared_functions():
    text = "\n".join(open(h).read() for h in HEADERS)
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nrx_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.EXPORTED)
    assert lib.nrx_abi_version() == 1


@pytest.mark.parametrize("variant,supported,kw", [
    ("single", (14,), {}),
    ("masking", (9, 14, 19), dict(d_s=56, num_iterations=2)),
    ("var_io", (9, 14, 19), dict(d_s=8, hidden_width=20)),
    ("single", (14,), dict(include_noise_plane=False, kernel_size=5)),
])
def test_weight_names_match_expected_shapes(variant, supported, kw):
    config = NrxConfig.from_table(default_mcs_table(), supported, variant=variant, **kw)
    names = _lib.weight_names(config)
    shapes = expected_shapes(config)
    assert set(names) == set(shapes) and len(names) == len(shapes)
    lib = _lib.load()
    m = _lib.model_desc(config)
    for i, n in enumerate(names):
        assert lib.nrx_weight_numel(ctypes.byref(m), i) == int(np.prod(shapes[n]))


def test_pack_weights_deterministic_and_sized():
    config = NrxConfig(d_s=56, num_iterations=2)
    w = init_weights(config, 0)
    for prec in ("fp32", "bf16", "fp16"):  # tensor-core blobs: deterministic too
        np.testing.assert_array_equal(pack_weights(config, w, prec),
                                      pack_weights(config, {k: v.copy() for k, v in w.items()}, prec))
    a = pack_weights(config, w, "fp32_simt")
    b = pack_weights(config, {k: v.copy() for k, v in w.items()}, "fp32_simt")
    np.testing.assert_array_equal(a, b)
    # every weight value lands somewhere in the packed blob (no value dropped)
    packed = a.view(np.float32)
    for name in ("iteration.update.conv0.w", "readout_chest.fc1.w"):
        vals = np.unique(w[name])
        assert np.isin(vals, packed).all()
    with pytest.raises(ValueError):
        pack_weights(config, {k: v for k, v in w.items() if k != "readout_chest.fc1.b"})


def test_validate_limits():
    lib = _lib.load()
    ok = _lib.model_desc(NrxConfig(d_s=56))
    s = _lib.slot_desc(SlotConfig(num_subcarriers=3276, num_ues=2))
    assert lib.nrx_validate(ctypes.byref(ok), ctypes.byref(s)) == 0
    too_deep = _lib.model_desc(NrxConfig(d_s=96))
    assert lib.nrx_validate(ctypes.byref(too_deep), None) == 2  # unsupported, not invalid
    bad = _lib.model_desc(NrxConfig(d_s=8))
    bad.kernel_size = 4
    assert lib.nrx_validate(ctypes.byref(bad), None) == 1
    assert "workspace" in _lib.status_text(3)


def test_workspace_and_geometry():
    config = NrxConfig(d_s=56, num_iterations=2)
    cfg = SlotConfig(num_subcarriers=3276, num_ues=2)
    lib = _lib.load()
    for prec, esz in (("fp32_simt", 4), ("fp32", 4), ("fp16", 2)):  # fp32x3: fp16 hi + lo planes
        geo = _lib.buffer_geometry(config, cfg, prec)
        assert geo["Tp"] == 15 and geo["rows_slab"] % 128 == 0 and geo["rows_slab"] >= 3276 * 15
        assert geo["Cs"] >= 58 and geo["Cf"] >= 19
        nb = lib.nrx_workspace_bytes(ctypes.byref(_lib.model_desc(config)), ctypes.byref(_lib.slot_desc(cfg)), 4,
                                     _lib.PRECISIONS[prec])
        assert nb >= 4 * 2 * geo["rows_slab"] * esz * (geo["Cf"] + geo["Cs"] + geo["Ch"] + geo["Ca"])


def test_pilot_comb_values_layout():
    cfg = SlotConfig(num_subcarriers=25, num_ues=2, comb_size=2, pilot_symbols=(2, 11))
    vals = np.arange(2 * 25 * 14).reshape(2, 25, 14).astype(np.complex128)
    p = pilot_comb_values(vals, cfg)
    assert p.shape == (2, 13, 2)
    assert p[1, 3, 1] == vals[1, 1 + 3 * 2, 11]
    assert p[0, 12, 0] == vals[0, 24, 2]


@pytest.mark.parametrize("precision,num_ues,n_it,expect", [
    ("fp16", 2, 2, 7),   # ls_feat, init.conv0, init.conv1+msg, 2 x (update.conv0, update.conv1+tail)
    ("bf16", 2, 8, 19),
    ("fp16", 1, 2, 9),   # U != 2: standalone message kernel per iteration
    ("fp32_simt", 2, 2, 10),  # SIMT parity path: ls_feat, 2 init convs, 3 per iteration, readout
    ("fp32", 2, 2, 10),       # fp32x3 tensor-core path: same sequence on CTA pairs
])
def test_forward_launch_count(precision, num_ues, n_it, expect):
    """nrx_forward_launch_count is the per-forward kernel count bench.py
    reports as gpu_launches; it must match the launch sequence of the path."""
    config = NrxConfig(d_s=56, num_iterations=8)
    cfg = SlotConfig(num_subcarriers=3276, num_ues=num_ues, comb_size=2)
    lib = _lib.load()
    m, s = _lib.model_desc(config), _lib.slot_desc(cfg)
    prec = _lib.PRECISIONS[precision]
    assert lib.nrx_forward_launch_count(ctypes.byref(m), ctypes.byref(s), prec, n_it) == expect
