"""CPU checks of the slot-generator path: the oracle and the host-side
variate recipe against the reference's own outputs (golden fixtures), the
Philox bijection against published known answers, and descriptor
validation through the C ABI (no GPU needed)."""

import ctypes

import numpy as np
import pytest

from oracle import slotgen_oracle as so
from paper_2409_02912_b200 import _lib, slotgen
from slotgen_cases import case_names, load_case

CASES = case_names()


@pytest.mark.parametrize("name", CASES)
def test_profiles_match_reference_declared_taps(name):
    c = load_case(name)
    for u, p in enumerate(c.profiles):
        np.testing.assert_array_equal(p.delays_s, c.a[f"delays_{u}"])
        np.testing.assert_array_equal(p.powers, c.a[f"powers_{u}"])


def test_qam_table_bit_identical_to_reference():
    c = load_case(CASES[0])
    table = slotgen.qam_table()
    off = {2: 0, 4: 4, 6: 20}
    for m in (2, 4, 6):
        np.testing.assert_array_equal(table[off[m]:off[m] + 2 ** m], c.a[f"qam_{m}"])
        np.testing.assert_array_equal(so.gray_points(m), c.a[f"qam_{m}"])
    assert table.shape == (_lib.NRX_SG_QAM_POINTS,)
    assert abs(np.mean(np.abs(table[84:]) ** 2) - 1.0) < 1e-12          # 256-QAM extension, unit energy


@pytest.mark.parametrize("name", CASES)
def test_reference_variates_recipe(name):
    """The product's host draw of the reference recipe reproduces the
    variates the reference consumed, bit for bit."""
    c = load_case(name)
    v = slotgen.reference_variates(c.cfg, c.profiles, c.orders, range(c.n), seed=c.seed)
    for k in ("angles", "phases", "labels", "noise", "pilots"):
        np.testing.assert_array_equal(v[k], c.a[k], err_msg=k)


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference_generator(name):
    c = load_case(name)
    for i in range(c.n):
        y, h_eff = so.synth_slot(c.cfg, c.profiles, c.orders, c.n0, c.a["angles"][i], c.a["phases"][i],
                                 c.a["labels"][i], c.a["noise"][i], c.a["pilots"][i])
        scale = np.abs(c.a["y"][i]).max()
        np.testing.assert_allclose(y, c.a["y"][i], rtol=0, atol=1e-13 * scale)
        np.testing.assert_allclose(h_eff, c.a["h_eff"][i], rtol=0, atol=1e-13 * np.abs(c.a["h_eff"][i]).max())


def test_labels_to_bits_round_trip():
    c = load_case("sg_mixed")
    bits = slotgen.labels_to_bits(c.a["labels"], c.cfg, c.orders)
    s_idx, t_idx = np.nonzero(c.cfg.data_mask)
    for u, m in enumerate(c.orders):
        assert bits[u].shape == (c.n, s_idx.size, m)
        lab = bits[u].astype(np.int64) @ (1 << np.arange(m - 1, -1, -1))
        np.testing.assert_array_equal(lab, c.a["labels"][:, u, s_idx, t_idx])


# Random123 known-answer vectors for Philox4x32-10 (ctr, key -> out).
PHILOX_KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,want", PHILOX_KAT)
def test_philox_known_answers(ctr, key, want):
    lib = _lib.load()
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib.nrx_philox4x32_10(c, k, o)
    assert tuple(o) == want


def test_synth_validate_and_workspace():
    from paper_2409_02912_b200.config import SlotConfig
    lib = _lib.load()
    cfg = SlotConfig(num_subcarriers=3276, num_ues=2)
    s = _lib.slot_desc(cfg)
    c = slotgen.channel_desc(cfg, slotgen.doubletdl())
    assert lib.nrx_synth_validate(ctypes.byref(s), ctypes.byref(c)) == 0
    nb = lib.nrx_synth_workspace_bytes(ctypes.byref(s), ctypes.byref(c), 8)
    assert nb == 8 * 2 * 14 * 4 * 5 * 16          # beamformed tap gains G[n][u][t][b][l], complex128
    # a tap beyond the cyclic prefix is rejected like sample_tdl (channel.py:135-138)
    late = slotgen.TdlProfile("late", np.array([0.0, 3e-6]), np.array([0.5, 0.5]), 10.0, 3e-6)
    bad = slotgen.channel_desc(cfg, [late, late])
    assert lib.nrx_synth_validate(ctypes.byref(s), ctypes.byref(bad)) == 1
    assert lib.nrx_synth_workspace_bytes(ctypes.byref(s), ctypes.byref(bad), 8) == 0
    many = slotgen.TdlProfile("many", np.linspace(0, 1e-6, 30), np.full(30, 1 / 30), 10.0, 1e-7)
    with pytest.raises(ValueError, match="taps"):
        slotgen.channel_desc(cfg, [many, many])
    with pytest.raises(ValueError, match="profiles"):
        slotgen.channel_desc(cfg, [slotgen.tdl_a()])


def test_profile_validation_texts():
    with pytest.raises(ValueError, match="sum to 1"):
        slotgen.TdlProfile("bad", np.array([0.0, 1e-9]), np.array([0.6, 0.6]), 10.0, 1e-9)
    with pytest.raises(ValueError, match="ascending"):
        slotgen.TdlProfile("bad", np.array([1e-9, 0.0]), np.array([0.5, 0.5]), 10.0, 1e-9)
