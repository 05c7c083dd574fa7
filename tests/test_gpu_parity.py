"""GPU parity of the CUDA path against the reference (golden vectors) and the
CPU oracle.  Gates (stated per test):

  fp32 mode:  max|dLLR| <= 1e-5 * max|LLR_ref|  (tensor-core fp32x3 and SIMT fp32_simt)
  bf16 mode:  max|dLLR| <= 2e-2 * max|LLR_ref|,  p99|dLLR| <= 5e-3 * max|LLR_ref|
  fp16 mode:  max|dLLR| <= 5e-3 * max|LLR_ref|,  p99|dLLR| <= 1.5e-3 * max|LLR_ref|
  hard bits (LLR > 0) bit-exact wherever |LLR_ref| exceeds the mode's bound.
"""

import ctypes
import threading

import numpy as np
import pytest

from golden_cases import case_names, load_case
from oracle import nrx_oracle as orc

pytestmark = pytest.mark.gpu

CASES = case_names()
GATES = {"fp32": dict(max=1e-5, p99=1e-5), "fp32_simt": dict(max=1e-5, p99=1e-5), "bf16": dict(max=2e-2, p99=5e-3), "fp16": dict(max=5e-3, p99=1.5e-3)}


def _gpu():
    import torch
    from paper_2409_02912_b200 import nrx as gnrx
    return torch, gnrx


def check_llrs(got_list, ref_list, precision, label="", depth=2):
    """The p99 gates are calibrated at the RT depth N_it = 2;
    rounding noise of the half-precision operands accumulates roughly like a
    random walk over the unrolled iterations, so the p99 gate is scaled by
    sqrt(depth / 2) for deeper models (bf16 at N_it = 8: 1e-2)."""
    gate = dict(GATES[precision])
    if depth > 2:
        gate["p99"] *= float(np.sqrt(depth / 2))
    scale = max(float(np.abs(r).max()) for r in ref_list)
    for got, ref in zip(got_list, ref_list):
        assert got.shape == ref.shape, (label, got.shape, ref.shape)
        assert got.dtype == np.float32
        err = np.abs(got.astype(np.float64) - ref)
        assert np.isfinite(got).all(), label
        assert err.max() <= gate["max"] * scale, (label, err.max() / scale)
        assert np.percentile(err, 99) <= gate["p99"] * scale, (label, np.percentile(err, 99) / scale)
        band = gate["max"] * scale
        sure = np.abs(ref) > band
        np.testing.assert_array_equal(got[sure] > 0, ref[sure] > 0)


def check_chest(got, ref, precision):
    gate = GATES[precision]
    scale = float(np.abs(ref).max())
    assert got.shape == ref.shape and got.dtype == np.complex64
    assert np.abs(got - ref).max() <= gate["max"] * scale


@pytest.mark.parametrize("precision", ["fp32", "fp32_simt", "bf16", "fp16"])
@pytest.mark.parametrize("name", CASES)
def test_golden_forward(name, precision):
    """Drop-in nrx_forward vs the reference's own outputs on reference inputs."""
    _, gnrx = _gpu()
    c = load_case(name)
    y, books, n0 = c.call_args()
    llrs, chest = gnrx.nrx_forward(y, books, c.cfg, c.mcs, c.weights, c.config, n0, precision=precision)
    check_llrs(llrs, c.llrs, precision, name)
    check_chest(chest, c.chest, precision)


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("name", CASES)
def test_golden_features(name, exact):
    """K1 (LS + features) vs the reference's assemble_features(ls_features(...)).
    complex128 inputs: equal to float32 rounding (<= 1 ulp); complex64
    inputs: the LS sees rounded samples, so 1e-6 relative."""
    torch, _ = _gpu()
    from paper_2409_02912_b200 import _lib
    from paper_2409_02912_b200.nrx import noise_features, stack_pilots
    c = load_case(name)
    n = c.y.shape[0]
    geo = _lib.buffer_geometry(c.config, c.cfg, "fp32_simt")
    lib = _lib.load()
    cdt = torch.complex128 if exact else torch.complex64
    y = torch.from_numpy(c.y).to(cdt).cuda()
    p = torch.from_numpy(stack_pilots(c.books, n, c.cfg)).to(cdt).cuda()
    nf = torch.from_numpy(noise_features(c.n0, n)).cuda()
    U = c.cfg.num_ues
    out = torch.zeros(n * U, geo["Cf"] // 4, geo["rows_slab"], 4, device="cuda")
    code = lib.nrx_ls_features(ctypes.byref(_lib.model_desc(c.config)), ctypes.byref(_lib.slot_desc(c.cfg)), n, 0,
                               y.data_ptr(), int(exact), p.data_ptr(), int(exact), p.shape[0], nf.data_ptr(),
                               out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert code == 0
    torch.cuda.synchronize()
    f = out.cpu().numpy().transpose(0, 2, 1, 3).reshape(n * U, geo["rows_slab"], geo["Cf"])
    S, T = c.cfg.num_subcarriers, c.cfg.num_symbols
    f = f[:, :S * geo["Tp"]].reshape(n, U, S, geo["Tp"], geo["Cf"])
    cin = c.features.shape[-1]
    assert not f[:, :, :, T:].any()                 # zero pad rows
    assert not f[..., cin:].any()                   # zero pad channels
    got = f[:, :, :, :T, :cin]
    if exact:
        np.testing.assert_allclose(got, c.features, rtol=2.5e-7, atol=1e-30)
    else:
        np.testing.assert_allclose(got, c.features, rtol=0, atol=1e-6 * np.abs(c.features).max())


@pytest.mark.parametrize("name", CASES[:3])
def test_golden_features_fp32x3_split(name):
    """K1 in the fp32x3 layout: hi plane (chunks [0, Cf/8)) + lo plane
    (chunks [Cf/8, Cf/4), scaled by 2^11) reconstruct the reference features
    to 2^-22 relative (+ 2^-25 absolute for the lo plane's subnormal floor)."""
    torch, _ = _gpu()
    from paper_2409_02912_b200 import _lib
    from paper_2409_02912_b200.nrx import noise_features, stack_pilots
    c = load_case(name)
    n = c.y.shape[0]
    geo = _lib.buffer_geometry(c.config, c.cfg, "fp32")
    assert geo["cw"] == 8
    lib = _lib.load()
    y = torch.from_numpy(c.y).to(torch.complex128).cuda()
    p = torch.from_numpy(stack_pilots(c.books, n, c.cfg)).to(torch.complex128).cuda()
    nf = torch.from_numpy(noise_features(c.n0, n)).cuda()
    U = c.cfg.num_ues
    nch = geo["Cf"] // 8
    out = torch.zeros(n * U, 2 * nch, geo["rows_slab"], 8, dtype=torch.float16, device="cuda")
    code = lib.nrx_ls_features(ctypes.byref(_lib.model_desc(c.config)), ctypes.byref(_lib.slot_desc(c.cfg)), n,
                               _lib.NRX_FP32X3, y.data_ptr(), 1, p.data_ptr(), 1, p.shape[0], nf.data_ptr(),
                               out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert code == 0
    torch.cuda.synchronize()
    o = out.float().cpu().numpy().astype(np.float64)
    rec = o[:, :nch] + o[:, nch:] / 2048.0
    f = rec.transpose(0, 2, 1, 3).reshape(n * U, geo["rows_slab"], geo["Cf"])
    S, T = c.cfg.num_subcarriers, c.cfg.num_symbols
    f = f[:, :S * geo["Tp"]].reshape(n, U, S, geo["Tp"], geo["Cf"])
    cin = c.features.shape[-1]
    assert not f[:, :, :, T:].any() and not f[..., cin:].any()
    want = c.features.astype(np.float64)
    err = np.abs(f[:, :, :, :T, :cin] - want)
    assert np.all(err <= 2.0 ** -22 * np.abs(want) + 2.0 ** -25)


def _c2_setup(d=56, n_it=2, U=2, S=3276, variant="single", supported=(14,), seed=0, bias=True):
    from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights
    from paper_2409_02912_b200.synth import synth_slots
    table = default_mcs_table()
    cfg = SlotConfig(num_subcarriers=S, num_ues=U, comb_size=max(2, U))
    config = NrxConfig.from_table(table, supported, variant=variant, d_s=d, num_iterations=n_it)
    w = init_weights(config, seed=0)
    if bias:
        w = orc.perturb_biases(w)
    return cfg, config, w, table


@pytest.mark.parametrize("precision", ["fp32", "fp32_simt", "bf16", "fp16"])
def test_c2_rt_slot_vs_oracle(precision):
    """273 PRB / 2 UE / 4 RX / RT model (d=56, N_it=2): the benchmark config."""
    _, gnrx = _gpu()
    from paper_2409_02912_b200.synth import synth_slots
    cfg, config, w, table = _c2_setup()
    mcs = (table[14], table[14])
    y, books, _ = synth_slots(cfg, [4, 4], 1, 0.1, seed=3)
    ref_llrs, ref_chest = orc.nrx_forward(y, books, cfg, mcs, w, config, 0.1, dtype=np.float64)
    llrs, chest = gnrx.nrx_forward(y, books, cfg, mcs, w, config, 0.1, precision=precision)
    check_llrs(llrs, ref_llrs, precision, "C2")
    check_chest(chest, ref_chest, precision)


def test_depth_control_and_errors():
    _, gnrx = _gpu()
    c = load_case("mu2_masking_bias")
    y, books, n0 = c.call_args()
    full, _ = gnrx.nrx_forward(y, books, c.cfg, c.mcs, c.weights, c.config, n0)
    explicit, _ = gnrx.nrx_forward(y, books, c.cfg, c.mcs, c.weights, c.config, n0,
                                   num_iterations=c.config.num_iterations)
    np.testing.assert_array_equal(full[0], explicit[0])            # deterministic
    shallow, _ = gnrx.nrx_forward(y, books, c.cfg, c.mcs, c.weights, c.config, n0, num_iterations=1)
    ref1, _ = orc.nrx_forward(y, books, c.cfg, c.mcs, c.weights, c.config, n0, num_iterations=1)
    check_llrs(shallow, ref1, "fp32", "depth1")
    with pytest.raises(ValueError, match="depth"):
        gnrx.nrx_forward(y, books, c.cfg, c.mcs, c.weights, c.config, n0,
                         num_iterations=c.config.num_iterations + 1)
    from paper_2409_02912_b200.config import McsEntry
    with pytest.raises(ValueError, match="supported set"):
        gnrx.nrx_forward(y, books, c.cfg, (McsEntry(5, 4, 0.5), c.mcs[1]), c.weights, c.config, n0)


def test_single_ue_independent_of_message_weights():
    """U=1: the aggregate is an empty sum, so perturbing the message MLP
    leaves the outputs bit-identical (test_nrx.py:86-98)."""
    _, gnrx = _gpu()
    cfg, config, w, table = _c2_setup(S=48, d=16, U=1)
    from paper_2409_02912_b200.config import SlotConfig
    cfg = SlotConfig(num_subcarriers=48, num_ues=1, comb_size=2)
    from paper_2409_02912_b200.synth import random_grid
    y, books = random_grid(cfg, 1, seed=5)
    out1, _ = gnrx.nrx_forward(y, books, cfg, (table[14],), w, config, 0.1)
    w2 = dict(w)
    w2["iteration.msg.fc1.w"] = w["iteration.msg.fc1.w"] + 0.7
    w2["iteration.msg.fc0.b"] = w["iteration.msg.fc0.b"] - 0.3
    out2, _ = gnrx.nrx_forward(y, books, cfg, (table[14],), w2, config, 0.1)
    np.testing.assert_array_equal(out1[0], out2[0])


def test_weight_cache_invalidation():
    """Weights mutated in place between calls are picked up (Adam updates
    p.data in place, autodiff.py:525)."""
    _, gnrx = _gpu()
    c = load_case("c1_small")
    y, books, n0 = c.call_args()
    w = {k: v.copy() for k, v in c.weights.items()}
    a, _ = gnrx.nrx_forward(y, books, c.cfg, c.mcs, w, c.config, n0)
    w["readout_llr.fc1.b"][...] += 1.0
    b, _ = gnrx.nrx_forward(y, books, c.cfg, c.mcs, w, c.config, n0)
    np.testing.assert_allclose(b[0], a[0] + 1.0, rtol=0, atol=1e-5)


def test_concurrent_threads_deterministic():
    """ReceiverBank calls nrx_forward from worker threads (evaluation.py:229-236):
    results must not depend on concurrency."""
    _, gnrx = _gpu()
    c = load_case("mu2_masking_bias")
    y, books, n0 = c.call_args()
    base, _ = gnrx.nrx_forward(y, books, c.cfg, c.mcs, c.weights, c.config, n0)
    results, errors = [None] * 6, []

    def work(i):
        try:
            results[i] = gnrx.nrx_forward(y, books, c.cfg, c.mcs, c.weights, c.config, n0)[0]
        except Exception as e:  # pragma: no cover
            errors.append(e)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors
    for r in results:
        for u in range(len(base)):
            np.testing.assert_array_equal(r[u], base[u])


def test_pdl_launch_bit_identical_to_stream_order(tmp_path):
    """The tensor-core layers (convolutions and the message / readout MLP
    kernels) are launched with programmatic dependent launch
    (each layer's prologue overlaps its predecessor; every activation access
    waits for the predecessor grid).  The results must be bit-identical to
    plain stream order (NRX_PDL=0, read once per process: run in a child)."""
    import os
    import subprocess
    import sys
    script = tmp_path / "fwd.py"
    script.write_text(
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        "from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights\n"
        "from paper_2409_02912_b200.nrx import nrx_forward\n"
        "from paper_2409_02912_b200.synth import synth_slots\n"
        "t = default_mcs_table()\n"
        "cfg = SlotConfig(num_subcarriers=3276, num_ues=2, comb_size=2)\n"
        "config = NrxConfig.from_table(t, (14,), d_s=56, num_iterations=2)\n"
        "w = init_weights(config, 0)\n"
        "rng = np.random.default_rng(5)\n"
        "w = {k: v + (0.05 * rng.standard_normal(v.shape).astype(np.float32) if v.ndim == 1 else 0) for k, v in w.items()}\n"
        "y, books, _ = synth_slots(cfg, [4, 4], 3, 0.1, seed=4)\n"
        "out = {}\n"
        "for p in ('fp32', 'fp16', 'bf16'):\n"
        "    llrs, chest = nrx_forward(y, books, cfg, (t[14], t[14]), w, config, 0.1, precision=p)\n"
        "    out[p + '_l0'], out[p + '_l1'], out[p + '_c'] = llrs[0], llrs[1], chest\n"
        "cfg1 = SlotConfig(num_subcarriers=288, num_ues=1, comb_size=2)\n"  # standalone message / readout kernels
        "y1, books1, _ = synth_slots(cfg1, [4], 3, 0.1, seed=6)\n"
        "for p in ('fp32', 'fp16'):\n"
        "    llrs, chest = nrx_forward(y1, books1, cfg1, (t[14],), w, config, 0.1, precision=p)\n"
        "    out[p + '_u1_l0'], out[p + '_u1_c'] = llrs[0], chest\n"
        "np.savez(sys.argv[1], **out)\n")
    res = {}
    for pdl in ("1", "0"):
        env = dict(os.environ, NRX_PDL=pdl)
        f = tmp_path / f"out{pdl}.npz"
        subprocess.run([sys.executable, str(script), str(f)], check=True, env=env, timeout=600)
        with np.load(f) as z:
            res[pdl] = {k: z[k] for k in z.files}
    for k in res["1"]:
        np.testing.assert_array_equal(res["1"][k], res["0"][k], err_msg=k)


@pytest.mark.parametrize("precision", ["fp32", "fp16"])
def test_range_guard_reruns_on_fp32_simt(precision):
    """Inputs far outside the fp16 operand range (received grid scaled by 1e5:
    features ~1e5 > 65504): the tensor-core readout flags the non-finite
    outputs (NRX_WS_FLAG_OFFSET) and the drop-in recomputes the call on the
    fp32 SIMT kernels with a RuntimeWarning -- results stay within the fp32
    gate of the float64 oracle instead of turning into NaN."""
    _, gnrx = _gpu()
    from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights
    from paper_2409_02912_b200.synth import synth_slots
    t = default_mcs_table()
    cfg = SlotConfig(num_subcarriers=96, num_ues=2, comb_size=2)
    config = NrxConfig.from_table(t, (14,), d_s=56, num_iterations=2)
    w = orc.perturb_biases(init_weights(config, 2))
    mcs = (t[14], t[14])
    y, books, _ = synth_slots(cfg, [4, 4], 1, 0.1, seed=8)
    y = y * 1e5
    ref, _ = orc.nrx_forward(y, books, cfg, mcs, w, config, 0.1, dtype=np.float64)
    with pytest.warns(RuntimeWarning, match="fp32_simt"):
        got, chest = gnrx.nrx_forward(y, books, cfg, mcs, w, config, 0.1, precision=precision)
    assert np.isfinite(chest).all()
    check_llrs(got, ref, "fp32_simt", "range guard")
