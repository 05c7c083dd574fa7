"""GPU training loop: batches from the GPU slot
generator through the LS/feature kernel into the torch training step; the
loss falls and the trained weights run on the inference kernels with a
lower uncoded BER than the initial ones."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_gpu_training_reduces_loss_and_ber():
    from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights
    from paper_2409_02912_b200.engine import NrxEngine
    from paper_2409_02912_b200.slotgen import GpuSlotSource, evaluate_uncoded
    from paper_2409_02912_b200.training import GpuTrainConfig, gpu_features, gpu_training_batch, train_gpu
    table = default_mcs_table()
    cfg = SlotConfig(num_subcarriers=48, num_ues=2)
    config = NrxConfig.from_table(table, (14,), d_s=16, num_iterations=2)
    w = init_weights(config, 3)
    src = GpuSlotSource(cfg)
    tcfg = GpuTrainConfig(batch_size=16, steps=300, snr_lo_db=5.0, snr_hi_db=20.0, learning_rate=3e-3, seed=1)
    # features of a generated batch equal the reference layout (N, U, S, T, Cin)
    sb, n0, mods, labels, mask, tgt = gpu_training_batch(src, config, table, tcfg, 0)
    f = gpu_features(config, cfg, sb, n0)
    assert tuple(f.shape) == (16, 2, 48, 14, 19)
    assert labels.shape[-1] == 4 and float(mask.sum()) == 16 * 2 * cfg.num_data_res * 4
    graph, adam, hist = train_gpu(config, w, src, table, tcfg, log_every=25)
    first = np.mean([h[1]["total"] for h in hist[:2]])
    last = np.mean([h[1]["total"] for h in hist[-2:]])
    assert last < 0.8 * first, (first, last)
    trained = graph.numpy_weights()
    mcs = (table[14], table[14])
    b0 = evaluate_uncoded(NrxEngine(config, w, "fp32"), src, mcs, [15.0], n_slots=32, batch=16, seed=9)[0].ber
    b1 = evaluate_uncoded(NrxEngine(config, trained, "fp32"), src, mcs, [15.0], n_slots=32, batch=16, seed=9)[0].ber
    assert b1 < 0.75 * b0, (b0, b1)


@pytest.mark.parametrize("kernels", ["nrx", "nrx_tc", "torch"])
@pytest.mark.parametrize("name", ["train_masking", "train_var_io"])
def test_gpu_train_step_matches_reference(name, kernels):
    """One training step on the GPU (kernels="nrx": the hand-written fp32
    convolution / dense / Adam kernels; "nrx_tc": the tcgen05 fp32x3 GEMMs;
    "torch": cuDNN / cuBLAS with TF32 off) against the
    reference's own train_step on the same batch (tests/golden/train_*.npz):
    the loss breakdown to 1e-5, the Adam step to 1e-3 relative (same gates
    as the CPU test)."""
    import torch
    from test_training_cpu import _config, _load
    from paper_2409_02912_b200.training import Adam, TorchNrxGraph, train_step
    a = _load(name)
    config = _config(name)
    w0 = {k[4:]: v for k, v in a.items() if k.startswith("w0::")}
    dev = "cuda"
    t = lambda x, dt=torch.float32: torch.as_tensor(x).to(dt).to(dev)
    args = (t(a["feats"]), t(a["labels"]), t(a["label_mask"]), t(a["chest_target"]), a["active"], a["mods"])
    g = TorchNrxGraph(config, w0, dev, kernels=kernels)
    res = train_step(g, Adam(lr=1e-3), *args, gamma=0.1)
    for key in ("total", "bce", "mse"):
        assert abs(res[key] - float(a[key])) <= 1e-5 * abs(float(a[key])), key
    w1 = {k[4:]: v for k, v in a.items() if k.startswith("w1::")}
    got = g.numpy_weights()
    for k, ref in w1.items():
        np.testing.assert_allclose(got[k] - w0[k], ref - w0[k], rtol=1e-3, atol=1e-6, err_msg=k)


@pytest.mark.parametrize("tc", [False, True])
@pytest.mark.parametrize("k,cin,cout,S,T,n", [(3, 19, 16, 24, 14, 3), (3, 114, 56, 20, 14, 2), (5, 8, 8, 11, 7, 2),
                                              (1, 56, 56, 300, 1, 1), (1, 56, 4, 1000, 1, 1),
                                              (3, 128, 128, 40, 14, 3), (3, 56, 114, 96, 14, 4)])
def test_train_conv_kernels_vs_float64(k, cin, cout, S, T, n, tc):
    """The hand-written training kernels (csrc/k_train.cu SIMT, or with tc the
    tcgen05 fp32x3 GEMMs of csrc/k_train_tc.cu) against float64 torch: 'same'
    convolution forward, input gradient and kernel gradient (k = 1, T = 1 is
    the dense layer), fp32-level error only."""
    import torch
    from paper_2409_02912_b200.training import _nrx_conv_fn, _nrx_conv_tc_fn
    g = torch.Generator().manual_seed(k * 1000 + cin)
    x = torch.randn(n, S, T, cin, generator=g, dtype=torch.float64)
    w = torch.randn(k, k, cin, cout, generator=g, dtype=torch.float64) / np.sqrt(k * k * cin)
    dy = torch.randn(n, S, T, cout, generator=g, dtype=torch.float64)
    xr, wr = x.clone().requires_grad_(), w.clone().requires_grad_()
    yr = torch.nn.functional.conv2d(xr.permute(0, 3, 1, 2), wr.permute(3, 2, 0, 1), padding=k // 2).permute(0, 2, 3, 1)
    yr.backward(dy)
    xc = x.float().cuda().requires_grad_()
    wc = w.float().cuda().requires_grad_()
    yc = (_nrx_conv_tc_fn() if tc else _nrx_conv_fn()).apply(xc, wc)
    yc.backward(dy.float().cuda())
    for got, ref in ((yc, yr), (xc.grad, xr.grad), (wc.grad, wr.grad)):
        ref = ref.detach()
        err = (got.detach().double().cpu() - ref).abs().max().item()
        assert err <= 2e-5 * max(1.0, ref.abs().max().item()), err


def test_train_adam_kernel_matches_formula():
    import torch
    from paper_2409_02912_b200.training import Adam
    g = torch.Generator().manual_seed(3)
    p0 = torch.randn(1000, generator=g)
    grads = [torch.randn(1000, generator=g) for _ in range(3)]
    ref = {"w": p0.clone()}
    dev = {"w": p0.clone().cuda()}
    a_ref, a_dev = Adam(lr=1e-2), Adam(lr=1e-2)
    for gr in grads:
        ref["w"].grad = gr.clone()
        dev["w"].grad = gr.clone().cuda()
        a_ref.step(ref, ["w"])   # torch elementwise on the CPU
        a_dev.step(dev, ["w"])   # nrx_train_adam
    np.testing.assert_allclose(dev["w"].cpu().numpy(), ref["w"].numpy(), rtol=1e-6, atol=1e-7)
