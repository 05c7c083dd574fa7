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


@pytest.mark.parametrize("name", ["train_masking", "train_var_io"])
def test_gpu_train_step_matches_reference(name):
    """One training step on the GPU (cuDNN / cuBLAS with TF32 off) against the
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
    g = TorchNrxGraph(config, w0, dev)
    res = train_step(g, Adam(lr=1e-3), *args, gamma=0.1)
    for key in ("total", "bce", "mse"):
        assert abs(res[key] - float(a[key])) <= 1e-5 * abs(float(a[key])), key
    w1 = {k[4:]: v for k, v in a.items() if k.startswith("w1::")}
    got = g.numpy_weights()
    for k, ref in w1.items():
        np.testing.assert_allclose(got[k] - w0[k], ref - w0[k], rtol=1e-3, atol=1e-6, err_msg=k)
