"""Training step parity on the CPU: the torch graph
+ loss + Adam of paper_2409_02912_b200/training.py against the reference's
own train_step on the same batch (tests/golden/train_*.npz, made by
tests/golden/make_golden_train.py): loss breakdown, every gradient and the
weights after one Adam update; masking and var_io variants, inactive UEs."""

import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def _config(name):
    from paper_2409_02912_b200.config import NrxConfig, default_mcs_table
    t = default_mcs_table()
    if name == "train_masking":
        return NrxConfig.from_table(t, (9, 14, 19), variant="masking", d_s=8, num_iterations=2)
    return NrxConfig.from_table(t, (9, 14, 19), variant="var_io", d_s=8, hidden_width=12, num_iterations=2)


@pytest.mark.parametrize("name", ["train_masking", "train_var_io"])
def test_train_step_matches_reference(name):
    torch = pytest.importorskip("torch")
    from paper_2409_02912_b200.training import Adam, TorchNrxGraph, train_step, training_loss
    a = _load(name)
    config = _config(name)
    w0 = {k[4:]: v for k, v in a.items() if k.startswith("w0::")}
    g = TorchNrxGraph(config, w0, "cpu")
    t = lambda x, dt=torch.float32: torch.as_tensor(x).to(dt)
    args = (t(a["feats"]), t(a["labels"]), t(a["label_mask"]), t(a["chest_target"]), a["active"], a["mods"])
    total, bce, mse = training_loss(g, *args, gamma=0.1)
    assert abs(float(total) - float(a["total"])) <= 1e-5 * abs(float(a["total"]))
    assert abs(float(bce) - float(a["bce"])) <= 1e-5 * abs(float(a["bce"]))
    assert abs(float(mse) - float(a["mse"])) <= 1e-5 * abs(float(a["mse"]))
    total.backward()
    grads = {k[3:]: v for k, v in a.items() if k.startswith("g::")}
    touched = {k for k, p in g.params.items() if p.grad is not None}
    assert touched == set(grads)
    for k, ref in grads.items():
        got = g.params[k].grad.numpy()
        np.testing.assert_allclose(got, ref, rtol=2e-4, atol=2e-6 * max(1.0, np.abs(ref).max()), err_msg=k)
    # one full step: weights after the Adam update
    g2 = TorchNrxGraph(config, w0, "cpu")
    res = train_step(g2, Adam(lr=1e-3), *args, gamma=0.1)
    assert abs(res["total"] - float(a["total"])) <= 1e-5 * abs(float(a["total"]))
    w1 = {k[4:]: v for k, v in a.items() if k.startswith("w1::")}
    got = g2.numpy_weights()
    for k, ref in w1.items():
        # Adam's first step moves every touched weight by ~lr * sign(g): compare the step itself
        step_ref, step_got = ref - w0[k], got[k] - w0[k]
        np.testing.assert_allclose(step_got, step_ref, rtol=1e-3, atol=1e-6, err_msg=k)


def test_adam_gradient_checks_mirror_reference():
    """adam_step (autodiff.py:497-525): parameters before the first missing /
    non-finite gradient are updated, then ValueError names the parameter."""
    import torch
    from paper_2409_02912_b200.training import Adam
    p = {k: torch.ones(3) for k in ("a", "b", "c")}
    p["a"].grad = torch.ones(3)
    p["b"].grad = torch.tensor([1.0, float("nan"), 1.0])
    p["c"].grad = torch.ones(3)
    with pytest.raises(ValueError, match="non-finite gradient for parameter 'b'"):
        Adam(lr=0.1).step(p, ["a", "b", "c"])
    assert not torch.equal(p["a"], torch.ones(3)) and torch.equal(p["b"], torch.ones(3))
    assert torch.equal(p["c"], torch.ones(3))
    p["b"].grad = None
    with pytest.raises(ValueError, match="missing gradient for parameter 'b'"):
        Adam(lr=0.1).step(p, ["a", "b", "c"])
