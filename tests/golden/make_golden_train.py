"""Golden vectors for one training step, made by the REFERENCE itself.

Run in the build container (where the read-only reference lives):

    PYTHONPATH=/root/reference/pkg/src python -B tests/golden/make_golden_train.py

Draws a training batch with the reference's sampler (training.py:112-171:
variable active-UE counts, mixed MCS, SNR offsets, LDPC-coded labels), runs
its train_step pieces (training.py:180-234): the training-mode forward with
per-iteration readouts, the multi-loss BCE + gamma * MSE, autodiff backward
and one Adam update (autodiff.py:485-525), and stores features, labels,
masks, targets, the weights before, every gradient and the weights after.
Two models: masking (d_s = 8, N_it = 2, supported MCS 9/14/19) and var_io
(d_s = 8, hidden 12, N_it = 2).
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = os.environ.get("NRX_REFERENCE_SRC", "/root/reference/pkg/src")
if REF not in sys.path:
    sys.path.insert(0, REF)

from nrxsim import autodiff as ad  # noqa: E402
from nrxsim import training as tr  # noqa: E402
from nrxsim.channel import doubletdl  # noqa: E402
from nrxsim.nrx import NrxConfig, assemble_features, init_weights, nrx_forward_graph  # noqa: E402
from nrxsim.slot import SlotConfig, default_mcs_table  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def make(name, config, seed):
    table = default_mcs_table()
    slot_cfg = SlotConfig()
    tcfg = tr.TrainConfig(batch_size=4, steps=1, snr_lo_db=0.0, snr_hi_db=10.0, supported_mcs=(9, 14, 19),
                          gamma=0.1, seed=seed)
    batch = tr.sample_training_batch(slot_cfg, doubletdl(), tcfg, table, config, 0)
    w = init_weights(config, seed)
    rng = np.random.default_rng(99)
    for k in sorted(w):
        if k.endswith(".b"):
            w[k].data[...] = rng.normal(scale=0.1, size=w[k].data.shape).astype(np.float32)
    before = {k: v.data.copy() for k, v in w.items()}
    feats = assemble_features(batch.y, batch.ls, batch.n0, slot_cfg, config)
    out = nrx_forward_graph(feats, w, config, slot_cfg, batch.mods, training=True, active=batch.active,
                            collect_chest=True)
    # the loss of train_step (training.py:189-222), kept to read the pieces
    adam = ad.AdamState(lr=1e-3)
    losses = tr.train_step(w, adam, batch, config, slot_cfg, tcfg)
    after = {k: v.data.copy() for k, v in w.items()}
    # gradients: re-run forward + loss on the saved weights and backward
    w2 = {k: ad.Tensor(v.copy(), requires_grad=True) for k, v in before.items()}
    adam2 = ad.AdamState(lr=1e-3)
    grads = {}
    orig = ad.adam_step

    def capture(params, g, state):
        for k, p in params.items():
            grads[k] = p.grad.copy()
        orig(params, g, state)

    ad.adam_step = capture
    try:
        tr.train_step(w2, adam2, batch, config, slot_cfg, tcfg)
    finally:
        ad.adam_step = orig
    arrays = dict(feats=feats, labels=batch.labels, label_mask=batch.label_mask, chest_target=batch.chest_target,
                  active=batch.active, mods=batch.mods, total=losses["total"], bce=losses["bce"], mse=losses["mse"])
    for k in before:
        arrays[f"w0::{k}"] = before[k]
        arrays[f"w1::{k}"] = after[k]
        if k in grads:
            arrays[f"g::{k}"] = grads[k]
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **arrays)
    print(name, losses, len(grads), "grads", batch.active.tolist(), batch.mods.tolist())


def main():
    table = default_mcs_table()
    make("train_masking", NrxConfig.from_table(table, (9, 14, 19), variant="masking", d_s=8, num_iterations=2), 11)
    make("train_var_io", NrxConfig.from_table(table, (9, 14, 19), variant="var_io", d_s=8, hidden_width=12,
                                              num_iterations=2), 12)


if __name__ == "__main__":
    main()
