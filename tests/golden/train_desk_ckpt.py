"""Train a small desk NRX with the REFERENCE trainer and save it as an NRXW
fixture (tests/golden/desk_d16_it2.nrxw) for the BER/BLER statistics test.

    PYTHONPATH=/root/reference/pkg/src python -B tests/golden/train_desk_ckpt.py

Random-init weights give BER ~ 0.5 on both receivers (a trivial match,
SURVEY.md §8c); a briefly trained model makes the uncoded-BER comparison
between the reference CPU path and the GPU path meaningful.  Uses the
reference's own train() loop (training.py:254-284) on its default desk slot
(24 subcarriers, 2 UEs, DoubleTDL), exactly like pkg/_scratch/smoke_train.py.
"""

import os
import sys
import time

sys.dont_write_bytecode = True
REF = os.environ.get("NRX_REFERENCE_SRC", "/root/reference/pkg/src")
if REF not in sys.path:
    sys.path.insert(0, REF)

from nrxsim import training as tr  # noqa: E402
from nrxsim.channel import doubletdl  # noqa: E402
from nrxsim.nrx import NrxConfig, checkpoint_save, init_weights  # noqa: E402
from nrxsim.slot import SlotConfig, default_mcs_table  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "desk_d16_it2.nrxw")
STEPS = int(os.environ.get("NRX_TRAIN_STEPS", "800"))


def main():
    table = default_mcs_table()
    slot_cfg = SlotConfig()
    config = NrxConfig.from_table(table, (14,), variant="single", d_s=16, num_iterations=2)
    w = init_weights(config, seed=42)
    tcfg = tr.TrainConfig(batch_size=16, steps=STEPS, snr_lo_db=0.0, snr_hi_db=12.0,
                          supported_mcs=(14,), seed=42, log_every=100)
    t0 = time.time()
    tr.train(w, config, slot_cfg, doubletdl(), tcfg, table)
    checkpoint_save(OUT, config, w)
    print(f"saved {OUT} after {STEPS} steps in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
