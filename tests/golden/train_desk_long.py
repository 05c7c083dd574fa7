"""Continue training the desk NRX (tests/golden/desk_d16_it2.nrxw) with the
REFERENCE trainer over a wider SNR range, for the coded (LDPC) TBLER test
that needs a receiver whose hard decisions are good enough to decode.

    PYTHONPATH=/root/reference/pkg/src python -B tests/golden/train_desk_long.py

Same reference train() loop (training.py:254-284) and desk slot as
train_desk_ckpt.py; output tests/golden/desk_d16_it2_long.nrxw.
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
from nrxsim.nrx import checkpoint_load, checkpoint_save  # noqa: E402
from nrxsim.slot import SlotConfig, default_mcs_table  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "desk_d16_it2.nrxw")
OUT = os.path.join(HERE, "desk_d16_it2_long.nrxw")
STEPS = int(os.environ.get("NRX_TRAIN_STEPS", "6000"))


def main():
    table = default_mcs_table()
    config, w = checkpoint_load(SRC)
    tcfg = tr.TrainConfig(batch_size=16, steps=STEPS, snr_lo_db=4.0, snr_hi_db=24.0, learning_rate=2e-3,
                          supported_mcs=(14,), seed=43, log_every=250)
    t0 = time.time()
    res = tr.train(w, config, SlotConfig(), doubletdl(), tcfg, table,
                   progress=lambda s, l: print(s, round(l['total'], 4), flush=True) if s % 250 == 0 else None)
    checkpoint_save(OUT, config, res.weights)
    print(f"saved {OUT} after {STEPS} steps in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
