"""Golden vectors for the LDPC decoder, made by the REFERENCE itself.

Run in the build container (where the read-only reference lives):

    PYTHONPATH=/root/reference/pkg/src python -B tests/golden/make_golden_ldpc.py

For a few of the reference's own codes (build_regular_code, rate_matched_code
with shortening and puncturing; ldpc.py:280-330) it stores the code structure
and batches of LLRs — noiseless, BPSK-over-AWGN at several noise levels (some
codewords do not converge), and a few random ones — together with the
reference decoder's outputs (info bits, success flags; ldpc.py:99-178) at 20
iterations and at 3 iterations (exercising the no-convergence exit).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = os.environ.get("NRX_REFERENCE_SRC", "/root/reference/pkg/src")
if REF not in sys.path:
    sys.path.insert(0, REF)

from nrxsim import ldpc  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
CASES = [
    dict(name="ldpc_648", kind="regular", args=(648, 324)),
    dict(name="ldpc_rm1152", kind="rate_matched", args=(1152, 553 / 1024)),   # desk 16-QAM slot (S=24)
    dict(name="ldpc_rm576", kind="rate_matched", args=(576, 679 / 1024)),     # desk QPSK slot
    dict(name="ldpc_rm900_033", kind="rate_matched", args=(900, 0.33)),       # shortening
]


def main():
    index = []
    for i, c in enumerate(CASES):
        code = ldpc.build_regular_code(*c["args"]) if c["kind"] == "regular" else ldpc.rate_matched_code(*c["args"])
        rng = np.random.default_rng((1234, i))
        info = (rng.random((24, code.k_eff)) < 0.5).astype(np.uint8)
        tx = code.encode(info).astype(np.float64)
        llrs = [20.0 * (2 * tx[:4] - 1)]
        for sigma in (0.5, 0.7, 0.9, 1.1):
            rx = (2 * tx[4:9] - 1) + sigma * rng.normal(size=tx[4:9].shape)
            llrs.append(np.clip(2.0 * rx / sigma ** 2, -20.0, 20.0))
        llrs.append(rng.normal(scale=3.0, size=(4, code.num_tx_bits)))
        llr = np.concatenate(llrs).astype(np.float32)
        dec20, ok20 = code.decode(llr, 20)
        dec3, ok3 = code.decode(llr, 3)
        np.savez_compressed(
            os.path.join(OUT, f"{c['name']}.npz"),
            n=code.n, k=code.k, row_cols=code.row_cols, col_rows=code.col_rows, col_slots=code.col_slots,
            info_positions=code.info_positions, punctured=code.punctured, shortened=code.shortened,
            tx_positions=code.tx_positions, info=info[:llr.shape[0]], llr=llr,
            dec20=dec20, ok20=ok20, dec3=dec3, ok3=ok3)
        index.append(dict(name=c["name"], kind=c["kind"], args=list(c["args"]), n=code.n, k=code.k,
                          k_eff=code.k_eff, num_tx_bits=code.num_tx_bits, ok20=int(ok20.sum()), ok3=int(ok3.sum()),
                          batch=int(llr.shape[0])))
        print(index[-1])
    with open(os.path.join(OUT, "ldpc_index.json"), "w") as f:
        json.dump(index, f, indent=1)


if __name__ == "__main__":
    main()
