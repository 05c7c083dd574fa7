"""Device time of the GPU LDPC layer at the C2 codeword size (273 PRB,
16-QAM: 157,248 coded bits, IRA mother code n = 169,840): encode, and
min-sum decode of BPSK-over-AWGN LLRs at a high SNR (early exit) and a low
SNR (all iterations).

  python scripts/profile_ldpc.py [--cw 64] [--iters 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2409_02912_b200.ldpc import GpuLdpc, rate_matched_ira_code  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cw", type=int, default=64)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    code = rate_matched_ira_code(3276 * 12 * 4, 553 / 1024)
    g = GpuLdpc(code)
    B = args.cw
    info = (torch.rand((B, code.k_eff), device="cuda") < 0.5).to(torch.uint8)
    ms = timed(lambda: g.encode(info))
    print(f"encode        {ms:8.3f} ms per {B} codewords  {ms * 1e3 / B:7.2f} us/codeword")
    tx = g.encode(info).float()
    for sigma in (0.5, 0.65, 0.72, 0.8, 1.2):
        llr = torch.clamp(2 * ((2 * tx - 1) + sigma * torch.randn_like(tx)) / sigma ** 2, -20, 20)
        ms = timed(lambda: g.decode(llr, args.iters))
        dec, ok = g.decode(llr, args.iters)
        ber = (dec != info).float().mean().item()
        print(f"decode s={sigma:.1f} {ms:8.3f} ms per {B} codewords  {ms * 1e3 / B:7.2f} us/codeword  "
              f"converged {ok.float().mean().item():.2f}  info BER {ber:.2e}")


if __name__ == "__main__":
    main()
