"""Where the host time of one drop-in nrx_forward call goes (C2, one slot)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2409_02912_b200 import nrx as gnrx
from paper_2409_02912_b200.synth import synth_slots

cfg, config, w, mcs = bench.c2_setup()
y, books, _ = synth_slots(cfg, [4, 4], 2, 0.1, seed=5)
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)) * 1e3


print("full call", timeit(lambda: gnrx.nrx_forward(y[0], books[0], cfg, mcs, w, config, 0.1, precision=prec)))
print("fingerprint", timeit(lambda: gnrx._fingerprint(w)))
yy = y[:1]
print("astype c64", timeit(lambda: yy.astype(np.complex64)))
print("stack_pilots", timeit(lambda: gnrx.stack_pilots(books[0], 1, cfg)))
h = torch.empty(yy.shape, dtype=torch.complex128, pin_memory=True)
print("memcpy c128 to pinned", timeit(lambda: h.numpy().__setitem__(Ellipsis, yy)))
d = torch.empty(yy.shape, dtype=torch.complex128, device="cuda")
print("H2D pinned c128", timeit(lambda: (d.copy_(h, non_blocking=True), torch.cuda.synchronize())))
print("H2D pageable c128", timeit(lambda: (d.copy_(torch.from_numpy(yy)), torch.cuda.synchronize())))
o = torch.empty((1, 2, 3276, 14, 4), dtype=torch.complex64, device="cuda")
ho = torch.empty(o.shape, dtype=torch.complex64, pin_memory=True)
print("D2H pinned chest", timeit(lambda: (ho.copy_(o, non_blocking=True), torch.cuda.synchronize())))
print("chest numpy copy", timeit(lambda: ho.numpy().copy()))
out = np.empty(o.shape, np.complex64)
print("D2H pageable chest", timeit(lambda: torch.from_numpy(out).copy_(o)))
