"""cProfile of the drop-in nrx_forward host path (C2, one slot)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2409_02912_b200 import nrx as gnrx
from paper_2409_02912_b200.synth import synth_slots

cfg, config, w, mcs = bench.c2_setup()
y, books, _ = synth_slots(cfg, [4, 4], 2, 0.1, seed=5)
prec = sys.argv[1] if len(sys.argv) > 1 else "fp16"
for _ in range(5):
    gnrx.nrx_forward(y[0], books[0], cfg, mcs, w, config, 0.1, precision=prec)
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    gnrx.nrx_forward(y[0], books[0], cfg, mcs, w, config, 0.1, precision=prec)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
