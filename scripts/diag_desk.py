"""Uncoded BER vs SNR of the desk checkpoints on the GPU pipeline (diagnostic)."""
import os, sys
sys.path.insert(0, os.getcwd())
from paper_2409_02912_b200.config import SlotConfig, checkpoint_load, default_mcs_table
from paper_2409_02912_b200.engine import NrxEngine
from paper_2409_02912_b200.slotgen import GpuSlotSource, evaluate_uncoded
from paper_2409_02912_b200.ldpc import evaluate_coded
t = default_mcs_table()
cfg = SlotConfig(num_subcarriers=96, num_ues=2)
src = GpuSlotSource(cfg)
for name in ("desk_d16_it2", "desk_d16_it2_long"):
    config, w = checkpoint_load(f"tests/golden/{name}.nrxw")
    eng = NrxEngine(config, w, precision="fp16")
    rec = evaluate_uncoded(eng, src, (t[14], t[14]), [5, 10, 15, 20, 25, 30], n_slots=64, batch=32)
    print(name, "uncoded", [(r.snr_db, round(r.ber, 4)) for r in rec])
    rec = evaluate_coded(eng, src, (t[14], t[14]), [10, 15, 20, 25, 30], n_slots=64, batch=32)
    print(name, "coded", [(r.snr_db, round(r.tbler, 3), round(r.ber, 4)) for r in rec])
