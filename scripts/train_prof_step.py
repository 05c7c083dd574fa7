import os, sys
sys.path.insert(0, '/root/repo')
import torch
from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights
from paper_2409_02912_b200.slotgen import GpuSlotSource
from paper_2409_02912_b200.training import Adam, GpuTrainConfig, TorchNrxGraph, train_gpu
table = default_mcs_table()
cfg = SlotConfig(num_subcarriers=96, num_ues=2)
config = NrxConfig.from_table(table, (14,), d_s=56, num_iterations=2)
w = init_weights(config, 0)
src = GpuSlotSource(cfg)
g = TorchNrxGraph(config, w, src.device, kernels=sys.argv[1] if len(sys.argv) > 1 else "nrx")
train_gpu(config, w, src, table, GpuTrainConfig(batch_size=32, steps=3, seed=1), graph=g, adam=Adam(lr=1e-3))
torch.cuda.synchronize()
