"""Multi-GPU plumbing for independent-slot throughput.

Slots are independent (no batch statistics or cross-slot term anywhere in
nrx.py), so ranks take contiguous slot ranges with replicated weights; the
only collectives are the final gather of per-slot results and the MAX of
the per-rank elapsed time.  Works with any torch.distributed backend (NCCL
on the GPU box, gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np


def shard_slots(n_slots: int, rank: int, world: int) -> range:
    """Contiguous shard of slot indices for `rank`: slot i -> rank floor(i*world/n)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    return range(rank * n_slots // world, (rank + 1) * n_slots // world)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (the job time is the slowest rank's time)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_slot_results(local: np.ndarray, n_slots: int, device=None, dst: int = 0):
    """Gather per-slot result rows (leading axis = this rank's shard) to
    `dst` in global slot order; returns the full array on dst, None elsewhere.
    `device` defaults to the rank's current CUDA device under NCCL and to the
    host under gloo."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    if device is None:  # NCCL moves device tensors only: this rank's GPU; gloo: host memory
        device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else "cpu"
    sizes = [len(shard_slots(n_slots, r, world)) for r in range(world)]
    row_shape = local.shape[1:]
    pad = max(sizes)
    buf = torch.zeros((pad,) + row_shape, dtype=torch.from_numpy(local[:0]).dtype, device=device)
    buf[: local.shape[0]] = torch.from_numpy(np.ascontiguousarray(local)).to(buf.device)
    gathered = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, gathered, dst=dst)
    if rank != dst:
        return None
    return np.concatenate([g[:sizes[r]].cpu().numpy() for r, g in enumerate(gathered)])


def sum_over_ranks(t):
    """All-reduce SUM of a counter tensor (the Monte-Carlo loops' ``reduce``
    argument: slotgen.evaluate_uncoded, ldpc.evaluate_coded)."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return t
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


class StepGather:
    """Gather of one step's per-rank result tensor (same shape on every rank,
    e.g. the (B, U, S, T, W) LLRs of a bench step) into rank dst's
    preallocated buffers — the "with gather" variant of SURVEY.md §8e, on
    NCCL over NVLink for CUDA tensors (gloo for CPU tensors)."""

    def __init__(self, like, dst: int = 0):
        import torch
        import torch.distributed as dist
        self.world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank() if self.world > 1 else 0
        self.dst = dst
        self.bufs = [torch.empty_like(like) for _ in range(self.world)] if self.rank == dst else None

    def __call__(self, t):
        import torch.distributed as dist
        if self.world == 1:
            return [t]
        dist.gather(t, self.bufs if self.rank == self.dst else None, dst=self.dst)
        return self.bufs

    def bytes_per_step(self, t) -> int:
        return t.numel() * t.element_size() * max(0, self.world - 1)
