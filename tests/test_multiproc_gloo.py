"""world_size-2 gloo test of the slot-sharding host logic (CPU only): each
rank runs the CPU oracle on its contiguous shard of slots, per-slot hard-bit
error counts are gathered to rank 0 and must equal the single-process run;
the job time is the MAX over ranks."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_02912_b200.shard import StepGather, gather_slot_results, max_over_ranks, shard_slots, sum_over_ranks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    from oracle import nrx_oracle as orc
    from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights
    from paper_2409_02912_b200.synth import synth_slots
    table = default_mcs_table()
    cfg = SlotConfig(num_subcarriers=24, num_ues=2, comb_size=2)
    config = NrxConfig.from_table(table, (14,), d_s=8, num_iterations=2)
    w = orc.perturb_biases(init_weights(config, 0))
    y, books, bits = synth_slots(cfg, [4, 4], 5, 0.1, seed=2)
    return orc, cfg, config, w, (table[14], table[14]), y, books, bits


def _errors(orc, cfg, config, w, mcs, y, books, bits, idx):
    s_idx, t_idx = np.nonzero(cfg.data_mask)
    out = []
    for i in idx:
        llrs, _ = orc.nrx_forward(y[i], books[i], cfg, mcs, w, config, 0.1)
        out.append([int(((llrs[u][s_idx, t_idx] > 0) != bits[u][i]).sum()) for u in range(2)])
    return np.asarray(out, dtype=np.int64).reshape(-1, 2)


def _worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc, cfg, config, w, mcs, y, books, bits = _problem()
    shard = shard_slots(len(y), rank, world)
    local = _errors(orc, cfg, config, w, mcs, y, books, bits, shard)
    full = gather_slot_results(local, len(y))
    t = max_over_ranks(float(rank + 1))
    if rank == 0:
        np.save(result_path, np.concatenate([full.reshape(-1), [int(t)]]))
    dist.destroy_process_group()


def test_shard_slots_partition():
    for n in (1, 5, 4096):
        for world in (1, 2, 3, 8):
            got = [i for r in range(world) for i in shard_slots(n, r, world)]
            assert got == list(range(n))
    with pytest.raises(ValueError):
        shard_slots(4, 2, 2)


def test_two_rank_gloo_gather_matches_single_process(tmp_path):
    path = str(tmp_path / "r.npy")
    mp.spawn(_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    res = np.load(path)
    orc, cfg, config, w, mcs, y, books, bits = _problem()
    ref = _errors(orc, cfg, config, w, mcs, y, books, bits, range(len(y)))
    np.testing.assert_array_equal(res[:-1].reshape(-1, 2), ref)
    assert res[-1] == 2  # max over ranks of (rank + 1)


def _worker_gather(rank, world, port, result_path):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    step = torch.full((3, 2, 4), float(rank + 1))
    g = StepGather(step)
    out = g(step)
    counts = sum_over_ranks(torch.tensor([rank + 1, 10 * (rank + 1)], dtype=torch.int64))
    if rank == 0:
        np.save(result_path, np.concatenate([torch.stack(out).reshape(-1).numpy(), counts.numpy(),
                                             [g.bytes_per_step(step)]]))
    dist.destroy_process_group()


def test_step_gather_and_counter_reduce_world2(tmp_path):
    """The bench's with-gather step (one result tensor per rank into rank 0)
    and the Monte-Carlo counter all-reduce, on gloo with world size 2."""
    path = str(tmp_path / "g.npy")
    mp.spawn(_worker_gather, args=(2, _free_port(), path), nprocs=2, join=True)
    r = np.load(path)
    got = r[:48].reshape(2, 3, 2, 4)
    assert (got[0] == 1).all() and (got[1] == 2).all()
    assert list(r[48:50]) == [3, 30]
    assert r[50] == 3 * 2 * 4 * 4
