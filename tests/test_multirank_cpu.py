"""The N > 1 path on CPU: two gloo ranks each solve their shard (FP64 oracle
standing in for the device kernel, which this container cannot run) and
all-reduce the three statistics exactly as bench.py / the sharded ABI do; the
reduced means must equal a single-process run over the whole batch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2304_12745_b200 as U
from paper_2304_12745_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O

    w = U.CONFIGS[1]
    lam, eta = w.layer_params()
    per = 96
    if mode == "weak":
        first, n = sharding.weak_shard(rank, per)
    else:
        first, n = sharding.strong_shard(rank, world, 2 * per + 1)
    H = U.make_inputs(w, first, n)
    r = O.forward_batch_f32(H, w.c, lam, eta, w0_mode=w.w0_mode, threads=1)
    # alpha = 1 (SystemConfig::uniform default): consumed power = ||W||_{2,1}
    stats = torch.tensor([float(np.nansum(r["l21"])), float(r["active"][r["diverged_at"] < 0].sum()),
                          float((r["diverged_at"] >= 0).sum())], dtype=torch.float64)
    sharding.reduce_stats(stats)
    if rank == 0:
        np.save(out_path, stats.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["weak", "strong"])
def test_two_gloo_ranks_reduce_to_single_process_totals(tmp_path, mode):
    from oracle import oracle as O

    out = str(tmp_path / "stats.npy")
    mp.spawn(_worker, args=(2, _free_port(), mode, out), nprocs=2, join=True)
    got = np.load(out)
    w = U.CONFIGS[1]
    lam, eta = w.layer_params()
    total = 2 * 96 if mode == "weak" else 2 * 96 + 1
    H = U.make_inputs(w, 0, total)
    r = O.forward_batch_f32(H, w.c, lam, eta, w0_mode=w.w0_mode, threads=2)
    ref = np.array([np.nansum(r["l21"]), r["active"].sum(), (r["diverged_at"] >= 0).sum()], dtype=float)
    assert got[2] == ref[2] == 0
    assert got[1] == ref[1]
    assert abs(got[0] - ref[0]) <= 1e-12 * ref[0]
    s = sharding.summarize(got, total)
    assert s["mean_active"] == ref[1] / total


def test_shard_layouts_cover_the_batch():
    for world in (1, 2, 3, 4, 8):
        for total in (0, 1, 7, 65536, 1048576):
            spans = [sharding.strong_shard(r, world, total) for r in range(world)]
            assert sum(n for _, n in spans) == total
            assert all(spans[i][0] + spans[i][1] == spans[i + 1][0] for i in range(world - 1))
    assert sharding.weak_shard(3, 65536) == (3 * 65536, 65536)
    with pytest.raises(ValueError):
        sharding.strong_shard(2, 2, 10)
