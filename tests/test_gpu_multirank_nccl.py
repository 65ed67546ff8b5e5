"""The bench's N > 1 path with real NCCL ranks: two processes, one GPU each,
each running the fused forward on its contiguous shard of one batch and
all-reducing the three statistics (sharding.reduce_stats, as bench.py does).
The reduced sums must equal one device's run over the whole batch, and every
shard must equal the same realizations run alone, bit for bit — the ordered
per-index-slot semantics of the reference's parallel_for
(proj/core/include/ufpgd/parallel.hpp:12-18). Skipped with fewer than two
GPUs (the gpurun box has one; the world-size-2 gloo test covers the host
logic on CPU)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    import paper_2304_12745_b200 as U
    from paper_2304_12745_b200 import sharding

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    w = U.CONFIGS[2]
    total = 20000 + 3
    first, n = sharding.strong_shard(rank, world, total)
    H = torch.from_numpy(U.make_inputs(w, first, n)).cuda()
    lam, eta = w.layer_params()
    out = U.unfolded_forward(H, lam, eta, w.c, w0_mode=w.w0_mode)
    sharding.reduce_stats(out["stats"])
    torch.cuda.synchronize()
    np.save(os.path.join(out_dir, f"W{rank}.npy"), out["W"].cpu().numpy())
    np.save(os.path.join(out_dir, f"stats{rank}.npy"), out["stats"].cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_nccl_ranks_match_one_device(tmp_path):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as mp

    import paper_2304_12745_b200 as U

    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    w = U.CONFIGS[2]
    total = 20000 + 3
    H = torch.from_numpy(U.make_inputs(w, 0, total)).cuda()
    lam, eta = w.layer_params()
    one = U.unfolded_forward(H, lam, eta, w.c, w0_mode=w.w0_mode)
    Wcat = np.concatenate([np.load(tmp_path / f"W{r}.npy") for r in range(2)])
    assert np.array_equal(Wcat, one["W"].cpu().numpy())
    ref = one["stats"].cpu().numpy()
    for r in range(2):
        st = np.load(tmp_path / f"stats{r}.npy")
        assert st[1] == ref[1] and st[2] == ref[2] == 0
        assert abs(st[0] - ref[0]) <= 1e-12 * ref[0]
