"""CPU, world_size 2 over gloo: the multi-GPU plumbing of SURVEY §8e.

Envs shard by contiguous global index range (sharding.shard_range); every
stream is keyed by the GLOBAL env index, so a shard reproduces its slice of the
whole batch bit for bit, and the only collective -- the all-reduce of the
episode statistics (sharding.allreduce_stats) -- reproduces the whole-batch
totals. The per-shard stepping here is the oracle (the GPU legs are covered by
test_gpu_parity.py::test_shards_equal_whole_batch); what is under test is the
partitioning and the collective."""
import os
import socket

import numpy as np
import pytest

from oracle_bindings import Oracle, default_config

N_TOTAL = 7
SEED = 11
STEPS = 9
CFG = dict(n_agents=2, n_targets=2, horizon=4, pf_n_particles=32)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_partitions():
    from paper_2505_08222_b200.sharding import shard_range
    for n in (0, 1, 7, 64, 65537):
        for world in (1, 2, 3, 8):
            ranges = [shard_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    from paper_2505_08222_b200.sharding import allreduce_stats, shard_range
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    lo, hi = shard_range(N_TOTAL, rank, world)
    env = Oracle(default_config(**CFG), hi - lo, SEED, env_index_offset=lo)
    env.step_policy(STEPS)
    total = allreduce_stats(env.stats()).numpy()
    blobs = np.stack([env.serialize(e) for e in range(hi - lo)])
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), total=total, blobs=blobs, lo=lo, hi=hi)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_reproduce_whole_batch(tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    whole = Oracle(default_config(**CFG), N_TOTAL, SEED)
    whole.step_policy(STEPS)
    want = whole.stats()
    for rank in range(world):
        r = np.load(tmp_path / f"rank{rank}.npz")
        for i, e in enumerate(range(int(r["lo"]), int(r["hi"]))):
            assert r["blobs"][i].tobytes() == whole.serialize(e).tobytes(), f"rank {rank} env {e}"
        # counts are exact; sums of fp64 differ only by the order of addition
        np.testing.assert_allclose(r["total"], want, rtol=1e-12, atol=0)
