"""Multi-process (gloo, world_size 2) tests of the probe-sweep sharding logic
used by bench.py --gpus N; CPU only."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1602_03207_b200 import sharding, workloads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    positions = workloads.config3().positions
    mine = sharding.shard(positions, rank, world)
    # fake per-position results (what solve_position returns), rank-specific timing
    pts = [{"z": z, "dz": [rank], "failed": False} for z in mine]
    el, work, failed, launches = sharding.reduce_timing(10.0 + rank, 100.0 * len(mine), 0, 3)
    merged = sharding.gather_points(pts)
    steps = [sharding.positions_for(s, rank, world, 2, positions) for s in range(3)]
    q.put((rank, el, work, failed, launches, merged, steps))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_sharding_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=100)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    positions = workloads.config3().positions
    for rank, el, work, failed, launches, merged, steps in res.values():
        assert el == 11.0                       # max over ranks
        assert work == 100.0 * len(positions)   # summed work
        assert launches == 6
    merged = res[0][5]
    assert [p["z"] for p in merged] == sorted(positions)      # complete, disjoint, z-sorted
    assert res[1][5] is None
    # per-step slots are disjoint across ranks and cover consecutive positions
    for s in range(3):
        a, b = res[0][6][s], res[1][6][s]
        assert not set(a) & set(b)
        assert sorted(a + b) == sorted(positions[4 * s: 4 * s + 4])


def test_shard_round_robin_matches_parallel_for():
    pos = list(range(10))
    assert sharding.shard(pos, 0, 3) == [0, 3, 6, 9]
    assert sorted(sum((sharding.shard(pos, r, 3) for r in range(3)), [])) == pos
