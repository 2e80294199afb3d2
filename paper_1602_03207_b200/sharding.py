"""Probe-position sharding over ranks (SURVEY.md §8(e), configs[3]).

Positions are independent given the matrices (scan.cpp:155-156), so each rank
(one per GPU) owns a disjoint round-robin subset and needs no collective on the
data path. The only cross-rank traffic is the end-of-run reduction of timings
and signals: `reduce_timing` (max time, summed work) and `gather_points`
(rank-0 trace in z order, as run_scan sorts, scan.cpp:160-161). Works on any
torch.distributed backend (NCCL on B200 ranks, gloo in the CPU tests).
"""
from __future__ import annotations


def positions_for(step: int, rank: int, world: int, per_rank: int, positions) -> list:
    """Positions of `rank` at `step`: global slot (step*world + rank)*per_rank + q."""
    n = len(positions)
    return [positions[((step * world + rank) * per_rank + q) % n] for q in range(per_rank)]


def shard(positions, rank: int, world: int) -> list:
    """Static round-robin split of a whole sweep: position i -> rank i % world
    (the reference's parallel_for assignment, worker_pool.hpp:12-14)."""
    return [z for i, z in enumerate(positions) if i % world == rank]


def reduce_timing(elapsed_ms: float, work: float, failed: int, launches: int, device=None):
    """(max elapsed, sum work, sum failed, sum launches) over ranks."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return elapsed_ms, work, failed, launches
    t = torch.tensor([elapsed_ms, work, float(failed), float(launches)], dtype=torch.float64,
                     device=device)
    mx = t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = t.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return float(mx[0]), float(sm[1]), int(sm[2]), int(sm[3])


def gather_points(points: list, root: int = 0):
    """All ranks' signal points on `root`, sorted by z (scan.cpp:160-161)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return sorted(points, key=lambda p: p["z"])
    out = [None] * dist.get_world_size() if dist.get_rank() == root else None
    dist.gather_object(points, out, dst=root)
    if dist.get_rank() != root:
        return None
    merged = [p for part in out for p in part]
    return sorted(merged, key=lambda p: p["z"])
