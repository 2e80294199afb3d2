"""The N>1 (row-partitioned) solve protocol on CPU with gloo.

Each rank builds ITS halo plan through the C ABI (ect_halo_plan_*, host-only
code the GPU ranks run too), exchanges ghost values with the neighbour ranks
exactly as ect_dist_solve does over NCCL (A values of the send nodes, then V
values of the conductor send nodes), applies its owned rows of the reference
matrix to the local + ghost vector, and all-reduces the COCG dot product. The
owned rows of A x and the dot must equal the single-process results.
"""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch.multiprocessing as mp

from oracle import port
from tests.helpers import golden, ref_matrix


def neighbours(n_nodes, tets):
    t = tets.astype(np.int64)
    pairs = np.concatenate([t[:, [a, b]] for a in range(4) for b in range(4)])
    key = np.unique(pairs[:, 0] * n_nodes + pairs[:, 1])
    src, dst = key // n_nodes, key % n_nodes
    off = np.zeros(n_nodes + 1, np.int64)
    np.add.at(off, src + 1, 1)
    return np.cumsum(off).astype(np.int32), dst.astype(np.int32)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def local_to_global(plan, n_nodes, cond_fwd):
    """Global dof of every local slot: [A owned | A ghost | V owned | V ghost]."""
    nodes = np.concatenate([np.arange(plan.n0, plan.n1), plan.ghost_nodes]).astype(np.int64)
    a = (3 * nodes[:, None] + np.arange(3)).ravel()
    v = np.full(plan.Vo + plan.Vg, -1, np.int64)
    m = plan.local_vdof >= 0
    v[plan.local_vdof[m]] = 3 * n_nodes + cond_fwd[nodes[m]]
    return np.concatenate([a, v])


def _worker(rank, world, mport, splits, q):
    import torch
    import torch.distributed as dist
    from paper_1602_03207_b200 import ect
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(mport))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = golden("small_6x6x12")
        n_nodes = len(g["xyz"])
        cond = port.conductor_map(n_nodes, g["tets"], g["region"])
        off, nbr = neighbours(n_nodes, g["tets"])
        plan = ect.HaloPlan(n_nodes, off, nbr, cond, splits, rank)
        A = ref_matrix(g).tocsr()
        n = A.shape[0]
        rng = np.random.default_rng(5)
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        l2g = local_to_global(plan, n_nodes, cond)
        xl = np.zeros(len(l2g), np.complex128)
        L, G, Vo = plan.L, plan.G, plan.Vo
        owned = np.r_[0:3 * L, 3 * (L + G):3 * (L + G) + Vo]
        xl[owned] = x[l2g[owned]]                      # only the owned rows are known
        # halo exchange: A of send nodes then V of conductor send nodes
        reqs, bufs = [], []
        for p in plan.peers:
            sn, sc = p["send_nodes"], p["send_cond_nodes"]
            msg = np.concatenate([xl[(3 * sn[:, None] + np.arange(3)).ravel()],
                                  xl[3 * (L + G) + plan.local_vdof[sc]]])
            reqs.append(dist.isend(torch.from_numpy(msg.view(np.float64).copy()), dst=int(p["part"])))
            rb = torch.empty(2 * (3 * p["recv_node_count"] + p["recv_v_count"]), dtype=torch.float64)
            reqs.append(dist.irecv(rb, src=int(p["part"])))
            bufs.append((p, rb))
        for r in reqs:
            r.wait()
        for p, rb in bufs:
            v = rb.numpy().view(np.complex128)
            na_cnt = 3 * p["recv_node_count"]
            a0 = 3 * (L + p["recv_node_begin"])
            xl[a0:a0 + na_cnt] = v[:na_cnt]
            v0 = 3 * (L + G) + Vo + p["recv_v_begin"]
            xl[v0:v0 + p["recv_v_count"]] = v[na_cnt:]
        # owned rows applied to local + ghost values only
        rows = l2g[owned]
        cols = sp.csr_matrix((np.ones(len(l2g)), (l2g, np.zeros(len(l2g), int))), shape=(n, 1))
        Ar = A[rows]
        assert set(Ar.indices) <= set(l2g.tolist()), "owned rows reference a column outside the halo"
        xg = np.zeros(n, np.complex128)
        xg[l2g] = xl
        y = Ar @ xg
        y_ref = (A @ x)[rows]
        err = np.max(np.abs(y - y_ref)) / np.max(np.abs(y_ref))
        # unconjugated COCG dot over owned rows, summed across ranks
        d = torch.tensor([np.sum(x[rows] * y).real, np.sum(x[rows] * y).imag], dtype=torch.float64)
        dist.all_reduce(d)
        dot_ref = np.sum(x * (A @ x))
        derr = abs(complex(d[0], d[1]) - dot_ref) / abs(dot_ref)
        q.put((rank, err, derr, plan.L, plan.G, plan.Vo, plan.Vg, len(plan.peers), int(cols.nnz)))
    except Exception as e:  # report instead of leaving the parent waiting
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
@pytest.mark.parametrize("splits", [[0, 300, 637], [0, 180, 400, 637]])
def test_halo_protocol_gloo(splits):
    world = len(splits) - 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_, splits, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=150) for _ in range(world)]
    assert all(len(r) > 2 for r in res), res
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    res.sort()
    assert sum(r[3] for r in res) == 637                   # owned nodes partition the mesh
    for rank, err, derr, L, G, Vo, Vg, npeer, _ in res:
        assert err <= 1e-13, (rank, err)
        assert derr <= 1e-13, (rank, derr)
        assert G > 0 and npeer == (1 if rank in (0, world - 1) else 2)


def test_halo_plan_contract():
    from paper_1602_03207_b200 import ect
    g = golden("small_4x4x8")
    n_nodes = len(g["xyz"])
    cond = port.conductor_map(n_nodes, g["tets"], g["region"])
    off, nbr = neighbours(n_nodes, g["tets"])
    splits = [0, 100, 225]
    plans = [ect.HaloPlan(n_nodes, off, nbr, cond, splits, r) for r in range(2)]
    # every ghost is owned by the peer it is received from; send == receive sizes
    for r, P in enumerate(plans):
        assert np.all(np.diff(P.ghost_nodes) > 0)
        for peer in P.peers:
            Q = plans[peer["part"]]
            back = next(p for p in Q.peers if p["part"] == r)
            assert back["recv_node_count"] == len(peer["send_nodes"])
            assert back["recv_v_count"] == len(peer["send_cond_nodes"])
            got = Q.ghost_nodes[back["recv_node_begin"]:back["recv_node_begin"] + back["recv_node_count"]]
            assert np.array_equal(got, P.n0 + peer["send_nodes"])
    with pytest.raises(ect.ConfigError):
        ect.HaloPlan(n_nodes, off, nbr, cond, [0, 300, 225], 0)
