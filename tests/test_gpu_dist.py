"""Row-partitioned (multi-GPU) solve on ONE GPU: every part runs in this
process with device-copy halos and a fixed-order cross-part sum — the same
kernels, partition and halo plan as the NCCL path. The
partitioned solution must match the single-part solve and the reference.
A 1-rank NCCL communicator exercises the NCCL transport (allreduce)."""
import numpy as np
import pytest

from paper_1602_03207_b200 import ect, workloads
from tests.helpers import GOLDEN, conductor_components, golden, solution_errors

pytestmark = pytest.mark.gpu


def _setup(ctx, g):
    m = ect.Mesh(ctx, g["xyz"], g["tets"], g["region"])
    p, r, _ = m.materials(workloads.Physics(sigma_defect=1e4, mu_r_defect=5.0))
    a = ect.Matrix(ctx, m).assemble(p)
    return m, a


@pytest.mark.parametrize("splits", [[0, 300, 637], [0, 150, 330, 500, 637], [0, 637]])
def test_partitioned_solve_matches_single(ctx, splits):
    g = golden("small_6x6x12")
    m, a = _setup(ctx, g)
    parts = [ect.Part(ctx, m, a, splits, r) for r in range(len(splits) - 1)]
    b = np.ascontiguousarray(g["rhs"].T)
    x1, r1 = a.solve(b, tol=1e-10, max_iter=20000)
    xd, rd = ect.dist_solve(parts, b, tol=1e-10, max_iter=20000)
    comp = conductor_components(g["tets"], g["region"], g["cond_forward"])
    for c in range(2):
        assert rd[c]["converged"] and rd[c]["residual"] <= 1e-10
        assert abs(rd[c]["iterations"] - r1[c]["iterations"]) <= 3
        ea, ev = solution_errors(xd[:, c], x1[:, c], m.n_nodes, comp)
        assert ea <= 1e-8 and ev <= 1e-8, (ea, ev)
        ea, ev = solution_errors(xd[:, c], g["primary_x"][c], m.n_nodes, comp)
        assert ea <= 1e-6 and ev <= 1e-6, (ea, ev)


def test_partitioned_configs0_vs_reference(ctx):
    w = workloads.config0()
    mm = w.mesh()
    m = ect.Mesh(ctx, mm.xyz, mm.tets, mm.region)
    p, _, _ = m.materials(w.physics)
    a = ect.Matrix(ctx, m).assemble(p)
    gold = np.load(GOLDEN / "cfg0.npz")
    b = mm_rhs = m.rhs(w.coil, [w.positions[0]] * 2, [1, 2], w.amplitude)
    splits = np.linspace(0, m.n_nodes, 5).astype(np.int64)   # 4 slabs of i-planes
    parts = [ect.Part(ctx, m, a, splits, r) for r in range(4)]
    xd, rd = ect.dist_solve(parts, b, tol=1e-8, max_iter=20000)
    comp = conductor_components(mm.tets, mm.region, m.export()["cond_forward"])
    for c in range(2):
        assert rd[c]["converged"]
        ea, ev = solution_errors(xd[:, c], gold["x"][c], m.n_nodes, comp)
        assert ea <= 1e-6 and ev <= 1e-6, (ea, ev)
    del mm_rhs


def test_nccl_transport_single_rank(ctx):
    g = golden("small_4x4x8")
    m, a = _setup(ctx, g)
    comm = ect.Comm(ctx, 0, 1, ect.comm_unique_id())
    part = ect.Part(ctx, m, a, [0, m.n_nodes], 0)
    b = np.ascontiguousarray(g["rhs"].T)
    xd, rd = ect.dist_solve([part], b, comm=comm, tol=1e-10, max_iter=20000)
    x1, r1 = a.solve(b, tol=1e-10, max_iter=20000)
    for c in range(2):
        assert rd[c]["converged"]
        assert np.linalg.norm(xd[:, c] - x1[:, c]) <= 1e-8 * np.linalg.norm(x1[:, c])
