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
    # the partitioned solve is Jacobi-COCG: compare against the same method
    a = ect.Matrix(ctx, m).assemble(p).set_preconditioner("jacobi")
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
        # the partitioned solve is the single-reduction (Chronopoulos-Gear)
        # form of the same Jacobi-COCG: equal in exact arithmetic
        assert abs(rd[c]["iterations"] - r1[c]["iterations"]) <= max(3, 0.03 * r1[c]["iterations"])
        ea, ev = solution_errors(xd[:, c], x1[:, c], m.n_nodes, comp)
        assert ea <= 1e-8 and ev <= 1e-8, (ea, ev)
        ea, ev = solution_errors(xd[:, c], g["primary_x"][c], m.n_nodes, comp)
        assert ea <= 1e-6 and ev <= 1e-6, (ea, ev)


@pytest.mark.parametrize("splits", [[0, 300, 637], [0, 150, 330, 500, 637]])
def test_slab_assembled_parts_equal_cut_parts(ctx, splits):
    """ect_part_create_assembled (only the slab's rows assembled) gives the same
    part as cutting the assembled global matrix: bitwise-equal solves."""
    g = golden("small_6x6x12")
    m, a = _setup(ctx, g)
    p, _, _ = m.materials(workloads.Physics(sigma_defect=1e4, mu_r_defect=5.0))
    cut = [ect.Part(ctx, m, a, splits, r) for r in range(len(splits) - 1)]
    own = [ect.Part(ctx, m, None, splits, r, mats=p) for r in range(len(splits) - 1)]
    assert [c.info for c in cut] == [o.info for o in own]
    b = np.ascontiguousarray(g["rhs"].T)
    x1, r1 = ect.dist_solve(cut, b, tol=1e-10, max_iter=20000)
    x2, r2 = ect.dist_solve(own, b, tol=1e-10, max_iter=20000)
    assert x1.tobytes() == x2.tobytes()
    assert [r["iterations"] for r in r1] == [r["iterations"] for r in r2]


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


def test_zslab_partition_of_relabelled_configs0(ctx):
    """configs[4]'s layout at configs[0] size: the mesh numbered z-slowest, cut
    into 4 contiguous node ranges = z-slabs; the partitioned solve, mapped back
    to the reference numbering, matches the reference's GMRES solution."""
    w = workloads.config0()
    ref_mesh = w.mesh()
    w.extra = dict(w.extra, node_order="kij")
    mm = w.mesh()
    m = ect.Mesh(ctx, mm.xyz, mm.tets, mm.region)
    p, _, _ = m.materials(w.physics)
    a = ect.Matrix(ctx, m).assemble(p)
    nx, ny, nz = w.dims
    ii, jj, kk = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    new_id = ((kk * (nx + 1) + ii) * (ny + 1) + jj).ravel()  # reference node -> relabelled node
    assert np.array_equal(new_id[ref_mesh.tets], mm.tets)
    per = (nx + 1) * (ny + 1)
    splits = np.array([0, 10, 20, 30, nz + 1]) * per   # 4 slabs of z-planes
    parts = [ect.Part(ctx, m, a, splits, r) for r in range(4)]
    b = m.rhs(w.coil, [w.positions[0]] * 2, [1, 2], w.amplitude)
    xd, rd = ect.dist_solve(parts, b, tol=1e-8, max_iter=20000)
    gold = np.load(GOLDEN / "cfg0.npz")
    fwd_ref = ect.Mesh(ctx, ref_mesh.xyz, ref_mesh.tets, ref_mesh.region).export()["cond_forward"]
    fwd_new = m.export()["cond_forward"]
    na = 3 * m.n_nodes
    back = np.empty(len(xd), np.int64)  # reference dof -> relabelled dof
    nodes = np.arange(m.n_nodes)
    for c in range(3):
        back[3 * nodes + c] = 3 * new_id + c
    cond = np.flatnonzero(fwd_ref >= 0)
    back[na + fwd_ref[cond]] = na + fwd_new[new_id[cond]]
    comp = conductor_components(ref_mesh.tets, ref_mesh.region, fwd_ref)
    for c in range(2):
        assert rd[c]["converged"]
        ea, ev = solution_errors(xd[back, c], gold["x"][c], m.n_nodes, comp)
        assert ea <= 1e-6 and ev <= 1e-6, (ea, ev)
