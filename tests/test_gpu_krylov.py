"""GPU Krylov recurrences against a numpy restatement, iteration by iteration.

The parity suite checks converged solutions against the reference; these tests
pin the batched Jacobi-COCG itself (krylov.cu cocg_solve): after exactly m
iterations (tolerance never met, max_iter = m) every column of x must equal
the plain COCG recurrence x_m -- which also checks that the x += alpha p the
p-update kernel owes for the final iteration lands (RhsState::xpend), that
padded batch columns (k = 3 runs as 4) stay inert and that a column with b = 0
does not disturb the others.  Test infrastructure: numpy is the checker only.
"""
import numpy as np
import pytest

from paper_1602_03207_b200 import ect
from tests.helpers import golden

pytestmark = pytest.mark.gpu


def cocg_numpy(row_ptr, col, val, b, m):
    """Jacobi-preconditioned COCG (unconjugated bilinear form), m iterations from
    x0 = 0: q = A p, alpha = rho / p^T q, x += alpha p, r -= alpha q,
    z = D^-1 r, beta = r^T z / rho, p = z + beta p."""
    n = len(row_ptr) - 1
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    diag = val[rows == col]
    dinv = 1.0 / diag
    x = np.zeros_like(b)
    r = b.copy()
    z = dinv * r
    p = z.copy()
    rho = r @ z
    for _ in range(m):
        q = np.zeros_like(b)
        np.add.at(q, rows, val * p[col])
        alpha = rho / (p @ q)
        x += alpha * p
        r -= alpha * q
        z = dinv * r
        rho_new = r @ z
        p = z + (rho_new / rho) * p
        rho = rho_new
    return x


@pytest.fixture(scope="module")
def system(ctx):
    from paper_1602_03207_b200 import workloads
    g = golden("small_6x6x12")
    mesh = ect.Mesh(ctx, g["xyz"], g["tets"], g["region"])
    p, _, _ = mesh.materials(workloads.Physics(sigma_defect=1e4, mu_r_defect=5.0))
    # node-block (NB-E) storage, the default path; Jacobi: the recurrence numpy restates
    a = ect.Matrix(ctx, mesh).assemble(p).set_preconditioner("jacobi")
    rp, ci, v = a.export()
    return a, rp, ci, v


@pytest.mark.parametrize("k", [1, 3, 8])
@pytest.mark.parametrize("m", [1, 6, 25])
def test_cocg_iterates_match_numpy(system, k, m):
    a, rp, ci, v = system
    rng = np.random.default_rng(100 * k + m)
    b = rng.uniform(-1, 1, (a.n, k)) + 1j * rng.uniform(-1, 1, (a.n, k))
    x, res = a.solve(b if k > 1 else b[:, 0], tol=1e-30, max_iter=m)
    x = x.reshape(a.n, k)
    for c in range(k):
        assert res[c]["iterations"] == m and not res[c]["converged"]
        xr = cocg_numpy(rp, ci, v, b[:, c], m)
        err = np.linalg.norm(x[:, c] - xr) / np.linalg.norm(xr)
        assert err <= 1e-9, (k, m, c, err)


def test_zero_column_is_inert(system):
    """A b = 0 column is converged at iteration 0 with x = 0 (iterative.cpp
    contract) and leaves the other columns' iterates unchanged."""
    a, rp, ci, v = system
    rng = np.random.default_rng(7)
    b = rng.uniform(-1, 1, (a.n, 2)) + 1j * rng.uniform(-1, 1, (a.n, 2))
    b[:, 1] = 0.0
    x, res = a.solve(b, tol=1e-30, max_iter=6)
    assert res[1]["converged"] and res[1]["iterations"] == 0 and np.all(x[:, 1] == 0)
    xr = cocg_numpy(rp, ci, v, b[:, 0], 6)
    assert np.linalg.norm(x[:, 0] - xr) / np.linalg.norm(xr) <= 1e-9


def test_profiled_launches_count_full_width_only(ctx, system):
    """ect_ctx_set_profiling: solver samples count toward spmv_ms_total only
    when every column of the batch is active (bench.py's roofline divides
    full-width algorithmic bytes by that mean)."""
    a, _, _, _ = system
    rng = np.random.default_rng(3)
    b = rng.uniform(-1, 1, (a.n, 2)) + 1j * rng.uniform(-1, 1, (a.n, 2))
    ctx.timings(reset=True)
    ctx.set_profiling(True)
    a.solve(b, tol=1e-30, max_iter=40)
    ctx.set_profiling(False)
    full = ctx.timings(reset=True)
    assert full["spmv_launches"] >= 40 // 8 and full["spmv_ms_total"] > 0
    b[:, 1] = 0.0  # one column never active: every sample is partial-width
    ctx.set_profiling(True)
    a.solve(b, tol=1e-30, max_iter=40)
    ctx.set_profiling(False)
    part = ctx.timings(reset=True)
    assert part["spmv_launches"] == 0 and part["spmv_partial_launches"] >= 40 // 8


def test_multigrid_iteration_graph_is_recaptured(ctx):
    """The multigrid COCG replays its iteration as a CUDA graph kept with the
    hierarchy (krylov.cu cocg_solve, IterGraph): kernel arguments bake in the
    batch width, the tolerance and max_iter. Alternating widths and stopping
    parameters on one matrix must re-capture, i.e. give bitwise the solutions
    of a fresh matrix solved once with the same parameters, and the plain
    launches (ECT_NO_GRAPH has the same arithmetic) agree through the residual."""
    from paper_1602_03207_b200 import workloads
    from tests.helpers import ref_matrix
    g = golden("small_6x6x12")
    mesh = ect.Mesh(ctx, g["xyz"], g["tets"], g["region"])
    p, _, _ = mesh.materials(workloads.Physics(sigma_defect=1e4, mu_r_defect=5.0))
    A = ref_matrix(g, "primary").tocsr()
    # consistent right-hand sides: the fixture's two coil vectors, scaled
    rhs = np.ascontiguousarray(g["rhs"].T)
    b8 = np.ascontiguousarray(np.stack([rhs[:, j & 1] * (1.0 + 0.25j * j) for j in range(8)],
                                       axis=1))
    b2 = np.ascontiguousarray(b8[:, :2])
    cases = [(b8, 1e-8, 500), (b2, 1e-10, 400), (b8, 1e-8, 500), (b8, 1e-6, 500), (b2, 1e-10, 400)]
    a = ect.Matrix(ctx, mesh).assemble(p)  # multigrid is the default preconditioner
    seq = [a.solve(b, tol=tol, max_iter=mi) for b, tol, mi in cases]
    for (b, tol, mi), (x, res) in zip(cases, seq):
        fresh = ect.Matrix(ctx, mesh).assemble(p)
        xf, rf = fresh.solve(b, tol=tol, max_iter=mi)
        assert [r["iterations"] for r in res] == [r["iterations"] for r in rf]
        assert x.tobytes() == xf.tobytes()
        assert all(r["converged"] for r in res)
        rr = np.linalg.norm(b - A @ x, axis=0) / np.linalg.norm(b, axis=0)
        assert np.all(rr <= tol * 1.01), rr
