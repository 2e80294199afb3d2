"""The drop-in boundary against the reference interface:

* ect_matrix_from_csc takes the reference's CscMatrix arrays as they are
  (sparse.hpp:56-66) and probes value symmetry, so a non-symmetric matrix
  (impedance surface terms) goes to BiCGStab, never to COCG;
* ect_physics_init mirrors RunConfig's defaults (config.hpp:25-39) and the
  parser's validation (config.cpp:218-236);
* the assemble_rhs overloads (support tets / coil region tag,
  assembly.hpp:84-87) and apply_pins_to_rhs (assembly.hpp:79);
* the multigrid preconditioner: same solution as Jacobi, bitwise repeatable.
"""
import math

import numpy as np
import pytest

from oracle import port
from paper_1602_03207_b200 import ect, workloads
from tests.helpers import IBC, conductor_components, golden, ref_matrix, solution_errors

pytestmark = pytest.mark.gpu


def _csc(g, key="primary"):
    return g[f"{key}_col_ptr"], g[f"{key}_row_idx"], g[f"{key}_values"]


def test_from_csc_matches_reference_matrix(ctx):
    g = golden("small_6x6x12")
    A = ref_matrix(g)
    a = ect.Matrix(ctx, csc=_csc(g))
    assert a.symmetric and a.n == A.shape[0] and a.nnz == A.nnz
    rng = np.random.default_rng(5)
    x = rng.standard_normal((a.n, 4)) + 1j * rng.standard_normal((a.n, 4))
    y = a.multiply(x)
    absA = abs(A)
    assert np.max(np.abs(y - A @ x) / (absA @ np.abs(x))) <= 1e-14
    comp = conductor_components(g["tets"], g["region"], g["cond_forward"])
    b = np.ascontiguousarray(g["rhs"].T)
    xs, res = a.solve(b, tol=1e-10, max_iter=20000)
    for c in range(2):
        assert res[c]["converged"]
        ea, ev = solution_errors(xs[:, c], g["primary_x"][c], len(g["xyz"]), comp)
        assert ea <= 1e-6 and ev <= 1e-6, (ea, ev)


@pytest.mark.parametrize("name", IBC)
def test_from_csc_nonsymmetric_goes_to_bicgstab(ctx, name):
    """Impedance surface terms make A != A^T (va = i omega av^T): the CSC
    entry point must detect it (COCG would silently solve the wrong system),
    and passing the CSC arrays as CSR (= A^T) must not be mistaken for A."""
    g = golden(name)
    A = ref_matrix(g)
    a = ect.Matrix(ctx, csc=_csc(g))
    assert not a.symmetric
    at = ect.Matrix(ctx, csr=_csc(g))  # A^T, still non-symmetric
    assert not at.symmetric
    b = np.ascontiguousarray(g["rhs"][0])
    x, res = a.solve(b, tol=1e-13, max_iter=40000)
    assert res[0]["converged"]
    rr = np.linalg.norm(b - A @ x) / np.linalg.norm(b)
    assert rr <= 2e-13, rr


def test_physics_init_and_validation(ctx):
    ph = ect.Physics.defaults()
    assert (ph.frequency, ph.sigma_tube, ph.mu_r_tube) == (100e3, 1e6, 1.0)
    assert math.isnan(ph.sigma_defect) and math.isnan(ph.mu_r_defect)  # std::optional unset
    assert (ph.sigma_eps_ratio, ph.delta_gauge, ph.bc_penalty) == (1e-6, 1e-6, 1e13)
    assert ph.mu_tilde_harmonic == 1 and ph.mu_tilde_fixed == 1.25663706212e-6
    assert (ph.sigma_tsp, ph.mu_r_tsp, ph.ibc_tsp, ph.l22_sigma_eps) == (5e6, 50.0, 0, 0)
    g = golden("small_4x4x8")
    m = ect.Mesh(ctx, g["xyz"], g["tets"], g["region"])
    # defaults == the workloads' physics with the deposit keys set
    ph.sigma_defect, ph.mu_r_defect = 1e4, 5.0
    p1, r1, two1 = m.materials(ph)
    p2, r2, two2 = m.materials(workloads.Physics(sigma_defect=1e4, mu_r_defect=5.0))
    assert bytes(p1) == bytes(p2) and bytes(r1) == bytes(r2) and two1 == two2
    # a zero-initialised struct is rejected instead of giving mu = 0
    with pytest.raises(ect.ConfigError):
        m.materials(ect.Physics())
    bad = ect.Physics.defaults()
    bad.mu_r_tsp = 0.0
    with pytest.raises(ect.ConfigError):
        m.materials(bad)
    bad = ect.Physics.defaults()
    bad.delta_gauge = 1.5
    with pytest.raises(ect.ConfigError):
        m.materials(bad)
    # l22_sigma_eps reaches the material table (config.cpp:331)
    ph = ect.Physics.defaults()
    ph.l22_sigma_eps = 1
    p3, _, _ = m.materials(ph)
    assert p3.l22_use_sigma_eps == 1


def test_rhs_overloads_and_pins(ctx):
    g = golden("small_6x6x12")
    m = ect.Mesh(ctx, g["xyz"], g["tets"], g["region"])
    z, coil = float(g["z"]), tuple(g["coil"])
    pins = m.export()["pinned_dofs"]
    for which in (1, 2):
        sup = port.coil_support(g["xyz"], g["tets"], coil, z, which)
        raw = m.rhs_support(sup, float(g["amplitude"]))  # assemble_rhs: not pinned
        ref = port.assemble_rhs(g["xyz"], g["tets"], g["region"], sup, float(g["amplitude"]),
                                m.n_dofs, np.zeros(0, np.int64))
        assert np.max(np.abs(raw - ref)) <= 1e-14 * np.max(np.abs(ref))
        pinned = m.apply_pins_to_rhs(raw.copy())
        assert np.all(pinned[pins] == 0)
        coil_rhs = m.rhs(coil, [z], [which], float(g["amplitude"]))[:, 0]
        assert np.array_equal(pinned, coil_rhs)  # = position_rhs (scan.cpp:87-93)
        # duplicates / any order in the support list do not change the result
        sup2 = np.concatenate([sup[::-1], sup[:3]])
        assert np.array_equal(m.rhs_support(sup2, float(g["amplitude"])), raw)
        # the region-tag overload: tag the support tets COIL1 / COIL2
        region = g["region"].copy()
        region[sup] = 2 + which
        mt = ect.Mesh(ctx, g["xyz"], g["tets"], region)
        assert np.array_equal(mt.rhs_region(2 + which, float(g["amplitude"])), raw)
    with pytest.raises(ect.MeshError):  # empty support
        m.rhs_support(np.zeros(0, np.int32), 1.0)
    cond = np.flatnonzero(g["region"] == 0)[:2]
    with pytest.raises(ect.MeshError):  # support in a conductor
        m.rhs_support(cond, 1.0)
    with pytest.raises(ect.MeshError):  # no tet carries the tag
        m.rhs_region(3, 1.0)
    with pytest.raises(ect.ConfigError):  # which / z length mismatch
        m.rhs(coil, [z, z], [1], 1.0)


def test_multigrid_matches_jacobi_and_repeats(ctx):
    g = golden("small_6x6x12")
    m = ect.Mesh(ctx, g["xyz"], g["tets"], g["region"])
    p, _, _ = m.materials(workloads.Physics(sigma_defect=1e4, mu_r_defect=5.0))
    aj = ect.Matrix(ctx, m).assemble(p).set_preconditioner("jacobi")
    am = ect.Matrix(ctx, m).assemble(p).set_preconditioner("amg")
    info = am.precond_info()
    assert info["levels"] >= 2 and 1.0 < info["op_complexity"] < 1.5
    b = np.ascontiguousarray(g["rhs"].T)
    xj, rj = aj.solve(b, tol=1e-11, max_iter=20000)
    xm, rm = am.solve(b, tol=1e-11, max_iter=20000)
    xm2, _ = am.solve(b, tol=1e-11, max_iter=20000)
    assert xm.tobytes() == xm2.tobytes()
    comp = conductor_components(g["tets"], g["region"], g["cond_forward"])
    for c in range(2):
        assert rm[c]["converged"] and rm[c]["iterations"] < rj[c]["iterations"]
        ea, ev = solution_errors(xm[:, c], xj[:, c], m.n_nodes, comp)
        assert ea <= 1e-8 and ev <= 1e-8, (ea, ev)
        ea, ev = solution_errors(xm[:, c], g["primary_x"][c], m.n_nodes, comp)
        assert ea <= 1e-6 and ev <= 1e-6, (ea, ev)
