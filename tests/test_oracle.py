"""CPU tests: pin the oracle before trusting it (no GPU needed).

1. The reference build (oracle/_ref: the unmodified ectsim core + our Eigen
   shim) reproduces the reference's own known-answer tests
   (test_elements.cpp:21-124) and the SURVEY's configs[0] counts.
2. The committed golden fixtures are exactly what the reference build produces.
3. The numpy restatement (oracle/port.py) matches the golden fixtures: pattern,
   pins and conductor map exactly, values bit for bit, rhs, impedance.
"""
import numpy as np
import pytest

from oracle import port
from paper_1602_03207_b200 import boxmesh, workloads
from tests.helpers import GOLDEN, SMALL, conductor_components, golden, ref_csr_values, solution_errors

KP = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)


# ---- 1. reference build vs the reference's own KATs --------------------------------
def test_reference_tet_frame_kat(ref_lib):
    g, vol = ref_lib.tet_frame(KP.ravel())
    assert vol == pytest.approx(1 / 6, rel=1e-15)                    # test_elements.cpp:21-28
    assert np.allclose(g, [[-1, -1, -1], [1, 0, 0], [0, 1, 0], [0, 0, 1]], atol=1e-14)


def test_reference_element_kats(ref_lib):
    l11, l12, l21, l22 = ref_lib.element_blocks(KP.ravel(), 1.0, 1.0, 0.0, 1.0, 0.0)
    assert l11[0, 0] == pytest.approx(0.5, rel=1e-14)                 # test_elements.cpp:34-38
    l11, l12, l21, l22 = ref_lib.element_blocks(KP.ravel(), 1.0, 1.0, 1.0, 1.0, 0.0)
    assert l12[0, 0].real == pytest.approx(1 / 24, rel=1e-14)         # :66-69
    assert l21[0, 0].real == pytest.approx(1 / 24, rel=1e-14)         # :92-95
    assert l22[0, 0] == pytest.approx(0.5j, rel=1e-14)                # :97-101
    assert np.array_equal(l21, l12.T)                                  # L21 = L12^T exactly
    # gauge mass delta*mu*sigma*|K|(1+d_ab)/20 (test_elements.cpp:112-124)
    _, _, _, g1 = ref_lib.element_blocks(KP.ravel(), 2.0, 1.0, 3.0, 1.0, 1e-6)
    _, _, _, g0 = ref_lib.element_blocks(KP.ravel(), 2.0, 1.0, 3.0, 1.0, 0.0)
    vol = 1 / 6
    expect = 1e-6 * 2.0 * 3.0 * vol * (np.ones((4, 4)) + np.eye(4)) / 20
    assert np.allclose((g1 - g0).real, expect, rtol=1e-12, atol=0)


def test_port_element_frames_bitwise_vs_reference(ref_lib):
    rng = np.random.default_rng(5)
    p = (KP[None] + rng.uniform(-0.1, 0.1, (200, 4, 3))) * 0.01
    xyz = p.reshape(-1, 3)
    tets = np.arange(800, dtype=np.int32).reshape(200, 4)
    g, vol = port.tet_frames(xyz, tets)
    for t in range(200):
        gr, vr = ref_lib.tet_frame(p[t].ravel())
        assert gr.tobytes() == g[t].tobytes() and vr == vol[t]


def test_reference_counts_configs0(ref_lib):
    """SURVEY §6 [probe] counts for configs[0]."""
    w = workloads.config0()
    m = w.mesh()
    rm = ref_lib.RefMesh(m.xyz, m.tets, m.region)
    assert (rm.n_nodes, rm.n_tets, rm.n_cond) == (18081, 96000, 4305)
    assert int((m.region == boxmesh.TUBE).sum()) == 19200
    assert np.array_equal(rm.export()["tets"], m.tets)  # generator output is canonical


# ---- 2. golden fixtures are the reference's output ----------------------------------
@pytest.mark.parametrize("name", ["small_4x4x8", "small_5x5x10_nodefect"])
def test_golden_fixture_regenerates(ref_lib, name):
    from oracle import make_golden
    kw = make_golden.SMALL_CASES[name]
    out = make_golden.reference_case(workloads.small(**kw), direct=True)
    g = golden(name)
    for key in ("cond_forward", "pins", "primary_col_ptr", "primary_row_idx", "primary_values",
                "rhs", "mats_primary"):
        # (older fixtures predate the trailing z_surface entries of mats_*)
        assert out[key][:len(g[key])].tobytes() == g[key].tobytes(), key
    assert np.allclose(out["primary_x"], g["primary_x"], rtol=0, atol=1e-12 * np.abs(g["primary_x"]).max())


# ---- 3. numpy port vs golden ----------------------------------------------------------
@pytest.mark.parametrize("name", SMALL)
def test_port_matches_golden(name):
    g = golden(name)
    xyz, tets, region = g["xyz"], g["tets"], g["region"]
    fwd = port.conductor_map(len(xyz), tets, region)
    assert np.array_equal(fwd, g["cond_forward"])
    pins = port.pinned_dofs(xyz, tets)
    assert np.array_equal(pins, g["pins"])
    keys = ["primary"] + (["reference"] if bool(g["two_configs"]) else [])
    for key in keys:
        mats = port.mats_dict(g[f"mats_{key}"])
        rp, ci, v = port.assemble(xyz, tets, region, mats, fwd, pins)
        assert np.array_equal(rp, g[f"{key}_col_ptr"]) and np.array_equal(ci, g[f"{key}_row_idx"])
        assert v.tobytes() == ref_csr_values(g, key).tobytes(), f"{key} values not bit-exact"
    z = float(g["z"])
    n = len(g["primary_col_ptr"]) - 1
    for c in (1, 2):
        sup = port.coil_support(xyz, tets, tuple(g["coil"]), z, c)
        b = port.assemble_rhs(xyz, tets, region, sup, float(g["amplitude"]), n, pins)
        assert b.tobytes() == g["rhs"][c - 1].tobytes()
    if bool(g["two_configs"]):
        pm, rm = port.mats_dict(g["mats_primary"]), port.mats_dict(g["mats_reference"])
        dz = [port.delta_impedance(xyz, tets, region, fwd, pm, rm, g["primary_x"][k],
                                   g["reference_x"][l]) for k in range(2) for l in range(2)]
        assert np.max(np.abs(np.array(dz) - g["dz"])) <= 1e-12 * np.max(np.abs(g["dz"]))


def test_port_direct_solution_matches_reference_lu():
    g = golden("small_4x4x8")
    rp, ci, v = port.assemble(g["xyz"], g["tets"], g["region"], port.mats_dict(g["mats_primary"]))
    comp = conductor_components(g["tets"], g["region"], g["cond_forward"])
    for c in range(2):
        x = port.solve_direct(rp, ci, v, g["rhs"][c])
        ea, ev = solution_errors(x, g["primary_x"][c], len(g["xyz"]), comp)
        assert ea <= 1e-8 and ev <= 1e-8, (ea, ev)


def test_port_configs0_pattern_hash():
    """configs[0] at full size: port pattern/values hash == reference build's."""
    import hashlib
    g = np.load(GOLDEN / "cfg0.npz")
    w = workloads.config0()
    m = w.mesh()
    mats = port.mats_dict(g["mats_primary"])
    rp, ci, v = port.assemble(m.xyz, m.tets, m.region, mats)
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    assert sha(rp) == str(g["sha_col_ptr"]) and sha(ci) == str(g["sha_row_idx"])
    import scipy.sparse as sp
    n = len(rp) - 1
    csc = sp.csr_matrix((v, ci, rp), shape=(n, n)).tocsc()
    csc.sort_indices()
    assert sha(csc.data) == str(g["sha_values"])


def test_box_generator_conventions():
    m = boxmesh.kuhn_box(2, 3, 4, seed=None)
    assert m.n_nodes == 3 * 4 * 5 and m.n_tets == 6 * 2 * 3 * 4
    assert np.all(boxmesh.signed_volumes(m.xyz, m.tets) > 0)
    # node id (i*(ny+1)+j)*(nz+1)+k  (test_meshes.hpp:18)
    i, j, k = 1, 2, 3
    nid = (i * 4 + j) * 5 + k
    assert np.allclose(m.xyz[nid], [(i / 2 - 0.2) * 0.01, (j / 3 - 0.5) * 0.01, (2 * k / 4) * 0.01])
    # jitter: deterministic, interior only, |d| <= 0.1 h
    a = boxmesh.kuhn_box(4, 4, 8, seed=3)
    b = boxmesh.kuhn_box(4, 4, 8, seed=3)
    c = boxmesh.kuhn_box(4, 4, 8, seed=None)
    assert np.array_equal(a.xyz, b.xyz)
    d = (a.xyz - c.xyz) / 0.01
    assert np.all(np.abs(d[:, 0]) <= 0.1 * 0.25 + 1e-15) and np.any(d != 0)
