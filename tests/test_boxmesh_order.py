"""configs[4]'s z-slowest node numbering (boxmesh.kuhn_box node_order="kij").

The row partition cuts contiguous node ranges; numbering the box z-slowest
makes those ranges the z-slabs BASELINE asks for. The relabelling must not
change the discrete problem: same geometry, tets and regions, and -- through
the numpy restatement of the reference assembly (oracle/port.py, bit-exact vs
the reference) -- a matrix that is exactly P A P^T of the reference-numbered
one (A-DOF 3 node + c, V-DOF by ascending conductor node id).
"""
import numpy as np
import pytest

from oracle import port
from paper_1602_03207_b200 import workloads
from paper_1602_03207_b200.boxmesh import kuhn_box
from tests.helpers import golden


def _dof_perm(n_nodes, fwd_a, fwd_b, new_id):
    """dof index in numbering A -> dof index in numbering B."""
    na = 3 * n_nodes
    nc = int(fwd_a.max()) + 1
    perm = np.empty(na + nc, np.int64)
    nodes = np.arange(n_nodes)
    for c in range(3):
        perm[3 * nodes + c] = 3 * new_id + c
    cond = np.flatnonzero(fwd_a >= 0)
    perm[na + fwd_a[cond]] = na + fwd_b[new_id[cond]]
    return perm


def test_kij_is_a_relabelling_with_z_slab_ranges():
    a = kuhn_box(5, 4, 7, seed=2)
    b = kuhn_box(5, 4, 7, seed=2, node_order="kij")
    assert np.array_equal(a.xyz[a.tets], b.xyz[b.tets])  # same tets, same vertex order
    assert np.array_equal(a.region, b.region)
    per = 6 * 5  # (nx + 1)(ny + 1) nodes per z-plane
    k_of = np.empty(len(b.xyz), np.int64)
    ii, jj, kk = np.meshgrid(np.arange(6), np.arange(5), np.arange(8), indexing="ij")
    k_of[((kk * 6 + ii) * 5 + jj).ravel()] = kk.ravel()
    assert np.array_equal(k_of, np.repeat(np.arange(8), per))  # range r*per.. = plane k = r
    with pytest.raises(ValueError):
        kuhn_box(2, 2, 2, node_order="zyx")


def test_kij_matrix_is_symmetric_permutation_of_reference_numbering():
    w = workloads.small(n=(4, 4, 8), seed=7, deposit=True)
    a = w.mesh()
    w.extra = dict(w.extra, node_order="kij")
    b = w.mesh()
    ii, jj, kk = np.meshgrid(np.arange(5), np.arange(5), np.arange(9), indexing="ij")
    new_id = ((kk * 5 + ii) * 5 + jj).ravel()
    assert np.array_equal(new_id[a.tets], b.tets)
    g = golden("small_4x4x8")
    mats = port.mats_dict(g["mats_primary"])
    fa = port.conductor_map(len(a.xyz), a.tets, a.region)
    fb = port.conductor_map(len(b.xyz), b.tets, b.region)
    rpa, ca, va = port.assemble(a.xyz, a.tets, a.region, mats, fa)
    rpb, cb, vb = port.assemble(b.xyz, b.tets, b.region, mats, fb)
    perm = _dof_perm(len(a.xyz), fa, fb, new_id)
    n = len(rpa) - 1
    ra = np.repeat(np.arange(n), np.diff(rpa))
    rb = np.repeat(np.arange(n), np.diff(rpb))
    # entries of A moved to (perm r, perm c), sorted like B's CSR
    key_a = perm[ra] * n + perm[ca]
    order = np.argsort(key_a, kind="stable")
    assert np.array_equal(key_a[order], rb.astype(np.int64) * n + cb)
    assert va[order].tobytes() == vb.tobytes(), "relabelled matrix is not exactly P A P^T"
