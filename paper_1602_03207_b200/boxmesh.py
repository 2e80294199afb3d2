"""Synthetic box meshes for the BASELINE configs (host-side input generator).

BASELINE.json's configs use a jittered Kuhn-split box, which the reference
does not ship: its only structured generator is the unit-cube test fixture
``test::unit_cube_mesh`` (/root/reference/proj/tests/support/test_meshes.hpp:15-54).
This module is that fixture generalised, keeping its

* node id ``(i*(ny+1)+j)*(nz+1)+k`` (test_meshes.hpp:18),
* cell-major / permutation-minor tet order with the kPerm path table
  (test_meshes.hpp:28-44),
* orientation fix "swap nodes 2,3 when the signed volume is negative"
  (Mesh::canonicalize_orientation, mesh.cpp:50-61, signed volume mesh.cpp:36-38),
* region-by-centroid tagging (test_meshes.hpp:46-49).

Additions fixed here (documented in DESIGN.md):

* box [0,Lx]x[0,Ly]x[0,Lz] with nx x ny x nz cells;
* interior nodes jittered by U(-0.1 h, 0.1 h) per axis, drawn with
  ``numpy.random.default_rng(seed).uniform(-0.1, 0.1, (n_nodes, 3))`` for ALL
  nodes and applied to interior ones only (reproducible on any host);
* coordinates translated so the coil axis sits at x = y = 0 (the reference's
  coil current is hard-wired azimuthal about the global z axis,
  assembly.cpp:351-358) and scaled by ``scale`` (0.01: metres);
* regions: slab x in [0.4, 0.6] -> TUBE, deposit boxes inside it -> DEFECT,
  everything else VACUUM (RegionTag values, types.hpp:22-29).

The oracle and the GPU path consume the SAME arrays produced here.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# RegionTag (types.hpp:22-29)
TUBE, TSP, DEFECT, COIL1, COIL2, VACUUM = 0, 1, 2, 3, 4, 5

# Kuhn path permutations (test_meshes.hpp:28)
KPERM = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))


@dataclass
class BoxMesh:
    xyz: np.ndarray          # float64 [n_nodes, 3], metres
    tets: np.ndarray         # int32 [n_tets, 4], positively oriented
    region: np.ndarray       # uint8 [n_tets]
    dims: tuple              # (nx, ny, nz)
    extent: tuple            # (Lx, Ly, Lz) in box units before scaling
    origin: tuple            # box-unit coordinate mapped to x = y = 0
    scale: float
    meta: dict = field(default_factory=dict)

    @property
    def n_nodes(self) -> int:
        return int(self.xyz.shape[0])

    @property
    def n_tets(self) -> int:
        return int(self.tets.shape[0])

    def to_metres(self, z_box: float) -> float:
        return z_box * self.scale


def signed_volumes(xyz: np.ndarray, tets: np.ndarray) -> np.ndarray:
    """(b-a) x (c-a) . (d-a) / 6 per tet (mesh.cpp:36-38)."""
    a, b, c, d = (xyz[tets[:, i]] for i in range(4))
    u, v, w = b - a, c - a, d - a
    cx = u[:, 1] * v[:, 2] - u[:, 2] * v[:, 1]
    cy = u[:, 2] * v[:, 0] - u[:, 0] * v[:, 2]
    cz = u[:, 0] * v[:, 1] - u[:, 1] * v[:, 0]
    return ((cx * w[:, 0] + cy * w[:, 1]) + cz * w[:, 2]) / 6.0


def centroids(xyz: np.ndarray, tets: np.ndarray) -> np.ndarray:
    """0.25 * (p0 + p1 + p2 + p3) (mesh.cpp:41-44)."""
    return 0.25 * (((xyz[tets[:, 0]] + xyz[tets[:, 1]]) + xyz[tets[:, 2]]) + xyz[tets[:, 3]])


def kuhn_box(nx: int, ny: int, nz: int, *, extent=(1.0, 1.0, 2.0), seed: int | None = 0,
             jitter: float = 0.1, origin=(0.2, 0.5), scale: float = 0.01,
             slab=(0.4, 0.6), deposits=((0.9, 1.1),), tsp_deposits=(),
             node_order: str = "ijk") -> BoxMesh:
    """Jittered Kuhn box; see module docstring for the conventions.

    node_order "ijk" (default) numbers nodes (i*(ny+1)+j)*(nz+1)+k as the
    reference's unit_cube_mesh does; "kij" renumbers the SAME geometry and tets
    as (k*(nx+1)+i)*(ny+1)+j, so that contiguous node ranges are z-slabs (the
    row partition of configs[4]). Geometry, tet order and orientation are
    identical; only the labels change (the reference numbers DOFs by node id,
    so its matrix for the relabelled mesh is P A P^T)."""
    if node_order not in ("ijk", "kij"):
        raise ValueError(f"node_order must be 'ijk' or 'kij', got {node_order!r}")
    lx, ly, lz = extent
    hx, hy, hz = lx / nx, ly / ny, lz / nz
    i = np.arange(nx + 1, dtype=np.int64)
    j = np.arange(ny + 1, dtype=np.int64)
    k = np.arange(nz + 1, dtype=np.int64)
    ii, jj, kk = np.meshgrid(i, j, k, indexing="ij")
    # node id (i*(ny+1)+j)*(nz+1)+k  -> C-order flattening of (i, j, k)
    x = (ii.astype(np.float64) / nx) * lx
    y = (jj.astype(np.float64) / ny) * ly
    z = (kk.astype(np.float64) / nz) * lz
    xyz = np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1)
    if seed is not None and jitter > 0.0:
        rng = np.random.default_rng(seed)
        u = rng.uniform(-jitter, jitter, size=xyz.shape)
        interior = ((ii > 0) & (ii < nx) & (jj > 0) & (jj < ny) & (kk > 0) & (kk < nz)).ravel()
        xyz[interior] += u[interior] * np.array([hx, hy, hz])

    def node(a, b, c):
        return (a * (ny + 1) + b) * (nz + 1) + c

    ci, cj, ck = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ci, cj, ck = ci.ravel(), cj.ravel(), ck.ravel()
    n_cells = ci.size
    tets = np.empty((n_cells, 6, 4), dtype=np.int64)
    for p, perm in enumerate(KPERM):
        corner = [ci.copy(), cj.copy(), ck.copy()]
        tets[:, p, 0] = node(*corner)
        for step in range(3):
            corner[perm[step]] = corner[perm[step]] + 1
            tets[:, p, step + 1] = node(*corner)
    tets = tets.reshape(-1, 4)
    # canonicalize_orientation (mesh.cpp:50-61) on the jittered coordinates
    vol = signed_volumes(xyz, tets)
    neg = vol < 0.0
    tets[neg, 2], tets[neg, 3] = tets[neg, 3].copy(), tets[neg, 2].copy()
    if np.any(vol == 0.0):
        raise ValueError("degenerate tet in box mesh")

    # regions from the centroid in box units (before translation/scaling)
    c = centroids(xyz, tets)
    region = np.full(tets.shape[0], VACUUM, dtype=np.uint8)
    in_slab = (c[:, 0] >= slab[0]) & (c[:, 0] <= slab[1])
    region[in_slab] = TUBE
    for z0, z1 in deposits:
        region[in_slab & (c[:, 2] >= z0) & (c[:, 2] <= z1)] = DEFECT
    # further deposits with their own (sigma, mu): the reference's MaterialTable
    # holds one pair per RegionTag, so they take the TSP tag (a conductor region,
    # types.hpp:46-48, excluded from dZ which integrates DEFECT only)
    for z0, z1 in tsp_deposits:
        region[in_slab & (c[:, 2] >= z0) & (c[:, 2] <= z1)] = TSP

    if node_order == "kij":
        new_id = ((kk * (nx + 1) + ii) * (ny + 1) + jj).ravel()  # indexed by the ijk id
        xyz_k = np.empty_like(xyz)
        xyz_k[new_id] = xyz
        xyz, tets = xyz_k, new_id[tets]

    xyz_m = np.empty_like(xyz)
    xyz_m[:, 0] = (xyz[:, 0] - origin[0]) * scale
    xyz_m[:, 1] = (xyz[:, 1] - origin[1]) * scale
    xyz_m[:, 2] = xyz[:, 2] * scale
    return BoxMesh(xyz=np.ascontiguousarray(xyz_m), tets=np.ascontiguousarray(tets.astype(np.int32)),
                   region=region, dims=(nx, ny, nz), extent=tuple(extent),
                   origin=tuple(origin), scale=scale,
                   meta={"seed": seed, "jitter": jitter, "slab": slab, "deposits": deposits,
                         "h": (hx, hy, hz), "node_order": node_order})
