"""BASELINE.json configs as concrete synthetic workloads.

Physics keys follow RunConfig's [materials] section (config.hpp:25-39); the
coil is a reference CoilPair (tube_mesh.hpp:13-21) whose support is selected
by coil_support's centroid rule (tube_mesh.cpp:272-288).

Fixed choices where BASELINE.json is silent or disagrees with the reference
(SURVEY.md D1-D12), all recorded in DESIGN.md:
* coil axis at box (x, y) = (0.2, 0.5), i.e. in the air left of the slab;
  ring r in [0.08, 0.13] box units, height = one z-cell, gap = 0, so coil 1 is
  the cell layer just below the probe plane and coil 2 the one just above;
* amplitude 1e6 A/m^2; f = 100 kHz; sigma_tube = 1e6; sigma_eps ratio 1e-6;
  delta_gauge = 1e-6; bc_penalty = 1e13; mu_tilde harmonic (config.hpp defaults);
* deposit: the full slab cross-section for z in [0.9, 1.1] box units,
  sigma = 1e4 S/m, mu_r = 5 (RegionTag::kDefect).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .boxmesh import BoxMesh, kuhn_box

SCALE = 0.01  # box units -> metres
COIL_AXIS = (0.2, 0.5)
COIL_R = (0.08, 0.13)


@dataclass
class Physics:
    """RunConfig [materials] subset (config.hpp:25-39)."""
    frequency: float = 100e3
    sigma_tube: float = 1e6
    mu_r_tube: float = 1.0
    sigma_defect: float = -1.0   # <0: unset -> tube value (config.cpp:333-334)
    mu_r_defect: float = -1.0
    sigma_eps_ratio: float = 1e-6
    delta_gauge: float = 1e-6
    bc_penalty: float = 1e13
    mu_tilde_harmonic: bool = True
    mu_tilde_fixed: float = 1.25663706212e-6
    sigma_tsp: float = -1.0      # <0: default (config.hpp:29)
    mu_r_tsp: float = -1.0
    ibc_tsp: bool = False        # plate as a surface impedance (config.hpp:38)


@dataclass
class Workload:
    name: str
    dims: tuple
    seed: int
    deposits: tuple
    physics: Physics
    coil: tuple              # CoilPair (r_inner, r_outer, height, gap) in metres
    amplitude: float
    positions: tuple         # probe z in metres
    tol: float = 1e-8
    extent: tuple = (1.0, 1.0, 2.0)
    notes: str = ""
    extra: dict = field(default_factory=dict)

    def mesh(self) -> BoxMesh:
        return kuhn_box(*self.dims, extent=self.extent, seed=self.seed, origin=COIL_AXIS,
                        scale=SCALE, deposits=self.deposits,
                        tsp_deposits=self.extra.get("tsp_deposits", ()),
                        node_order=self.extra.get("node_order", "ijk"))


def _coil(nz: int, lz: float = 2.0) -> tuple:
    hz = lz / nz
    return (COIL_R[0] * SCALE, COIL_R[1] * SCALE, hz * SCALE, 0.0)


def positions(z_start: float, z_end: float, count: int) -> tuple:
    """RunConfig::positions (config.cpp:316-323)."""
    return tuple(z_start if count == 1 else z_start + (z_end - z_start) * i / (count - 1)
                 for i in range(count))


def config0() -> Workload:
    return Workload("configs[0]", (20, 20, 40), 0, (), Physics(), _coil(40), 1e6,
                    (1.0 * SCALE,), notes="small A-V solve, no deposit (DeltaZ == 0)")


def config1() -> Workload:
    return Workload("configs[1]", (64, 64, 128), 1, ((0.9, 1.1),),
                    Physics(sigma_defect=1e4, mu_r_defect=5.0), _coil(128), 1e6,
                    (1.0 * SCALE,), notes="single-position medium mesh, deposit at z in [0.9,1.1]")


def config3() -> Workload:
    w = config1()
    w.name = "configs[3]"
    w.positions = positions(0.3 * SCALE, 1.7 * SCALE, 64)
    w.notes = "probe sweep, 64 positions over z in [0.3,1.7]"
    return w


def config4() -> Workload:
    """configs[4]: 128x128x512 cells (50.3M tets) on a [0,1]x[0,1]x[0,4] box so
    that h_z = h_x and the second deposit z in [2.5, 2.7] lies inside (SURVEY
    §8(d)); second deposit sigma = 5e3, mu_r = 2 via the TSP tag. Nodes are
    numbered z-slowest (node_order "kij") so that the contiguous node ranges of
    the row partition are the z-slabs BASELINE asks for."""
    return Workload("configs[4]", (128, 128, 512), 3, ((0.9, 1.1),),
                    Physics(sigma_defect=1e4, mu_r_defect=5.0, sigma_tsp=5e3, mu_r_tsp=2.0),
                    _coil(512, 4.0), 1e6, (1.0 * SCALE,), extent=(1.0, 1.0, 4.0),
                    notes="large mesh, z-slab row partition",
                    extra={"tsp_deposits": ((2.5, 2.7),), "node_order": "kij"})


def small(n=(4, 4, 8), seed=7, deposit=True) -> Workload:
    """Small configs[1]-like case for golden fixtures and fast tests."""
    nx, ny, nz = n
    deps = ((0.9, 1.1),) if deposit else ()
    phys = Physics(sigma_defect=1e4, mu_r_defect=5.0) if deposit else Physics()
    return Workload(f"small{nx}x{ny}x{nz}", n, seed, deps, phys, _coil(nz), 1e6,
                    (1.0 * SCALE,))


BY_NAME = {"configs[0]": config0, "configs[1]": config1, "configs[3]": config3,
           "configs[4]": config4}
