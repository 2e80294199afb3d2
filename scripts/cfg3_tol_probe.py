"""Dev probe: ScanSession at the configs[3] golden position on the configs[1] mesh
for several tolerances -- iterations, failure flag and how much dZ moves with
the tolerance (what tolerance a 1e-6 impedance comparison needs)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_1602_03207_b200 import ect, workloads  # noqa: E402

w = workloads.config3()
z = w.positions[31]
m = w.mesh()
ctx = ect.Context(0)
mesh = ect.Mesh(ctx, m.xyz, m.tets, m.region)
ref = None
for tol in (1e-12, 1e-11, 1e-10, 1e-9, 1e-8):
    s = ect.Session(ctx, mesh, w.physics, w.coil, w.amplitude, tol=tol, max_iter=200000)
    pt = s.solve_positions([z])[0]
    if ref is None:
        ref = pt["dz"]
    dev = np.max(np.abs(pt["dz"] - ref)) / np.max(np.abs(ref))
    print(f"tol {tol:.0e}: failed={pt['failed']} iterations={pt['iterations']} "
          f"dz={np.round(pt['dz'], 12)} max dev vs tol 1e-12: {dev:.2e}", flush=True)
    del s
