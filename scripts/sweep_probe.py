"""Dev: per-position iterations / time over the configs[3] sweep (ppb batches)."""
import os
import sys
import time
sys.path.insert(0, ".")
from paper_1602_03207_b200 import ect, workloads  # noqa: E402

ppb = int(sys.argv[1]) if len(sys.argv) > 1 else 4
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-8
w = workloads.config3()
m = w.mesh()
ctx = ect.Context(0)
if os.environ.get("PRECOND"):
    ctx.set_preconditioner(os.environ["PRECOND"])
mesh = ect.Mesh(ctx, m.xyz, m.tets, m.region)
s = ect.Session(ctx, mesh, w.physics, w.coil, w.amplitude, tol=tol, max_iter=20000)
print(s.matrix().precond_info(), flush=True)
pos = list(w.positions)
sel = [int(v) for v in os.environ.get("IDX", "").split(",") if v] or list(range(len(pos)))
for i0 in range(0, len(sel), ppb):
    zs = [pos[i] for i in sel[i0:i0 + ppb]]
    ctx.synchronize()
    t = time.perf_counter()
    pts = s.solve_positions(zs, positions_per_batch=ppb)
    dt = time.perf_counter() - t
    print(f"positions {sel[i0:i0 + ppb]}: {dt * 1e3 / len(zs):.0f} ms/pos its="
          f"{[p['iterations'] for p in pts]} failed={[p['failed'] for p in pts]}", flush=True)
