"""Per-phase setup timing at growing mesh sizes (dev tool)."""
import sys
import time
sys.path.insert(0, ".")
from paper_1602_03207_b200 import ect, workloads, boxmesh  # noqa: E402

sizes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1:]] or [(64, 64, 256)]
ctx = ect.Context(0)
for (nx, ny, nz) in sizes:
    t = time.time()
    m = boxmesh.kuhn_box(nx, ny, nz, extent=(1.0, 1.0, nz / nx), seed=3)
    print(f"{nx}x{ny}x{nz}: gen {time.time() - t:.1f}s tets={m.n_tets}", flush=True)
    t = time.time(); mesh = ect.Mesh(ctx, m.xyz, m.tets, m.region); ctx.synchronize()
    print(f"  mesh {time.time() - t:.2f}s", flush=True)
    ph = workloads.Physics(sigma_defect=1e4, mu_r_defect=5.0)
    t = time.time(); p, r, two = mesh.materials(ph); print(f"  materials {time.time() - t:.2f}s", flush=True)
    t = time.time(); a = ect.Matrix(ctx, mesh); ctx.synchronize(); print(f"  pattern {time.time() - t:.2f}s nnz={a.nnz}", flush=True)
    t = time.time(); a.assemble(p); ctx.synchronize(); print(f"  assemble {time.time() - t:.2f}s fmt={a.format}", flush=True)
    del a, mesh
