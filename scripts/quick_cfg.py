"""Quick timing probe of one probe position on a BASELINE config (dev tool)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1602_03207_b200 import ect, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "configs[1]"
w = workloads.BY_NAME[name]()
t0 = time.time()
m = w.mesh()
print(f"{name}: mesh gen {time.time() - t0:.2f}s nodes={m.n_nodes} tets={m.n_tets}", flush=True)
ctx = ect.Context(0)
t0 = time.time()
mesh = ect.Mesh(ctx, m.xyz, m.tets, m.region)
print(f"mesh upload+prep {time.time() - t0:.2f}s N={mesh.n_dofs} pins={mesh.n_pins} "
      f"defect={mesh.n_defect}", flush=True)
t0 = time.time()
s = ect.Session(ctx, mesh, w.physics, w.coil, w.amplitude, tol=w.tol, max_iter=20000)
ctx.synchronize()
print(f"session (2x pattern+assembly) {time.time() - t0:.2f}s", ctx.timings(reset=True), flush=True)
a = s.matrix()
print("nnz", a.nnz, flush=True)
for rep in range(2):
    ctx.set_profiling(True)
    t0 = time.time()
    pts = s.solve_positions([w.positions[0]])
    dt = time.time() - t0
    tm = ctx.timings(reset=True)
    its = pts[0]["iterations"]
    print(f"position solve {dt:.3f}s iterations={its} failed={pts[0]['failed']} dz={pts[0]['dz']}")
    B = 20 * a.nnz + 4 * (a.n + 1) + 32 * 2 * a.n
    avg = tm["spmv_ms_total"] / max(1, tm["spmv_launches"])
    print(f"  spmv launches={tm['spmv_launches']} avg={avg:.4f} ms  -> {B / avg / 1e6:.0f} GB/s (k=2)"
          f"  solve_ms={tm['solve_ms']:.1f} launches={tm['kernel_launches']}")
    dofit = a.n * sum(its)
    print(f"  DOF*iter/s = {dofit / dt:.3e}", flush=True)
