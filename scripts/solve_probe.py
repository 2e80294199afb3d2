"""Dev probe: per-iteration cost of the batched COCG on configs[1]."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1602_03207_b200 import ect, workloads

max_iter = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
w = workloads.config1()
m = w.mesh()
ctx = ect.Context(0)
mesh = ect.Mesh(ctx, m.xyz, m.tets, m.region)
s = ect.Session(ctx, mesh, w.physics, w.coil, w.amplitude, tol=1e-8, max_iter=20000)
a = s.matrix()
z = w.positions[0]
b = torch.from_numpy(mesh.rhs(w.coil, [z, z], [1, 2], w.amplitude)).cuda()
x = torch.empty_like(b)
for prof in (False, True, False):
    ctx.set_profiling(prof)
    ctx.timings(reset=True)
    t0 = time.perf_counter()
    ctx.mark(0)
    _, res = a.solve(b, tol=1e-8, max_iter=max_iter, out=x)
    ctx.mark(1)
    ms = ctx.elapsed_ms(0, 1)
    wall = time.perf_counter() - t0
    tm = ctx.timings()
    it = max(r["iterations"] for r in res)
    print(f"profiling={prof} its={[r['iterations'] for r in res]} dev_ms={ms:.1f} wall_ms={wall*1e3:.1f} "
          f"ms/iter={ms/it:.4f} spmv_avg={tm['spmv_ms_total']/max(1,tm['spmv_launches']):.4f} "
          f"launches={tm['kernel_launches']}", flush=True)
