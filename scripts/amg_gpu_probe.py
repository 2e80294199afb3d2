"""Dev probe (B200): COCG iterations and device time with the multigrid
preconditioner against point Jacobi on the configs[1] matrix, k right-hand
sides (4 configs[3] positions x 2 coils by default), plus the A-part
agreement of the two solutions.

  python scripts/amg_gpu_probe.py [k] [tol] [omega] [oc] [wcycle]
"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_03207_b200 import ect, workloads  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-8
w = workloads.config3()
if os.environ.get("DIMS"):  # a smaller configs[1]-like box, e.g. DIMS=16,16,32
    dims = tuple(int(v) for v in os.environ["DIMS"].split(","))
    w = workloads.Workload("probe", dims, 1, ((0.9, 1.1),), w.physics, workloads._coil(dims[2]),
                           1e6, w.positions)
m = w.mesh()
ctx = ect.Context(0)
mesh = ect.Mesh(ctx, m.xyz, m.tets, m.region)
p, r, two = mesh.materials(w.physics)
zs = [w.positions[i] for i in (20, 26, 31, 36, 10, 44, 5, 58)][: max(1, k // 2)]
zz = [z for z in zs for _ in (1, 2)][:k]
which = [c for _ in zs for c in (1, 2)][:k]
b = torch.from_numpy(mesh.rhs(w.coil, zz, which, w.amplitude)).cuda()
if k == 1:
    b = b[:, 0].contiguous()
sols = {}
for pc in os.environ.get("PRECONDS", "jacobi,amg").split(","):
    a = ect.Matrix(ctx, mesh).assemble(p).set_preconditioner(pc)
    info = a.precond_info()
    x = torch.empty_like(b)
    a.solve(b, tol=tol, max_iter=20000, out=x)  # warm (builds the hierarchy once)
    ctx.set_profiling(True)
    ctx.timings(reset=True)
    ctx.mark(0)
    _, res = a.solve(b, tol=tol, max_iter=20000, out=x)
    ctx.mark(1)
    ms = ctx.elapsed_ms(0, 1)
    tm = ctx.timings()
    ctx.set_profiling(False)
    its = [rr["iterations"] for rr in res]
    sp = tm["spmv_ms_total"] / max(1, tm["spmv_launches"])
    vc = tm["vec_ms_total"] / max(1, tm["vec_launches"])
    pcm = tm["precond_ms_total"] / max(1, tm["precond_launches"])
    print(f"{pc:7s} k={k} tol={tol:g} its={its} conv={[rr['converged'] for rr in res]} "
          f"res={max(rr['residual'] for rr in res):.2e} solve {ms:.1f} ms, {ms / max(its):.3f} ms/it "
          f"(spmv {sp:.3f} vec {vc:.3f} cycle {pcm:.3f}) info={info}", flush=True)
    sols[pc] = x.cpu().numpy()
if len(sols) == 2:
    xa, xb = sols["jacobi"], sols["amg"]
    na = 3 * mesh.n_nodes
    d = np.linalg.norm(xa[:na] - xb[:na]) / np.linalg.norm(xa[:na])
    print(f"A-part relative difference jacobi vs amg: {d:.2e}")
