"""Dev probe: NB SpMV time per batch width k on the configs[1] primary matrix
(kernel variant from ECT_NB_VARIANT).  python scripts/spmv_sweep.py [k,k,...]"""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1602_03207_b200 import ect, workloads  # noqa: E402

ks = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [2, 4, 8]
w = workloads.config1()
m = w.mesh()
ctx = ect.Context(0)
mesh = ect.Mesh(ctx, m.xyz, m.tets, m.region)
p, r, two = mesh.materials(w.physics)
a = ect.Matrix(ctx, mesh).assemble(p)
for k in ks:
    x = torch.randn(a.n, k, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    xs = x[:, 0].contiguous() if k == 1 else x
    ys = y[:, 0].contiguous() if k == 1 else y
    for _ in range(3):
        a.multiply(xs, out=ys)
    ctx.synchronize()
    ctx.mark(0)
    reps = 20
    for _ in range(reps):
        a.multiply(xs, out=ys)
    ctx.mark(1)
    ms = ctx.elapsed_ms(0, 1) / reps
    print(f"variant {os.environ.get('ECT_NB_VARIANT', '0')} k={k}: {ms:.4f} ms "
          f"({ms / k:.4f} ms per column)", flush=True)
