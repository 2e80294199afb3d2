"""Dev probe: SpMV time per batch width k on the configs[1] primary matrix for the
kernel variant in ECT_NB_VARIANT, and the max deviation from the CSR kernel
(same matrix, same x).  python scripts/nbw_probe.py [k,k,...]"""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1602_03207_b200 import ect, workloads  # noqa: E402

ks = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [8]
w = workloads.config1()
m = w.mesh()
ctx = ect.Context(0)
mesh = ect.Mesh(ctx, m.xyz, m.tets, m.region)
p, r, two = mesh.materials(w.physics)
a = ect.Matrix(ctx, mesh).assemble(p)
ctx.set_format("csr")
c = ect.Matrix(ctx, mesh).assemble(p)
var = os.environ.get("ECT_NB_VARIANT", "0")
g = torch.Generator(device="cuda").manual_seed(2)
for k in ks:
    x = torch.complex(torch.rand(a.n, k, device="cuda", dtype=torch.float64, generator=g) * 2 - 1,
                      torch.rand(a.n, k, device="cuda", dtype=torch.float64, generator=g) * 2 - 1)
    y = torch.empty_like(x)
    yc = torch.empty_like(x)
    c.multiply(x, out=yc)
    for _ in range(3):
        a.multiply(x, out=y)
    ctx.synchronize()
    dev = ((y - yc).abs().max() / yc.abs().max()).item()
    ctx.mark(0)
    reps = 20
    for _ in range(reps):
        a.multiply(x, out=y)
    ctx.mark(1)
    ms = ctx.elapsed_ms(0, 1) / reps
    print(f"variant {var} k={k}: {ms:.4f} ms ({ms / k:.4f} ms per column) "
          f"max|y-y_csr|/max|y|={dev:.2e}", flush=True)
