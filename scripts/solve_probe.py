"""Dev probe: SpMV and per-iteration cost on configs[1], NB vs CSR storage."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1602_03207_b200 import ect, workloads  # noqa: E402

max_iter = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
formats = sys.argv[2].split(",") if len(sys.argv) > 2 else ["nb", "csr"]
w = workloads.config1()
m = w.mesh()
ctx = ect.Context(0)
mesh = ect.Mesh(ctx, m.xyz, m.tets, m.region)
p, r, two = mesh.materials(w.physics)
z = w.positions[0]
b = torch.from_numpy(mesh.rhs(w.coil, [z, z], [1, 2], w.amplitude)).cuda()
for fmt in formats:
    ctx.set_format(fmt)
    a = ect.Matrix(ctx, mesh).assemble(p)
    print(f"== format {a.format}", flush=True)
    for k in (1, 2, 4, 8):
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
        B = 20 * a.nnz + 4 * (a.n + 1) + 32 * k * a.n
        print(f"  spmv k={k}: {ms:.4f} ms  algorithmic {B / ms / 1e6:.0f} GB/s", flush=True)
    x = torch.empty_like(b)
    for prof in (False, True):
        ctx.set_profiling(prof)
        ctx.timings(reset=True)
        ctx.mark(0)
        _, res = a.solve(b, tol=1e-8, max_iter=max_iter, out=x)
        ctx.mark(1)
        ms = ctx.elapsed_ms(0, 1)
        tm = ctx.timings()
        it = max(rr["iterations"] for rr in res)
        print(f"  solve k=2 profiling={prof} its={[rr['iterations'] for rr in res]} dev_ms={ms:.1f} "
              f"ms/iter={ms / it:.4f} spmv_avg={tm['spmv_ms_total'] / max(1, tm['spmv_launches']):.4f}"
              f" vec_avg={tm['vec_ms_total'] / max(1, tm['vec_launches']):.4f} n_spmv={tm['spmv_launches']}",
              flush=True)
    ctx.set_profiling(False)
    del a
