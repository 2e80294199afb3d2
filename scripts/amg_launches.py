"""Dev: a short multigrid-COCG solve (fixed iterations) on the configs[1]
matrix for an ncu launch list of the cycle's kernels."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_1602_03207_b200 import ect, workloads  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
its = int(sys.argv[2]) if len(sys.argv) > 2 else 6
w = workloads.config3()
m = w.mesh()
ctx = ect.Context(0)
mesh = ect.Mesh(ctx, m.xyz, m.tets, m.region)
p, r, two = mesh.materials(w.physics)
zs = [w.positions[i] for i in (20, 26, 31, 36)]
b = torch.from_numpy(mesh.rhs(w.coil, [z for z in zs for _ in (1, 2)][:k],
                              [c for _ in zs for c in (1, 2)][:k], w.amplitude)).cuda()
a = ect.Matrix(ctx, mesh).assemble(p)
print(a.precond_info())
x = torch.empty_like(b)
a.solve(b, tol=1e-30, max_iter=its, out=x)
ctx.synchronize()
