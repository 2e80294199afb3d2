"""Dev probe: recurrence-residual history (ECT_TRACE_SOLVE=1) of the multigrid
COCG at a tight tolerance on the configs[1] matrices, golden-trace positions."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_1602_03207_b200 import ect, workloads  # noqa: E402

tol = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-12
max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 400
w = workloads.config3()
mm = w.mesh()
ctx = ect.Context(0)
m = ect.Mesh(ctx, mm.xyz, mm.tets, mm.region)
p, r, two = m.materials(w.physics)
idx = [0, 13, 20, 26, 31, 36, 45, 63]
for tag, mats in (("primary", p), ("reference", r)):
    a = ect.Matrix(ctx, m).assemble(mats)
    for grp in (idx[:4], idx[4:]):
        zs = [w.positions[i] for i in grp for _ in (0, 1)]
        b = m.rhs(w.coil, zs, [1, 2] * len(grp), w.amplitude)
        x, res = a.solve(b, tol=tol, max_iter=max_iter)
        print(tag, grp, [(q["iterations"], f"{q['residual']:.1e}", q["converged"]) for q in res], flush=True)
    del a
