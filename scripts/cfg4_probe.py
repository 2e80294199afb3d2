"""Dev probe: where the true residual of the multigrid COCG sits on configs[4]
(A part, V part, per-conductor-component mean of the V part) when the solve
stalls at tight tolerances."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1602_03207_b200 import ect, workloads  # noqa: E402
from tests.helpers import conductor_components  # noqa: E402

w = workloads.config4()
mm = w.mesh()
ctx = ect.Context(0)
m = ect.Mesh(ctx, mm.xyz, mm.tets, mm.region)
p, r, two = m.materials(w.physics)
comp = conductor_components(mm.tets, mm.region, m.export()["cond_forward"])
print("V components:", np.bincount(comp), flush=True)
b = m.rhs(w.coil, [w.positions[0]] * 2, [1, 2], w.amplitude)
na = 3 * m.n_nodes
a = ect.Matrix(ctx, m).assemble(r)
for tol, mi in ((1e-8, 2000), (1e-10, 600), (1e-10, 3000)):
    t0 = time.time()
    x, res = a.solve(b, tol=tol, max_iter=mi)
    print("reference", tol, mi, f"{time.time() - t0:.1f}s", res, flush=True)
    rr = b - a.multiply(x)
    for c in range(2):
        bn = np.linalg.norm(b[:, c])
        rv = rr[na:, c]
        means = [rv[comp == q].sum() / np.sqrt((comp == q).sum()) for q in range(comp.max() + 1)]
        print(f"  col {c}: |r|/|b| {np.linalg.norm(rr[:, c]) / bn:.2e}  A part {np.linalg.norm(rr[:na, c]) / bn:.2e}"
              f"  V part {np.linalg.norm(rv) / bn:.2e}  V const-per-component part "
              f"{np.linalg.norm(means) / bn:.2e}  |x| {np.linalg.norm(x[:, c]):.2e} "
              f"|xV| {np.linalg.norm(x[na:, c]):.2e} xV comp means "
              f"{[abs(x[na:, c][comp == q].mean()) for q in range(comp.max() + 1)]}", flush=True)
