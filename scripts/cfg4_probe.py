"""Dev probe: multigrid COCG on configs[4] at tight tolerances (env knobs
ECT_AMG_F32 / ECT_AMG_OC / ... select the cycle variant)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1602_03207_b200 import ect, workloads  # noqa: E402

w = workloads.config4()
mm = w.mesh()
ctx = ect.Context(0)
m = ect.Mesh(ctx, mm.xyz, mm.tets, mm.region)
p, r, two = m.materials(w.physics)
b = m.rhs(w.coil, [w.positions[0]] * 2, [1, 2], w.amplitude)
print("env", {k: v for k, v in os.environ.items() if k.startswith("ECT_")}, flush=True)
for tag, mats in (("reference", r), ("primary", p)):
    a = ect.Matrix(ctx, m).assemble(mats)
    for tol, mi in ((1e-10, 1000), (1e-12, 1000)):
        t0 = time.time()
        x, res = a.solve(b, tol=tol, max_iter=mi)
        print(tag, tol, mi, f"{time.time() - t0:.1f}s", res, flush=True)
    del a
