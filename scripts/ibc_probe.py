"""Dev probe: BiCGStab on the impedance-boundary fixture with a given library build."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from pathlib import Path  # noqa: E402

from paper_1602_03207_b200 import ect, workloads  # noqa: E402

if os.environ.get("ECT_PROBE_LIB"):
    ect.LIB_PATH = Path(os.environ["ECT_PROBE_LIB"]).resolve()
from tests.helpers import golden  # noqa: E402

g = golden("tube_ibc_r4")
ctx = ect.Context(0)
m = ect.Mesh(ctx, g["xyz"], g["tets"], g["region"])
p, r, two = m.materials(workloads.Physics(sigma_defect=1e4, mu_r_defect=5.0, ibc_tsp=True))
b = np.ascontiguousarray(g["rhs"].T)
for key, mats in (("primary", p), ("reference", r)):
    a = ect.Matrix(ctx, m).assemble(mats)
    for tol in (1e-10, 1e-13):
        try:
            x, res = a.solve(b, tol=tol, max_iter=8000)
            print(os.environ.get("ECT_PROBE_LIB", "current"), key, tol, res, flush=True)
        except Exception as e:  # noqa: BLE001
            print(os.environ.get("ECT_PROBE_LIB", "current"), key, tol, "error", e, flush=True)
