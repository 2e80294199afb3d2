import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1602_03207_b200 import ect, workloads
from tests.helpers import golden
g = golden("small_4x4x8")
ctx = ect.Context(0)
for fmt in ("nb", "csr"):
    ctx.set_format(fmt)
    m = ect.Mesh(ctx, g["xyz"], g["tets"], g["region"])
    for tol in (1e-10, 1e-11):
        s = ect.Session(ctx, m, workloads.Physics(sigma_defect=1e4, mu_r_defect=5.0), tuple(g["coil"]), float(g["amplitude"]), tol=tol, max_iter=20000)
        pt = s.solve_positions([float(g["z"])])[0]
        print(fmt, tol, pt["failed"], pt["iterations"], pt["dz"][:2])
        sol = np.empty((4, m.n_dofs), np.complex128)
        pt = s.solve_positions([float(g["z"])], solutions=sol)[0]
        b = m.rhs(tuple(g["coil"]), [float(g["z"])]*2, [1,2], float(g["amplitude"]))
        print("  rhs diff", np.abs(b.T - g["rhs"]).max())
