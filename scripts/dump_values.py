import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1602_03207_b200 import ect, workloads
from tests.helpers import golden
g = golden("small_4x4x8")
ctx = ect.Context(0)
m = ect.Mesh(ctx, g["xyz"], g["tets"], g["region"])
p, r, two = m.materials(workloads.Physics(sigma_defect=1e4, mu_r_defect=5.0))
out = {}
for key, mats in (("primary", p), ("reference", r)):
    a = ect.Matrix(ctx, m).assemble(mats)
    out[key] = a.export()[2]
np.savez("gpurun_out/values_small4.npz", **out)
print("dumped")
