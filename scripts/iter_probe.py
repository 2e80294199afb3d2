"""Dev probe: per-iteration wall time of a fixed-length k-column COCG solve on
the configs[1] matrix (tolerance never met), with and without the sampled
per-kernel event profiling, against the profiled kernel means.
python scripts/iter_probe.py [k] [iters]"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1602_03207_b200 import ect, workloads  # noqa: E402

import os  # noqa: E402
if os.environ.get("ECT_PROBE_LIB"):  # dev: compare against another build
    ect.LIB_PATH = ect.LIB_PATH.parent / os.environ["ECT_PROBE_LIB"]

k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 320
w = workloads.config1()
m = w.mesh()
ctx = ect.Context(0)
mesh = ect.Mesh(ctx, m.xyz, m.tets, m.region)
p, r, two = mesh.materials(w.physics)
a = ect.Matrix(ctx, mesh).assemble(p)
b = mesh.rhs(w.coil, [w.positions[0]] * k, [1, 2] * (k // 2), w.amplitude)
bt = torch.from_numpy(b).cuda() if not hasattr(b, "data_ptr") else b
for prof in (False, True, False):
    ctx.set_profiling(prof)
    ctx.timings(reset=True)
    ctx.synchronize()
    ctx.mark(0)
    x, res = a.solve(bt, tol=1e-30, max_iter=iters)
    ctx.mark(1)
    ms = ctx.elapsed_ms(0, 1)
    tm = ctx.timings(reset=True)
    its = res[0]["iterations"]
    print(f"k={k} profiling={prof}: {ms / its:.4f} ms/iteration over {its} iterations; "
          f"timings={ {kk: round(v, 4) if isinstance(v, float) else v for kk, v in tm.items()} }",
          flush=True)
