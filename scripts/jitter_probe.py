"""Dev probe: wall time of every ect_session_solve_positions call (4 positions
per call) over many calls -- looks for sporadic host-side stalls."""
import sys
import time

sys.path.insert(0, ".")
from paper_1602_03207_b200 import ect, sharding, workloads  # noqa: E402

w = workloads.config1()
pos = workloads.config3().positions
m = w.mesh()
ctx = ect.Context(0)
mesh = ect.Mesh(ctx, m.xyz, m.tets, m.region)
sess = ect.Session(ctx, mesh, w.physics, w.coil, w.amplitude, tol=1e-8, max_iter=20000)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
out = []
for s in range(n):
    zs = sharding.positions_for(s, 0, 1, 4, pos)
    t0 = time.perf_counter()
    pts = sess.solve_positions(zs, positions_per_batch=4)
    dt = time.perf_counter() - t0
    tm = ctx.timings(reset=True)
    out.append((dt * 1e3, sum(sum(p["iterations"]) for p in pts), tm["solve_ms"], tm["rhs_ms"]))
for i, o in enumerate(out):
    print(i, " ".join(f"{v:.1f}" for v in o), flush=True)
