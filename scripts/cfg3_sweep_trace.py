"""Dev: the configs[3] 64-position sweep on the GPU written as reference-format
traces at solver tolerances 1e-9 and 1e-12 (gpurun_out/gpu_cfg3_tol*.csv), with
the sweep wall time -- the positions/s figure BASELINE configs[3] asks for."""
import sys
import time

sys.path.insert(0, ".")
from paper_1602_03207_b200 import ect, trace, workloads  # noqa: E402

w = workloads.config3()
mm = w.mesh()
ctx = ect.Context(0)
m = ect.Mesh(ctx, mm.xyz, mm.tets, mm.region)
for tol in (1e-9, 1e-12):
    s = ect.Session(ctx, m, w.physics, w.coil, w.amplitude, tol=tol, max_iter=200000)
    s.solve_positions(list(w.positions[:4]), positions_per_batch=4)  # warm
    ctx.synchronize()
    t0 = time.time()
    pts = s.solve_positions(list(w.positions), positions_per_batch=4)
    ctx.synchronize()
    dt = time.time() - t0
    trace.write_trace_csv(f"gpurun_out/gpu_cfg3_tol{tol:g}.csv", pts,
                          config_hash=f"configs[3] GPU tol {tol:g}")
    its = [sum(p["iterations"]) for p in pts]
    print(f"tol {tol:g}: 64 positions in {dt:.2f} s = {64 / dt:.2f} positions/s "
          f"({1e3 * dt / 64:.0f} ms per position), iterations per position "
          f"{min(its)}..{max(its)}, failed {sum(p['failed'] for p in pts)}", flush=True)
    del s
