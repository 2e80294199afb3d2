"""Benchmark: A–V eddy-current probe-position solves on B200 (BASELINE.json metric).

Step = one probe position of the configs[1] mesh (64x64x128 Kuhn box, 3.15M
tets, N = 1,760,464 complex DOFs) exactly as ScanSession::solve_position
(scan.cpp:95-143) does it: coil-1 and coil-2 right-hand sides, solved against
the primary AND the reference (defect -> vacuum) matrix to tol 1e-8, then the
four impedance variations and the signal modes. Positions follow configs[3]'s
sweep (64 positions, z in [0.3, 1.7] cm), round-robin over ranks and steps
(weak scaling: one position per GPU per step).

  value    : complex DOF*iterations/s over all ranks = sum(N * Krylov iterations
             of every right-hand side) / max-over-ranks device time of the K steps
  e2e      : the same metric through the public C ABI with HOST buffers
             (ect_solve: pinned b -> device, 4 solves, 4 solutions -> host)
  roofline : dominant kernel = complex SpMV (K4) on 2 interleaved right-hand
             sides; algorithmic bytes 20*nnz + 4*(N+1) + 32*k*N
             / mean CUDA-event duration of its launches in the timed region
  cpu_baseline: the reference's solve_iterative (GMRES(80)+ILU(0), oracle/_ref)
             on the same matrix, bounded sample, rank 0 at N=1

--impl reference: the reference's own CPU path (oracle/_ref, assembled by the
reference itself) on the same config/metric, timed on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "complex DOF*iterations/s of the A-V Krylov solve"
UNIT = "DOF*iter/s"
TOL = 1e-8
MAX_ITER = 20000
PROFILE_SUMMARY = ROOT / "profiles" / "spmv_ncu_summary.json"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ppb", type=int, default=4,
                    help="probe positions per batched solve (their 2*ppb right-hand sides "
                         "share each matrix pass)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--workload", default="sweep", choices=["sweep", "large", "micro"],
                    help="sweep: configs[1] mesh, configs[3] positions sharded over GPUs (weak); "
                         "large: configs[4] one system row-partitioned over GPUs (strong)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def sweep_positions():
    from paper_1602_03207_b200 import workloads
    return workloads.config3().positions


# --------------------------------------------------------------------------- ours
def run_ours(args):
    world, rank, local = dist_env()
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1602_03207_b200 import ect, workloads

    w = workloads.config1()
    positions = sweep_positions()
    t0 = time.time()
    m = w.mesh()
    t_mesh = time.time() - t0
    ctx = ect.Context(local)
    mesh = ect.Mesh(ctx, m.xyz, m.tets, m.region)
    ctx.timings(reset=True)
    sess = ect.Session(ctx, mesh, w.physics, w.coil, w.amplitude, tol=TOL, max_iter=MAX_ITER)
    setup = ctx.timings(reset=True)
    a = sess.matrix()
    N, nnz = a.n, a.nnz
    ppb = max(1, args.ppb)

    from paper_1602_03207_b200 import sharding

    def step_positions(s):
        return sharding.positions_for(s, rank, world, ppb, positions)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # warm-up
    for s in range(args.warmup):
        sess.solve_positions(step_positions(s), positions_per_batch=ppb)
    ctx.synchronize()
    barrier()
    ctx.timings(reset=True)
    ctx.set_profiling(True)
    iters = 0
    failed = 0
    with ClockSampler(local) as clk:
        ctx.mark(0)
        for s in range(args.steps):
            pts = sess.solve_positions(step_positions(args.warmup + s), positions_per_batch=ppb)
            for p in pts:
                iters += sum(p["iterations"])
                failed += int(p["failed"])
        ctx.mark(1)
        ctx.synchronize()
        elapsed_ms = ctx.elapsed_ms(0, 1)
    ctx.set_profiling(False)
    barrier()
    tm = ctx.timings(reset=True)
    clocks = clk.summary()

    dofit = float(N) * iters
    elapsed_max, dofit_all, failed_all, launches_all = sharding.reduce_timing(
        elapsed_ms, dofit, failed, int(tm["kernel_launches"]),
        device=f"cuda:{local}" if world > 1 else None)
    value = dofit_all / (elapsed_max / 1e3)

    # roofline of the dominant kernel (SpMV on k = 2*ppb interleaved vectors)
    k = 2 * ppb
    spmv_ms = tm["spmv_ms_total"] / max(1, tm["spmv_launches"])
    b_spmv = 20 * nnz + 4 * (N + 1) + 32 * k * N
    achieved = b_spmv / (spmv_ms / 1e3) / 1e9
    nb = a.nb_stats()
    # bytes the node-block format must move per launch: blocks 96+4 B, couplings
    # 64+8 B, two node pointers + cond map, x read + q written + p re-read (dot)
    b_fmt = (100 * nb["blocks"] + 72 * nb["couplings"] + 12 * (mesh.n_nodes + 1)
             + 48 * k * N) if nb["format"] != "csr" else b_spmv
    peak, peak_src = measured_peak()
    traffic = None
    if PROFILE_SUMMARY.exists():
        try:
            traffic = json.loads(PROFILE_SUMMARY.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    e2e = None
    if not args.no_e2e:
        e2e = e2e_leg(ect, ctx, sess, mesh, w, positions, max(1, args.steps), rank, world, ppb,
                      step_positions)

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_leg(a, mesh, w, positions, args.cpu_threads)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded jittered Kuhn box, BASELINE configs[1]/[3])",
            "config": {
                "workload": f"configs[1] mesh 64x64x128 Kuhn box (3,145,728 tets), {ppb} probe "
                            f"position(s) of the configs[3] sweep per GPU per step, batched",
                "n_dofs": N, "nnz": nnz, "solves_per_position": 4,
                "rhs_per_matrix_pass": k, "tol": TOL, "solver": "Jacobi-COCG (complex symmetric)",
                "ms_per_probe_position": elapsed_max / (args.steps * ppb),
                "probe_positions_per_s": world * args.steps * ppb / (elapsed_max / 1e3),
                "krylov_iterations_timed": int(iters),
                "failed_positions": failed_all,
                "parallelism": f"positions round-robin over {world} GPU(s)",
                "l2": "inputs larger than L2 (matrix 1.68 GB x2 >> 126 MB)",
                "setup_ms": {"mesh_generation_host": t_mesh * 1e3,
                             "pattern_x2": setup["pattern_ms"], "assembly_x2": setup["assemble_ms"]},
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": f"k_nb_spmv (node-block, k={k} interleaved RHS, fused p^T q)"
                                   if nb["format"] != "csr" else f"k_spmv (CSR, k={k})",
                         "mean_launch_ms": spmv_ms,
                         "launches_timed": int(tm["spmv_launches"]),
                         "launch_sampling": "CUDA events on every 8th solver iteration; only "
                                            "iterations with all k columns still active "
                                            f"({int(tm['spmv_partial_launches'])} partial-width "
                                            "samples excluded)",
                         "algorithmic_bytes": b_spmv,
                         "algorithmic_bytes_note": "SURVEY 8(d) CSR formula 20*nnz+4*(N+1)+32*k*N; "
                                                   "NB stores the same matrix in fewer bytes",
                         "format_bytes": b_fmt,
                         "format_frac": b_fmt / (spmv_ms / 1e3) / 1e9 / peak,
                         "vector_ops_mean_ms": tm["vec_ms_total"] / max(1, tm["vec_launches"]),
                         "peak_source": peak_src},
            "gpu_launches": launches_all,
            "clocks": clocks,
        }
        if e2e:
            line["e2e"] = e2e
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def e2e_leg(ect, ctx, sess, mesh, w, positions, steps, rank, world, ppb, step_positions):
    """Same metric through the public ABI with host buffers (pinned).

    Headline: ect_session_solve_positions (ScanSession::solve_position) with the
    probe positions from host memory and, every step, the 4 solution vectors of
    the step's last position copied back into pinned host memory. Beside it:
    ect_solve (solve_iterative) per matrix with pinned host b and x."""
    import torch
    N = mesh.n_dofs
    sol = torch.empty((4, N), dtype=torch.complex128, pin_memory=True)
    sess.solve_positions(step_positions(0), positions_per_batch=ppb, solutions=sol)
    iters_s = 0
    t0 = time.perf_counter()
    for s in range(steps):
        pts = sess.solve_positions(step_positions(s), positions_per_batch=ppb, solutions=sol)
        iters_s += sum(sum(p["iterations"]) for p in pts)
    dt_s = time.perf_counter() - t0
    session = {"value": N * iters_s / dt_s, "unit": UNIT, "h2d_bytes_per_step": 8 * ppb,
               "d2h_bytes_per_step": 4 * N * 16 + ppb * 128,
               "path": "ect_session_solve_positions with host z and pinned host solutions "
                       "(4 x n_dofs complex) + signal points"}
    a_p = sess.matrix(False)
    a_r = sess.matrix(True)
    b_pin = torch.empty((N, 2), dtype=torch.complex128, pin_memory=True)
    x_pin = [torch.empty((N, 2), dtype=torch.complex128, pin_memory=True) for _ in range(2)]
    z = positions[rank % len(positions)]
    b_np = mesh.rhs(w.coil, [z, z], [1, 2], w.amplitude)  # the user's inputs, on the host
    b_pin.copy_(torch.from_numpy(b_np))
    iters = 0
    a_p.solve(b_pin, tol=TOL, max_iter=MAX_ITER, out=x_pin[0])  # warm
    t0 = time.perf_counter()
    for _ in range(steps):
        for j, a in enumerate((a_p, a_r)):
            _, res = a.solve(b_pin, tol=TOL, max_iter=MAX_ITER, out=x_pin[j])
            iters += sum(r["iterations"] for r in res)
    dt = time.perf_counter() - t0
    session["ect_solve"] = {"value": N * iters / dt, "unit": UNIT,
                            "h2d_bytes_per_step": 2 * N * 2 * 16,
                            "d2h_bytes_per_step": 2 * N * 2 * 16,
                            "path": "ect_solve (C ABI) with pinned host b/x, primary + reference "
                                    "matrices solved separately, 2 coils"}
    return session


def cpu_baseline_leg(a, mesh, w, positions, threads):
    """Reference solve_iterative (GMRES(80)+ILU(0)) on the same matrix, bounded."""
    try:
        from oracle import ref
        if not ref.available():
            return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                    "sample": "oracle/_ref not built"}
        cp, ri, v = a.export_csc()  # bit-identical to the reference's own build_global
        rs = ref.system_from_csc(cp, ri, v)
        nthreads = threads or min(os.cpu_count() or 1, 8)
        zs = [positions[i % len(positions)] for i in range(nthreads)]
        b = mesh.rhs(w.coil, zs, [1] * nthreads, w.amplitude)
        bs = np.ascontiguousarray(b.T)
        max_iter = 8
        out = rs.solve_iterative_batch(bs, tol=TOL, max_iter=max_iter, restart=80,
                                       threads=nthreads)
        its = int(out["iterations"].sum())
        # the reference's CscMatrix::multiply, single thread
        # dense x as configs[2] (re, im uniform [-1, 1], seed 2): the reference
        # skips x_j = 0 (sparse.cpp:115-124), so a coil RHS would time mostly zeros
        rng = np.random.default_rng(2)
        xs = rng.uniform(-1, 1, a.n) + 1j * rng.uniform(-1, 1, a.n)
        _, t_mv = rs.multiply(xs, repeat=3)
        b_mv = 20 * a.nnz + 4 * (a.n + 1) + 32 * a.n
        return {"value": a.n * its / out["seconds"], "unit": UNIT, "cores": nthreads,
                "kind": "reference",
                "spmv_single_thread_GBps": b_mv / (t_mv / 3) / 1e9,
                "spmv_single_thread_ms": t_mv / 3 * 1e3,
                "spmv_sample": "CscMatrix::multiply x3, dense seeded x (configs[2] distribution)",
                "sample": f"{nthreads} concurrent solve_iterative calls (GMRES(80)+ILU(0), "
                          f"ILU rebuilt per call as iterative.cpp:126) x {max_iter} iterations "
                          f"on the configs[1] primary matrix; {out['seconds']:.1f} s wall"}
    except Exception as e:  # never let the baseline kill the GPU line
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": f"failed: {e}"}


# --------------------------------------------------------------------- reference arm
def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return
    from oracle import ref
    from paper_1602_03207_b200 import workloads
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    w = workloads.config1()
    positions = sweep_positions()
    nthreads = args.cpu_threads or (os.cpu_count() or 1)
    t0 = time.time()
    m = w.mesh()
    rm = ref.RefMesh(m.xyz, m.tets, m.region)
    prim, refm, two = rm.materials(w.physics)
    parts = max(1, min(nthreads, 64))
    s = ref.RefSystem(rm, prim, parts=parts, workers=parts)
    setup_s = time.time() - t0
    zs = [positions[i % len(positions)] for i in range(nthreads)]
    bs = np.stack([s.position_rhs(w.coil, z, 1, w.amplitude) for z in zs])
    max_iter = 8  # amortises the per-call ILU(0) rebuild over a few GMRES iterations
    for _ in range(args.warmup):
        s.solve_iterative_batch(bs[:1], tol=TOL, max_iter=1, restart=80, threads=1)
    its = 0
    secs = 0.0
    for _ in range(args.steps):
        out = s.solve_iterative_batch(bs, tol=TOL, max_iter=max_iter, restart=80, threads=nthreads)
        its += int(out["iterations"].sum())
        secs += out["seconds"]
    value = s.n * its / secs
    sample = (f"{nthreads} concurrent solve_iterative calls (GMRES(80)+ILU(0), ILU rebuilt per "
              f"call) x {max_iter} iterations per step on the reference-assembled configs[1] "
              f"primary matrix")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded jittered Kuhn box, BASELINE configs[1])",
        "config": {"workload": "configs[1] mesh 64x64x128, reference CPU path (oracle/_ref)",
                   "n_dofs": s.n, "nnz": s.nnz, "reference_setup_s": setup_s,
                   "reference_assembly_s": s.timings, "parts": parts},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_micro(args):
    """configs[2]: 200 fixed Krylov iterations on the assembled configs[1]
    matrix, right-hand side re/im uniform [-1, 1] from seed 2: CSR vs SELL-32-sigma
    (the storage pair configs[2] names) vs the node-block format (NB)."""
    import torch
    from paper_1602_03207_b200 import ect, workloads
    w = workloads.config1()
    m = w.mesh()
    ctx = ect.Context(0)
    mesh = ect.Mesh(ctx, m.xyz, m.tets, m.region)
    p, _, _ = mesh.materials(w.physics)
    rng = np.random.default_rng(2)
    out = {}
    for fmt in ("nb", "sell", "csr"):
        ctx.set_format(fmt)
        a = ect.Matrix(ctx, mesh).assemble(p)
        n = a.n
        b = torch.from_numpy(rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)).cuda()
        x = torch.empty_like(b)
        a.solve(b, tol=1e-30, max_iter=20, out=x)  # warm
        ctx.timings(reset=True)
        ctx.set_profiling(True)
        ctx.mark(0)
        _, res = a.solve(b, tol=1e-30, max_iter=200, out=x)
        ctx.mark(1)
        ms = ctx.elapsed_ms(0, 1)
        ctx.set_profiling(False)
        tm = ctx.timings(reset=True)
        spmv = tm["spmv_ms_total"] / max(1, tm["spmv_launches"])
        B = 20 * a.nnz + 4 * (n + 1) + 32 * n
        out[fmt] = {"iterations": res[0]["iterations"], "ms_per_iteration": ms / res[0]["iterations"],
                    "spmv_ms": spmv, "spmv_algorithmic_GBps": B / spmv / 1e6,
                    "dof_iter_per_s": n * res[0]["iterations"] / (ms / 1e3)}
        del a
    peak, src = measured_peak()
    nbv = out["nb"]
    print(json.dumps({"metric": METRIC, "value": nbv["dof_iter_per_s"], "unit": UNIT, "n_gpus": 1,
                      "steps": 1, "warmup": 1, "ms_per_step": nbv["ms_per_iteration"] * 200,
                      "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                      "dtype": "f64", "data": "synthetic (configs[2]: x re/im U[-1,1], seed 2)",
                      "config": {"workload": "configs[2] 200 fixed Jacobi-COCG iterations on the "
                                             "configs[1] matrix", "formats": out,
                                 "peak_GBps": peak, "peak_source": src}}), flush=True)


def run_large(args):
    """configs[4]: one 27.4M-DOF system, rows partitioned by z-slabs (the mesh is
    numbered z-slowest, so contiguous node ranges are slabs of z-planes)
    over the GPUs (NCCL halo per SpMV + allreduce per dot), strong scaling."""
    world, rank, local = dist_env()
    import torch
    from paper_1602_03207_b200 import ect, workloads
    comm = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = workloads.config4()
    m = w.mesh()
    ctx = ect.Context(local)
    mesh = ect.Mesh(ctx, m.xyz, m.tets, m.region)
    p, _, _ = mesh.materials(w.physics)
    a = ect.Matrix(ctx, mesh).assemble(p)
    splits = np.linspace(0, mesh.n_nodes, world + 1).astype(np.int64)
    if world > 1:
        import torch.distributed as dist
        uid = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{local}")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(ect.comm_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        comm = ect.Comm(ctx, rank, world, bytes(uid.cpu().numpy()))
    part = ect.Part(ctx, mesh, a, splits, rank)
    del a  # the global matrix is only needed to cut the part
    b = torch.from_numpy(mesh.rhs(w.coil, [w.positions[0]] * 2, [1, 2], w.amplitude)).cuda(local)
    x = torch.zeros_like(b)
    for _ in range(args.warmup):
        ect.dist_solve([part], b, comm=comm, tol=TOL, max_iter=MAX_ITER, out=x)
    ctx.synchronize()
    if world > 1:
        torch.distributed.barrier()
    iters = 0
    with ClockSampler(local) as clk:
        ctx.mark(0)
        for _ in range(args.steps):
            _, res = ect.dist_solve([part], b, comm=comm, tol=TOL, max_iter=MAX_ITER, out=x)
            iters += sum(r["iterations"] for r in res)
        ctx.mark(1)
        ctx.synchronize()
        el = ctx.elapsed_ms(0, 1)
    from paper_1602_03207_b200 import sharding
    el_max, _, _, launches = sharding.reduce_timing(el, 0.0, 0, 0,
                                                    device=f"cuda:{local}" if world > 1 else None)
    N = mesh.n_dofs
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": N * iters / (el_max / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded jittered Kuhn box, BASELINE configs[4])",
            "config": {"workload": "configs[4] 128x128x512 (50.3M tets, N=%d), coil pair at z=1 cm, "
                                   "rows split in z-slabs (nodes numbered z-slowest)" % N,
                       "parallelism": f"row partition over {world} GPU(s), NCCL halo + allreduce",
                       "krylov_iterations_timed": iters, "part": part.info},
            "clocks": clk.summary(),
        }), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.workload == "large":
        run_large(a)
    elif a.workload == "micro":
        run_micro(a)
    else:
        run_ours(a)
