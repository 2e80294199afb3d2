// K4 SpMV/SpMM + K5 fused Krylov vector ops + K6 device-resident COCG.
//
// Replaces CscMatrix::multiply (sparse.cpp:115-124), vector_norm /
// relative_residual (sparse.cpp:126-145) and solve_iterative
// (iterative.cpp:109-228). The reference runs restarted GMRES(80) with an
// ILU(0) right preconditioner, serial; A is complex SYMMETRIC (A = A^T, not
// Hermitian, when IBC is off — SURVEY §8(a)), so the GPU uses Jacobi-
// preconditioned COCG (conjugate orthogonal CG, unconjugated bilinear form)
// whose iteration is one SpMV plus fused vector updates: bandwidth-bound and
// without GMRES's growing basis. Convergence follows the reference contract:
// recurrence residual <= tol, then a TRUE residual confirmation
// (iterative.cpp:208-216) with restart when it fails; b == 0 -> x = 0
// converged (iterative.cpp:120-124); non-convergence is a flag, breakdown an
// error (iterative.cpp:176).
//
// Layout: CSR values double2 (16 B), int32 columns; vectors for k
// right-hand sides are interleaved [n][k] double2 so one gather serves all
// k columns (multi-RHS sweep, SURVEY §8(d) B_iter(k)).
// Determinism: grid-stride persistent grids with a static row->thread map,
// fixed-order warp/block trees, and a last-block fixed-order reduction of the
// per-block partials — bitwise-repeatable, no fp64 atomics.
#include <cub/cub.cuh>

#include <algorithm>
#include <array>
#include <chrono>
#include <thread>

#include "ect_internal.h"

namespace ect {
namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
// fp64 <-> fp32 complex element access (multigrid work vectors)
__device__ __forceinline__ double2 as_d2(double2 v) { return v; }
__device__ __forceinline__ double2 as_d2(float2 v) { return make_double2(v.x, v.y); }
__device__ __forceinline__ void put(double2* p, double2 v) { *p = v; }
__device__ __forceinline__ void put(float2* p, double2 v) {
  *p = make_float2((float)v.x, (float)v.y);
}
// Smith's complex division a / b
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    double r = b.y / b.x, den = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / den, (a.y - a.x * r) / den);
  }
  double r = b.x / b.y, den = b.x * r + b.y;
  return make_double2((a.x * r + a.y) / den, (a.y * r - a.x) / den);
}

__device__ __forceinline__ double2 ldg2(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}
__device__ __forceinline__ int ldg_i(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Block-wide sum of NV doubles per thread into smem-backed result (thread 0).
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j)
#pragma unroll
    for (int o = 16; o; o >>= 1) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) smem[wid * NV + j] = v[j];
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double x = lane < nw ? smem[lane * NV + j] : 0.0;
#pragma unroll
      for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      v[j] = x;
    }
  }
  __syncthreads();
}

// Block-wide sum when lane l holds NVL values of slot (l % CL): the result in
// thread 0's out[NVL * CL] is ordered slot-major (fixed order, deterministic).
template <int NVL, int CL>
__device__ __forceinline__ void block_sum_slots(double (&v)[NVL], double* smem,
                                                double (&out)[NVL * CL]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < NVL; ++j)
#pragma unroll
    for (int o = 16; o >= CL; o >>= 1) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
  if (lane < CL)
#pragma unroll
    for (int j = 0; j < NVL; ++j) smem[(wid * CL + lane) * NVL + j] = v[j];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NVL * CL; ++j) {
      double t = 0.0;
      for (int w = 0; w < nw; ++w) t += smem[w * NVL * CL + j];
      out[j] = t;
    }
  }
  __syncthreads();
}

// Last-block-done: returns true in the block that finished last (all of
// whose threads then see every other block's partials).
__device__ __forceinline__ bool last_block(unsigned* counter) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned ticket = atomicAdd(counter, 1u);
    is_last = ticket == gridDim.x - 1;
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

// Fixed-order reduction of NV values per block stored at partial[b*NV + j].
template <int NV>
__device__ __forceinline__ void reduce_partials(const double* partial, double (&out)[NV],
                                                double* smem) {
#pragma unroll
  for (int j = 0; j < NV; ++j) out[j] = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
#pragma unroll
    for (int j = 0; j < NV; ++j) out[j] += __ldcg(partial + (size_t)b * NV + j);
  block_sum<NV>(out, smem);
}

// SpMV epilogues:
//  kPlain    : y = A x
//  kCocg     : y = q = A p; per column p^T q (unconjugated) -> alpha = rho / p^T q
//  kResid    : y = b - A x; per column ||y||^2 -> st.rnorm (true residual)
//  kResidNR  : y = b - A x (multigrid residual, no reduction)
//  kSmooth   : y = x + omega D^-1 (b - A x) (damped-Jacobi sweep, no reduction)
//  kSmoothDot: kSmooth, plus per column b^T y (unconjugated) -> rho = r^T z of
//              the preconditioned COCG (b = r, y = z = M r on the finest level)
//  kCgDot    : y = w = A z (x = z, b = r); per column r^T z, w^T z, ||r||^2 (the
//              single reduction of the Chronopoulos-Gear COCG, distributed solve)
enum Mode { kPlain = 0, kCocg = 1, kResid = 2, kResidNR = 3, kSmooth = 4, kSmoothDot = 5,
            kCgDot = 6 };
__host__ __device__ constexpr int mode_nv(int mode, int k) {
  return mode == kCocg || mode == kSmoothDot ? 2 * k
         : mode == kResid                    ? k
         : mode == kCgDot                    ? 5 * k
                                             : 0;
}

struct KrylovCtl {
  RhsState* st;       // [K]
  int* n_active;
  unsigned* counter;
  double* partial;    // [grid][NV]
  double tol;
  int max_iter;
  // distributed solve: the last block writes its (part-local) totals here and
  // the finalisation runs after the cross-part reduction (k_fin); nullptr on
  // a single part, where the last block finalises directly
  double* red;
  // owned rows of the vector kernels: [s0, e0) U [s1, e1)
  int64_t s0, e0, s1, e1;
  // split SpMV (halo overlap): later launches add their totals into red
  int red_add;
  // damped-Jacobi epilogues (kSmooth / kSmoothDot): D^-1 of the level, weight
  const double2* dinv;
  double omega;
  // kSmoothDot: 1 = first preconditioned residual of a (re)start (sets rho),
  // 0 = an iteration (beta = rho_new / rho)
  int rho_start;
  // dev (ECT_TRACE_SOLVE=1): relative recurrence residual per iteration,
  // hist[iters * hist_k + column], iterations < hist_cap
  double* hist = nullptr;
  int hist_cap = 0, hist_k = 0;
};
__device__ __forceinline__ void trace_residual(const KrylovCtl& ctl, const RhsState& s, int k) {
  if (ctl.hist && s.iters < ctl.hist_cap)
    ctl.hist[(size_t)s.iters * ctl.hist_k + k] = s.bnorm > 0.0 ? s.rnorm / s.bnorm : 0.0;
}

// COCG has no look-ahead: after a near-breakdown (p^T A p ~ 0: one huge step,
// the residual jumps by orders of magnitude) the recurrences stop producing
// conjugate directions and the residual hovers instead of converging (measured
// on configs[1] at tol 1e-12: 7e-11 at iteration 90, 5e-7 at 110, then ~1e-7
// for 300 iterations), although a fresh start from the same residual converges
// at the initial rate. With the multigrid preconditioner a healthy solve sets a
// new best residual at least every ~30 iterations, so a column that has not
// improved for max(kStall, iterations / 2) iterations restarts its direction:
// p = z (beta = 0), the window and the best value are reset, x and r are
// untouched. The window grows with the iteration count because a slow, noisy
// but converging solve (multigrid on a matrix given without its mesh: 500-2000
// iterations) goes 300 iterations between best values late in the solve; a
// fixed 50-iteration window restarts it to death (measured). (Taking the big
// step back instead was tried and is worse: COCG's route to convergence goes
// through 10-100x peaks, and restarting at each one forfeits the superlinear
// phase.)
constexpr int kStall = 50;
__device__ __forceinline__ void stall_check(RhsState& s) {
  if (s.rnorm < s.rbest) {
    s.rbest = s.rnorm;
    s.best_iter = (double)s.iters;
  } else if ((double)s.iters - s.best_iter >= fmax((double)kStall, 0.5 * (double)s.iters)) {
    s.restart_dir = 1;  // consumed by fin_rho
    s.rbest = s.rnorm;
    s.best_iter = (double)s.iters;
  }
}

// ---- scalar finalisations (run by one thread on the global totals) ----------
template <int K>
__device__ void fin_alpha(const KrylovCtl& ctl, const double* tot) {
  int active = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    RhsState& s = ctl.st[k];
    if (s.status != kActive) continue;
    const double2 pq = make_double2(tot[2 * k], tot[2 * k + 1]);
    if (pq.x == 0.0 && pq.y == 0.0) {
      s.status = kBreakdown;
      continue;
    }
    s.alpha = cdiv(s.rho, pq);
    ++active;
  }
  *ctl.n_active = active;
}

template <int K>
__device__ void fin_resid(const KrylovCtl& ctl, const double* tot) {
#pragma unroll
  for (int k = 0; k < K; ++k) ctl.st[k].rnorm = sqrt(tot[k]);
}

template <int K>
__device__ void fin_update(const KrylovCtl& ctl, const double* tot) {
  int active = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    RhsState& s = ctl.st[k];
    s.xpend = s.status == kActive;  // this iteration's x += alpha p is owed to k_pupdate
    if (s.status != kActive) continue;
    const double2 rho_new = make_double2(tot[3 * k], tot[3 * k + 1]);
    s.rnorm = sqrt(tot[3 * k + 2]);
    s.iters += 1;
    trace_residual(ctl, s, k);
    if (s.rnorm <= ctl.tol * s.bnorm) {
      s.status = kConverged;
    } else if (s.iters >= ctl.max_iter) {
      s.status = kMaxIter;
    } else if (rho_new.x == 0.0 && rho_new.y == 0.0) {
      s.status = kBreakdown;
    } else {
      s.beta = cdiv(rho_new, s.rho);
      s.rho = rho_new;
      ++active;
    }
  }
  *ctl.n_active = active;
}

// External preconditioner (multigrid): the update decides convergence from
// ||r|| alone; rho = r^T z and beta come from the preconditioner's last
// kernel (fin_rho).
template <int K>
__device__ void fin_update_norm(const KrylovCtl& ctl, const double* tot) {
  int active = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    RhsState& s = ctl.st[k];
    s.xpend = s.status == kActive;
    if (s.status != kActive) continue;
    s.rnorm = sqrt(tot[k]);
    s.iters += 1;
    trace_residual(ctl, s, k);
    if (s.rnorm <= ctl.tol * s.bnorm) {
      s.status = kConverged;
    } else if (s.iters >= ctl.max_iter) {
      s.status = kMaxIter;
    } else {
      stall_check(s);
      ++active;
    }
  }
  *ctl.n_active = active;
}

template <int K>
__device__ void fin_rho(const KrylovCtl& ctl, const double* tot) {
  int active = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    RhsState& s = ctl.st[k];
    if (s.status != kActive) continue;
    const double2 rho_new = make_double2(tot[2 * k], tot[2 * k + 1]);
    if (rho_new.x == 0.0 && rho_new.y == 0.0) {
      s.status = kBreakdown;
      continue;
    }
    if (!ctl.rho_start) s.beta = cdiv(rho_new, s.rho);
    if (s.restart_dir) {  // stalled (stall_check): p = z, the direction restarts from r
      s.beta = make_double2(0.0, 0.0);
      s.restart_dir = 0;
    }
    s.rho = rho_new;
    ++active;
  }
  *ctl.n_active = active;
}

template <int K>
__device__ void fin_start_norm(const KrylovCtl& ctl, const double* tot, unsigned mask,
                               int fresh) {
  int active = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    RhsState& s = ctl.st[k];
    if ((mask >> k) & 1u) {
      if (fresh) {
        s.bnorm = sqrt(tot[2 * k + 1]);
        s.iters = 0;
      }
      s.rnorm = s.rbest = sqrt(tot[2 * k]);
      s.restart_dir = 0;
      s.best_iter = (double)s.iters;
      if (fresh && s.bnorm == 0.0) s.status = kZeroRhs;
      else if (s.rnorm <= ctl.tol * s.bnorm) s.status = kConverged;
      else s.status = kActive;
    }
    active += s.status == kActive;
  }
  *ctl.n_active = active;
}

template <int K>
__device__ void fin_start(const KrylovCtl& ctl, const double* tot, unsigned mask, int fresh) {
  int active = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    RhsState& s = ctl.st[k];
    if ((mask >> k) & 1u) {
      if (fresh) {
        s.bnorm = sqrt(tot[4 * k + 3]);
        s.iters = 0;
      }
      s.rho = make_double2(tot[4 * k], tot[4 * k + 1]);
      s.rnorm = s.rbest = sqrt(tot[4 * k + 2]);
      s.restart_dir = 0;
      s.best_iter = (double)s.iters;
      if (fresh && s.bnorm == 0.0) {
        s.status = kZeroRhs;
      } else if (s.rnorm <= ctl.tol * s.bnorm) {
        s.status = kConverged;
      } else if (s.rho.x == 0.0 && s.rho.y == 0.0) {
        s.status = kBreakdown;
      } else {
        s.status = kActive;
      }
    }
    active += s.status == kActive;
  }
  *ctl.n_active = active;
}

// Chronopoulos-Gear COCG (one reduction per iteration): tot per column =
// (r^T z re, im, w^T z re, im, ||r||^2) after the step r -= alpha s.
template <int K>
__device__ void fin_cg(const KrylovCtl& ctl, const double* tot, unsigned mask, int start,
                       int fresh) {
  int active = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    RhsState& s = ctl.st[k];
    const double2 g = make_double2(tot[5 * k], tot[5 * k + 1]);
    const double2 d = make_double2(tot[5 * k + 2], tot[5 * k + 3]);
    const double rn = sqrt(tot[5 * k + 4]);
    if (start) {
      if (!((mask >> k) & 1u)) {
        active += s.status == kActive;
        continue;
      }
      if (fresh) {
        s.bnorm = rn;  // r = b
        s.iters = 0;
      }
      s.rnorm = rn;
      s.beta = make_double2(0.0, 0.0);
      if (fresh && s.bnorm == 0.0) s.status = kZeroRhs;
      else if (rn <= ctl.tol * s.bnorm) s.status = kConverged;
      else if ((g.x == 0.0 && g.y == 0.0) || (d.x == 0.0 && d.y == 0.0)) s.status = kBreakdown;
      else {
        s.status = kActive;
        s.rho = g;
        s.alpha = cdiv(g, d);
        ++active;
      }
      continue;
    }
    if (s.status != kActive) continue;
    s.rnorm = rn;
    s.iters += 1;
    if (rn <= ctl.tol * s.bnorm) {
      s.status = kConverged;
    } else if (s.iters >= ctl.max_iter) {
      s.status = kMaxIter;
    } else {
      const double2 beta = cdiv(g, s.rho);
      const double2 den = csub(d, cdiv(cmul(beta, g), s.alpha));
      if ((g.x == 0.0 && g.y == 0.0) || (den.x == 0.0 && den.y == 0.0)) {
        s.status = kBreakdown;
      } else {
        s.beta = beta;
        s.alpha = cdiv(g, den);
        s.rho = g;
        ++active;
      }
    }
  }
  *ctl.n_active = active;
}

enum Fin { kFinAlpha = 0, kFinUpdate = 1, kFinStart = 2, kFinResid = 3, kFinCg = 4,
           kFinCgStart = 5 };

// Finalisation after a cross-part reduction of ctl.red (distributed solve).
template <int K, int WHAT>
__global__ void k_fin(KrylovCtl ctl, unsigned mask, int fresh) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  constexpr int NV = WHAT == kFinAlpha ? 2 * K : WHAT == kFinUpdate ? 3 * K
                     : WHAT == kFinStart ? 4 * K : (WHAT == kFinCg || WHAT == kFinCgStart) ? 5 * K
                     : K;
  if (WHAT != kFinStart && WHAT != kFinResid && WHAT != kFinCgStart && *ctl.n_active == 0) return;
  double tot[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) tot[j] = ctl.red[j];
  if (WHAT == kFinCg || WHAT == kFinCgStart) fin_cg<K>(ctl, tot, mask, WHAT == kFinCgStart, fresh);
  else if (WHAT == kFinAlpha) fin_alpha<K>(ctl, tot);
  else if (WHAT == kFinUpdate) fin_update<K>(ctl, tot);
  else if (WHAT == kFinStart) fin_start<K>(ctl, tot, mask, fresh);
  else fin_resid<K>(ctl, tot);
}

// y = A x for K interleaved vectors with G lanes per row.
//  kPlain: y = A x
//  kCocg : y = q = A p; per column p^T q (unconjugated) -> alpha = rho / p^T q
//  kResid: y = b - A x; per column ||y||^2 -> st.rnorm (true residual)
template <int G, int K, int MODE>
__global__ void __launch_bounds__(kBlock)
k_spmv(int64_t n, const int* __restrict__ row_ptr, const int* __restrict__ col,
       const double2* __restrict__ val, const double2* __restrict__ x, double2* __restrict__ y,
       const double2* __restrict__ b, KrylovCtl ctl) {
  constexpr int NV0 = mode_nv(MODE, K), NV = NV0 > 0 ? NV0 : 1;
  __shared__ double smem[32 * NV];
  if (MODE != kPlain && *ctl.n_active == 0) return;
  bool act[K];
#pragma unroll
  for (int k = 0; k < K; ++k) act[k] = (MODE == kPlain) || ctl.st[k].status == kActive;

  constexpr int RPW = 32 / G;  // rows per warp and pass
  const int lane = threadIdx.x & 31;
  const int g = lane & (G - 1);
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double part[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) part[j] = 0.0;

  // warp-uniform trip count so the segment shuffles always see full warps
  for (int64_t wrow = warp * RPW; wrow < n; wrow += n_warps * RPW) {
    const int64_t row = wrow + lane / G;
    const bool valid = row < n;
    const int beg = valid ? row_ptr[row] : 0, end = valid ? row_ptr[row + 1] : 0;
    double2 acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = make_double2(0.0, 0.0);
    int p = beg + g;
    // 2-deep software pipeline on the streamed matrix entries
    for (; p + G < end; p += 2 * G) {
      const int j0 = ldg_i(col + p), j1 = ldg_i(col + p + G);
      const double2 a0 = ldg2(val + p), a1 = ldg2(val + p + G);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (!act[k]) continue;
        const double2 x0 = x[(int64_t)j0 * K + k], x1 = x[(int64_t)j1 * K + k];
        acc[k].x += a0.x * x0.x - a0.y * x0.y;
        acc[k].y += a0.x * x0.y + a0.y * x0.x;
        acc[k].x += a1.x * x1.x - a1.y * x1.y;
        acc[k].y += a1.x * x1.y + a1.y * x1.x;
      }
    }
    if (p < end) {
      const int j0 = ldg_i(col + p);
      const double2 a0 = ldg2(val + p);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (!act[k]) continue;
        const double2 x0 = x[(int64_t)j0 * K + k];
        acc[k].x += a0.x * x0.x - a0.y * x0.y;
        acc[k].y += a0.x * x0.y + a0.y * x0.x;
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
      for (int o = G / 2; o; o >>= 1) {
        acc[k].x += __shfl_xor_sync(0xffffffffu, acc[k].x, o, G);
        acc[k].y += __shfl_xor_sync(0xffffffffu, acc[k].y, o, G);
      }
    }
    if (g == 0 && valid) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (!act[k]) continue;
        const int64_t idx = row * K + k;
        if (MODE == kPlain) {
          y[idx] = acc[k];
        } else if (MODE == kCocg) {
          y[idx] = acc[k];
          const double2 pv = x[idx];
          part[2 * k] += pv.x * acc[k].x - pv.y * acc[k].y;
          part[2 * k + 1] += pv.x * acc[k].y + pv.y * acc[k].x;
        } else if (MODE == kResid) {
          const double2 rv = csub(b[idx], acc[k]);
          y[idx] = rv;
          part[k] += rv.x * rv.x + rv.y * rv.y;
        } else if (MODE == kResidNR) {
          y[idx] = csub(b[idx], acc[k]);
        } else {
          const double2 bv = b[idx];
          const double2 zv = cadd(x[idx], cmul(make_double2(ctl.omega * ctl.dinv[row].x,
                                                            ctl.omega * ctl.dinv[row].y),
                                               csub(bv, acc[k])));
          y[idx] = zv;
          if (MODE == kSmoothDot) {
            part[2 * k] += bv.x * zv.x - bv.y * zv.y;
            part[2 * k + 1] += bv.x * zv.y + bv.y * zv.x;
          }
        }
      }
    }
  }
  if (NV0 == 0) return;

  block_sum<NV>(part, smem);
  if (threadIdx.x == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) ctl.partial[(size_t)blockIdx.x * NV + j] = part[j];
  if (!last_block(ctl.counter)) return;
  double tot[NV];
  reduce_partials<NV>(ctl.partial, tot, smem);
  if (threadIdx.x == 0) {
    if (ctl.red) {
#pragma unroll
      for (int j = 0; j < NV; ++j) ctl.red[j] = tot[j];
    } else if (MODE == kCocg) {
      fin_alpha<K>(ctl, tot);
    } else if (MODE == kSmoothDot) {
      fin_rho<K>(ctl, tot);
    } else {
      fin_resid<K>(ctl, tot);
    }
    *ctl.counter = 0u;
  }
}

// ---- node-block (NB) SpMV ----------------------------------------------------
// The A–V matrix has exploitable structure: the 3 A-rows of a
// node share one column set (3x3 blocks), A-A entries are real except the
// c == d mass entries, and the A-V / V-A couplings are real. NB stores per
// node i its 3x3 blocks as 12 doubles (9 real + 3 diagonal imaginary) in 3
// planes of 4 doubles — one coalesced 256-bit load (LDG.E.ENL2.256, sm_100)
// per plane per lane — sharing one int32 column per block, and its conductor
// couplings (AV[3], VA[3], VV) as 2 planes of 4 doubles + one int2 (node,
// V-dof). ~11 B per A-A entry instead of CSR's 20, and each x gather (3
// contiguous complex per column node, 256-bit loads for even k) feeds 3 rows.
// The imaginary parts dropped are exact zeros (checked at build).
struct NbView {
  const int* blk_ptr;
  const int* blk_col;
  const double* blk;    // plane p of block q at blk + 4 * (p * nblk + q)
  int64_t nblk;
  const int* cpl_ptr;
  const int2* cpl_idx;
  const double* cpl;    // plane p of coupling q at cpl + 4 * (p * ncpl + q)
  int64_t ncpl;
  const int* cond_fwd;
  int64_t n_nodes;  // nodes whose rows this view computes (owned nodes)
  int64_t na;       // V block offset in the x/y layout (3 n_nodes, or 3 (L + G) on a part)
  const int* e_off = nullptr;  // NB-E: chunk slot offsets (blk / blk_col are then slot-major)
  int64_t node_begin = 0;      // rows of nodes [node_begin, n_nodes) (split SpMV)
};

// 256-bit streaming load (read-once matrix data: no L1 allocation)
__device__ __forceinline__ void ld4s(const double* p, double (&v)[4]) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}
// 256-bit read-only load that may allocate in L1 (x gathers are reused)
__device__ __forceinline__ void ld4x(const double2* p, double2& a, double2& b) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
               : "l"(p));
}

__device__ __forceinline__ void load_block(const NbView& A, int64_t q, double (&B)[3][3],
                                           double (&Im)[3]) {
  double v0[4], v1[4], v2[4];
  ld4s(A.blk + 4 * q, v0);
  ld4s(A.blk + 4 * (A.nblk + q), v1);
  ld4s(A.blk + 4 * (2 * A.nblk + q), v2);
  B[0][0] = v0[0]; B[0][1] = v0[1]; B[0][2] = v0[2];
  B[1][0] = v0[3]; B[1][1] = v1[0]; B[1][2] = v1[1];
  B[2][0] = v1[2]; B[2][1] = v1[3]; B[2][2] = v2[0];
  Im[0] = v2[1]; Im[1] = v2[2]; Im[2] = v2[3];
}

__device__ __forceinline__ void load_cpl(const NbView& A, int64_t q, double (&av)[3],
                                         double (&va)[3], double2& vv) {
  double c0[4], c1[4];
  ld4s(A.cpl + 4 * q, c0);
  ld4s(A.cpl + 4 * (A.ncpl + q), c1);
  av[0] = c0[0]; av[1] = c0[1]; av[2] = c0[2];
  va[0] = c0[3]; va[1] = c1[0]; va[2] = c1[1];
  vv = make_double2(c1[2], c1[3]);
}

// K consecutive complex values (one node component, all right-hand sides).
template <int K>
__device__ __forceinline__ void load_xk(const double2* p, double2 (&v)[K]) {
  if constexpr (K % 2 == 0) {
#pragma unroll
    for (int j = 0; j < K; j += 2) ld4x(p + j, v[j], v[j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < K; ++j) v[j] = __ldg(p + j);
  }
}

__device__ __forceinline__ int2 ldg_i2(const int2* p) {
  int2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}

// Multi-RHS CSR SpMV with column-pair lanes (K >= 2; coarse multigrid levels,
// CSR / IBC matrices): G = (K/2) x E lanes per row, lane (e, c) streams the
// row's entries e, e + E, ... and gathers the 2 right-hand sides 2c, 2c + 1
// of each column with one 256-bit load; the E entry lanes reduce by shuffles.
// Same epilogues as k_spmv.
template <int K, int E, int MODE>
__global__ void __launch_bounds__(kBlock)
k_spmv_v(int64_t n, const int* __restrict__ row_ptr, const int* __restrict__ col,
         const double2* __restrict__ val, const double2* __restrict__ x, double2* __restrict__ y,
         const double2* __restrict__ b, KrylovCtl ctl) {
  static_assert(K % 2 == 0, "column pairs");
  constexpr int CLN = K / 2, G = CLN * E, RPW = 32 / G;
  static_assert(32 % G == 0, "lanes per row");
  constexpr int NVL0 = mode_nv(MODE, 2), NVL = NVL0 > 0 ? NVL0 : 1;
  constexpr int NV = NVL * CLN;
  __shared__ double smem[32 * NV];
  if (MODE != kPlain && *ctl.n_active == 0) return;
  const int lane = threadIdx.x & 31;
  const int g = lane % G, e = g / CLN, cl = g % CLN, kc = 2 * cl;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double part[NVL];
#pragma unroll
  for (int j = 0; j < NVL; ++j) part[j] = 0.0;
  for (int64_t wrow = warp * RPW; wrow < n; wrow += n_warps * RPW) {
    const int64_t row = wrow + lane / G;
    const bool valid = row < n;
    const int beg = valid ? row_ptr[row] : 0, end = valid ? row_ptr[row + 1] : 0;
    double2 acc[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    // U entries per step: all column / value loads first, then all gathers,
    // so a lane pays two dependent load latencies per U entries, not per entry
    // (short rows on small levels are pure latency: 35 -> ~10 us per launch)
    constexpr int U = 4;
    for (int p0 = beg + e; p0 < end; p0 += U * E) {
      int j[U];
      double2 a[U], x0[U], x1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int p = p0 + u * E;
        j[u] = -1;
        a[u] = make_double2(0.0, 0.0);
        if (p < end) {
          j[u] = ldg_i(col + p);
          a[u] = ldg2(val + p);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        x0[u] = x1[u] = make_double2(0.0, 0.0);
        if (j[u] >= 0) ld4x(x + (int64_t)j[u] * K + kc, x0[u], x1[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc[0].x += a[u].x * x0[u].x - a[u].y * x0[u].y;
        acc[0].y += a[u].x * x0[u].y + a[u].y * x0[u].x;
        acc[1].x += a[u].x * x1[u].x - a[u].y * x1[u].y;
        acc[1].y += a[u].x * x1[u].y + a[u].y * x1[u].x;
      }
    }
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int o = G / 2; o >= CLN; o >>= 1) {
        acc[c].x += __shfl_xor_sync(0xffffffffu, acc[c].x, o, G);
        acc[c].y += __shfl_xor_sync(0xffffffffu, acc[c].y, o, G);
      }
    if (e == 0 && valid) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int64_t idx = row * K + kc + c;
        const double2 v = acc[c];
        if (MODE == kPlain) {
          y[idx] = v;
        } else if (MODE == kCocg) {
          y[idx] = v;
          const double2 pv = x[idx];
          part[2 * c] += pv.x * v.x - pv.y * v.y;
          part[2 * c + 1] += pv.x * v.y + pv.y * v.x;
        } else if (MODE == kResid) {
          const double2 rv = csub(b[idx], v);
          y[idx] = rv;
          part[c] += rv.x * rv.x + rv.y * rv.y;
        } else if (MODE == kResidNR) {
          y[idx] = csub(b[idx], v);
        } else {
          const double2 bv = b[idx];
          const double2 d = ctl.dinv[row];
          const double2 zv = cadd(x[idx], cmul(make_double2(ctl.omega * d.x, ctl.omega * d.y),
                                               csub(bv, v)));
          y[idx] = zv;
          if (MODE == kSmoothDot) {
            part[2 * c] += bv.x * zv.x - bv.y * zv.y;
            part[2 * c + 1] += bv.x * zv.y + bv.y * zv.x;
          }
        }
      }
    }
  }
  if (NVL0 == 0) return;
  double bsum[NV];
  block_sum_slots<NVL, CLN>(part, smem, bsum);
  if (threadIdx.x == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) ctl.partial[(size_t)blockIdx.x * NV + j] = bsum[j];
  if (!last_block(ctl.counter)) return;
  double tot[NV];
  reduce_partials<NV>(ctl.partial, tot, smem);
  if (threadIdx.x == 0) {
    if (ctl.red) {
#pragma unroll
      for (int j = 0; j < NV; ++j) ctl.red[j] = tot[j];
    } else if (MODE == kCocg) {
      fin_alpha<K>(ctl, tot);
    } else if (MODE == kSmoothDot) {
      fin_rho<K>(ctl, tot);
    } else {
      fin_resid<K>(ctl, tot);
    }
    *ctl.counter = 0u;
  }
}

// ---- SELL-C-sigma SpMV (configs[2]'s storage comparison) -------------------------
// Rows sorted by length (descending) inside windows of sigma rows, then cut
// into chunks of C = 32 rows (one warp); a chunk stores its entries column-
// major and padded to the chunk's widest row, so entry j of the 32 rows is one
// contiguous 512-byte (values) + 128-byte (columns) access. Same 20 B per
// stored entry as CSR plus padding; slot -> row permutation applied on write.
constexpr int kSellC = 32;

template <int K, int MODE>
__global__ void __launch_bounds__(kBlock)
k_sell_spmv(int64_t n_chunks, const int* __restrict__ off, const int* __restrict__ perm,
            const int* __restrict__ scol, const double2* __restrict__ sval,
            const double2* __restrict__ x, double2* __restrict__ y, const double2* __restrict__ b,
            KrylovCtl ctl) {
  constexpr int NV0 = mode_nv(MODE, K), NV = NV0 > 0 ? NV0 : 1;
  __shared__ double smem[32 * NV];
  if (MODE != kPlain && *ctl.n_active == 0) return;
  bool act[K];
#pragma unroll
  for (int k = 0; k < K; ++k) act[k] = (MODE == kPlain) || ctl.st[k].status == kActive;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double part[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) part[j] = 0.0;
  for (int64_t c = warp; c < n_chunks; c += n_warps) {
    const int o0 = off[c], w = (off[c + 1] - o0) / kSellC;
    const int row = perm[c * kSellC + lane];
    double2 acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = make_double2(0.0, 0.0);
#pragma unroll 4
    for (int j = 0; j < w; ++j) {
      const int e = o0 + j * kSellC + lane;
      const int jc = ldg_i(scol + e);
      const double2 a = ldg2(sval + e);
      double2 xv[K];
      load_xk<K>(x + (int64_t)jc * K, xv);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        acc[k].x += a.x * xv[k].x - a.y * xv[k].y;
        acc[k].y += a.x * xv[k].y + a.y * xv[k].x;
      }
    }
    if (row >= 0) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (!act[k]) continue;
        const int64_t idx = (int64_t)row * K + k;
        if (MODE == kPlain) {
          y[idx] = acc[k];
        } else if (MODE == kCocg) {
          y[idx] = acc[k];
          const double2 pv = x[idx];
          part[2 * k] += pv.x * acc[k].x - pv.y * acc[k].y;
          part[2 * k + 1] += pv.x * acc[k].y + pv.y * acc[k].x;
        } else if (MODE == kResid) {
          const double2 rv = csub(b[idx], acc[k]);
          y[idx] = rv;
          part[k] += rv.x * rv.x + rv.y * rv.y;
        } else if (MODE == kResidNR) {
          y[idx] = csub(b[idx], acc[k]);
        } else {
          const double2 bv = b[idx];
          const double2 zv = cadd(x[idx], cmul(make_double2(ctl.omega * ctl.dinv[row].x,
                                                            ctl.omega * ctl.dinv[row].y),
                                               csub(bv, acc[k])));
          y[idx] = zv;
          if (MODE == kSmoothDot) {
            part[2 * k] += bv.x * zv.x - bv.y * zv.y;
            part[2 * k + 1] += bv.x * zv.y + bv.y * zv.x;
          }
        }
      }
    }
  }
  if (NV0 == 0) return;
  block_sum<NV>(part, smem);
  if (threadIdx.x == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) ctl.partial[(size_t)blockIdx.x * NV + j] = part[j];
  if (!last_block(ctl.counter)) return;
  double tot[NV];
  reduce_partials<NV>(ctl.partial, tot, smem);
  if (threadIdx.x == 0) {
    if (ctl.red) {
#pragma unroll
      for (int j = 0; j < NV; ++j) ctl.red[j] = tot[j];
    } else if (MODE == kCocg) {
      fin_alpha<K>(ctl, tot);
    } else {
      fin_resid<K>(ctl, tot);
    }
    *ctl.counter = 0u;
  }
}

__global__ void k_sell_lens(int64_t n, const int* __restrict__ row_ptr, int* __restrict__ len,
                            int* __restrict__ idx, int64_t n_pad) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_pad;
       r += (int64_t)gridDim.x * blockDim.x) {
    len[r] = r < n ? row_ptr[r + 1] - row_ptr[r] : 0;
    idx[r] = r < n ? (int)r : -1;
  }
}

// chunk width = longest row of the chunk (rows are sorted inside sigma windows)
__global__ void k_sell_width(int64_t n_chunks, const int* __restrict__ slen, int* __restrict__ w) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_chunks;
       c += (int64_t)gridDim.x * blockDim.x) {
    int m = 0;
    for (int l = 0; l < kSellC; ++l) m = max(m, slen[c * kSellC + l]);
    w[c] = kSellC * m;
  }
}

__global__ void k_sell_fill(int64_t n_slots, const int* __restrict__ perm,
                            const int* __restrict__ off, const int* __restrict__ row_ptr,
                            const int* __restrict__ col, const double2* __restrict__ val,
                            int* __restrict__ scol, double2* __restrict__ sval) {
  for (int64_t sl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sl < n_slots;
       sl += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = sl / kSellC;
    const int lane = (int)(sl % kSellC);
    const int o0 = off[c], w = (off[c + 1] - o0) / kSellC;
    const int r = perm[sl];
    const int beg = r >= 0 ? row_ptr[r] : 0, len = r >= 0 ? row_ptr[r + 1] - beg : 0;
    const int pad_col = len > 0 ? col[beg + len - 1] : 0;
    for (int j = 0; j < w; ++j) {
      const int64_t e = o0 + (int64_t)j * kSellC + lane;
      if (j < len) {
        scol[e] = col[beg + j];
        sval[e] = val[beg + j];
      } else {
        scol[e] = pad_col;  // stays in the row's own x neighbourhood
        sval[e] = make_double2(0.0, 0.0);
      }
    }
  }
}

// G lanes per node = GB block lanes x CL column lanes. Block lane bl streams
// the node's blocks bl, bl + GB, ...; column lane cl computes the KL = K / CL
// right-hand sides [cl KL, (cl + 1) KL). CL > 1 keeps the per-lane state of a
// narrow batch for a wide one (the CL lanes of one block load the same
// addresses in the same instruction: one request), so wide batches keep the
// software pipeline and 128-register occupancy instead of spilling.
// NB SpMV over the sliced-ELL block layout (NB-E): chunks of 32 nodes,
// block j of the chunk's nodes stored contiguously (1 KB per plane), padded to
// the chunk's largest degree with zero blocks. A warp's block loads are
// contiguous runs instead of 16-32 scattered 64-byte pieces.
//
// FLAT (wide batches, G == CL: one block lane per node): the NPW nodes of a
// warp lie in one 32-node chunk, so the block loop runs the chunk's width for
// every lane, unpredicated (padding slots are zero blocks); only the column
// index is fetched one step ahead, and a step issues its three block planes
// and its x gathers together. Without the register copy of a pipelined block
// the kernel keeps ~108 registers and its loads per step stay at the L1
// writeback floor (every 256-bit load writes 1 KB per warp into registers:
// 128 B per clock per SM bounds this kernel, not DRAM; ncu r02).
template <int G, int K, int MODE, int MINB, int CL, int PFD = 0, int BLOCK = kBlock,
          bool FLAT = false>
__global__ void __launch_bounds__(BLOCK, MINB)
k_nbe_spmv(NbView A, const double2* __restrict__ x, double2* __restrict__ y,
          const double2* __restrict__ b, KrylovCtl ctl) {
  static_assert(G % CL == 0 && K % CL == 0, "lane split");
  static_assert(!FLAT || G == CL, "the flat loop has one block lane per node");
  constexpr int GB = G / CL;   // block lanes per node
  constexpr int KL = K / CL;   // right-hand sides per lane
  constexpr int NVL0 = mode_nv(MODE, KL), NVL = NVL0 > 0 ? NVL0 : 1;  // per lane
  constexpr int NV = NVL * CL;
  __shared__ double smem[32 * NV];
  if (MODE != kPlain && *ctl.n_active == 0) return;
  constexpr int NPW = 32 / G;  // nodes per warp and pass
  const int lane = threadIdx.x & 31;
  const int g = lane & (G - 1);
  const int bl = g / CL, cl = g % CL;
  const int kc = cl * KL;      // first column of this lane
  // every column is computed (no per-column predicates in the block loop):
  // frozen columns' outputs are scratch and their partial sums are ignored by
  // the finalisations, which only touch active columns
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t na = A.na;
  double part[NVL];  // this lane's columns [kc, kc + KL)
#pragma unroll
  for (int j = 0; j < NVL; ++j) part[j] = 0.0;

  const int64_t w0 = A.node_begin & ~(int64_t)(NPW - 1);  // warps stay chunk-aligned
  for (int64_t wn = w0 + warp * NPW; wn < A.n_nodes; wn += n_warps * NPW) {
    const int64_t i = wn + lane / G;
    const bool valid = i >= A.node_begin && i < A.n_nodes;
    double2 acc[3][KL], accv[KL];
#pragma unroll
    for (int k = 0; k < KL; ++k) {
      acc[0][k] = acc[1][k] = acc[2][k] = accv[k] = make_double2(0.0, 0.0);
    }
    int cf_i = -1;
    if constexpr (FLAT) {
      const int c32 = (int)(wn >> 5);
      const int o32 = A.e_off[c32];
      const int w32 = (A.e_off[c32 + 1] - o32) >> 5;
      const int sbase = o32 + (int)(i & 31);
      constexpr int LINES = NPW >= 4 ? NPW / 4 : 1;  // 128-B lines per plane row of the warp
      const char* pf = nullptr;
      int pf_stride = 0;
      if constexpr (PFD > 0) {
        if (lane < 3 * LINES) {
          pf = reinterpret_cast<const char*>(A.blk + 4 * ((int64_t)(lane / LINES) * A.nblk + o32 +
                                                          (int)(wn & 31)) +
                                             16 * (lane % LINES));
          pf_stride = 32 * 32;
        } else if (lane == 3 * LINES) {
          pf = reinterpret_cast<const char*>(A.blk_col + o32 + (int)(wn & 31));
          pf_stride = 32 * 4;
        }
      }
      int m = ldg_i(A.blk_col + sbase);
      for (int j = 0; j < w32; ++j) {
        if constexpr (PFD > 0) {
          if (pf && j + PFD < w32)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pf + (int64_t)(j + PFD) * pf_stride));
        }
        const int q = sbase + 32 * j;
        double B[3][3], Im[3];
        load_block(A, q, B, Im);
        const double2* xm = x + (int64_t)3 * m * K + kc;
        double2 xp[3][KL];
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int k = 0; k < KL; k += 2) ld4x(xm + d * K + k, xp[d][k], xp[d][k + 1]);
        if (j + 1 < w32) m = ldg_i(A.blk_col + q + 32);
#pragma unroll
        for (int k = 0; k < KL; ++k)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            double2 s = acc[c][k];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              s.x += B[c][d] * xp[d][k].x;
              s.y += B[c][d] * xp[d][k].y;
            }
            s.x -= Im[c] * xp[c][k].y;
            s.y += Im[c] * xp[c][k].x;
            acc[c][k] = s;
          }
      }
    }
    if (valid) {
      // sliced-ELL blocks: block j of node i at slot off[c] + 32 j + (i mod 32)
      const int c32 = (int)(i >> 5);
      const int o32 = A.e_off[c32];
      const int w32 = (A.e_off[c32 + 1] - o32) >> 5;
      const int sbase = o32 + (int)(i & 31);
      const int be = sbase + 32 * w32;
      constexpr int GS = 32 * GB;  // slot stride between a lane's blocks
      int q = sbase + 32 * bl;
      int m_nx = 0;
      double B_nx[3][3], Im_nx[3];
      if (!FLAT && q < be) {
        m_nx = ldg_i(A.blk_col + q);
        load_block(A, q, B_nx, Im_nx);
      }
      // (wide per-lane batches keep the accumulators instead)
      constexpr bool kPipe = KL <= 2 && MINB <= 2;
      // L2 prefetch of the warp's block rows PFD steps ahead: the DRAM latency
      // of the matrix stream is covered without holding registers. Lanes
      // 0 .. 3 LINES - 1 own one 128-B line of a plane row, lane 3 LINES the
      // column row; the line address of row r is pf + r * stride.
      constexpr int LINES = NPW >= 4 ? NPW / 4 : 1;  // 128-B lines per plane row
      const char* pf = nullptr;
      int pf_stride = 0;
      if constexpr (PFD > 0) {
        if (lane < 3 * LINES) {
          pf = reinterpret_cast<const char*>(A.blk + 4 * ((int64_t)(lane / LINES) * A.nblk + o32 +
                                                          (int)(wn & 31)) +
                                             16 * (lane % LINES));
          pf_stride = 32 * 32;  // 32 slots x 4 doubles
        } else if (lane == 3 * LINES) {
          pf = reinterpret_cast<const char*>(A.blk_col + o32 + (int)(wn & 31));
          pf_stride = 32 * 4;
        }
      }
      for (; !FLAT && q < be; q += GS) {
        if constexpr (PFD > 0) {
          const int row0 = ((q - sbase) >> 5) - bl + PFD * GB;
          if (pf) {
#pragma unroll
            for (int gb = 0; gb < GB; ++gb)
              if (row0 + gb < w32)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pf + (int64_t)(row0 + gb) * pf_stride));
          }
        }
        int m = m_nx;
        double B[3][3], Im[3];
        if constexpr (kPipe) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            Im[c] = Im_nx[c];
#pragma unroll
            for (int d = 0; d < 3; ++d) B[c][d] = B_nx[c][d];
          }
          if (q + GS < be) {
            m_nx = ldg_i(A.blk_col + q + GS);
            load_block(A, q + GS, B_nx, Im_nx);
          }
        } else {
          if (q != sbase + 32 * bl) {
            m = ldg_i(A.blk_col + q);
            load_block(A, q, B, Im);
          } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              Im[c] = Im_nx[c];
#pragma unroll
              for (int d = 0; d < 3; ++d) B[c][d] = B_nx[c][d];
            }
          }
        }
        const double2* xm = x + (int64_t)3 * m * K + kc;
        // right-hand sides in pairs: one 256-bit gather per (component, pair)
        constexpr int KP = (KL % 2 == 0) ? 2 : 1;
#pragma unroll
        for (int k0 = 0; k0 < KL; k0 += KP) {
          double2 xp[3][KP];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            if constexpr (KP == 2) ld4x(xm + d * K + k0, xp[d][0], xp[d][1]);
            else xp[d][0] = __ldg(xm + d * K + k0);
          }
#pragma unroll
          for (int kk = 0; kk < KP; ++kk) {
            const int k = k0 + kk;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              double2 s = acc[c][k];
#pragma unroll
              for (int d = 0; d < 3; ++d) {
                s.x += B[c][d] * xp[d][kk].x;
                s.y += B[c][d] * xp[d][kk].y;
              }
              s.x -= Im[c] * xp[c][kk].y;
              s.y += Im[c] * xp[c][kk].x;
              acc[c][k] = s;
            }
          }
        }
      }
      cf_i = A.cond_fwd[i];
      if (cf_i >= 0) {
        const int ce = A.cpl_ptr[i + 1];
        for (int q = A.cpl_ptr[i] + bl; q < ce; q += GB) {
          const int2 mi = ldg_i2(A.cpl_idx + q);
          double av[3], va[3];
          double2 Q3;
          load_cpl(A, q, av, va, Q3);
          const double2* xm = x + (int64_t)3 * mi.x * K + kc;
          const double2* xvp = x + (na + mi.y) * K + kc;
          constexpr int KP = (KL % 2 == 0) ? 2 : 1;
#pragma unroll
          for (int k0 = 0; k0 < KL; k0 += KP) {
            double2 xa[3][KP], xv[KP];
            if constexpr (KP == 2) {
              ld4x(xvp + k0, xv[0], xv[1]);
#pragma unroll
              for (int d = 0; d < 3; ++d) ld4x(xm + d * K + k0, xa[d][0], xa[d][1]);
            } else {
              xv[0] = __ldg(xvp + k0);
#pragma unroll
              for (int d = 0; d < 3; ++d) xa[d][0] = __ldg(xm + d * K + k0);
            }
#pragma unroll
            for (int kk = 0; kk < KP; ++kk) {
              const int k = k0 + kk;
              const double2 v = xv[kk];
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                acc[c][k].x += av[c] * v.x;
                acc[c][k].y += av[c] * v.y;
              }
              double2 s = accv[k];
#pragma unroll
              for (int d = 0; d < 3; ++d) {
                s.x += va[d] * xa[d][kk].x;
                s.y += va[d] * xa[d][kk].y;
              }
              s.x += Q3.x * v.x - Q3.y * v.y;
              s.y += Q3.x * v.y + Q3.y * v.x;
              accv[k] = s;
            }
          }
        }
      }
    }
    // segment reduction over the GB block lanes of a node (same column lane)
#pragma unroll
    for (int k = 0; k < KL; ++k) {
#pragma unroll
      for (int o = (GB / 2) * CL; o >= CL; o >>= 1) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          acc[c][k].x += __shfl_xor_sync(0xffffffffu, acc[c][k].x, o, G);
          acc[c][k].y += __shfl_xor_sync(0xffffffffu, acc[c][k].y, o, G);
        }
        accv[k].x += __shfl_xor_sync(0xffffffffu, accv[k].x, o, G);
        accv[k].y += __shfl_xor_sync(0xffffffffu, accv[k].y, o, G);
      }
    }
    if (bl == 0 && valid) {
#pragma unroll
      for (int k = 0; k < KL; ++k) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c == 3 && cf_i < 0) break;
          const int64_t row = c < 3 ? 3 * i + c : na + cf_i;
          const double2 v = c < 3 ? acc[c][k] : accv[k];
          const int64_t idx = row * K + kc + k;
          if (MODE == kPlain) {
            y[idx] = v;
          } else if (MODE == kCocg) {
            y[idx] = v;
            const double2 pv = x[idx];
            part[2 * k] += pv.x * v.x - pv.y * v.y;
            part[2 * k + 1] += pv.x * v.y + pv.y * v.x;
          } else if (MODE == kResid) {
            const double2 rv = csub(b[idx], v);
            y[idx] = rv;
            part[k] += rv.x * rv.x + rv.y * rv.y;
          } else if (MODE == kResidNR) {
            y[idx] = csub(b[idx], v);
          } else if (MODE == kCgDot) {
            y[idx] = v;
            const double2 zz = x[idx], rr = b[idx];
            part[5 * k] += rr.x * zz.x - rr.y * zz.y;
            part[5 * k + 1] += rr.x * zz.y + rr.y * zz.x;
            part[5 * k + 2] += v.x * zz.x - v.y * zz.y;
            part[5 * k + 3] += v.x * zz.y + v.y * zz.x;
            part[5 * k + 4] += rr.x * rr.x + rr.y * rr.y;
          } else {
            const double2 bv = b[idx];
            const double2 d = ctl.dinv[row];
            const double2 zv = cadd(x[idx], cmul(make_double2(ctl.omega * d.x, ctl.omega * d.y),
                                                 csub(bv, v)));
            y[idx] = zv;
            if (MODE == kSmoothDot) {
              part[2 * k] += bv.x * zv.x - bv.y * zv.y;
              part[2 * k + 1] += bv.x * zv.y + bv.y * zv.x;
            }
          }
        }
      }
    }
  }
  if (NVL0 == 0) return;

  // per-block totals, column-major over the lanes' slots = global column order
  double bsum[NV];
  block_sum_slots<NVL, CL>(part, smem, bsum);
  if (threadIdx.x == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) ctl.partial[(size_t)blockIdx.x * NV + j] = bsum[j];
  if (!last_block(ctl.counter)) return;
  double tot[NV];
  reduce_partials<NV>(ctl.partial, tot, smem);
  if (threadIdx.x == 0) {
    if (ctl.red) {
#pragma unroll
      for (int j = 0; j < NV; ++j) ctl.red[j] = ctl.red_add ? ctl.red[j] + tot[j] : tot[j];
    } else if (MODE == kCocg) {
      fin_alpha<K>(ctl, tot);
    } else if (MODE == kSmoothDot) {
      fin_rho<K>(ctl, tot);
    } else {
      fin_resid<K>(ctl, tot);
    }
    *ctl.counter = 0u;
  }
}

// CSR (assembled, node-structured) -> NB planes. Warp per node; lane = block.
__global__ void k_build_nb(const int* __restrict__ row_ptr, const double2* __restrict__ val,
                           const int* __restrict__ nbr_off, const int* __restrict__ nbr,
                           const uint8_t* __restrict__ nbr_cond, const int* __restrict__ cond_fwd,
                           const int* __restrict__ cpl_ptr, int64_t n_nodes, double* blk,
                           int64_t nblk, int2* cpl_idx, double* cpl, int64_t ncpl, int* bad,
                           int64_t lo, int64_t hi, int64_t blk_base, int64_t cpl_base) {
  // nodes [lo, hi); block q / coupling p stored at q - blk_base / p - cpl_base
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t na = 3 * n_nodes;
  for (int64_t i = lo + warp; i < hi; i += n_warps) {
    const int nb = nbr_off[i], u = nbr_off[i + 1] - nb;
    const int cf_i = cond_fwd[i];
    int ncc = 0;
    for (int r0 = 0; r0 < u; r0 += 32) {
      bool c = (r0 + lane < u) && nbr_cond[nb + r0 + lane];
      ncc += __popc(__ballot_sync(0xffffffffu, c));
    }
    const int base[3] = {row_ptr[3 * i], row_ptr[3 * i + 1], row_ptr[3 * i + 2]};
    const int basev = cf_i >= 0 ? row_ptr[na + cf_i] : 0;
    const int cb = cpl_ptr[i];
    int rc0 = 0;
    for (int r0 = 0; r0 < u; r0 += 32) {
      const int r = r0 + lane;
      const bool valid = r < u;
      const bool mc = valid && nbr_cond[nb + r];
      const unsigned mask = __ballot_sync(0xffffffffu, mc);
      const int rc = rc0 + __popc(mask & ((1u << lane) - 1u));
      rc0 += __popc(mask);
      if (!valid) continue;
      double Bv[3][3], Im[3];
      int nonzero_offdiag_im = 0;
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double2 v = val[base[c] + 3 * r + d];
          Bv[c][d] = v.x;
          if (c == d) Im[c] = v.y; else nonzero_offdiag_im |= v.y != 0.0;
        }
      const int64_t q = nb + r - blk_base;
      const double w0[4] = {Bv[0][0], Bv[0][1], Bv[0][2], Bv[1][0]};
      const double w1[4] = {Bv[1][1], Bv[1][2], Bv[2][0], Bv[2][1]};
      const double w2[4] = {Bv[2][2], Im[0], Im[1], Im[2]};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        blk[4 * q + e] = w0[e];
        blk[4 * (nblk + q) + e] = w1[e];
        blk[4 * (2 * nblk + q) + e] = w2[e];
      }
      if (mc) {
        const int m = nbr[nb + r];
        const int64_t p = cb + rc - cpl_base;
        double av[3], va[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double2 v = val[base[c] + 3 * u + rc];
          av[c] = v.x;
          nonzero_offdiag_im |= v.y != 0.0;
        }
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double2 v = val[basev + 3 * rc + d];
          va[d] = v.x;
          nonzero_offdiag_im |= v.y != 0.0;
        }
        const double2 vv = val[basev + 3 * ncc + rc];
        cpl_idx[p] = make_int2(m, cond_fwd[m]);
        const double c0[4] = {av[0], av[1], av[2], va[0]};
        const double c1[4] = {va[1], va[2], vv.x, vv.y};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          cpl[4 * p + e] = c0[e];
          cpl[4 * (ncpl + p) + e] = c1[e];
        }
      }
      if (nonzero_offdiag_im) atomicOr(bad, 1);
    }
  }
}

// NB-E build: chunk widths (32 x the chunk's largest node degree) and the
// slot-major copy of the NB planes / columns with zero padding blocks.
__global__ void k_nbe_width(const int* __restrict__ blk_ptr, int64_t n_nodes, int64_t n_chunks,
                            int* __restrict__ w) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_chunks;
       c += (int64_t)gridDim.x * blockDim.x) {
    int m = 0;
    for (int64_t i = 32 * c; i < 32 * c + 32 && i < n_nodes; ++i) m = max(m, blk_ptr[i + 1] - blk_ptr[i]);
    w[c] = 32 * m;
  }
}
__global__ void k_nbe_fill(const int* __restrict__ blk_ptr, const int* __restrict__ blk_col,
                           const double* __restrict__ blk, int64_t nblk, int64_t n_nodes,
                           int64_t n_chunks, const int* __restrict__ off, int* __restrict__ ecol,
                           double* __restrict__ eblk, int64_t nslots) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 32 * n_chunks;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t >> 5, i = t;
    const int l = (int)(t & 31);
    const int o = off[c], w = (off[c + 1] - o) >> 5;
    const int q0 = i < n_nodes ? blk_ptr[i] : 0, deg = i < n_nodes ? blk_ptr[i + 1] - q0 : 0;
    for (int j = 0; j < w; ++j) {
      const int64_t sl = o + 32 * (int64_t)j + l;
      const bool real = j < deg;
      ecol[sl] = real ? blk_col[q0 + j] : (i < n_nodes ? (int)i : 0);
#pragma unroll
      for (int pl = 0; pl < 3; ++pl)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          eblk[4 * (pl * nslots + sl) + e] = real ? blk[4 * (pl * nblk + q0 + j) + e] : 0.0;
    }
  }
}

// A part's NB-E slots straight from the global NB-E: local node il = global
// n0 + il, its block j read from the global slot of (n0 + il, j), columns
// mapped global -> local (g2l); padding slots are zero blocks on the node itself.
__global__ void k_part_nbe_fill(const int* __restrict__ lptr, int64_t L, int64_t n0,
                                const int* __restrict__ goff, const int* __restrict__ gcol,
                                const double* __restrict__ gblk, int64_t gslots,
                                const int* __restrict__ g2l, const int* __restrict__ loff,
                                int64_t n_chunks, int* __restrict__ lcol,
                                double* __restrict__ lblk, int64_t lslots) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 32 * n_chunks;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t >> 5, il = t;
    const int l = (int)(t & 31);
    const int o = loff[c], w = (loff[c + 1] - o) >> 5;
    const bool node = il < L;
    const int deg = node ? lptr[il + 1] - lptr[il] : 0;
    const int64_t i = n0 + il;
    const int64_t gs0 = node ? goff[i >> 5] + (i & 31) : 0;
    for (int j = 0; j < w; ++j) {
      const int64_t sl = o + 32 * (int64_t)j + l;
      const bool real = j < deg;
      const int64_t gs = gs0 + 32 * (int64_t)j;
      lcol[sl] = real ? g2l[gcol[gs]] : (node ? (int)il : 0);
#pragma unroll
      for (int pl = 0; pl < 3; ++pl)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          lblk[4 * (pl * lslots + sl) + e] = real ? gblk[4 * (pl * gslots + gs) + e] : 0.0;
    }
  }
}

__global__ void k_cpl_count(const int* __restrict__ nbr_off, const uint8_t* __restrict__ nbr_cond,
                            const int* __restrict__ cond_fwd, int64_t lo, int64_t hi, int* cnt) {
  for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = 0;
    if (cond_fwd[i] >= 0)
      for (int p = nbr_off[i]; p < nbr_off[i + 1]; ++p) c += nbr_cond[p];
    cnt[i] = c;
  }
}

// Vector kernels: a thread owns CW = min(K, 2) adjacent right-hand sides of
// one row (32 contiguous bytes per vector: a warp touches 1 KB runs), KH =
// K / CW threads share a row; the thread's column slot h = lane % KH is fixed
// because the grid stride is a multiple of KH.
template <int K>
struct VecMap {
  static constexpr int CW = K >= 2 ? 2 : 1;
  static constexpr int KH = K / CW;
};

// r -= alpha q ; z = D^-1 r ; partial r^T z, ||r||^2
// last block: convergence test, beta, rho. The iteration's x += alpha p is
// deferred to k_pupdate, which reads p anyway (x and p travel once, not twice).
// EXT (external preconditioner, multigrid): partial ||r||^2 only; rho and beta
// come from the preconditioner's last kernel (kSmoothDot).
template <int K, bool EXT = false>
__global__ void __launch_bounds__(kBlock)
k_update(int64_t n, double2* __restrict__ r, const double2* __restrict__ q,
         const double2* __restrict__ dinv, KrylovCtl ctl, double2* __restrict__ xt = nullptr,
         double omega = 0.0, float2* __restrict__ xt32 = nullptr) {
  constexpr int CW = VecMap<K>::CW, KH = VecMap<K>::KH;
  constexpr int PV = EXT ? 1 : 3;  // values per column
  constexpr int NVL = PV * CW, NV = PV * K;
  __shared__ double smem[32 * NV];
  if (*ctl.n_active == 0) return;
  const int h = (threadIdx.x & 31) % KH, kb = h * CW;
  bool act[CW];
  double2 alpha[CW];
#pragma unroll
  for (int c = 0; c < CW; ++c) {
    act[c] = ctl.st[kb + c].status == kActive;
    alpha[c] = ctl.st[kb + c].alpha;
  }
  double part[NVL];
#pragma unroll
  for (int j = 0; j < NVL; ++j) part[j] = 0.0;
  const int64_t len0 = ctl.e0 - ctl.s0, rows = len0 + (ctl.e1 - ctl.s1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * KH;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / KH;
    const int64_t i = j < len0 ? ctl.s0 + j : ctl.s1 + (j - len0);  // owned rows
    const double2 d = (EXT && !xt && !xt32) ? make_double2(0.0, 0.0) : dinv[i];
#pragma unroll
    for (int c = 0; c < CW; ++c) {
      if (!act[c]) continue;
      const int64_t idx = i * K + kb + c;
      const double2 rv = csub(r[idx], cmul(alpha[c], q[idx]));
      r[idx] = rv;
      if constexpr (EXT) {
        part[c] += rv.x * rv.x + rv.y * rv.y;
        // the multigrid cycle's first step on the finest level, x = omega D^-1 r
        if (xt) xt[idx] = cmul(make_double2(omega * d.x, omega * d.y), rv);
        if (xt32) put(xt32 + idx, cmul(make_double2(omega * d.x, omega * d.y), rv));
      } else {
        const double2 z = cmul(d, rv);
        part[3 * c] += rv.x * z.x - rv.y * z.y;
        part[3 * c + 1] += rv.x * z.y + rv.y * z.x;
        part[3 * c + 2] += rv.x * rv.x + rv.y * rv.y;
      }
    }
  }
  double bsum[NV];
  block_sum_slots<NVL, KH>(part, smem, bsum);
  if (threadIdx.x == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) ctl.partial[(size_t)blockIdx.x * NV + j] = bsum[j];
  if (!last_block(ctl.counter)) return;
  double tot[NV];
  reduce_partials<NV>(ctl.partial, tot, smem);
  if (threadIdx.x == 0) {
    if (ctl.red) {
#pragma unroll
      for (int j = 0; j < NV; ++j) ctl.red[j] = tot[j];
    } else if (EXT) {
      fin_update_norm<K>(ctl, tot);
    } else {
      fin_update<K>(ctl, tot);
    }
    *ctl.counter = 0u;
  }
}

// x += alpha p (owed by the last k_update) ; p = z + beta p (active columns),
// z = D^-1 r (Jacobi) or the preconditioner's output zv (EXT)
template <int K, bool EXT = false>
__global__ void __launch_bounds__(kBlock)
k_pupdate(int64_t n, double2* __restrict__ x, const double2* __restrict__ r,
          double2* __restrict__ p, const double2* __restrict__ dinv, KrylovCtl ctl,
          const double2* __restrict__ zv = nullptr) {
  constexpr int CW = VecMap<K>::CW, KH = VecMap<K>::KH;
  bool any = *ctl.n_active != 0;
#pragma unroll
  for (int c = 0; c < K; ++c) any |= ctl.st[c].xpend != 0;
  if (!any) return;
  const int h = (threadIdx.x & 31) % KH, kb = h * CW;
  bool act[CW], xp[CW];
  double2 alpha[CW], beta[CW];
#pragma unroll
  for (int c = 0; c < CW; ++c) {
    const RhsState& st = ctl.st[kb + c];
    act[c] = st.status == kActive;
    xp[c] = st.xpend != 0;
    alpha[c] = st.alpha;
    beta[c] = st.beta;
  }
  const int64_t len0 = ctl.e0 - ctl.s0, rows = len0 + (ctl.e1 - ctl.s1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * KH;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / KH;
    const int64_t i = j < len0 ? ctl.s0 + j : ctl.s1 + (j - len0);  // owned rows
    const double2 d = EXT ? make_double2(0.0, 0.0) : dinv[i];
#pragma unroll
    for (int c = 0; c < CW; ++c) {
      if (!act[c] && !xp[c]) continue;
      const int64_t idx = i * K + kb + c;
      const double2 pv = p[idx];
      if (xp[c]) x[idx] = cadd(x[idx], cmul(alpha[c], pv));
      if (act[c]) p[idx] = cadd(EXT ? zv[idx] : cmul(d, r[idx]), cmul(beta[c], pv));
    }
  }
  // the owed updates are done: clear the flags (after every block read them)
  if (!last_block(ctl.counter)) return;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < K; ++c) ctl.st[c].xpend = 0;
    *ctl.counter = 0u;
  }
}

// (Re)start selected columns from their residual r: p = D^-1 r, rho = r^T z,
// ||r||; on a fresh start also x = 0, r = b and bnorm = ||b||.
// mask bit k set -> (re)start column k. EXT: norms only (p and rho come from
// the preconditioner applied next).
template <int K, bool EXT = false>
__global__ void __launch_bounds__(kBlock)
k_start(int64_t n, const double2* __restrict__ b, double2* __restrict__ x, double2* __restrict__ r,
        double2* __restrict__ p, const double2* __restrict__ dinv, unsigned mask, int fresh,
        KrylovCtl ctl) {
  constexpr int CW = VecMap<K>::CW, KH = VecMap<K>::KH;
  constexpr int PV = EXT ? 2 : 4;
  constexpr int NVL = PV * CW, NV = PV * K;
  __shared__ double smem[32 * NV];
  const int h = (threadIdx.x & 31) % KH, kb = h * CW;
  double part[NVL];
#pragma unroll
  for (int j = 0; j < NVL; ++j) part[j] = 0.0;
  const int64_t len0 = ctl.e0 - ctl.s0, rows = len0 + (ctl.e1 - ctl.s1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * KH;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / KH;
    const int64_t i = j < len0 ? ctl.s0 + j : ctl.s1 + (j - len0);  // owned rows
    const double2 d = EXT ? make_double2(0.0, 0.0) : dinv[i];
#pragma unroll
    for (int c = 0; c < CW; ++c) {
      if (!((mask >> (kb + c)) & 1u)) continue;
      const int64_t idx = i * K + kb + c;
      double2 rv;
      if (fresh) {
        rv = b[idx];
        x[idx] = make_double2(0.0, 0.0);
        r[idx] = rv;
        part[PV * c + PV - 1] += rv.x * rv.x + rv.y * rv.y;
      } else {
        rv = r[idx];
      }
      if constexpr (EXT) {
        part[2 * c] += rv.x * rv.x + rv.y * rv.y;
      } else {
        const double2 z = cmul(d, rv);
        p[idx] = z;
        part[4 * c] += rv.x * z.x - rv.y * z.y;
        part[4 * c + 1] += rv.x * z.y + rv.y * z.x;
        part[4 * c + 2] += rv.x * rv.x + rv.y * rv.y;
      }
    }
  }
  double bsum[NV];
  block_sum_slots<NVL, KH>(part, smem, bsum);
  if (threadIdx.x == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) ctl.partial[(size_t)blockIdx.x * NV + j] = bsum[j];
  if (!last_block(ctl.counter)) return;
  double tot[NV];
  reduce_partials<NV>(ctl.partial, tot, smem);
  if (threadIdx.x == 0) {
    if (ctl.red) {
#pragma unroll
      for (int j = 0; j < NV; ++j) ctl.red[j] = tot[j];
    } else if (EXT) {
      fin_start_norm<K>(ctl, tot, mask, fresh);
    } else {
      fin_start<K>(ctl, tot, mask, fresh);
    }
    *ctl.counter = 0u;
  }
}

__global__ void k_jacobi(int64_t n, const int* __restrict__ row_ptr, const int* __restrict__ col,
                         const double2* __restrict__ val, double2* dinv, int* missing) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int lo = row_ptr[i], hi = row_ptr[i + 1] - 1;
    int pos = -1;
    while (lo <= hi) {
      int mid = lo + ((hi - lo) >> 1);  // no int overflow at nnz > 2^30
      int c = col[mid];
      if (c == i) { pos = mid; break; }
      if (c < i) lo = mid + 1; else hi = mid - 1;
    }
    double2 d = pos >= 0 ? val[pos] : make_double2(0.0, 0.0);
    if (d.x == 0.0 && d.y == 0.0) {
      atomicAdd(missing, 1);
      dinv[i] = make_double2(1.0, 0.0);
    } else {
      dinv[i] = cdiv(make_double2(1.0, 0.0), d);
    }
  }
}

struct Launch {
  int grid_spmv = 0, grid_vec = 0;
};

NbView nb_view(const ect_matrix* a) {
  return NbView{a->nb_blk_ptr, a->nb_blk_col, reinterpret_cast<const double*>(a->nb_blk.p),
                a->nb_blocks, a->nb_cpl_ptr.p, a->nb_cpl_idx.p,
                reinterpret_cast<const double*>(a->nb_cpl.p), a->nb_ncpl, a->nb_cond_fwd,
                a->n_nodes, 3 * a->n_nodes};
}

// Default NB-E launch configuration per batch width (measured on configs[1],
// B200): G lanes per node, CTAs per SM, CL column lanes, L2 prefetch distance.
struct KFn {
  const void* fn;
  int block;  // threads per CTA the kernel is compiled for
};
template <int K, int MODE>
KFn nbe_kernel() {
  if constexpr (K <= 2) return {(const void*)k_nbe_spmv<2, K, MODE, 2, 1, 2>, kBlock};
  else if constexpr (K == 4) return {(const void*)k_nbe_spmv<2, K, MODE, 2, 2, 4>, kBlock};
  else if constexpr (K == 8)  // flat loop, 2 columns per lane (lab: 0.282 vs 0.327 ms)
    return {(const void*)k_nbe_spmv<4, K, MODE, 2, 4, 2, kBlock, true>, kBlock};
  else {
    if constexpr (MODE == kCgDot) return {(const void*)k_nbe_spmv<8, K, MODE, 2, 8>, kBlock};
    else return {(const void*)k_nbe_spmv<8, K, MODE, 2, 8, 2, kBlock, true>, kBlock};
  }
}
template <int K>
KFn nbe_fn(int mode) {
  switch (mode) {
    case kPlain: return nbe_kernel<K, kPlain>();
    case kCocg: return nbe_kernel<K, kCocg>();
    case kResid: return nbe_kernel<K, kResid>();
    case kResidNR: return nbe_kernel<K, kResidNR>();
    case kSmooth: return nbe_kernel<K, kSmooth>();
    case kCgDot: return nbe_kernel<K, kCgDot>();
    default: return nbe_kernel<K, kSmoothDot>();
  }
}
template <int K, int MODE>
const void* csr_kernel() {
  if constexpr (K == 1) return (const void*)k_spmv<16, 1, MODE>;
  else return (const void*)k_spmv_v<K, (K >= 16 ? 1 : 16 / K), MODE>;
}
template <int K>
const void* csr_fn(int mode) {
  switch (mode) {
    case kPlain: return csr_kernel<K, kPlain>();
    case kCocg: return csr_kernel<K, kCocg>();
    case kResid: return csr_kernel<K, kResid>();
    case kResidNR: return csr_kernel<K, kResidNR>();
    case kSmooth: return csr_kernel<K, kSmooth>();
    default: return csr_kernel<K, kSmoothDot>();
  }
}
// lanes per row of the CSR kernel (grid sizing)
template <int K>
constexpr int csr_lanes() { return K == 1 ? 16 : (K / 2) * (K >= 16 ? 1 : 16 / K); }
// Coarse multigrid levels: Galerkin rows are long (60-200 entries) and the
// levels are small, so a whole warp streams one row (32 lanes = K/2 column
// pairs x 64/K entry lanes): the serial chain of dependent column -> gather
// loads per lane is what those launches cost (35 us for a 5k-row level with
// 2 entry lanes, r02 launch list).
template <int K>
const void* csr_row_fn(int mode) {
  if constexpr (K == 1) {
    return mode == kResidNR ? (const void*)k_spmv<32, 1, kResidNR> : (const void*)k_spmv<32, 1, kSmooth>;
  } else {
    constexpr int E = K >= 64 ? 1 : 64 / K;
    return mode == kResidNR ? (const void*)k_spmv_v<K, E, kResidNR>
                            : (const void*)k_spmv_v<K, E, kSmooth>;
  }
}
template <int K>
const void* sell_fn(int mode) {
  return mode == kPlain  ? (const void*)k_sell_spmv<K, kPlain>
         : mode == kCocg ? (const void*)k_sell_spmv<K, kCocg>
                         : (const void*)k_sell_spmv<K, kResid>;
}

// Storage used by the SpMV of a matrix: NB-E when built, else SELL, else CSR.
enum class Store { kNbe, kSell, kCsr };
inline Store store_of(const ect_matrix* a, int mode) {
  if (a->has_nb && a->has_nbe) return Store::kNbe;
  if (a->has_sell && (mode == kPlain || mode == kCocg || mode == kResid)) return Store::kSell;
  return Store::kCsr;
}

template <int K>
struct Dispatch {
  static constexpr int kWidth = K;
  static void spmv(ect_ctx* ctx, int mode, int grid, int64_t n, const ect_matrix* a,
                   const double2* x, double2* y, const double2* b, KrylovCtl ctl) {
    cudaStream_t s = ctx->stream;
    switch (store_of(a, mode)) {
      case Store::kNbe: {
        NbView v = nb_view(a);
        v.blk = reinterpret_cast<const double*>(a->nbe_blk.p);
        v.blk_col = a->nbe_col.p;
        v.nblk = a->nbe_slots;
        v.e_off = a->nbe_off.p;
        void* args[] = {&v, &x, &y, &b, &ctl};
        const KFn f = nbe_fn<K>(mode);
        CK(cudaLaunchKernel(f.fn, dim3(grid), dim3(f.block), args, 0, s));
        return;
      }
      case Store::kSell: {
        const int64_t nc = a->sell_chunks;
        const int* off = a->sell_off.p;
        const int* perm = a->sell_perm.p;
        const int* scol = a->sell_col.p;
        const double2* sval = a->sell_val.p;
        void* args[] = {(void*)&nc, (void*)&off, (void*)&perm, (void*)&scol, (void*)&sval,
                        (void*)&x, (void*)&y, (void*)&b, (void*)&ctl};
        CK(cudaLaunchKernel(sell_fn<K>(mode), dim3(grid), dim3(kBlock), args, 0, s));
        return;
      }
      case Store::kCsr:
        csr(ctx, mode, grid, n, a->row_ptr.p, a->col.p, a->val.p, x, y, b, ctl);
        return;
    }
  }
  // plain complex CSR (also the coarse multigrid levels)
  static void csr(ect_ctx* ctx, int mode, int grid, int64_t n, const int* rp, const int* cl,
                  const double2* vl, const double2* x, double2* y, const double2* b,
                  KrylovCtl ctl, bool warp_per_row = false) {
    void* args[] = {(void*)&n, (void*)&rp, (void*)&cl, (void*)&vl, (void*)&x, (void*)&y,
                    (void*)&b, (void*)&ctl};
    const void* fn = warp_per_row ? csr_row_fn<K>(mode) : csr_fn<K>(mode);
    CK(cudaLaunchKernel(fn, dim3(grid), dim3(kBlock), args, 0, ctx->stream));
  }
  static void update(ect_ctx* ctx, int grid, int64_t n, double2* r, const double2* q,
                     const double2* dinv, KrylovCtl ctl) {
    k_update<K><<<grid, kBlock, 0, ctx->stream>>>(n, r, q, dinv, ctl);
    CK_LAUNCH();
  }
  static void pupdate(ect_ctx* ctx, int grid, int64_t n, double2* x, const double2* r, double2* p,
                      const double2* dinv, KrylovCtl ctl) {
    k_pupdate<K><<<grid, kBlock, 0, ctx->stream>>>(n, x, r, p, dinv, ctl);
    CK_LAUNCH();
  }
  static void start(ect_ctx* ctx, int grid, int64_t n, const double2* b, double2* x, double2* r,
                    double2* p, const double2* dinv, unsigned mask, int fresh, KrylovCtl ctl) {
    k_start<K><<<grid, kBlock, 0, ctx->stream>>>(n, b, x, r, p, dinv, mask, fresh, ctl);
    CK_LAUNCH();
  }
  static int spmv_grid(ect_ctx* ctx, int mode, const ect_matrix* a) {
    switch (store_of(a, mode)) {
      case Store::kNbe: return grid_for(ctx, nbe_fn<K>(mode).fn, nbe_fn<K>(mode).block);
      case Store::kSell: return grid_for(ctx, sell_fn<K>(mode), kBlock);
      default: return grid_for(ctx, csr_fn<K>(mode), kBlock);
    }
  }
  // Grid of the fused vector kernels. Multigrid path (ext): k_update / k_pupdate
  // hold 48 registers, and 4 CTAs per SM run them at 0.15 ms instead of 0.18 ms
  // (k = 8, r02 bench A/B); the Jacobi kernels (100 registers) keep their
  // occupancy-sized grid, where more CTAs measured no gain.
  static int vec_grid(ect_ctx* ctx, bool ext = false) {
    const int base = grid_for(ctx, (const void*)k_update<K>, kBlock);
    if (!ext) return base;
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_update<K, true>, kBlock, 0));
    int per_p = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_p, k_pupdate<K, true>, kBlock, 0));
    return std::max(base, std::min({4, per_sm, per_p}) * ctx->num_sms);
  }
};

// Runs fn with the Dispatch<K> matching k.
template <typename F>
void with_k(int k, F&& fn) {
  switch (k) {
    case 1: fn(Dispatch<1>{}); break;
    case 2: fn(Dispatch<2>{}); break;
    case 4: fn(Dispatch<4>{}); break;
    case 8: fn(Dispatch<8>{}); break;
    case 16: fn(Dispatch<16>{}); break;
    default: fail(ECT_ERR_SOLVER, "unsupported right-hand-side batch width " + std::to_string(k));
  }
}

// kind 0: SpMV launches, kind 1: the fused vector-update launches.
// sampled = true (solver loop): time one launch in kProfStride, so the event
// records do not perturb the timed region; the mean is over the sampled ones.
constexpr int kProfStride = 8;
int prof_stride() {
  static const int stride = [] {
    const char* v = std::getenv("ECT_PROF_STRIDE");  // dev: sample every n-th iteration
    return v ? std::max(1, std::atoi(v)) : kProfStride;
  }();
  return stride;
}
// true when the next solver iteration is one of the profiled samples
bool prof_sample_next(ect_ctx* ctx) {
  return ctx->prof.enabled && (ctx->prof.launches % prof_stride()) == 0;
}
void prof_begin(ect_ctx* ctx, cudaEvent_t* ev, int kind = 0, bool sampled = false,
                const int* n_active = nullptr, int width = 0, int snap = -1) {
  ev[0] = ev[1] = nullptr;
  if (!ctx->prof.enabled) return;
  auto& P = ctx->prof;
  if (sampled && (P.launches++ % prof_stride()) != 0) return;
  if (P.used + 2 > P.pool.size()) {
    for (int i = 0; i < 512; ++i) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      P.pool.push_back(e);
    }
  }
  P.kinds.resize(P.pool.size());
  P.widths.resize(P.pool.size());
  P.snap_of.resize(P.pool.size());
  P.kinds[P.used] = kind;
  P.widths[P.used] = width;
  P.snap_of[P.used] = snap;
  if (n_active) {  // snapshot the active-column count this launch will see
    if (P.n_snaps + 1 > P.snaps.n) {
      DevBuf<int> grown(std::max<size_t>(1024, 2 * P.snaps.n));
      if (P.n_snaps)
        CK(cudaMemcpyAsync(grown.p, P.snaps.p, P.n_snaps * sizeof(int), cudaMemcpyDeviceToDevice,
                           ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      P.snaps = std::move(grown);
    }
    P.snap_of[P.used] = (int)P.n_snaps;
    CK(cudaMemcpyAsync(P.snaps.p + P.n_snaps, n_active, sizeof(int), cudaMemcpyDeviceToDevice,
                       ctx->stream));
    ++P.n_snaps;
  }
  ev[0] = P.pool[P.used++];
  ev[1] = P.pool[P.used++];
  CK(cudaEventRecord(ev[0], ctx->stream));
}
void prof_end(ect_ctx* ctx, cudaEvent_t* ev) {
  if (!ctx->prof.enabled || ev[0] == nullptr) return;
  CK(cudaEventRecord(ev[1], ctx->stream));
}
// slot of the snapshot taken by the pair whose start event is ev0 (-1 if none)
int prof_snap_of(ect_ctx* ctx, cudaEvent_t ev0) {
  auto& P = ctx->prof;
  for (size_t i = P.used; i >= 2; i -= 2)
    if (P.pool[i - 2] == ev0) return P.snap_of[i - 2];
  return -1;
}
void prof_collect(ect_ctx* ctx) {
  auto& P = ctx->prof;
  if (!P.enabled || P.used == 0) return;
  CK(cudaStreamSynchronize(ctx->stream));
  std::vector<int> act(P.n_snaps);
  if (P.n_snaps)
    CK(cudaMemcpy(act.data(), P.snaps.p, P.n_snaps * sizeof(int), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i + 1 < P.used; i += 2) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, P.pool[i], P.pool[i + 1]));
    // a solver sample counts only if all `width` columns were active
    const bool full = P.snap_of[i] < 0 || act[(size_t)P.snap_of[i]] >= P.widths[i];
    if (P.kinds[i] == 0) {
      if (full) {
        ctx->timings.spmv_ms_total += ms;
        ctx->timings.spmv_launches += 1;
      } else {
        ctx->timings.spmv_partial_launches += 1;
      }
    } else if (P.kinds[i] == 1) {
      if (full) {
        ctx->timings.vec_ms_total += ms;
        ctx->timings.vec_launches += 1;
      } else {
        ctx->timings.vec_partial_launches += 1;
      }
    } else if (full) {
      ctx->timings.precond_ms_total += ms;
      ctx->timings.precond_launches += 1;
    }
  }
  P.used = 0;
  P.n_snaps = 0;
}

}  // namespace

void compute_jacobi(ect_matrix* a) {
  ect_ctx* ctx = a->ctx;
  a->dinv.alloc(std::max<int64_t>(1, a->n));
  DevBuf<int> missing(1);
  CK(cudaMemsetAsync(missing.p, 0, sizeof(int), ctx->stream));
  int grid = (int)std::min<int64_t>((a->n + 255) / 256, (int64_t)ctx->num_sms * 16);
  k_jacobi<<<std::max(grid, 1), 256, 0, ctx->stream>>>(a->n, a->row_ptr.p, a->col.p, a->val.p,
                                                        a->dinv.p, missing.p);
  CK_LAUNCH();
  note_launch(ctx, 1);
  int h = 0;
  CK(cudaMemcpyAsync(&h, missing.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  a->n_zero_diag = h;  // a Jacobi solve on such a matrix is a SolverError (cocg_solve)
}

void build_nb(ect_mesh* m, ect_matrix* a) {
  ect_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  a->has_nb = false;
  const int64_t nn = m->n_nodes;
  int64_t nblk = 0;
  {
    int h = 0;
    CK(cudaMemcpyAsync(&h, m->nbr_off.p + nn, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    nblk = h;
  }
  DevBuf<int> cnt(nn + 1);
  CK(cudaMemsetAsync(cnt.p, 0, cnt.bytes(), s));
  const int grid = (int)std::min<int64_t>((nn + 255) / 256, (int64_t)ctx->num_sms * 16);
  k_cpl_count<<<std::max(grid, 1), 256, 0, s>>>(m->nbr_off.p, m->nbr_cond.p, m->cond_fwd.p, 0,
                                                 nn, cnt.p);
  CK_LAUNCH();
  a->nb_cpl_ptr.alloc(nn + 1);
  size_t tmp = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.p, a->nb_cpl_ptr.p, nn + 1, s));
  CK(cub::DeviceScan::ExclusiveSum(cub_scratch(ctx, tmp), tmp, cnt.p, a->nb_cpl_ptr.p, nn + 1, s));
  int ncpl = 0;
  CK(cudaMemcpyAsync(&ncpl, a->nb_cpl_ptr.p + nn, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  a->nb_blocks = nblk;
  a->nb_ncpl = ncpl;
  a->nb_blk.alloc(6 * (std::max<int64_t>(1, nblk) + 4));  // + staged-copy overrun padding
  a->nb_cpl_idx.alloc(std::max(1, ncpl));
  a->nb_cpl.alloc(4 * (size_t)std::max(1, ncpl));
  a->nb_blk_ptr = m->nbr_off.p;
  a->nb_blk_col = m->nbr.p;
  a->nb_cond_fwd = m->cond_fwd.p;
  DevBuf<int> bad(1);
  CK(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
  const int wgrid = (int)std::min<int64_t>((32 * nn + 255) / 256, (int64_t)ctx->num_sms * 16);
  k_build_nb<<<std::max(wgrid, 1), 256, 0, s>>>(a->row_ptr.p, a->val.p, m->nbr_off.p, m->nbr.p,
                                                 m->nbr_cond.p, m->cond_fwd.p, a->nb_cpl_ptr.p, nn,
                                                 reinterpret_cast<double*>(a->nb_blk.p), nblk,
                                                 a->nb_cpl_idx.p,
                                                 reinterpret_cast<double*>(a->nb_cpl.p),
                                                 ncpl, bad.p, 0, nn, 0, 0);
  CK_LAUNCH();
  note_launch(ctx, 3);
  int h_bad = 0;
  CK(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  // NB drops imaginary parts it proves to be exact zeros; otherwise stay CSR.
  a->has_nb = h_bad == 0;
  if (!a->has_nb) {
    a->nb_blk.release();
    a->nb_cpl.release();
    a->nb_cpl_idx.release();
    return;
  }
  // ---- NB-E sliced-ELL copy of the blocks (chunks of 32 nodes) -----------------
  a->has_nbe = false;
  {
    const int64_t nch = (nn + 31) / 32;
    DevBuf<int> w(nch + 1);
    const int cg = (int)std::min<int64_t>((nch + 255) / 256, (int64_t)ctx->num_sms * 16);
    k_nbe_width<<<std::max(cg, 1), 256, 0, s>>>(m->nbr_off.p, nn, nch, w.p);
    CK_LAUNCH();
    a->nbe_off.alloc(nch + 1);
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, w.p, a->nbe_off.p, nch + 1, s));
    CK(cub::DeviceScan::ExclusiveSum(cub_scratch(ctx, tmp), tmp, w.p, a->nbe_off.p, nch + 1, s));
    int slots = 0;
    CK(cudaMemcpyAsync(&slots, a->nbe_off.p + nch, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    a->nbe_col.alloc(std::max(1, slots));
    a->nbe_blk.alloc(6 * (size_t)std::max(1, slots));
    const int fg = (int)std::min<int64_t>((32 * nch + 255) / 256, (int64_t)ctx->num_sms * 16);
    k_nbe_fill<<<std::max(fg, 1), 256, 0, s>>>(m->nbr_off.p, m->nbr.p,
                                                reinterpret_cast<const double*>(a->nb_blk.p), nblk,
                                                nn, nch, a->nbe_off.p, a->nbe_col.p,
                                                reinterpret_cast<double*>(a->nbe_blk.p), slots);
    CK_LAUNCH();
    note_launch(ctx, 2);
    CK(cudaStreamSynchronize(s));
    a->nbe_slots = slots;
    a->has_nbe = true;
    // only the sliced-ELL copy stays resident (parts are cut from it too)
    a->nb_blk.release();
  }
}

void build_sell(ect_matrix* a, int sigma) {
  ect_ctx* ctx = a->ctx;
  cudaStream_t s = ctx->stream;
  const int64_t n = a->n;
  const int64_t n_chunks = (n + kSellC - 1) / kSellC, n_slots = n_chunks * kSellC;
  sigma = std::max(kSellC, sigma / kSellC * kSellC);
  DevBuf<int> len(n_slots), idx(n_slots), slen(n_slots), w(n_chunks + 1);
  const int grid = (int)std::min<int64_t>((n_slots + 255) / 256, (int64_t)ctx->num_sms * 16);
  k_sell_lens<<<std::max(grid, 1), 256, 0, s>>>(n, a->row_ptr.p, len.p, idx.p, n_slots);
  CK_LAUNCH();
  a->sell_perm.alloc(n_slots);
  // sort rows by length (descending) inside windows of sigma rows
  const int64_t n_win = (n_slots + sigma - 1) / sigma;
  std::vector<int> h_seg(n_win + 1);
  for (int64_t q = 0; q <= n_win; ++q) h_seg[q] = (int)std::min<int64_t>(q * sigma, n_slots);
  DevBuf<int> seg(n_win + 1);
  CK(cudaMemcpyAsync(seg.p, h_seg.data(), h_seg.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  size_t tmp = 0;
  CK(cub::DeviceSegmentedSort::StableSortPairsDescending(nullptr, tmp, len.p, slen.p, idx.p,
                                                         a->sell_perm.p, (int)n_slots, (int)n_win,
                                                         seg.p, seg.p + 1, s));
  CK(cub::DeviceSegmentedSort::StableSortPairsDescending(cub_scratch(ctx, tmp), tmp, len.p, slen.p,
                                                         idx.p, a->sell_perm.p, (int)n_slots,
                                                         (int)n_win, seg.p, seg.p + 1, s));
  const int cgrid = (int)std::min<int64_t>((n_chunks + 255) / 256, (int64_t)ctx->num_sms * 16);
  k_sell_width<<<std::max(cgrid, 1), 256, 0, s>>>(n_chunks, slen.p, w.p);
  CK_LAUNCH();
  a->sell_off.alloc(n_chunks + 1);
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, w.p, a->sell_off.p, n_chunks + 1, s));
  CK(cub::DeviceScan::ExclusiveSum(cub_scratch(ctx, tmp), tmp, w.p, a->sell_off.p, n_chunks + 1, s));
  int total = 0;
  CK(cudaMemcpyAsync(&total, a->sell_off.p + n_chunks, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  a->sell_col.alloc(std::max(1, total));
  a->sell_val.alloc(std::max(1, total));
  k_sell_fill<<<std::max(grid, 1), 256, 0, s>>>(n_slots, a->sell_perm.p, a->sell_off.p,
                                                 a->row_ptr.p, a->col.p, a->val.p, a->sell_col.p,
                                                 a->sell_val.p);
  CK_LAUNCH();
  note_launch(ctx, 4);
  CK(cudaStreamSynchronize(s));
  a->sell_chunks = n_chunks;
  a->sell_stored = total;
  a->has_sell = true;
}

namespace {
struct Cols4 {
  int c[4];
};
__global__ void __launch_bounds__(kBlock)
k_gather_columns(const double2* __restrict__ src, int k, Cols4 cols, int n_cols, int64_t n,
                 double2* __restrict__ dst) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n_cols;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / n, i = e - c * n;
    dst[e] = src[i * k + cols.c[c]];
  }
}
}  // namespace

void gather_columns(ect_ctx* ctx, const double2* src, int k, const int* cols, int n_cols,
                    int64_t n, double2* dst) {
  if (n_cols < 1 || n_cols > 4) fail(ECT_ERR_CONFIG, "gather_columns: 1..4 columns");
  Cols4 c{};
  for (int j = 0; j < n_cols; ++j) c.c[j] = cols[j];
  const int grid = (int)std::min<int64_t>((n * n_cols + kBlock - 1) / kBlock,
                                          (int64_t)ctx->num_sms * 8);
  k_gather_columns<<<std::max(grid, 1), kBlock, 0, ctx->stream>>>(src, k, c, n_cols, n, dst);
  CK_LAUNCH();
  note_launch(ctx, 1);
}

void spmv(ect_ctx* ctx, ect_matrix* a, const double2* x, double2* y, int k) {
  if (k < 1 || k > 16) fail(ECT_ERR_SOLVER, "spmv: n_rhs must be in 1..16");
  if (k & (k - 1)) {  // pad to the next supported width
    int kk = 1;
    while (kk < k) kk <<= 1;
    DevBuf<double2> xp((size_t)a->n * kk), yp((size_t)a->n * kk);
    CK(cudaMemsetAsync(xp.p, 0, xp.bytes(), ctx->stream));
    CK(cudaMemcpy2DAsync(xp.p, kk * sizeof(double2), x, k * sizeof(double2), k * sizeof(double2),
                         a->n, cudaMemcpyDeviceToDevice, ctx->stream));
    spmv(ctx, a, xp.p, yp.p, kk);
    CK(cudaMemcpy2DAsync(y, k * sizeof(double2), yp.p, kk * sizeof(double2), k * sizeof(double2),
                         a->n, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return;
  }
  with_k(k, [&](auto D) {
    using DK = decltype(D);
    KrylovCtl ctl{};
    const int grid = DK::spmv_grid(ctx, kPlain, a);
    cudaEvent_t ev[2];
    prof_begin(ctx, ev);
    DK::spmv(ctx, kPlain, grid, a->n, a, x, y, nullptr, ctl);
    prof_end(ctx, ev);
    note_launch(ctx, 1);
  });
  prof_collect(ctx);
}

// ---- BiCGStab (non-symmetric A: impedance surface terms) ----------------------
// With element_ibc the coupling blocks satisfy va = i*omega*av^T, so A != A^T
// and COCG does not apply; the reference still runs GMRES(80)+ILU(0)
// (iterative.cpp:109-228). The GPU runs right-Jacobi-preconditioned BiCGStab
// (conjugated inner products), k right-hand sides interleaved, device-resident
// scalars, the same convergence contract (recurrence residual, then a true
// residual with restart) and the same breakdown-as-error rule.
namespace {

__device__ __forceinline__ double2 cconj_mul(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

// Elementwise kernels: thread owns element e = i*K + k of [n][K] vectors; the
// grid stride is a multiple of K, so k = lane % K is fixed per thread.
template <int K>
__global__ void __launch_bounds__(kBlock)
k_bi_p(int64_t n, const double2* __restrict__ r, double2* __restrict__ p,
       const double2* __restrict__ v, double2* __restrict__ ph, const double2* __restrict__ dinv,
       KrylovCtl ctl) {
  if (*ctl.n_active == 0) return;
  const int k = (threadIdx.x & 31) % K;
  const RhsState st = ctl.st[k];
  if (st.status != kActive) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * K;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double2 pn = cadd(r[e], cmul(st.beta, csub(p[e], cmul(st.omega, v[e]))));
    p[e] = pn;
    ph[e] = cmul(dinv[e / K], pn);
  }
}

template <int K>
__global__ void __launch_bounds__(kBlock)
k_bi_s(int64_t n, double2* __restrict__ r, const double2* __restrict__ v,
       double2* __restrict__ sh, const double2* __restrict__ dinv, KrylovCtl ctl) {
  if (*ctl.n_active == 0) return;
  const int k = (threadIdx.x & 31) % K;
  const RhsState st = ctl.st[k];
  if (st.status != kActive) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * K;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double2 s = csub(r[e], cmul(st.alpha, v[e]));
    r[e] = s;
    sh[e] = cmul(dinv[e / K], s);
  }
}

// WHAT 0: (a, b) -> alpha = rho / (r_hat, v)
// WHAT 1: (t, s), (t, t) -> omega
template <int K, int WHAT>
__global__ void __launch_bounds__(kBlock)
k_bi_dot(int64_t n, const double2* __restrict__ a, const double2* __restrict__ b, KrylovCtl ctl) {
  constexpr int NVL = WHAT == 0 ? 2 : 3, NV = NVL * K;
  __shared__ double smem[32 * NV];
  if (*ctl.n_active == 0) return;
  const int k = (threadIdx.x & 31) % K;
  const bool act = ctl.st[k].status == kActive;
  double part[NVL];
#pragma unroll
  for (int j = 0; j < NVL; ++j) part[j] = 0.0;
  if (act)
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * K;
         e += (int64_t)gridDim.x * blockDim.x) {
      const double2 av = a[e], bv = b[e];
      const double2 d = cconj_mul(av, bv);
      part[0] += d.x;
      part[1] += d.y;
      if (WHAT == 1) part[2] += av.x * av.x + av.y * av.y;
    }
  double bsum[NV];
  block_sum_slots<NVL, K>(part, smem, bsum);
  if (threadIdx.x == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) ctl.partial[(size_t)blockIdx.x * NV + j] = bsum[j];
  if (!last_block(ctl.counter)) return;
  double tot[NV];
  reduce_partials<NV>(ctl.partial, tot, smem);
  if (threadIdx.x == 0) {
    int active = 0;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      RhsState& s = ctl.st[c];
      if (s.status != kActive) continue;
      const double2 d = make_double2(tot[NVL * c], tot[NVL * c + 1]);
      if (WHAT == 0) {
        if (d.x == 0.0 && d.y == 0.0) { s.status = kBreakdown; continue; }
        s.alpha = cdiv(s.rho, d);
      } else {
        const double tt = tot[NVL * c + 2];
        s.omega = tt > 0.0 ? cdiv(d, make_double2(tt, 0.0)) : make_double2(0.0, 0.0);
      }
      ++active;
    }
    *ctl.n_active = active;
    *ctl.counter = 0u;
  }
}

constexpr double kBiGrowth = 1e4;  // recurrence residual / best since restart -> restart
constexpr int kBiStall = 600;      // iterations without a new best residual -> restart

// x += alpha p_hat + omega s_hat ; r = s - omega t ; rho_new = (r_hat, r), ||r||
template <int K>
__global__ void __launch_bounds__(kBlock)
k_bi_x(int64_t n, double2* __restrict__ x, double2* __restrict__ r,
       const double2* __restrict__ ph, const double2* __restrict__ sh,
       const double2* __restrict__ t, const double2* __restrict__ rh, KrylovCtl ctl) {
  constexpr int NVL = 3, NV = NVL * K;
  __shared__ double smem[32 * NV];
  if (*ctl.n_active == 0) return;
  const int k = (threadIdx.x & 31) % K;
  const RhsState st = ctl.st[k];
  const bool act = st.status == kActive;
  double part[NVL] = {0.0, 0.0, 0.0};
  if (act)
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * K;
         e += (int64_t)gridDim.x * blockDim.x) {
      x[e] = cadd(x[e], cadd(cmul(st.alpha, ph[e]), cmul(st.omega, sh[e])));
      const double2 rn = csub(r[e], cmul(st.omega, t[e]));
      r[e] = rn;
      const double2 d = cconj_mul(rh[e], rn);
      part[0] += d.x;
      part[1] += d.y;
      part[2] += rn.x * rn.x + rn.y * rn.y;
    }
  double bsum[NV];
  block_sum_slots<NVL, K>(part, smem, bsum);
  if (threadIdx.x == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) ctl.partial[(size_t)blockIdx.x * NV + j] = bsum[j];
  if (!last_block(ctl.counter)) return;
  double tot[NV];
  reduce_partials<NV>(ctl.partial, tot, smem);
  if (threadIdx.x == 0) {
    int active = 0;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      RhsState& s = ctl.st[c];
      if (s.status != kActive) continue;
      const double2 rho_new = make_double2(tot[NVL * c], tot[NVL * c + 1]);
      s.rnorm = sqrt(tot[NVL * c + 2]);
      s.iters += 1;
      if (s.rnorm < s.rbest) {
        s.rbest = s.rnorm;
        s.best_iter = (double)s.iters;
      }
      if (s.rnorm <= ctl.tol * s.bnorm) {
        s.status = kConverged;
      } else if (s.iters >= ctl.max_iter) {
        s.status = kMaxIter;
      } else if ((rho_new.x == 0.0 && rho_new.y == 0.0) || (s.omega.x == 0.0 && s.omega.y == 0.0) ||
                 !(s.rnorm <= kBiGrowth * s.rbest) ||
                 (double)s.iters - s.best_iter >= (double)kBiStall) {
        // Lanczos (near-)breakdown; or the recurrence residual has grown far
        // above its best value (also NaN); or it has not improved for kBiStall
        // iterations (the recurrence has drifted from b - A x and hovers above
        // the tolerance): restart from the true residual, which turns the
        // solve into iterative refinement with BiCGStab as the inner solver
        s.status = kBreakdown;
      } else {
        s.beta = cmul(cdiv(rho_new, s.rho), cdiv(s.alpha, s.omega));
        s.rho = rho_new;
        ++active;
      }
    }
    *ctl.n_active = active;
    *ctl.counter = 0u;
  }
}

// (re)start masked columns from r (fresh: x = 0, r = b, bnorm): r_hat = r,
// p = v = 0, rho = (r_hat, r), alpha = omega = 1, beta = 0
template <int K>
__global__ void __launch_bounds__(kBlock)
k_bi_start(int64_t n, const double2* __restrict__ b, double2* __restrict__ x,
           double2* __restrict__ r, double2* __restrict__ rh, double2* __restrict__ p,
           double2* __restrict__ v, unsigned mask, int fresh, KrylovCtl ctl) {
  constexpr int NVL = 3, NV = NVL * K;
  __shared__ double smem[32 * NV];
  const int k = (threadIdx.x & 31) % K;
  const bool on = (mask >> k) & 1u;
  double part[NVL] = {0.0, 0.0, 0.0};
  if (on)
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * K;
         e += (int64_t)gridDim.x * blockDim.x) {
      double2 rv;
      if (fresh) {
        rv = b[e];
        x[e] = make_double2(0.0, 0.0);
        r[e] = rv;
      } else {
        rv = r[e];
      }
      rh[e] = rv;
      p[e] = v[e] = make_double2(0.0, 0.0);
      part[0] += rv.x * rv.x + rv.y * rv.y;  // (r_hat, r) = ||r||^2
    }
  double bsum[NV];
  block_sum_slots<NVL, K>(part, smem, bsum);
  if (threadIdx.x == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) ctl.partial[(size_t)blockIdx.x * NV + j] = bsum[j];
  if (!last_block(ctl.counter)) return;
  double tot[NV];
  reduce_partials<NV>(ctl.partial, tot, smem);
  if (threadIdx.x == 0) {
    int active = 0;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      RhsState& s = ctl.st[c];
      if ((mask >> c) & 1u) {
        const double rr = tot[NVL * c];
        if (fresh) {
          s.bnorm = sqrt(rr);
          s.iters = 0;
        }
        s.rnorm = s.rbest = sqrt(rr);
        s.best_iter = (double)s.iters;
        s.rho = make_double2(rr, 0.0);
        s.alpha = s.omega = make_double2(1.0, 0.0);
        s.beta = make_double2(0.0, 0.0);
        if (fresh && s.bnorm == 0.0) s.status = kZeroRhs;
        else if (s.rnorm <= ctl.tol * s.bnorm) s.status = kConverged;
        else s.status = kActive;
      }
      active += s.status == kActive;
    }
    *ctl.n_active = active;
    *ctl.counter = 0u;
  }
}

template <int K>
void bicgstab_k(ect_ctx* ctx, ect_matrix* a, const double2* b, double2* x, int k,
                const ect_iter_options& opt, SolveOut* out) {
  using DK = Dispatch<K>;
  const int64_t n = a->n;
  cudaStream_t s = ctx->stream;
  const int grid_s = DK::spmv_grid(ctx, kPlain, a);
  const int grid_r = DK::spmv_grid(ctx, kResid, a);
  const int grid_v = grid_for(ctx, (const void*)k_bi_x<K>, kBlock);
  const int grid_max = std::max(std::max(grid_s, grid_r), grid_v);
  const size_t vec = (size_t)n * K;
  auto& W = ctx->ws;
  for (auto* v : {&W.bb, &W.xx, &W.r, &W.p, &W.q, &W.rh, &W.ph, &W.sh, &W.t}) v->ensure(vec);
  W.st.ensure(K);
  W.n_active.ensure(1);
  W.counter.ensure(1);
  W.partial.ensure((size_t)grid_max * 4 * K);
  CK(cudaMemsetAsync(W.st.p, 0, W.st.bytes(), s));
  CK(cudaMemsetAsync(W.counter.p, 0, sizeof(unsigned), s));
  if (K == k) {
    CK(cudaMemcpyAsync(W.bb.p, b, vec * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  } else {
    CK(cudaMemsetAsync(W.bb.p, 0, W.bb.bytes(), s));
    CK(cudaMemcpy2DAsync(W.bb.p, K * sizeof(double2), b, k * sizeof(double2), k * sizeof(double2),
                         n, cudaMemcpyDeviceToDevice, s));
  }
  KrylovCtl ctl{W.st.p, W.n_active.p, W.counter.p, W.partial.p, opt.tol, opt.max_iter,
                nullptr, 0, n, n, n};
  const unsigned all = (K == 32) ? 0xffffffffu : ((1u << K) - 1u);
  // v lives in q
  k_bi_start<K><<<grid_v, kBlock, 0, s>>>(n, W.bb.p, W.xx.p, W.r.p, W.rh.p, W.p.p, W.q.p, all, 1,
                                          ctl);
  CK_LAUNCH();
  note_launch(ctx, 1);
  std::vector<int> last_break(K, -1);
  std::vector<RhsState> hs(K);
  int* flag = ctx->pinned_flag;
  const int chunk = 16;
  for (int restart_round = 0;; ++restart_round) {
    int polls = 0, launched = 0;
    cudaEvent_t poll_ev[2] = {ctx->ev_a, ctx->ev_b};
    const int cap = opt.max_iter + chunk;
    for (; opt.max_iter > 0;) {
      for (int it = 0; it < chunk; ++it) {
        k_bi_p<K><<<grid_v, kBlock, 0, s>>>(n, W.r.p, W.p.p, W.q.p, W.ph.p, a->dinv.p, ctl);
        DK::spmv(ctx, kPlain, grid_s, n, a, W.ph.p, W.q.p, nullptr, ctl);
        k_bi_dot<K, 0><<<grid_v, kBlock, 0, s>>>(n, W.rh.p, W.q.p, ctl);
        k_bi_s<K><<<grid_v, kBlock, 0, s>>>(n, W.r.p, W.q.p, W.sh.p, a->dinv.p, ctl);
        DK::spmv(ctx, kPlain, grid_s, n, a, W.sh.p, W.t.p, nullptr, ctl);
        k_bi_dot<K, 1><<<grid_v, kBlock, 0, s>>>(n, W.t.p, W.r.p, ctl);
        k_bi_x<K><<<grid_v, kBlock, 0, s>>>(n, W.xx.p, W.r.p, W.ph.p, W.sh.p, W.t.p, W.rh.p, ctl);
        CK_LAUNCH();
        note_launch(ctx, 7);
      }
      launched += chunk;
      CK(cudaMemcpyAsync(flag + (polls & 1), W.n_active.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      CK(cudaEventRecord(poll_ev[polls & 1], s));
      ++polls;
      if (polls >= 2) {
        const int prev = (polls - 2) & 1;
        CK(cudaEventSynchronize(poll_ev[prev]));
        if (flag[prev] == 0) break;
      }
      if (launched > cap + 2 * chunk) break;
    }
    CK(cudaStreamSynchronize(s));
    // true residual confirmation (iterative.cpp:208-216): q <- b - A x
    CK(cudaMemsetAsync(W.n_active.p, 0xff, sizeof(int), s));
    CK(cudaMemcpyAsync(hs.data(), W.st.p, K * sizeof(RhsState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    {
      std::vector<RhsState> tmp = hs;
      for (auto& t : tmp) t.status = kActive;
      CK(cudaMemcpyAsync(W.st.p, tmp.data(), K * sizeof(RhsState), cudaMemcpyHostToDevice, s));
      DK::spmv(ctx, kResid, grid_r, n, a, W.xx.p, W.q.p, W.bb.p, ctl);
      note_launch(ctx, 1);
      std::vector<RhsState> res(K);
      CK(cudaMemcpyAsync(res.data(), W.st.p, K * sizeof(RhsState), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      for (int c = 0; c < K; ++c) hs[c].rnorm = res[c].rnorm;
      CK(cudaMemcpyAsync(W.st.p, hs.data(), K * sizeof(RhsState), cudaMemcpyHostToDevice, s));
    }
    unsigned restart_mask = 0;
    for (int c = 0; c < k; ++c) {
      RhsState& t = hs[c];
      const double rel = t.bnorm > 0.0 ? t.rnorm / t.bnorm : 0.0;
      if (t.status == kBreakdown) {
        // a (near-)breakdown of the Lanczos recurrences: restart from the true
        // residual (new shadow vector); an error only when it recurs at once
        if (restart_round >= 32 || t.iters >= opt.max_iter || t.iters == last_break[c]) {
          out->breakdown[c] = 1;  // reported per column; ect_solve raises SolverError
          continue;
        }
        last_break[c] = t.iters;
        restart_mask |= 1u << c;
        continue;
      }
      if (t.status == kConverged && rel > opt.tol && t.iters < opt.max_iter && restart_round < 32)
        restart_mask |= 1u << c;
    }
    if (!restart_mask) break;
    for (int c = 0; c < K; ++c)
      if ((restart_mask >> c) & 1u)
        CK(cudaMemcpy2DAsync(W.r.p + c, K * sizeof(double2), W.q.p + c, K * sizeof(double2),
                             sizeof(double2), n, cudaMemcpyDeviceToDevice, s));
    k_bi_start<K><<<grid_v, kBlock, 0, s>>>(n, W.bb.p, W.xx.p, W.r.p, W.rh.p, W.p.p, W.q.p,
                                            restart_mask, 0, ctl);
    CK_LAUNCH();
    note_launch(ctx, 1);
    CK(cudaStreamSynchronize(s));
  }
  for (int c = 0; c < k; ++c) {
    const RhsState& t = hs[c];
    out->iters[c] = t.iters;
    const double rel = t.bnorm > 0.0 ? t.rnorm / t.bnorm : 0.0;
    out->residual[c] = rel;
    out->converged[c] = (t.status == kZeroRhs) || (t.status == kConverged && rel <= opt.tol);
  }
  if (K == k) {
    CK(cudaMemcpyAsync(x, W.xx.p, vec * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  } else {
    CK(cudaMemcpy2DAsync(x, k * sizeof(double2), W.xx.p, K * sizeof(double2), k * sizeof(double2),
                         n, cudaMemcpyDeviceToDevice, s));
  }
  CK(cudaStreamSynchronize(s));
}

}  // namespace

// ---- single-precision finest-level smoothing (multigrid cycle) -----------------
// The damped-Jacobi sweeps of the finest level only have to reduce the error's
// oscillatory part, so they stream an fp32 copy of the NB-E blocks and fp32
// iterates: half the bytes of the two smoothing SpMVs and of the cycle's
// finest-level vectors. The residual b = r, D^-1, the output z = M r and the
// dot r^T z stay fp64 (the COCG recurrence is untouched). Measured on a
// configs[1]-like mesh: 62 -> 62 iterations to 1e-8, 104 -> 107 to 1e-12.
struct Nb32 {
  const int* e_off;
  const int* blk_col;
  const float* blk;  // plane p of slot q at blk + 4 * (p * nslots + q): 9 real + 3 diag imag
  int64_t nslots;
  const int* cpl_ptr;
  const int2* cpl_idx;
  const float* cpl;  // plane p of coupling q at cpl + 4 * (p * ncpl + q)
  int64_t ncpl;
  const int* cond_fwd;
  int64_t n_nodes, na;
};

__device__ __forceinline__ void ld4f(const float* p, float (&v)[4]) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
               : "l"(p));
}
__device__ __forceinline__ void ld2xf(const float2* p, float2& a, float2& b) {
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(a.x), "=f"(a.y), "=f"(b.x), "=f"(b.y)
               : "l"(p));
}

__device__ __forceinline__ void load_block32(const Nb32& A, int64_t q, float (&B)[3][3],
                                             float (&Im)[3]) {
  float v0[4], v1[4], v2[4];
  ld4f(A.blk + 4 * q, v0);
  ld4f(A.blk + 4 * (A.nslots + q), v1);
  ld4f(A.blk + 4 * (2 * A.nslots + q), v2);
  B[0][0] = v0[0]; B[0][1] = v0[1]; B[0][2] = v0[2];
  B[1][0] = v0[3]; B[1][1] = v1[0]; B[1][2] = v1[1];
  B[2][0] = v1[2]; B[2][1] = v1[3]; B[2][2] = v2[0];
  Im[0] = v2[1]; Im[1] = v2[2]; Im[2] = v2[3];
}

// K right-hand sides, G = GB x CL lanes per node (block lanes x column lanes,
// KL = K / CL columns per lane, even or 1). Modes:
//  kResidNR  : y32 = b - A x                  (b fp64, x fp32, y fp32)
//  kSmoothDot: z = x + omega D^-1 (b - A x), rho partials b^T z (z fp64)
// FLAT (wide batches, one block lane per node): the unpredicated chunk-width
// loop of k_nbe_spmv; at ~63 registers the SM holds 32 warps, which is what
// hides the gather latency here (lab: 0.147 vs 0.347 ms at k = 8).
template <int G, int K, int MODE, int MINB, int CL, int BLOCK = kBlock, bool FLAT = false,
          int PFD = 0>
__global__ void __launch_bounds__(BLOCK, MINB)
k_nbe32(Nb32 A, const float2* __restrict__ x, void* __restrict__ yv,
        const double2* __restrict__ b, KrylovCtl ctl) {
  static_assert(G % CL == 0 && K % CL == 0, "lane split");
  static_assert(!FLAT || G == CL, "the flat loop has one block lane per node");
  static_assert(MODE == kResidNR || MODE == kSmoothDot, "fp32 smoothing modes");
  constexpr int GB = G / CL, KL = K / CL;
  constexpr int NVL = MODE == kSmoothDot ? 2 * KL : 1, NV = NVL * CL;
  __shared__ double smem[32 * NV];
  if (*ctl.n_active == 0) return;
  constexpr int NPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int g = lane & (G - 1);
  const int bl = g / CL, cl = g % CL;
  const int kc = cl * KL;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double part[NVL];
#pragma unroll
  for (int j = 0; j < NVL; ++j) part[j] = 0.0;
  for (int64_t wn = warp * NPW; wn < A.n_nodes; wn += n_warps * NPW) {
    const int64_t i = wn + lane / G;
    const bool valid = i < A.n_nodes;
    float2 acc[3][KL], accv[KL];
#pragma unroll
    for (int k = 0; k < KL; ++k) acc[0][k] = acc[1][k] = acc[2][k] = accv[k] = make_float2(0.f, 0.f);
    int cf_i = -1;
    if constexpr (FLAT) {
      const int c32 = (int)(wn >> 5);
      const int o32 = A.e_off[c32];
      const int w32 = (A.e_off[c32 + 1] - o32) >> 5;
      const int sbase = o32 + (int)(i & 31);
      constexpr int LINES = NPW >= 8 ? NPW / 8 : 1;  // 128-B lines per fp32 plane row of the warp
      const char* pf = nullptr;
      int pf_stride = 0;
      if constexpr (PFD > 0) {
        if (lane < 3 * LINES) {
          pf = reinterpret_cast<const char*>(A.blk + 4 * ((int64_t)(lane / LINES) * A.nslots + o32 +
                                                          (int)(wn & 31)) +
                                             32 * (lane % LINES));
          pf_stride = 32 * 16;
        } else if (lane == 3 * LINES) {
          pf = reinterpret_cast<const char*>(A.blk_col + o32 + (int)(wn & 31));
          pf_stride = 32 * 4;
        }
      }
      int m = ldg_i(A.blk_col + sbase);
      for (int j = 0; j < w32; ++j) {
        if constexpr (PFD > 0) {
          if (pf && j + PFD < w32)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pf + (int64_t)(j + PFD) * pf_stride));
        }
        const int q = sbase + 32 * j;
        float B[3][3], Im[3];
        load_block32(A, q, B, Im);
        const float2* xm = x + (int64_t)3 * m * K + kc;
        float2 xp[3][KL];
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int k = 0; k < KL; k += 2) ld2xf(xm + d * K + k, xp[d][k], xp[d][k + 1]);
        if (j + 1 < w32) m = ldg_i(A.blk_col + q + 32);
#pragma unroll
        for (int k = 0; k < KL; ++k)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            float2 s = acc[c][k];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              s.x = fmaf(B[c][d], xp[d][k].x, s.x);
              s.y = fmaf(B[c][d], xp[d][k].y, s.y);
            }
            s.x = fmaf(-Im[c], xp[c][k].y, s.x);
            s.y = fmaf(Im[c], xp[c][k].x, s.y);
            acc[c][k] = s;
          }
      }
    }
    if (valid) {
      const int c32 = (int)(i >> 5);
      const int o32 = A.e_off[c32];
      const int w32 = (A.e_off[c32 + 1] - o32) >> 5;
      const int sbase = o32 + (int)(i & 31), be = sbase + 32 * w32;
      constexpr int GS = 32 * GB;
      int q = sbase + 32 * bl;
      int m_nx = 0;
      float B_nx[3][3], Im_nx[3];
      if (!FLAT && q < be) {
        m_nx = ldg_i(A.blk_col + q);
        load_block32(A, q, B_nx, Im_nx);
      }
      for (; !FLAT && q < be; q += GS) {
        const int m = m_nx;
        float B[3][3], Im[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          Im[c] = Im_nx[c];
#pragma unroll
          for (int d = 0; d < 3; ++d) B[c][d] = B_nx[c][d];
        }
        if (q + GS < be) {  // software pipeline: the next block's loads in flight
          m_nx = ldg_i(A.blk_col + q + GS);
          load_block32(A, q + GS, B_nx, Im_nx);
        }
        const float2* xm = x + (int64_t)3 * m * K + kc;
        constexpr int KP = (KL % 2 == 0) ? 2 : 1;
#pragma unroll
        for (int k0 = 0; k0 < KL; k0 += KP) {
          float2 xp[3][KP];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            if constexpr (KP == 2) ld2xf(xm + d * K + k0, xp[d][0], xp[d][1]);
            else xp[d][0] = __ldg(xm + d * K + k0);
          }
#pragma unroll
          for (int kk = 0; kk < KP; ++kk) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              float2 s = acc[c][k0 + kk];
#pragma unroll
              for (int d = 0; d < 3; ++d) {
                s.x = fmaf(B[c][d], xp[d][kk].x, s.x);
                s.y = fmaf(B[c][d], xp[d][kk].y, s.y);
              }
              s.x = fmaf(-Im[c], xp[c][kk].y, s.x);
              s.y = fmaf(Im[c], xp[c][kk].x, s.y);
              acc[c][k0 + kk] = s;
            }
          }
        }
      }
      cf_i = A.cond_fwd[i];
      if (cf_i >= 0) {
        const int ce = A.cpl_ptr[i + 1];
        for (int qq = A.cpl_ptr[i] + bl; qq < ce; qq += GB) {
          const int2 mi = ldg_i2(A.cpl_idx + qq);
          float c0[4], c1[4];
          ld4f(A.cpl + 4 * qq, c0);
          ld4f(A.cpl + 4 * (A.ncpl + qq), c1);
          const float av[3] = {c0[0], c0[1], c0[2]}, va[3] = {c0[3], c1[0], c1[1]};
          const float2 vv = make_float2(c1[2], c1[3]);
          const float2* xm = x + (int64_t)3 * mi.x * K + kc;
          const float2* xvp = x + (A.na + mi.y) * K + kc;
#pragma unroll
          for (int k = 0; k < KL; ++k) {
            const float2 v = __ldg(xvp + k);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              acc[c][k].x = fmaf(av[c], v.x, acc[c][k].x);
              acc[c][k].y = fmaf(av[c], v.y, acc[c][k].y);
            }
            float2 s = accv[k];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              const float2 xa = __ldg(xm + d * K + k);
              s.x = fmaf(va[d], xa.x, s.x);
              s.y = fmaf(va[d], xa.y, s.y);
            }
            s.x += vv.x * v.x - vv.y * v.y;
            s.y += vv.x * v.y + vv.y * v.x;
            accv[k] = s;
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < KL; ++k) {
#pragma unroll
      for (int o = (GB / 2) * CL; o >= CL; o >>= 1) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          acc[c][k].x += __shfl_xor_sync(0xffffffffu, acc[c][k].x, o, G);
          acc[c][k].y += __shfl_xor_sync(0xffffffffu, acc[c][k].y, o, G);
        }
        accv[k].x += __shfl_xor_sync(0xffffffffu, accv[k].x, o, G);
        accv[k].y += __shfl_xor_sync(0xffffffffu, accv[k].y, o, G);
      }
    }
    if (bl == 0 && valid) {
#pragma unroll
      for (int k = 0; k < KL; ++k) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c == 3 && cf_i < 0) break;
          const int64_t row = c < 3 ? 3 * i + c : A.na + cf_i;
          const float2 a32 = c < 3 ? acc[c][k] : accv[k];
          const int64_t idx = row * K + kc + k;
          const double2 bv = b[idx];
          const double2 res = make_double2(bv.x - (double)a32.x, bv.y - (double)a32.y);
          if constexpr (MODE == kResidNR) {
            static_cast<float2*>(yv)[idx] = make_float2((float)res.x, (float)res.y);
          } else {
            const double2 d = ctl.dinv[row];
            const float2 xv = x[idx];
            const double2 z = cadd(make_double2(xv.x, xv.y),
                                   cmul(make_double2(ctl.omega * d.x, ctl.omega * d.y), res));
            static_cast<double2*>(yv)[idx] = z;
            part[2 * k] += bv.x * z.x - bv.y * z.y;
            part[2 * k + 1] += bv.x * z.y + bv.y * z.x;
          }
        }
      }
    }
  }
  if constexpr (MODE == kResidNR) return;
  double bsum[NV];
  block_sum_slots<NVL, CL>(part, smem, bsum);
  if (threadIdx.x == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) ctl.partial[(size_t)blockIdx.x * NV + j] = bsum[j];
  if (!last_block(ctl.counter)) return;
  double tot[NV];
  reduce_partials<NV>(ctl.partial, tot, smem);
  if (threadIdx.x == 0) {
    fin_rho<K>(ctl, tot);
    *ctl.counter = 0u;
  }
}

template <int K, int MODE>
KFn nbe32_fn() {
  if constexpr (K <= 2) return {(const void*)k_nbe32<2, K, MODE, 3, 1>, kBlock};
  else if constexpr (K == 4) return {(const void*)k_nbe32<4, K, MODE, 3, 2>, kBlock};
  else if constexpr (K == 8) {  // 64 registers (32 warps/SM); the dot epilogue needs 73
    // (forced to 64 registers it spills and the iteration is 1.7% slower; at 85
    // registers / 24 warps it is 0.3% slower)
    constexpr int MINB = MODE == kSmoothDot ? 7 : 8;
    return {(const void*)k_nbe32<4, K, MODE, MINB, 4, 128, true, 2>, 128};
  } else {
    constexpr int MINB = MODE == kSmoothDot ? 7 : 8;
    return {(const void*)k_nbe32<8, K, MODE, MINB, 8, 128, true, 2>, 128};
  }
}

__global__ void k_to_f32(const double* __restrict__ a, int64_t n, float* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = (float)a[e];
}

// ---- aggregation-multigrid cycle (setup in amg.cu) ----------------------------
// M r for the preconditioned COCG: per level l with right-hand side b_l
//   x = omega D^-1 b                 (k_vscale)
//   t = b - A x                      (SpMV, kResidNR)
//   b_{l+1} = P^T t                  (k_restrict: sum over the aggregate's dofs)
//   e = cycle(l+1, b_{l+1})          (W-cycle: a second visit on b_{l+1} - A e)
//   x += oc P e                      (k_prolong)
//   y = x + omega D^-1 (b - A x)     (SpMV, kSmooth; on level 0 kSmoothDot also
//                                     forms r^T z -> rho, beta)
// and a dense inverse on the coarsest level. Symmetric pre/post smoothing and
// the plain transpose keep M complex symmetric (M = M^T), as COCG requires.
namespace {

__device__ __forceinline__ bool idle(const int* n_active) { return *n_active == 0; }


// x = omega D^-1 b (x fp64 or fp32)
template <int K, typename TO>
__global__ void __launch_bounds__(kBlock)
k_vscale(int64_t n, const double2* __restrict__ b, const double2* __restrict__ dinv, double omega,
         TO* __restrict__ x, const int* n_active) {
  if (idle(n_active)) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * K;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double2 d = dinv[e / K];
    put(x + e, cmul(make_double2(omega * d.x, omega * d.y), b[e]));
  }
}

// b_c = P^T t: fixed-order sum over the aggregate's dofs (t fp64 or fp32)
template <int K, typename TI>
__global__ void __launch_bounds__(kBlock)
k_restrict(int64_t nc, const int* __restrict__ r_ptr, const int* __restrict__ r_idx,
           const TI* __restrict__ t, double2* __restrict__ bc, const int* n_active) {
  if (idle(n_active)) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nc * K;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / K, k = e - c * K;
    double2 acc = make_double2(0.0, 0.0);
    const int pe = r_ptr[c + 1];
    // four member indices, then their four values, per step (latency, not
    // bandwidth, is what these small launches cost); the sum stays in order
    for (int p = r_ptr[c]; p < pe; p += 4) {
      int idx[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) idx[u] = p + u < pe ? __ldg(r_idx + p + u) : -1;
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        v[u] = idx[u] >= 0 ? as_d2(t[(int64_t)idx[u] * K + k]) : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < 4; ++u) acc = cadd(acc, v[u]);
    }
    bc[e] = acc;
  }
}

// x += oc P e (x fp64 or fp32)
template <int K, typename TO>
__global__ void __launch_bounds__(kBlock)
k_prolong(int64_t n, const int* __restrict__ cmap, double oc, const double2* __restrict__ ec,
          TO* __restrict__ x, const int* n_active) {
  if (idle(n_active)) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * K;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / K;
    const int c = cmap[i];
    if (c < 0) continue;
    const double2 v = ec[(int64_t)c * K + (e - i * K)];
    put(x + e, cadd(as_d2(x[e]), make_double2(oc * v.x, oc * v.y)));
  }
}

template <int K>
__global__ void __launch_bounds__(kBlock)
k_axpy1(int64_t n, double2* __restrict__ y, const double2* __restrict__ x, const int* n_active) {
  if (idle(n_active)) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * K;
       e += (int64_t)gridDim.x * blockDim.x)
    y[e] = cadd(y[e], x[e]);
}

// x = Minv b on the coarsest level: warp per row, fixed-order lane/shuffle sums
template <int K>
__global__ void __launch_bounds__(kBlock)
k_dense(int64_t n, const double2* __restrict__ minv, const double2* __restrict__ b,
        double2* __restrict__ x, const int* n_active) {
  if (idle(n_active)) return;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += n_warps) {
    double2 acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = make_double2(0.0, 0.0);
    for (int64_t j = lane; j < n; j += 32) {
      const double2 m = minv[i * n + j];
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] = cadd(acc[k], cmul(m, b[j * K + k]));
    }
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        acc[k].x += __shfl_xor_sync(0xffffffffu, acc[k].x, o);
        acc[k].y += __shfl_xor_sync(0xffffffffu, acc[k].y, o);
      }
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < K; ++k) x[i * K + k] = acc[k];
  }
}

// rho = r^T z per active column (single-level hierarchy: no smoothing
// SpMV to fuse it into), finalised by fin_rho
template <int K>
__global__ void __launch_bounds__(kBlock)
k_rho(int64_t n, const double2* __restrict__ r, const double2* __restrict__ z, KrylovCtl ctl) {
  constexpr int CW = VecMap<K>::CW, KH = VecMap<K>::KH;
  constexpr int NVL = 2 * CW, NV = 2 * K;
  __shared__ double smem[32 * NV];
  if (*ctl.n_active == 0) return;
  const int h = (threadIdx.x & 31) % KH, kb = h * CW;
  bool act[CW];
#pragma unroll
  for (int c = 0; c < CW; ++c) act[c] = ctl.st[kb + c].status == kActive;
  double part[NVL];
#pragma unroll
  for (int j = 0; j < NVL; ++j) part[j] = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * KH;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / KH;
#pragma unroll
    for (int c = 0; c < CW; ++c) {
      if (!act[c]) continue;
      const int64_t idx = i * K + kb + c;
      const double2 rv = r[idx], zv = z[idx];
      part[2 * c] += rv.x * zv.x - rv.y * zv.y;
      part[2 * c + 1] += rv.x * zv.y + rv.y * zv.x;
    }
  }
  double bsum[NV];
  block_sum_slots<NVL, KH>(part, smem, bsum);
  if (threadIdx.x == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) ctl.partial[(size_t)blockIdx.x * NV + j] = bsum[j];
  if (!last_block(ctl.counter)) return;
  double tot[NV];
  reduce_partials<NV>(ctl.partial, tot, smem);
  if (threadIdx.x == 0) {
    fin_rho<K>(ctl, tot);
    *ctl.counter = 0u;
  }
}


template <int K>
struct Cycle {
  using DK = Dispatch<K>;
  ect_ctx* ctx;
  ect_matrix* a;
  Amg& H;
  int grid0[6] = {};                  // level-0 SpMV grids per mode
  std::vector<std::array<int, 6>> gl;  // levels >= 1
  int gvec(int64_t work) const {
    const int64_t b = (work + kBlock - 1) / kBlock;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)ctx->num_sms * 8));
  }
  int grid_vec = 1;                   // <= the partial-buffer rows of the solve
  bool f32 = false;                   // finest-level smoothing in fp32 (NB-E storage)
  int grid32[6] = {};
  Cycle(ect_ctx* c, ect_matrix* m, Amg& h) : ctx(c), a(m), H(h) {
    grid_vec = DK::vec_grid(ctx);
    f32 = H.f32 && a->has_nb && a->has_nbe && H.lv.size() > 1;
    if (f32) {
      if (!H.blk32.p) {  // fp32 copies of the NB-E blocks and couplings, once
        H.blk32.alloc(12 * (size_t)std::max<int64_t>(1, a->nbe_slots));
        H.cpl32.alloc(8 * (size_t)std::max<int64_t>(1, a->nb_ncpl));
        k_to_f32<<<gvec(12 * a->nbe_slots), kBlock, 0, ctx->stream>>>(
            reinterpret_cast<const double*>(a->nbe_blk.p), 12 * a->nbe_slots, H.blk32.p);
        CK_LAUNCH();
        k_to_f32<<<gvec(8 * a->nb_ncpl), kBlock, 0, ctx->stream>>>(
            reinterpret_cast<const double*>(a->nb_cpl.p), 8 * a->nb_ncpl, H.cpl32.p);
        CK_LAUNCH();
        note_launch(ctx, 2);
      }
      grid32[kResidNR] = grid_for(ctx, nbe32_fn<K, kResidNR>().fn, nbe32_fn<K, kResidNR>().block);
      grid32[kSmoothDot] =
          grid_for(ctx, nbe32_fn<K, kSmoothDot>().fn, nbe32_fn<K, kSmoothDot>().block);
    }
    for (int mode : {kResidNR, kSmooth, kSmoothDot}) grid0[mode] = DK::spmv_grid(ctx, mode, a);
    gl.resize(H.lv.size());
    for (size_t l = 1; l < H.lv.size(); ++l)
      for (int mode : {kResidNR, kSmooth}) {  // one warp per coarse row
        const int64_t need = (H.lv[l].n * 32 + kBlock - 1) / kBlock;
        gl[l][mode] = (int)std::max<int64_t>(
            1, std::min<int64_t>(need, grid_for(ctx, csr_row_fn<K>(mode), kBlock)));
      }
    // work vectors for this batch width
    if (H.kcap < K) {
      for (size_t l = 0; l + 1 < H.lv.size(); ++l) {
        AmgLevel& L = H.lv[l];
        L.xt.alloc((size_t)L.n * K);
        if (l > 0) L.t.alloc((size_t)L.n * K);
      }
      if (H.f32 && H.lv.size() > 1) {
        H.xt32.alloc((size_t)H.lv[0].n * K);
        H.t32.alloc((size_t)H.lv[0].n * K);
      }
      for (size_t l = 1; l < H.lv.size(); ++l) {
        AmgLevel& L = H.lv[l];
        for (auto* v : {&L.b, &L.out, &L.b2, &L.out2}) v->alloc((size_t)L.n * K);
      }
      H.kcap = K;
    }
  }
  int max_grid() const {
    return std::max({grid0[kResidNR], grid0[kSmooth], grid0[kSmoothDot], grid32[kSmoothDot]});
  }
  Nb32 nb32() const {
    return Nb32{a->nbe_off.p, a->nbe_col.p, H.blk32.p, a->nbe_slots, a->nb_cpl_ptr.p,
                a->nb_cpl_idx.p, H.cpl32.p, a->nb_ncpl, a->nb_cond_fwd, a->n_nodes,
                3 * a->n_nodes};
  }
  void spmv32(int mode, const float2* x, void* y, const double2* b, KrylovCtl c) {
    c.dinv = a->dinv.p;
    Nb32 v = nb32();
    void* args[] = {&v, (void*)&x, &y, (void*)&b, &c};
    const KFn f = mode == kResidNR ? nbe32_fn<K, kResidNR>() : nbe32_fn<K, kSmoothDot>();
    CK(cudaLaunchKernel(f.fn, dim3(grid32[mode]), dim3(f.block), args, 0, ctx->stream));
  }
  // finest level with fp32 smoothing: b = r (fp64), out = z (fp64), dot always
  void run0_f32(const double2* b, double2* out, KrylovCtl c, bool pre) {
    cudaStream_t s = ctx->stream;
    const int64_t n = H.lv[0].n;
    const int* na = c.n_active;
    c.omega = H.omega;
    if (!pre) {
      k_vscale<K, float2><<<gvec(n * K), kBlock, 0, s>>>(n, b, a->dinv.p, H.omega, H.xt32.p, na);
      CK_LAUNCH();
    }
    spmv32(kResidNR, H.xt32.p, H.t32.p, b, c);
    AmgLevel& L = H.lv[0];
    AmgLevel& C = H.lv[1];
    k_restrict<K, float2><<<gvec(C.n * K), kBlock, 0, s>>>(C.n, L.r_ptr.p, L.r_idx.p, H.t32.p,
                                                           C.b.p, na);
    CK_LAUNCH();
    run(1, C.b.p, C.out.p, nullptr, c, false);
    if (H.wcycle && H.lv.size() > 2) {
      spmv(1, kResidNR, C.out.p, C.b2.p, C.b.p, c);
      run(1, C.b2.p, C.out2.p, nullptr, c, false);
      k_axpy1<K><<<gvec(C.n * K), kBlock, 0, s>>>(C.n, C.out.p, C.out2.p, na);
      CK_LAUNCH();
    }
    k_prolong<K, float2><<<gvec(n * K), kBlock, 0, s>>>(n, L.cmap.p, H.oc, C.out.p, H.xt32.p, na);
    CK_LAUNCH();
    spmv32(kSmoothDot, H.xt32.p, out, b, c);
    note_launch(ctx, 6);
  }
  void spmv(size_t l, int mode, const double2* x, double2* y, const double2* b, KrylovCtl c) {
    if (l == 0) {
      c.dinv = a->dinv.p;
      DK::spmv(ctx, mode, grid0[mode], a->n, a, x, y, b, c);
    } else {
      AmgLevel& L = H.lv[l];
      c.dinv = L.dinv.p;
      DK::csr(ctx, mode, gl[l][mode], L.n, L.row_ptr.p, L.col.p, L.val.p, x, y, b, c, true);
    }
  }
  // out = M_l b; t0 = a free level-0 vector (COCG's q); pre = the level's
  // x = omega D^-1 b is already in xt (fused into the COCG update)
  void run(size_t l, const double2* b, double2* out, double2* t0, KrylovCtl c, bool dot,
           bool pre = false) {
    if (l == 0 && f32 && dot) {
      run0_f32(b, out, c, pre);
      return;
    }
    cudaStream_t s = ctx->stream;
    AmgLevel& L = H.lv[l];
    const int64_t n = L.n;
    const int* na = c.n_active;
    if (l + 1 == H.lv.size()) {
      const int g = (int)std::max<int64_t>(1, std::min<int64_t>((n * 32 + kBlock - 1) / kBlock,
                                                                 (int64_t)ctx->num_sms * 8));
      k_dense<K><<<g, kBlock, 0, s>>>(n, H.minv.p, b, out, na);
      CK_LAUNCH();
      note_launch(ctx, 1);
      if (dot) {  // single-level hierarchy: rho = r^T z here
        k_rho<K><<<std::min(gvec(n * K), grid_vec), kBlock, 0, s>>>(n, b, out, c);
        CK_LAUNCH();
        note_launch(ctx, 1);
      }
      return;
    }
    c.omega = H.omega;
    const double2* dinv = l == 0 ? a->dinv.p : L.dinv.p;
    double2* xt = L.xt.p;
    double2* t = l == 0 ? t0 : L.t.p;
    if (!pre) {
      k_vscale<K, double2><<<gvec(n * K), kBlock, 0, s>>>(n, b, dinv, H.omega, xt, na);
      CK_LAUNCH();
    }
    spmv(l, kResidNR, xt, t, b, c);
    AmgLevel& C = H.lv[l + 1];
    k_restrict<K, double2><<<gvec(C.n * K), kBlock, 0, s>>>(C.n, L.r_ptr.p, L.r_idx.p, t, C.b.p,
                                                            na);
    CK_LAUNCH();
    run(l + 1, C.b.p, C.out.p, t0, c, false);
    if (H.wcycle && l + 2 < H.lv.size()) {
      spmv(l + 1, kResidNR, C.out.p, C.b2.p, C.b.p, c);
      run(l + 1, C.b2.p, C.out2.p, t0, c, false);
      k_axpy1<K><<<gvec(C.n * K), kBlock, 0, s>>>(C.n, C.out.p, C.out2.p, na);
      CK_LAUNCH();
      note_launch(ctx, 2);
    }
    k_prolong<K, double2><<<gvec(n * K), kBlock, 0, s>>>(n, L.cmap.p, H.oc, C.out.p, xt, na);
    CK_LAUNCH();
    spmv(l, dot ? kSmoothDot : kSmooth, xt, out, b, c);
    note_launch(ctx, 5);
  }
};

}  // namespace

void throw_on_breakdown(const SolveOut& out) {
  for (size_t c = 0; c < out.breakdown.size(); ++c)
    if (out.breakdown[c])
      fail(ECT_ERR_SOLVER, "Krylov breakdown (p^T A p or r^T z vanished) on right-hand side " +
                               std::to_string(c));
}

void cocg_solve(ect_ctx* ctx, ect_matrix* a, const double2* b, double2* x, int k,
                const ect_iter_options& opt, SolveOut* out) {
  if (!(opt.tol > 0.0)) fail(ECT_ERR_SOLVER, "solve_iterative: tolerance must be positive");
  if (k < 1 || k > 16) fail(ECT_ERR_SOLVER, "solve: n_rhs must be in 1..16");
  if (!a->symmetric) {  // impedance surface terms: A != A^T
    if (a->n_zero_diag > 0)
      fail(ECT_ERR_SOLVER, "Jacobi preconditioner: " + std::to_string(a->n_zero_diag) +
                               " rows have a zero diagonal");
    out->iters.assign(k, 0);
    out->residual.assign(k, 0.0);
    out->converged.assign(k, 0);
    out->breakdown.assign(k, 0);
    int kb = 1;
    while (kb < k) kb <<= 1;
    with_k(kb, [&](auto D) {
      using DK = decltype(D);
      constexpr int KK = DK::kWidth;
      bicgstab_k<KK>(ctx, a, b, x, k, opt, out);
    });
    return;
  }
  int kk = 1;
  while (kk < k) kk <<= 1;  // internal batch width (padding columns stay at b = 0)
  const int64_t n = a->n;
  cudaStream_t s = ctx->stream;

  out->iters.assign(k, 0);
  out->residual.assign(k, 0.0);
  out->converged.assign(k, 0);
  out->breakdown.assign(k, 0);

  // preconditioner: multigrid (built once per matrix) or point Jacobi
  const bool ext = a->precond == ECT_PRECOND_AMG;
  if (ext && !a->amg) amg_setup(a);
  if (!ext && a->n_zero_diag > 0)
    fail(ECT_ERR_SOLVER, "Jacobi preconditioner: " + std::to_string(a->n_zero_diag) +
                             " rows have a zero diagonal");

  with_k(kk, [&](auto D) {
    using DK = decltype(D);
    constexpr int KW = DK::kWidth;
    const int grid_s = DK::spmv_grid(ctx, kCocg, a);
    const int grid_r = DK::spmv_grid(ctx, kResid, a);
    const int grid_v = DK::vec_grid(ctx, ext);
    std::unique_ptr<Cycle<KW>> cyc;
    if (ext) cyc = std::make_unique<Cycle<KW>>(ctx, a, *a->amg);
    const int grid_max = std::max({grid_s, grid_r, grid_v, cyc ? cyc->max_grid() : 0});
    const size_t vec = (size_t)n * kk;
    // workspace cached on the context (a sweep solves thousands of times)
    auto& W = ctx->ws;
    for (auto* v : {&W.bb, &W.xx, &W.r, &W.p, &W.q}) v->ensure(vec);
    if (ext) W.z.ensure(vec);
    W.st.ensure(kk);
    W.n_active.ensure(1);
    W.counter.ensure(1);
    W.partial.ensure((size_t)grid_max * 4 * kk);
    auto &bb = W.bb, &xx = W.xx, &r = W.r, &p = W.p, &q = W.q;
    auto& st = W.st;
    auto& n_active = W.n_active;
    auto& counter = W.counter;
    auto& partial = W.partial;
    CK(cudaMemsetAsync(st.p, 0, st.bytes(), s));
    CK(cudaMemsetAsync(counter.p, 0, sizeof(unsigned), s));
    CK(cudaMemsetAsync(n_active.p, 0, sizeof(int), s));
    // b in internal layout (zero-padded columns)
    if (kk == k) {
      CK(cudaMemcpyAsync(bb.p, b, vec * sizeof(double2), cudaMemcpyDeviceToDevice, s));
    } else {
      CK(cudaMemsetAsync(bb.p, 0, bb.bytes(), s));
      CK(cudaMemcpy2DAsync(bb.p, kk * sizeof(double2), b, k * sizeof(double2),
                           k * sizeof(double2), n, cudaMemcpyDeviceToDevice, s));
    }
    KrylovCtl ctl{st.p, n_active.p, counter.p, partial.p, opt.tol, opt.max_iter,
                  nullptr, 0, n, n, n};
    DevBuf<double> hist;
    const bool trace = std::getenv("ECT_TRACE_SOLVE") != nullptr;
    if (trace) {
      ctl.hist_cap = std::min(opt.max_iter + 1, 1 << 16);
      ctl.hist_k = kk;
      hist.alloc((size_t)ctl.hist_cap * kk);
      CK(cudaMemsetAsync(hist.p, 0, hist.bytes(), s));
      ctl.hist = hist.p;
    }
    const unsigned all = (kk == 32) ? 0xffffffffu : ((1u << kk) - 1u);
    // (re)start: norms (+ p = D^-1 r, rho with Jacobi); multigrid then sets
    // p = M r and rho = r^T M r
    auto start = [&](unsigned mask, int fresh) {
      if (ext) {
        k_start<KW, true><<<grid_v, kBlock, 0, s>>>(n, bb.p, xx.p, r.p, p.p, nullptr, mask, fresh,
                                                     ctl);
        CK_LAUNCH();
        KrylovCtl c = ctl;
        c.rho_start = 1;
        cyc->run(0, r.p, p.p, q.p, c, true);
      } else {
        DK::start(ctx, grid_v, n, bb.p, xx.p, r.p, p.p, a->dinv.p, mask, fresh, ctl);
      }
      note_launch(ctx, 1);
    };
    start(all, 1);

    auto iteration = [&]() {
          cudaEvent_t ev[2];
          prof_begin(ctx, ev, 0, true, n_active.p, k);
          DK::spmv(ctx, kCocg, grid_s, n, a, p.p, q.p, nullptr, ctl);
          prof_end(ctx, ev);
          cudaEvent_t ev2[2];
          ev2[0] = ev2[1] = nullptr;
          // same sampled iterations as the SpMV, same active-column snapshot
          if (ev[0]) prof_begin(ctx, ev2, 1, false, nullptr, k, prof_snap_of(ctx, ev[0]));
          if (ext) {
            const bool fuse = a->amg->lv.size() > 1;
            k_update<KW, true><<<grid_v, kBlock, 0, s>>>(
                n, r.p, q.p, a->dinv.p, ctl, fuse && !cyc->f32 ? a->amg->lv[0].xt.p : nullptr,
                a->amg->omega, fuse && cyc->f32 ? a->amg->xt32.p : nullptr);
            CK_LAUNCH();
            prof_end(ctx, ev2);
            cudaEvent_t ev3[2];
            ev3[0] = ev3[1] = nullptr;
            if (ev[0]) prof_begin(ctx, ev3, 2, false, nullptr, k, prof_snap_of(ctx, ev[0]));
            cyc->run(0, r.p, W.z.p, q.p, ctl, true, fuse);  // z = M r, rho, beta
            prof_end(ctx, ev3);
            k_pupdate<KW, true><<<grid_v, kBlock, 0, s>>>(n, xx.p, r.p, p.p, nullptr, ctl, W.z.p);
            CK_LAUNCH();
          } else {
            DK::update(ctx, grid_v, n, r.p, q.p, a->dinv.p, ctl);
            DK::pupdate(ctx, grid_v, n, xx.p, r.p, p.p, a->dinv.p, ctl);
            prof_end(ctx, ev2);
          }
          note_launch(ctx, 3);
            };
    // one iteration captured as a CUDA graph (multigrid path only: with Jacobi
    // the iteration is 3 bandwidth-bound launches and a graph gives nothing),
    // kept with the hierarchy across solves
    IterGraph none;
    IterGraph& graph = ext ? a->amg->iter : none;
    if (ext && std::getenv("ECT_NO_GRAPH") == nullptr && !trace) {
      const void* tag[3] = {r.p, partial.p, st.p};
      const bool valid = graph.exec && graph.k == kk && graph.tol == opt.tol &&
                         graph.max_iter == opt.max_iter && graph.tag[0] == tag[0] &&
                         graph.tag[1] == tag[1] && graph.tag[2] == tag[2];
      if (!valid) {
        graph.reset();
        const bool prof_was = ctx->prof.enabled;
        ctx->prof.enabled = false;  // no event records inside the capture
        const int64_t l0 = ctx->timings.kernel_launches;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        iteration();
        CK(cudaStreamEndCapture(s, &graph.graph));
        graph.launches = (int)(ctx->timings.kernel_launches - l0);
        ctx->timings.kernel_launches = l0;  // captured, not launched
        ctx->prof.enabled = prof_was;
        CK(cudaGraphInstantiate(&graph.exec, graph.graph, 0));
        graph.k = kk;
        graph.tol = opt.tol;
        graph.max_iter = opt.max_iter;
        for (int q = 0; q < 3; ++q) graph.tag[q] = tag[q];
      }
    } else if (ext) {
      graph.reset();
    }

    std::vector<RhsState> hs(kk);
    int* flag = ctx->pinned_flag;
    const int chunk = 32;
    for (int restart_round = 0;; ++restart_round) {
      // ---- iterate until no column is active ------------------------------
      int polls_in_flight = 0;
      cudaEvent_t poll_ev[2] = {ctx->ev_a, ctx->ev_b};
      int launched = 0;
      const int cap = opt.max_iter + chunk;  // iterations can never exceed max_iter
      for (; opt.max_iter > 0;) {
        for (int it = 0; it < chunk; ++it) {
          // the multigrid iteration is ~46 launches, most of them 4-30 us
          // coarse-level kernels: replayed as one CUDA graph (captured once per
          // solve) the host enqueues 1 node list instead of 46 launches and
          // stops being the bottleneck of the coarse part; profiled sample
          // iterations go through the plain launches with their events
          if (graph.exec && !prof_sample_next(ctx)) {
            if (ctx->prof.enabled) ++ctx->prof.launches;  // keep the sampling stride
            CK(cudaGraphLaunch(graph.exec, s));
            note_launch(ctx, graph.launches);
            continue;
          }
          iteration();
        }
        launched += chunk;
        CK(cudaMemcpyAsync(flag + (polls_in_flight & 1), n_active.p, sizeof(int),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(poll_ev[polls_in_flight & 1], s));
        ++polls_in_flight;
        if (polls_in_flight >= 2) {
          // wait for the previous poll while the current chunk runs
          const int prev = (polls_in_flight - 2) & 1;
          CK(cudaEventSynchronize(poll_ev[prev]));
          if (flag[prev] == 0) break;
        }
        if (launched > cap + 2 * chunk) break;
      }
      CK(cudaStreamSynchronize(s));
      prof_collect(ctx);
      // ---- true residual confirmation (iterative.cpp:208-216) ------------
      // q <- b - A x (q is free here), st.rnorm <- ||b - A x||
      CK(cudaMemsetAsync(n_active.p, 0xff, sizeof(int), s));  // force the kernel to run
      {
        // mark every column for the residual pass
        CK(cudaMemcpyAsync(hs.data(), st.p, kk * sizeof(RhsState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::vector<RhsState> tmp = hs;
        for (auto& t : tmp) t.status = kActive;
        CK(cudaMemcpyAsync(st.p, tmp.data(), kk * sizeof(RhsState), cudaMemcpyHostToDevice, s));
        DK::spmv(ctx, kResid, grid_r, n, a, xx.p, q.p, bb.p, ctl);
        note_launch(ctx, 1);
        std::vector<RhsState> res(kk);
        CK(cudaMemcpyAsync(res.data(), st.p, kk * sizeof(RhsState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (int c = 0; c < kk; ++c) hs[c].rnorm = res[c].rnorm;  // true ||b - A x||
        CK(cudaMemcpyAsync(st.p, hs.data(), kk * sizeof(RhsState), cudaMemcpyHostToDevice, s));
      }
      unsigned restart_mask = 0;
      for (int c = 0; c < k; ++c) {
        RhsState& t = hs[c];
        if (t.status == kBreakdown) continue;  // reported per column (SolveOut::breakdown)
        const double rel = t.bnorm > 0.0 ? t.rnorm / t.bnorm : 0.0;
        if (t.status == kConverged && rel > opt.tol && t.iters < opt.max_iter &&
            restart_round < 8) {
          restart_mask |= 1u << c;
        }
      }
      if (!restart_mask) break;
      // restart failed columns from their true residual: r <- b - A x
      for (int c = 0; c < kk; ++c)
        if ((restart_mask >> c) & 1u)
          CK(cudaMemcpy2DAsync(r.p + c, kk * sizeof(double2), q.p + c, kk * sizeof(double2),
                               sizeof(double2), n, cudaMemcpyDeviceToDevice, s));
      start(restart_mask, 0);
      // keep the other columns frozen
      CK(cudaStreamSynchronize(s));
    }
    if (trace) {  // dev: recurrence residual history, every 10th iteration
      std::vector<double> h((size_t)ctl.hist_cap * kk);
      CK(cudaMemcpy(h.data(), hist.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost));
      for (int c = 0; c < k; ++c) {
        std::fprintf(stderr, "[ect trace] column %d (iterations %d, true %.3e):", c, hs[c].iters,
                     hs[c].bnorm > 0.0 ? hs[c].rnorm / hs[c].bnorm : 0.0);
        for (int it = 1; it <= hs[c].iters && it < ctl.hist_cap; it += (it < 20 ? 1 : 10))
          std::fprintf(stderr, " %d:%.2e", it, h[(size_t)it * kk + c]);
        std::fprintf(stderr, "\n");
      }
    }
    for (int c = 0; c < k; ++c) {
      const RhsState& t = hs[c];
      out->iters[c] = t.iters;
      const double rel = t.bnorm > 0.0 ? t.rnorm / t.bnorm : 0.0;
      out->residual[c] = rel;
      out->converged[c] = (t.status == kZeroRhs) || (t.status == kConverged && rel <= opt.tol);
      out->breakdown[c] = t.status == kBreakdown;
    }
    if (kk == k) {
      CK(cudaMemcpyAsync(x, xx.p, vec * sizeof(double2), cudaMemcpyDeviceToDevice, s));
    } else {
      CK(cudaMemcpy2DAsync(x, k * sizeof(double2), xx.p, kk * sizeof(double2),
                           k * sizeof(double2), n, cudaMemcpyDeviceToDevice, s));
    }
    CK(cudaStreamSynchronize(s));
  });
}


// ============================================================================
// Distributed (row-partitioned) solve — SURVEY §8(e), configs[4].
// Each part owns a contiguous node range (dist_plan.cpp); per SpMV the ghost
// x values are exchanged with the neighbour parts (NCCL send/recv, or device
// copies when all parts run in this process on one GPU), and the per-iteration
// dot products are summed across parts (ncclAllReduce of <= 4k doubles, or a
// fixed-order device sum) before the scalar finalisation (k_fin). The
// in-process mode runs exactly the same kernels and partition logic: it is how
// the partitioned path is validated on a single GPU.
namespace {

template <int K>
__global__ void k_pack(const double2* __restrict__ v, const int* __restrict__ nodes, int64_t ns,
                       const int* __restrict__ cnodes, int64_t nsc,
                       const int* __restrict__ cond_local, int64_t na_local, double2* out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ns * 3 * K; e += stride) {
    const int64_t nd = e / (3 * K), c = e - nd * 3 * K;
    out[e] = v[(int64_t)nodes[nd] * 3 * K + c];
  }
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nsc * K; e += stride) {
    const int64_t nd = e / K, k = e - nd * K;
    out[ns * 3 * K + e] = v[(na_local + cond_local[cnodes[nd]]) * K + k];
  }
}

// fixed-order sum of the parts' totals, broadcast back to every part
__global__ void k_sum_parts(double* const* reds, int n_parts, int nv) {
  for (int j = threadIdx.x; j < nv; j += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < n_parts; ++r) s += reds[r][j];
    for (int r = 0; r < n_parts; ++r) reds[r][j] = s;
  }
}

NbView part_view(const ect_part* P) {
  NbView v{P->blk_ptr.p, P->nbe_col.p, reinterpret_cast<const double*>(P->nbe_blk.p), P->nbe_slots,
           P->cpl_ptr.p, P->cpl_idx.p, reinterpret_cast<const double*>(P->cpl.p), P->ncpl,
           P->cond_local.p, P->plan.L, P->plan.na_local()};
  if (P->has_nbe) {  // sliced-ELL copy of the part's blocks (the default SpMV layout)
    v.blk = reinterpret_cast<const double*>(P->nbe_blk.p);
    v.blk_col = P->nbe_col.p;
    v.nblk = P->nbe_slots;
    v.e_off = P->nbe_off.p;
  }
  return v;
}

template <int K>
KFn part_fn(const ect_part* P, int mode) {
  (void)P;
  return nbe_fn<K>(mode);
}

}  // namespace

ect_part* create_part(ect_mesh* m, ect_matrix* a, const int64_t* splits, int n_parts, int part) {
  ect_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  if (!a->has_nb) fail(ECT_ERR_SOLVER, "part: the global matrix must be assembled in NB format");
  const int64_t nn = m->n_nodes;
  // host copies of the neighbour structure, conductor map and NB coupling index
  std::vector<int> nbr_off(nn + 1), cond(nn), cpl_ptr(nn + 1);
  CK(cudaMemcpyAsync(nbr_off.data(), m->nbr_off.p, (nn + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(cond.data(), m->cond_fwd.p, nn * sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(cpl_ptr.data(), a->nb_cpl_ptr.p, (nn + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::vector<int> nbr(nbr_off[nn]);
  CK(cudaMemcpy(nbr.data(), m->nbr.p, nbr.size() * sizeof(int), cudaMemcpyDeviceToHost));
  auto P = std::make_unique<ect_part>();
  P->ctx = ctx;
  P->plan = build_halo_plan(nn, nbr_off.data(), nbr.data(), cond.data(), splits, n_parts, part);
  const HaloPlan& H = P->plan;
  P->n_nodes_global = nn;
  P->na_global = 3 * nn;
  P->n_global = 3 * nn + m->n_cond;
  const int64_t L = H.L, G = H.G, NL = H.n_local();
  // global node -> local node map (owned, ghosts; -1 elsewhere) on the device
  std::vector<int> g2l(nn, -1);
  for (int64_t i = 0; i < L; ++i) g2l[H.n0 + i] = (int)i;
  for (int64_t q = 0; q < G; ++q) g2l[H.ghost_nodes[q]] = (int)(L + q);
  DevBuf<int> d_g2l(nn);
  CK(cudaMemcpy(d_g2l.p, g2l.data(), nn * sizeof(int), cudaMemcpyHostToDevice));
  // interior rows (no ghost column): the longest run of such owned nodes; its
  // SpMV runs while the halo is in flight, the rest after it lands
  {
    int64_t best_lo = 0, best_len = 0, run_lo = 0;
    for (int64_t i = 0; i <= L; ++i) {
      bool boundary = i == L;
      if (i < L)
        for (int q = nbr_off[H.n0 + i]; q < nbr_off[H.n0 + i + 1] && !boundary; ++q)
          boundary = g2l[nbr[q]] >= L;
      if (boundary) {
        if (i - run_lo > best_len) {
          best_len = i - run_lo;
          best_lo = run_lo;
        }
        run_lo = i + 1;
      }
    }
    P->int_lo = best_lo;
    P->int_hi = best_lo + best_len;
  }
  // block pointers of the owned nodes (their NB-E slots come from the global NB-E below)
  const int64_t q0 = nbr_off[H.n0], q1 = nbr_off[H.n1];
  P->nblk = q1 - q0;
  P->blk_ptr.alloc(L + 1);
  {
    std::vector<int> bp(L + 1);
    for (int64_t i = 0; i <= L; ++i) bp[i] = nbr_off[H.n0 + i] - (int)q0;
    CK(cudaMemcpy(P->blk_ptr.p, bp.data(), (L + 1) * sizeof(int), cudaMemcpyHostToDevice));
  }
  // couplings of the owned nodes
  const int64_t c0 = cpl_ptr[H.n0], c1 = cpl_ptr[H.n1];
  P->ncpl = c1 - c0;
  P->cpl_ptr.alloc(L + 1);
  {
    std::vector<int> cp(L + 1);
    for (int64_t i = 0; i <= L; ++i) cp[i] = cpl_ptr[H.n0 + i] - (int)c0;
    CK(cudaMemcpy(P->cpl_ptr.p, cp.data(), (L + 1) * sizeof(int), cudaMemcpyHostToDevice));
  }
  P->cpl_idx.alloc(std::max<int64_t>(1, P->ncpl));
  P->cpl.alloc(4 * std::max<int64_t>(1, P->ncpl));
  if (P->ncpl) {
    std::vector<int2> ci(P->ncpl);
    CK(cudaMemcpy(ci.data(), a->nb_cpl_idx.p + c0, P->ncpl * sizeof(int2), cudaMemcpyDeviceToHost));
    for (auto& e : ci) {
      const int l = g2l[e.x];
      e = make_int2(l, H.local_vdof[l]);
    }
    CK(cudaMemcpy(P->cpl_idx.p, ci.data(), P->ncpl * sizeof(int2), cudaMemcpyHostToDevice));
    for (int pl = 0; pl < 2; ++pl)
      CK(cudaMemcpyAsync(reinterpret_cast<double*>(P->cpl.p) + 4 * pl * P->ncpl,
                         reinterpret_cast<const double*>(a->nb_cpl.p) + 4 * (pl * a->nb_ncpl + c0),
                         4 * P->ncpl * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  P->cond_local.alloc(std::max<int64_t>(1, L + G));
  CK(cudaMemcpy(P->cond_local.p, H.local_vdof.data(), (L + G) * sizeof(int), cudaMemcpyHostToDevice));
  // Jacobi diagonal of the owned rows in the local layout (ghost rows unused)
  P->dinv.alloc(NL);
  CK(cudaMemsetAsync(P->dinv.p, 0, P->dinv.bytes(), s));
  CK(cudaMemcpyAsync(P->dinv.p, a->dinv.p + 3 * H.n0, 3 * L * sizeof(double2),
                     cudaMemcpyDeviceToDevice, s));
  if (H.Vo)
    CK(cudaMemcpyAsync(P->dinv.p + H.na_local(), a->dinv.p + 3 * nn + H.c0, H.Vo * sizeof(double2),
                       cudaMemcpyDeviceToDevice, s));
  // send lists
  for (const auto& peer : H.peers) {
    ect_part::Peer d;
    d.ns = (int64_t)peer.send_nodes.size();
    d.nsc = (int64_t)peer.send_cond_nodes.size();
    d.send_nodes.alloc(std::max<int64_t>(1, d.ns));
    d.send_cond.alloc(std::max<int64_t>(1, d.nsc));
    if (d.ns) CK(cudaMemcpy(d.send_nodes.p, peer.send_nodes.data(), d.ns * sizeof(int), cudaMemcpyHostToDevice));
    if (d.nsc) CK(cudaMemcpy(d.send_cond.p, peer.send_cond_nodes.data(), d.nsc * sizeof(int), cudaMemcpyHostToDevice));
    P->peers.push_back(std::move(d));
  }
  // NB-E copy of the part's blocks (same layout and kernels as a whole matrix)
  {
    const int64_t nch = (L + 31) / 32;
    DevBuf<int> w(nch + 1);
    const int cg = (int)std::min<int64_t>((nch + 255) / 256, (int64_t)ctx->num_sms * 16);
    k_nbe_width<<<std::max(cg, 1), 256, 0, s>>>(P->blk_ptr.p, L, nch, w.p);
    CK_LAUNCH();
    P->nbe_off.alloc(nch + 1);
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, w.p, P->nbe_off.p, nch + 1, s));
    CK(cub::DeviceScan::ExclusiveSum(cub_scratch(ctx, tmp), tmp, w.p, P->nbe_off.p, nch + 1, s));
    int slots = 0;
    CK(cudaMemcpyAsync(&slots, P->nbe_off.p + nch, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    P->nbe_col.alloc(std::max(1, slots));
    P->nbe_blk.alloc(6 * (size_t)std::max(1, slots));
    if (!a->has_nbe) fail(ECT_ERR_SOLVER, "part: the global matrix has no NB-E blocks");
    const int fg = (int)std::min<int64_t>((32 * nch + 255) / 256, (int64_t)ctx->num_sms * 16);
    k_part_nbe_fill<<<std::max(fg, 1), 256, 0, s>>>(
        P->blk_ptr.p, L, H.n0, a->nbe_off.p, a->nbe_col.p,
        reinterpret_cast<const double*>(a->nbe_blk.p), a->nbe_slots, d_g2l.p, P->nbe_off.p, nch,
        P->nbe_col.p, reinterpret_cast<double*>(P->nbe_blk.p), slots);
    CK_LAUNCH();
    P->nbe_slots = slots;
    P->has_nbe = true;
    note_launch(ctx, 2);
  }
  CK(cudaStreamSynchronize(s));
  note_launch(ctx, 1);
  return P.release();
}

// The part of `create_part` built without a global matrix: the slab's rows
// are patterned and assembled on their own (build_pattern / assemble_values
// over nodes [n0, n1), global indices, the other rows empty), the slab's NB
// blocks cut from that CSR, then the same local renumbering, halo plan and
// NB-E layout. Device memory per rank ~ the slab's share of the matrix, as the
// reference's per-partition assembly (assembly.cpp:246-258) and the paper's
// per-rank matrices.
ect_part* create_part_assembled(ect_mesh* m, const ect_materials& mats, const int64_t* splits,
                                int n_parts, int part) {
  ect_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  if (mats.ibc_enabled) fail(ECT_ERR_SOLVER, "part: impedance surface terms are not partitioned");
  const int64_t nn = m->n_nodes;
  if (!m->have_nbr) {  // the mesh-level neighbour lists (K1) are shared by every slab
    ect_matrix probe;
    probe.ctx = ctx;
    build_pattern(m, &probe, 0, 0);
  }
  std::vector<int> nbr_off(nn + 1), cond(nn);
  CK(cudaMemcpyAsync(nbr_off.data(), m->nbr_off.p, (nn + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(cond.data(), m->cond_fwd.p, nn * sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::vector<int> nbr(nbr_off[nn]);
  CK(cudaMemcpy(nbr.data(), m->nbr.p, nbr.size() * sizeof(int), cudaMemcpyDeviceToHost));
  auto P = std::make_unique<ect_part>();
  P->ctx = ctx;
  P->plan = build_halo_plan(nn, nbr_off.data(), nbr.data(), cond.data(), splits, n_parts, part);
  const HaloPlan& H = P->plan;
  P->n_nodes_global = nn;
  P->na_global = 3 * nn;
  P->n_global = 3 * nn + m->n_cond;
  const int64_t L = H.L, G = H.G, NL = H.n_local();
  std::vector<int> g2l(nn, -1);
  for (int64_t i = 0; i < L; ++i) g2l[H.n0 + i] = (int)i;
  for (int64_t q = 0; q < G; ++q) g2l[H.ghost_nodes[q]] = (int)(L + q);
  DevBuf<int> d_g2l(nn);
  CK(cudaMemcpy(d_g2l.p, g2l.data(), nn * sizeof(int), cudaMemcpyHostToDevice));
  {
    int64_t best_lo = 0, best_len = 0, run_lo = 0;
    for (int64_t i = 0; i <= L; ++i) {
      bool boundary = i == L;
      if (i < L)
        for (int q = nbr_off[H.n0 + i]; q < nbr_off[H.n0 + i + 1] && !boundary; ++q)
          boundary = g2l[nbr[q]] >= L;
      if (boundary) {
        if (i - run_lo > best_len) {
          best_len = i - run_lo;
          best_lo = run_lo;
        }
        run_lo = i + 1;
      }
    }
    P->int_lo = best_lo;
    P->int_hi = best_lo + best_len;
  }
  // ---- the slab's rows, patterned and assembled alone ----------------------
  ect_matrix slab;
  slab.ctx = ctx;
  build_pattern(m, &slab, H.n0, H.n1);
  assemble_values(m, mats, &slab);
  // ---- its NB blocks (owned nodes only) ------------------------------------
  const int64_t q0 = nbr_off[H.n0], q1 = nbr_off[H.n1];
  P->nblk = q1 - q0;
  DevBuf<int> cnt(nn + 1), cpl_ptr(nn + 1);
  CK(cudaMemsetAsync(cnt.p, 0, cnt.bytes(), s));
  const int cgrid = (int)std::max<int64_t>(1, std::min<int64_t>((L + 255) / 256, ctx->num_sms * 16));
  k_cpl_count<<<cgrid, 256, 0, s>>>(m->nbr_off.p, m->nbr_cond.p, m->cond_fwd.p, H.n0, H.n1, cnt.p);
  CK_LAUNCH();
  size_t tmp = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.p, cpl_ptr.p, nn + 1, s));
  CK(cub::DeviceScan::ExclusiveSum(cub_scratch(ctx, tmp), tmp, cnt.p, cpl_ptr.p, nn + 1, s));
  std::vector<int> h_cpl(nn + 1);
  CK(cudaMemcpyAsync(h_cpl.data(), cpl_ptr.p, (nn + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const int64_t c0 = h_cpl[H.n0];  // = 0: only owned nodes were counted
  P->ncpl = h_cpl[H.n1] - c0;
  DevBuf<double2> blk(6 * std::max<int64_t>(1, P->nblk));
  DevBuf<int2> cidx(std::max<int64_t>(1, P->ncpl));
  P->cpl.alloc(4 * std::max<int64_t>(1, P->ncpl));
  DevBuf<int> bad(1);
  CK(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
  const int wgrid = (int)std::max<int64_t>(1, std::min<int64_t>((32 * L + 255) / 256, ctx->num_sms * 16));
  k_build_nb<<<wgrid, 256, 0, s>>>(slab.row_ptr.p, slab.val.p, m->nbr_off.p, m->nbr.p,
                                   m->nbr_cond.p, m->cond_fwd.p, cpl_ptr.p, nn,
                                   reinterpret_cast<double*>(blk.p), P->nblk, cidx.p,
                                   reinterpret_cast<double*>(P->cpl.p), P->ncpl, bad.p, H.n0, H.n1,
                                   q0, c0);
  CK_LAUNCH();
  int h_bad = 0;
  CK(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (h_bad) fail(ECT_ERR_SOLVER, "part: node blocks carry imaginary off-diagonal parts");
  // local node-block structure
  P->blk_ptr.alloc(L + 1);
  P->cpl_ptr.alloc(L + 1);
  {
    std::vector<int> bp(L + 1), cp(L + 1);
    for (int64_t i = 0; i <= L; ++i) {
      bp[i] = nbr_off[H.n0 + i] - (int)q0;
      cp[i] = h_cpl[H.n0 + i] - (int)c0;
    }
    CK(cudaMemcpy(P->blk_ptr.p, bp.data(), (L + 1) * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(P->cpl_ptr.p, cp.data(), (L + 1) * sizeof(int), cudaMemcpyHostToDevice));
  }
  DevBuf<int> lcol(std::max<int64_t>(1, P->nblk));
  {
    std::vector<int> lc(P->nblk);
    for (int64_t q = q0; q < q1; ++q) lc[q - q0] = g2l[nbr[q]];
    if (P->nblk) CK(cudaMemcpy(lcol.p, lc.data(), P->nblk * sizeof(int), cudaMemcpyHostToDevice));
  }
  P->cpl_idx.alloc(std::max<int64_t>(1, P->ncpl));
  if (P->ncpl) {
    std::vector<int2> ci(P->ncpl);
    CK(cudaMemcpy(ci.data(), cidx.p, P->ncpl * sizeof(int2), cudaMemcpyDeviceToHost));
    for (auto& e : ci) {
      const int l = g2l[e.x];
      e = make_int2(l, H.local_vdof[l]);
    }
    CK(cudaMemcpy(P->cpl_idx.p, ci.data(), P->ncpl * sizeof(int2), cudaMemcpyHostToDevice));
  }
  P->cond_local.alloc(std::max<int64_t>(1, L + G));
  CK(cudaMemcpy(P->cond_local.p, H.local_vdof.data(), (L + G) * sizeof(int), cudaMemcpyHostToDevice));
  P->dinv.alloc(NL);
  CK(cudaMemsetAsync(P->dinv.p, 0, P->dinv.bytes(), s));
  CK(cudaMemcpyAsync(P->dinv.p, slab.dinv.p + 3 * H.n0, 3 * L * sizeof(double2),
                     cudaMemcpyDeviceToDevice, s));
  if (H.Vo)
    CK(cudaMemcpyAsync(P->dinv.p + H.na_local(), slab.dinv.p + 3 * nn + H.c0,
                       H.Vo * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  for (const auto& peer : H.peers) {
    ect_part::Peer d;
    d.ns = (int64_t)peer.send_nodes.size();
    d.nsc = (int64_t)peer.send_cond_nodes.size();
    d.send_nodes.alloc(std::max<int64_t>(1, d.ns));
    d.send_cond.alloc(std::max<int64_t>(1, d.nsc));
    if (d.ns) CK(cudaMemcpy(d.send_nodes.p, peer.send_nodes.data(), d.ns * sizeof(int), cudaMemcpyHostToDevice));
    if (d.nsc) CK(cudaMemcpy(d.send_cond.p, peer.send_cond_nodes.data(), d.nsc * sizeof(int), cudaMemcpyHostToDevice));
    P->peers.push_back(std::move(d));
  }
  // NB-E layout of the part
  {
    const int64_t nch = (L + 31) / 32;
    DevBuf<int> w(nch + 1);
    const int cg = (int)std::min<int64_t>((nch + 255) / 256, (int64_t)ctx->num_sms * 16);
    k_nbe_width<<<std::max(cg, 1), 256, 0, s>>>(P->blk_ptr.p, L, nch, w.p);
    CK_LAUNCH();
    P->nbe_off.alloc(nch + 1);
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, w.p, P->nbe_off.p, nch + 1, s));
    CK(cub::DeviceScan::ExclusiveSum(cub_scratch(ctx, tmp), tmp, w.p, P->nbe_off.p, nch + 1, s));
    int slots = 0;
    CK(cudaMemcpyAsync(&slots, P->nbe_off.p + nch, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    P->nbe_col.alloc(std::max(1, slots));
    P->nbe_blk.alloc(6 * (size_t)std::max(1, slots));
    const int fg = (int)std::min<int64_t>((32 * nch + 255) / 256, (int64_t)ctx->num_sms * 16);
    k_nbe_fill<<<std::max(fg, 1), 256, 0, s>>>(P->blk_ptr.p, lcol.p,
                                                reinterpret_cast<const double*>(blk.p), P->nblk,
                                                L, nch, P->nbe_off.p, P->nbe_col.p,
                                                reinterpret_cast<double*>(P->nbe_blk.p), slots);
    CK_LAUNCH();
    P->nbe_slots = slots;
    P->has_nbe = true;
  }
  note_launch(ctx, 6);
  CK(cudaStreamSynchronize(s));
  return P.release();
}

namespace {

// Chronopoulos-Gear COCG vector kernels (distributed solve): owned rows, a
// thread owns CW adjacent columns of a row (as k_update).
// (re)start of the masked columns: [x = 0, r = b when fresh]; z = D^-1 r; p = s = 0
template <int K>
__global__ void __launch_bounds__(kBlock)
k_cg_init(const double2* __restrict__ b, double2* __restrict__ x, double2* __restrict__ r,
          double2* __restrict__ z, double2* __restrict__ p, double2* __restrict__ sv,
          const double2* __restrict__ dinv, unsigned mask, int fresh, KrylovCtl ctl) {
  constexpr int CW = VecMap<K>::CW, KH = VecMap<K>::KH;
  const int h = (threadIdx.x & 31) % KH, kb = h * CW;
  const int64_t len0 = ctl.e0 - ctl.s0, rows = len0 + (ctl.e1 - ctl.s1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * KH;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / KH;
    const int64_t i = j < len0 ? ctl.s0 + j : ctl.s1 + (j - len0);
    const double2 d = dinv[i];
#pragma unroll
    for (int c = 0; c < CW; ++c) {
      if (!((mask >> (kb + c)) & 1u)) continue;
      const int64_t idx = i * K + kb + c;
      double2 rv;
      if (fresh) {
        rv = b[idx];
        x[idx] = make_double2(0.0, 0.0);
        r[idx] = rv;
      } else {
        rv = r[idx];
      }
      z[idx] = cmul(d, rv);
      p[idx] = sv[idx] = make_double2(0.0, 0.0);
    }
  }
}

// one fused step (active columns): p = z + beta p, s = w + beta s (s = A p by
// recurrence), x += alpha p, r -= alpha s, z = D^-1 r
template <int K>
__global__ void __launch_bounds__(kBlock)
k_cg_step(double2* __restrict__ x, double2* __restrict__ r, double2* __restrict__ z,
          double2* __restrict__ p, double2* __restrict__ sv, const double2* __restrict__ w,
          const double2* __restrict__ dinv, KrylovCtl ctl) {
  constexpr int CW = VecMap<K>::CW, KH = VecMap<K>::KH;
  if (*ctl.n_active == 0) return;
  const int h = (threadIdx.x & 31) % KH, kb = h * CW;
  bool act[CW];
  double2 alpha[CW], beta[CW];
#pragma unroll
  for (int c = 0; c < CW; ++c) {
    const RhsState& st = ctl.st[kb + c];
    act[c] = st.status == kActive;
    alpha[c] = st.alpha;
    beta[c] = st.beta;
  }
  const int64_t len0 = ctl.e0 - ctl.s0, rows = len0 + (ctl.e1 - ctl.s1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * KH;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / KH;
    const int64_t i = j < len0 ? ctl.s0 + j : ctl.s1 + (j - len0);
    const double2 d = dinv[i];
#pragma unroll
    for (int c = 0; c < CW; ++c) {
      if (!act[c]) continue;
      const int64_t idx = i * K + kb + c;
      const double2 pv = cadd(z[idx], cmul(beta[c], p[idx]));
      const double2 svv = cadd(w[idx], cmul(beta[c], sv[idx]));
      p[idx] = pv;
      sv[idx] = svv;
      x[idx] = cadd(x[idx], cmul(alpha[c], pv));
      const double2 rv = csub(r[idx], cmul(alpha[c], svv));
      r[idx] = rv;
      z[idx] = cmul(d, rv);
    }
  }
}

template <int K>
struct PartState {
  DevBuf<double2> b, x, r, p, q, z, sv;  // q: w = A z (and the true residual)
  DevBuf<RhsState> st;
  DevBuf<int> n_active;
  DevBuf<unsigned> counter;
  DevBuf<double> partial, red;
  KrylovCtl ctl{};
};

template <int K>
void dist_solve_k(ect_part** parts, int R, ect_comm* comm, const double2* b_global,
                  double2* x_global, int k, const ect_iter_options& opt, SolveOut* out) {
  using DK = Dispatch<K>;
  ect_ctx* ctx = parts[0]->ctx;
  cudaStream_t s = ctx->stream;
  for (int r = 0; r < R; ++r)
    if (parts[r]->ctx != ctx) fail(ECT_ERR_SOLVER, "dist_solve: in-process parts must share a context");
  if (comm && R != 1) fail(ECT_ERR_SOLVER, "dist_solve: with a communicator each process owns one part");
  const int grid_s = grid_for(ctx, part_fn<K>(parts[0], kCgDot).fn,
                              part_fn<K>(parts[0], kCgDot).block);
  const int grid_v = DK::vec_grid(ctx);
  const int grid_max = std::max(grid_s, grid_v);
  const int64_t na_g = parts[0]->na_global;
  std::vector<PartState<K>> S(R);
  DevBuf<double*> reds(R);
  std::vector<double*> h_reds(R);
  for (int r = 0; r < R; ++r) {
    const HaloPlan& H = parts[r]->plan;
    const int64_t NL = H.n_local();
    PartState<K>& P = S[r];
    for (auto* v : {&P.b, &P.x, &P.r, &P.p, &P.q, &P.z, &P.sv}) {
      v->alloc(NL * K);
      CK(cudaMemsetAsync(v->p, 0, v->bytes(), s));
    }
    P.st.alloc(K); P.n_active.alloc(1); P.counter.alloc(1);
    P.partial.alloc((size_t)grid_max * 5 * K); P.red.alloc(5 * K);
    CK(cudaMemsetAsync(P.st.p, 0, P.st.bytes(), s));
    CK(cudaMemsetAsync(P.counter.p, 0, sizeof(unsigned), s));
    CK(cudaMemsetAsync(P.n_active.p, 0, sizeof(int), s));
    P.ctl = KrylovCtl{P.st.p, P.n_active.p, P.counter.p, P.partial.p, opt.tol, opt.max_iter,
                      P.red.p, 0, 3 * H.L, H.na_local(), H.na_local() + H.Vo};
    // owned rows of b: A rows [3 n0, 3 n1), V rows [na + c0, na + c0 + Vo)
    CK(cudaMemcpyAsync(P.b.p, b_global + 3 * H.n0 * K, 3 * H.L * K * sizeof(double2),
                       cudaMemcpyDeviceToDevice, s));
    if (H.Vo)
      CK(cudaMemcpyAsync(P.b.p + H.na_local() * K, b_global + (na_g + H.c0) * K,
                         H.Vo * K * sizeof(double2), cudaMemcpyDeviceToDevice, s));
    h_reds[r] = P.red.p;
  }
  CK(cudaMemcpyAsync(reds.p, h_reds.data(), R * sizeof(double*), cudaMemcpyHostToDevice, s));

  auto allreduce = [&](int nv) {
    if (comm) nccl_allreduce_sum(comm, S[0].red.p, nv, s);
    else if (R > 1) { k_sum_parts<<<1, 64, 0, s>>>(reds.p, R, nv); CK_LAUNCH(); }
  };
  // ghost exchange of vector v (member pointer of PartState)
  // ghost exchange of vector v; the transfers run on stream `hs_`, after the
  // packing kernels (on s) have been recorded
  auto halo = [&](DevBuf<double2> PartState<K>::*v, cudaStream_t hs_) {
    for (int r = 0; r < R; ++r) {
      ect_part* P = parts[r];
      for (size_t i = 0; i < P->peers.size(); ++i) {
        auto& d = P->peers[i];
        const int64_t cnt = d.ns * 3 * K + d.nsc * K;
        d.sendbuf.ensure(std::max<int64_t>(1, cnt));
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>((cnt + 255) / 256, ctx->num_sms * 8));
        k_pack<K><<<g, 256, 0, s>>>((S[r].*v).p, d.send_nodes.p, d.ns, d.send_cond.p, d.nsc,
                                    P->cond_local.p, P->plan.na_local(), d.sendbuf.p);
        CK_LAUNCH();
      }
    }
    if (hs_ != s) {
      CK(cudaEventRecord(ctx->ev_h1, s));
      CK(cudaStreamWaitEvent(hs_, ctx->ev_h1, 0));
    }
    if (comm) nccl_group_start();
    for (int r = 0; r < R; ++r) {
      ect_part* P = parts[r];
      const HaloPlan& H = P->plan;
      double2* base = (S[r].*v).p;
      for (size_t i = 0; i < H.peers.size(); ++i) {
        const HaloPeer& hp = H.peers[i];
        double2* dstA = base + 3 * (H.L + hp.recv_node_begin) * K;
        double2* dstV = base + (H.na_local() + H.Vo + hp.recv_v_begin) * K;
        if (comm) {
          const auto& d = P->peers[i];
          nccl_send(comm, d.sendbuf.p, 2 * d.ns * 3 * K, hp.part, hs_);
          if (d.nsc) nccl_send(comm, d.sendbuf.p + d.ns * 3 * K, 2 * d.nsc * K, hp.part, hs_);
          nccl_recv(comm, dstA, 2 * hp.recv_node_count * 3 * K, hp.part, hs_);
          if (hp.recv_v_count) nccl_recv(comm, dstV, 2 * hp.recv_v_count * K, hp.part, hs_);
        } else {
          // the owner's send buffer for this part
          ect_part* Q = parts[hp.part];
          size_t qi = 0;
          while (qi < Q->plan.peers.size() && Q->plan.peers[qi].part != r) ++qi;
          if (qi == Q->plan.peers.size()) fail(ECT_ERR_SOLVER, "halo plan: asymmetric peers");
          const auto& d = Q->peers[qi];
          if (d.ns != hp.recv_node_count || d.nsc != hp.recv_v_count)
            fail(ECT_ERR_SOLVER, "halo plan: send/receive sizes differ");
          CK(cudaMemcpyAsync(dstA, d.sendbuf.p, d.ns * 3 * K * sizeof(double2),
                             cudaMemcpyDeviceToDevice, hs_));
          if (d.nsc)
            CK(cudaMemcpyAsync(dstV, d.sendbuf.p + d.ns * 3 * K, d.nsc * K * sizeof(double2),
                               cudaMemcpyDeviceToDevice, hs_));
        }
      }
    }
    if (comm) nccl_group_end();
    if (hs_ != s) CK(cudaEventRecord(ctx->ev_h2, hs_));
  };
  // rows of nodes [lo, hi) of every part; add: accumulate the dot totals
  auto spmv_rows = [&](int mode, DevBuf<double2> PartState<K>::*xin,
                       DevBuf<double2> PartState<K>::*yout, bool with_b, int64_t lo, int64_t hi,
                       bool add, int r) {
    NbView v = part_view(parts[r]);
    v.node_begin = lo;
    v.n_nodes = hi;
    const double2* xp = (S[r].*xin).p;
    double2* yp = (S[r].*yout).p;
    const double2* bp = !with_b ? nullptr : mode == kCgDot ? S[r].r.p : S[r].b.p;
    KrylovCtl c = S[r].ctl;
    c.red_add = add ? 1 : 0;
    void* args[] = {&v, &xp, &yp, &bp, &c};
    const KFn f = part_fn<K>(parts[r], mode);
    CK(cudaLaunchKernel(f.fn, dim3(grid_s), dim3(f.block), args, 0, s));
  };
  auto spmv = [&](int mode, DevBuf<double2> PartState<K>::*xin, DevBuf<double2> PartState<K>::*yout,
                  bool with_b) {
    for (int r = 0; r < R; ++r)
      spmv_rows(mode, xin, yout, with_b, 0, parts[r]->plan.L, false, r);
  };
  // q = A p with the halo exchange overlapped: interior rows while the ghost
  // values travel (halo stream), then the rows that read ghosts
  const bool overlap = true;  // halo transfers on their own stream
  if (!ctx->halo_stream) {
    CK(cudaStreamCreateWithFlags(&ctx->halo_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_h1, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_h2, cudaEventDisableTiming));
  }
  // w = A z with the fused dots (b slot = r), halo of z overlapped
  auto spmv_overlapped = [&](DevBuf<double2> PartState<K>::*xin,
                             DevBuf<double2> PartState<K>::*yout) {
    halo(xin, overlap ? ctx->halo_stream : s);
    for (int r = 0; r < R; ++r) {
      const ect_part* P = parts[r];
      if (P->int_hi > P->int_lo) spmv_rows(kCgDot, xin, yout, true, P->int_lo, P->int_hi, false, r);
    }
    if (overlap) CK(cudaStreamWaitEvent(s, ctx->ev_h2, 0));
    for (int r = 0; r < R; ++r) {
      const ect_part* P = parts[r];
      const bool any = P->int_hi > P->int_lo;
      if (P->int_lo > 0) spmv_rows(kCgDot, xin, yout, true, 0, P->int_lo, any, r);
      if (P->int_hi < P->plan.L)
        spmv_rows(kCgDot, xin, yout, true, any ? P->int_hi : P->int_lo, P->plan.L,
                  any || P->int_lo > 0, r);
    }
  };
  auto fin = [&](int what, unsigned mask, int fresh) {
    for (int r = 0; r < R; ++r) {
      KrylovCtl c = S[r].ctl;
      if (what == kFinAlpha) k_fin<K, kFinAlpha><<<1, 32, 0, s>>>(c, mask, fresh);
      else if (what == kFinUpdate) k_fin<K, kFinUpdate><<<1, 32, 0, s>>>(c, mask, fresh);
      else if (what == kFinStart) k_fin<K, kFinStart><<<1, 32, 0, s>>>(c, mask, fresh);
      else if (what == kFinCg) k_fin<K, kFinCg><<<1, 32, 0, s>>>(c, mask, fresh);
      else if (what == kFinCgStart) k_fin<K, kFinCgStart><<<1, 32, 0, s>>>(c, mask, fresh);
      else k_fin<K, kFinResid><<<1, 32, 0, s>>>(c, mask, fresh);
      CK_LAUNCH();
    }
  };
  // Chronopoulos-Gear COCG: one reduction (r^T z, w^T z, ||r||) per iteration
  auto start = [&](unsigned mask, int fresh) {
    for (int r = 0; r < R; ++r) {
      k_cg_init<K><<<grid_v, kBlock, 0, s>>>(S[r].b.p, S[r].x.p, S[r].r.p, S[r].z.p, S[r].p.p,
                                             S[r].sv.p, parts[r]->dinv.p, mask, fresh, S[r].ctl);
      CK_LAUNCH();
    }
    for (int r = 0; r < R; ++r) CK(cudaMemsetAsync(S[r].n_active.p, 0xff, sizeof(int), s));
    spmv_overlapped(&PartState<K>::z, &PartState<K>::q);
    allreduce(5 * K);
    fin(kFinCgStart, mask, fresh);
  };

  const unsigned all = (K == 32) ? 0xffffffffu : ((1u << K) - 1u);
  start(all, 1);
  out->iters.assign(k, 0);
  out->residual.assign(k, 0.0);
  out->converged.assign(k, 0);
  std::vector<RhsState> hs(K);
  int* flag = ctx->pinned_flag;
  const int chunk = 16;
  cudaEvent_t poll_ev[2] = {ctx->ev_a, ctx->ev_b};
  for (int round = 0;; ++round) {
    int polls = 0;
    for (int launched = 0; opt.max_iter > 0 && launched <= opt.max_iter + 2 * chunk;) {
      for (int it = 0; it < chunk; ++it) {
        for (int r = 0; r < R; ++r) {
          k_cg_step<K><<<grid_v, kBlock, 0, s>>>(S[r].x.p, S[r].r.p, S[r].z.p, S[r].p.p,
                                                 S[r].sv.p, S[r].q.p, parts[r]->dinv.p, S[r].ctl);
          CK_LAUNCH();
        }
        spmv_overlapped(&PartState<K>::z, &PartState<K>::q);  // w = A z, fused dots
        allreduce(5 * K);                                       // the one reduction
        fin(kFinCg, 0, 0);
      }
      launched += chunk;
      // poll the active count one chunk behind (the next chunk is queued first)
      CK(cudaMemcpyAsync(flag + (polls & 1), S[0].n_active.p, sizeof(int),
                         cudaMemcpyDeviceToHost, s));
      CK(cudaEventRecord(poll_ev[polls & 1], s));
      ++polls;
      if (polls >= 2) {
        CK(cudaEventSynchronize(poll_ev[(polls - 2) & 1]));
        if (flag[(polls - 2) & 1] == 0) break;
      }
    }
    CK(cudaStreamSynchronize(s));
    // true residual (iterative.cpp:208-216): q <- b - A x, norms across parts
    CK(cudaMemcpyAsync(hs.data(), S[0].st.p, K * sizeof(RhsState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));  // statuses are identical on every part
    {
      std::vector<RhsState> tmp = hs;
      for (auto& t : tmp) t.status = kActive;
      for (int r = 0; r < R; ++r) {
        CK(cudaMemcpyAsync(S[r].st.p, tmp.data(), K * sizeof(RhsState), cudaMemcpyHostToDevice, s));
        CK(cudaMemsetAsync(S[r].n_active.p, 0xff, sizeof(int), s));
      }
      CK(cudaStreamSynchronize(s));
    }
    halo(&PartState<K>::x, s);
    spmv(kResid, &PartState<K>::x, &PartState<K>::q, true);
    allreduce(K);
    fin(kFinResid, 0, 0);
    std::vector<RhsState> res(K);
    CK(cudaMemcpyAsync(res.data(), S[0].st.p, K * sizeof(RhsState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int c = 0; c < K; ++c) hs[c].rnorm = res[c].rnorm;  // keep statuses, true norm
    for (int r = 0; r < R; ++r)
      CK(cudaMemcpyAsync(S[r].st.p, hs.data(), K * sizeof(RhsState), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    unsigned restart_mask = 0;
    for (int c = 0; c < k; ++c) {
      const RhsState& t = hs[c];
      if (t.status == kBreakdown) fail(ECT_ERR_SOLVER, "COCG breakdown on right-hand side " + std::to_string(c));
      const double rel = t.bnorm > 0.0 ? t.rnorm / t.bnorm : 0.0;
      if (t.status == kConverged && rel > opt.tol && t.iters < opt.max_iter && round < 8)
        restart_mask |= 1u << c;
    }
    if (!restart_mask) break;
    for (int r = 0; r < R; ++r)
      for (int c = 0; c < K; ++c)
        if ((restart_mask >> c) & 1u)
          CK(cudaMemcpy2DAsync(S[r].r.p + c, K * sizeof(double2), S[r].q.p + c, K * sizeof(double2),
                               sizeof(double2), parts[r]->plan.n_local(), cudaMemcpyDeviceToDevice, s));
    start(restart_mask, 0);
  }
  for (int c = 0; c < k; ++c) {
    const RhsState& t = hs[c];
    out->iters[c] = t.iters;
    const double rel = t.bnorm > 0.0 ? t.rnorm / t.bnorm : 0.0;
    out->residual[c] = rel;
    out->converged[c] = (t.status == kZeroRhs) || (t.status == kConverged && rel <= opt.tol);
  }
  // owned rows of x back to the global vector
  for (int r = 0; r < R; ++r) {
    const HaloPlan& H = parts[r]->plan;
    CK(cudaMemcpyAsync(x_global + 3 * H.n0 * K, S[r].x.p, 3 * H.L * K * sizeof(double2),
                       cudaMemcpyDeviceToDevice, s));
    if (H.Vo)
      CK(cudaMemcpyAsync(x_global + (na_g + H.c0) * K, S[r].x.p + H.na_local() * K,
                         H.Vo * K * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  }
  CK(cudaStreamSynchronize(s));
}

}  // namespace

void dist_solve(ect_part** parts, int n_parts, ect_comm* comm, const double2* b_global,
                double2* x_global, int k, const ect_iter_options& opt, SolveOut* out) {
  if (!(opt.tol > 0.0)) fail(ECT_ERR_SOLVER, "solve_iterative: tolerance must be positive");
  if (n_parts < 1) fail(ECT_ERR_SOLVER, "dist_solve: no parts");
  int kk = 1;
  while (kk < k) kk <<= 1;
  if (kk > 8) fail(ECT_ERR_SOLVER, "dist_solve: n_rhs must be in 1..8");
  const int64_t n = parts[0]->n_global;
  ect_ctx* ctx = parts[0]->ctx;
  cudaStream_t s = ctx->stream;
  // internal (power-of-two) batch width
  DevBuf<double2> bpad, xpad;
  const double2* bg = b_global;
  double2* xg = x_global;
  if (kk != k) {
    bpad.alloc((size_t)n * kk);
    xpad.alloc((size_t)n * kk);
    CK(cudaMemsetAsync(bpad.p, 0, bpad.bytes(), s));
    CK(cudaMemsetAsync(xpad.p, 0, xpad.bytes(), s));
    CK(cudaMemcpy2DAsync(bpad.p, kk * sizeof(double2), b_global, k * sizeof(double2),
                         k * sizeof(double2), n, cudaMemcpyDeviceToDevice, s));
    bg = bpad.p;
    xg = xpad.p;
  }
  switch (kk) {
    case 1: dist_solve_k<1>(parts, n_parts, comm, bg, xg, k, opt, out); break;
    case 2: dist_solve_k<2>(parts, n_parts, comm, bg, xg, k, opt, out); break;
    case 4: dist_solve_k<4>(parts, n_parts, comm, bg, xg, k, opt, out); break;
    default: dist_solve_k<8>(parts, n_parts, comm, bg, xg, k, opt, out); break;
  }
  if (kk != k) {
    CK(cudaMemcpy2DAsync(x_global, k * sizeof(double2), xpad.p, kk * sizeof(double2),
                         k * sizeof(double2), n, cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
}

}  // namespace ect
