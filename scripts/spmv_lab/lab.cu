// Dev lab (not part of the library): k = 8 node-block sliced-ELL (NB-E) SpMV
// kernel structures on a synthetic configs[1]-like node graph (65 x 65 x 129
// nodes numbered z-fastest, 15-point Kuhn stencil, random 3x3 real blocks + 3
// diagonal imaginary parts). Times each variant with CUDA events and checks it
// against the first one. Build: nvcc -O3 -std=c++20 -gencode
// arch=compute_100a,code=sm_100a -lineinfo lab.cu -o lab
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                 \
    }                                                                               \
  } while (0)

struct View {
  const int* off;     // chunk slot offsets (n_chunks + 1), multiples of 32
  const int* col;     // per slot
  const double* blk;  // plane p of slot q at blk + 4 * (p * nslots + q)
  int64_t nslots;
  int64_t n_nodes;
};
struct View32 {
  const int* off;
  const int* col;
  const float* blk;
  int64_t nslots;
  int64_t n_nodes;
};

__device__ __forceinline__ void ld4s(const double* p, double (&v)[4]) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}
__device__ __forceinline__ void ld4x(const double2* p, double2& a, double2& b) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
               : "l"(p));
}
__device__ __forceinline__ int ldg_i(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void ld4f(const float* p, float (&v)[4]) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
               : "l"(p));
}
// 4 float2 (4 right-hand sides) in one 256-bit load
__device__ __forceinline__ void ld8xf(const float2* p, float2 (&v)[4]) {
  asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(v[0].x), "=f"(v[0].y), "=f"(v[1].x), "=f"(v[1].y), "=f"(v[2].x),
                 "=f"(v[2].y), "=f"(v[3].x), "=f"(v[3].y)
               : "l"(p));
}
__device__ __forceinline__ void ld4xf(const float2* p, float2& a, float2& b) {
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(a.x), "=f"(a.y), "=f"(b.x), "=f"(b.y)
               : "l"(p));
}

struct Blk {
  double B[3][3], Im[3];
};
__device__ __forceinline__ void load_block(const View& A, int64_t q, Blk& b) {
  double v0[4], v1[4], v2[4];
  ld4s(A.blk + 4 * q, v0);
  ld4s(A.blk + 4 * (A.nslots + q), v1);
  ld4s(A.blk + 4 * (2 * A.nslots + q), v2);
  b.B[0][0] = v0[0]; b.B[0][1] = v0[1]; b.B[0][2] = v0[2];
  b.B[1][0] = v0[3]; b.B[1][1] = v1[0]; b.B[1][2] = v1[1];
  b.B[2][0] = v1[2]; b.B[2][1] = v1[3]; b.B[2][2] = v2[0];
  b.Im[0] = v2[1]; b.Im[1] = v2[2]; b.Im[2] = v2[3];
}
struct Blk32 {
  float B[3][3], Im[3];
};
__device__ __forceinline__ void load_block32(const View32& A, int64_t q, Blk32& b) {
  float v0[4], v1[4], v2[4];
  ld4f(A.blk + 4 * q, v0);
  ld4f(A.blk + 4 * (A.nslots + q), v1);
  ld4f(A.blk + 4 * (2 * A.nslots + q), v2);
  b.B[0][0] = v0[0]; b.B[0][1] = v0[1]; b.B[0][2] = v0[2];
  b.B[1][0] = v0[3]; b.B[1][1] = v1[0]; b.B[1][2] = v1[1];
  b.B[2][0] = v1[2]; b.B[2][1] = v1[3]; b.B[2][2] = v2[0];
  b.Im[0] = v2[1]; b.Im[1] = v2[2]; b.Im[2] = v2[3];
}

template <int KL>
struct XV {
  double2 v[3][KL];
};
template <int K, int KL>
__device__ __forceinline__ void load_x(const double2* x, int m, int kc, XV<KL>& X) {
  const double2* xm = x + (int64_t)3 * m * K + kc;
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int k = 0; k < KL; k += 2) ld4x(xm + d * K + k, X.v[d][k], X.v[d][k + 1]);
}
template <int KL>
__device__ __forceinline__ void fma_block(const Blk& b, const XV<KL>& X, double2 (&acc)[3][KL]) {
#pragma unroll
  for (int k = 0; k < KL; ++k)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double2 s = acc[c][k];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        s.x += b.B[c][d] * X.v[d][k].x;
        s.y += b.B[c][d] * X.v[d][k].y;
      }
      s.x -= b.Im[c] * X.v[c][k].y;
      s.y += b.Im[c] * X.v[c][k].x;
      acc[c][k] = s;
    }
}

// ---------------------------------------------------------------------------
// wide<KL, BLOCK, MINB, PIPE, PFD>: CL = 8 / KL lanes per node, 32 / CL nodes
// per warp (all in one 32-node chunk, so the block loop is warp-uniform and
// unpredicated). PIPE: 0 = column one step ahead, block + x loads issued
// together; 1 = block one step ahead too (register copy); 2 = block and x one
// step ahead (ping-pong, unrolled by two).
template <int KL, int BLOCK, int MINB, int PIPE, int PFD>
__global__ void __launch_bounds__(BLOCK, MINB)
k_wide(View A, const double2* __restrict__ x, double2* __restrict__ y) {
  constexpr int K = 8, CL = K / KL, NPW = 32 / CL;
  const int lane = threadIdx.x & 31;
  const int cl = lane % CL, kc = cl * KL;
  const int64_t warp = (blockIdx.x * (int64_t)BLOCK + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * BLOCK) >> 5;
  const int64_t n_groups = (A.n_nodes + NPW - 1) / NPW;
  for (int64_t gidx = warp; gidx < n_groups; gidx += n_warps) {
    const int64_t wn = gidx * NPW;
    const int64_t i = wn + lane / CL;
    const int c32 = (int)(wn >> 5);
    const int o32 = A.off[c32];
    const int w32 = (A.off[c32 + 1] - o32) >> 5;
    const int sbase = o32 + (int)(i & 31);
    double2 acc[3][KL];
#pragma unroll
    for (int k = 0; k < KL; ++k) acc[0][k] = acc[1][k] = acc[2][k] = make_double2(0.0, 0.0);
    // L2 prefetch of the warp's block rows PFD steps ahead
    constexpr int LINES = NPW >= 4 ? NPW / 4 : 1;  // 128-B lines per plane row of the warp
    const char* pf = nullptr;
    int pf_stride = 0;
    if constexpr (PFD > 0) {
      if (lane < 3 * LINES) {
        pf = reinterpret_cast<const char*>(A.blk + 4 * ((int64_t)(lane / LINES) * A.nslots + o32 +
                                                        (int)(wn & 31))) + 128 * (lane % LINES);
        pf_stride = 32 * 32;
      } else if (lane == 3 * LINES) {
        pf = reinterpret_cast<const char*>(A.col + o32 + (int)(wn & 31));
        pf_stride = 32 * 4;
      }
    }
    auto prefetch = [&](int row) {
      if constexpr (PFD > 0) {
        if (pf && row < w32)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(pf + (int64_t)row * pf_stride));
      }
    };
    if constexpr (PIPE == 0) {
      int m = ldg_i(A.col + sbase);
      for (int j = 0; j < w32; ++j) {
        prefetch(j + PFD);
        const int q = sbase + 32 * j;
        Blk b;
        load_block(A, q, b);
        XV<KL> X;
        load_x<K, KL>(x, m, kc, X);
        if (j + 1 < w32) m = ldg_i(A.col + q + 32);
        fma_block<KL>(b, X, acc);
      }
    } else if constexpr (PIPE == 1) {
      int m_nx = ldg_i(A.col + sbase);
      Blk b_nx;
      load_block(A, sbase, b_nx);
      for (int j = 0; j < w32; ++j) {
        prefetch(j + PFD);
        const int q = sbase + 32 * j;
        const int m = m_nx;
        Blk b = b_nx;
        XV<KL> X;
        load_x<K, KL>(x, m, kc, X);
        if (j + 1 < w32) {
          m_nx = ldg_i(A.col + q + 32);
          load_block(A, q + 32, b_nx);
        }
        fma_block<KL>(b, X, acc);
      }
    } else {
      // ping-pong: buffers 0/1 hold steps j / j + 1; columns two steps ahead
      Blk b0, b1;
      XV<KL> X0, X1;
      int m1 = 0, m2 = 0;
      {
        const int m0 = ldg_i(A.col + sbase);
        if (w32 > 1) m1 = ldg_i(A.col + sbase + 32);
        load_block(A, sbase, b0);
        load_x<K, KL>(x, m0, kc, X0);
      }
      int j = 0;
      for (; j + 1 < w32; j += 2) {
        prefetch(j + PFD);
        prefetch(j + 1 + PFD);
        const int q = sbase + 32 * j;
        // step j + 1 loads in flight while step j computes
        load_block(A, q + 32, b1);
        load_x<K, KL>(x, m1, kc, X1);
        if (j + 2 < w32) m2 = ldg_i(A.col + q + 64);
        fma_block<KL>(b0, X0, acc);
        if (j + 2 < w32) {
          load_block(A, q + 64, b0);
          load_x<K, KL>(x, m2, kc, X0);
          if (j + 3 < w32) m1 = ldg_i(A.col + q + 96);
        }
        fma_block<KL>(b1, X1, acc);
      }
      if (j < w32) fma_block<KL>(b0, X0, acc);
    }
    if (i < A.n_nodes) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double2* yr = y + (3 * i + c) * K + kc;
#pragma unroll
        for (int k = 0; k < KL; k += 2) {
          asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(yr + k), "d"(acc[c][k].x),
                       "d"(acc[c][k].y), "d"(acc[c][k + 1].x), "d"(acc[c][k + 1].y)
                       : "memory");
        }
      }
    }
  }
}


// ---------------------------------------------------------------------------
// k_shfl: CL = 4 / KL = 2 lanes as k_wide, but the block is loaded ONCE per
// node (lane cl < 3 loads plane cl) and broadcast with shuffles, so the L1
// writeback carries each matrix byte once instead of CL times.
template <int BLOCK, int MINB, int PFD>
__global__ void __launch_bounds__(BLOCK, MINB)
k_shfl(View A, const double2* __restrict__ x, double2* __restrict__ y) {
  constexpr int K = 8, KL = 2, CL = 4, NPW = 8;
  const int lane = threadIdx.x & 31;
  const int cl = lane % CL, kc = cl * KL;
  const int lbase = lane & ~3;
  const int64_t warp = (blockIdx.x * (int64_t)BLOCK + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * BLOCK) >> 5;
  const int64_t n_groups = (A.n_nodes + NPW - 1) / NPW;
  for (int64_t gidx = warp; gidx < n_groups; gidx += n_warps) {
    const int64_t wn = gidx * NPW;
    const int64_t i = wn + lane / CL;
    const int c32 = (int)(wn >> 5);
    const int o32 = A.off[c32];
    const int w32 = (A.off[c32 + 1] - o32) >> 5;
    const int sbase = o32 + (int)(i & 31);
    double2 acc[3][KL];
#pragma unroll
    for (int k = 0; k < KL; ++k) acc[0][k] = acc[1][k] = acc[2][k] = make_double2(0.0, 0.0);
    constexpr int LINES = 2;
    const char* pf = nullptr;
    int pf_stride = 0;
    if constexpr (PFD > 0) {
      if (lane < 3 * LINES) {
        pf = reinterpret_cast<const char*>(A.blk + 4 * ((int64_t)(lane / LINES) * A.nslots + o32 +
                                                        (int)(wn & 31))) + 128 * (lane % LINES);
        pf_stride = 32 * 32;
      } else if (lane == 3 * LINES) {
        pf = reinterpret_cast<const char*>(A.col + o32 + (int)(wn & 31));
        pf_stride = 32 * 4;
      }
    }
    // this lane's plane (cl = 3 re-reads plane 2: same address as lane 2, no extra sector)
    const double* mine = A.blk + 4 * ((int64_t)(cl < 3 ? cl : 2) * A.nslots + sbase);
    int m_nx = ldg_i(A.col + sbase);
    double v_nx[4];
    ld4s(mine, v_nx);
    for (int j = 0; j < w32; ++j) {
      if constexpr (PFD > 0) {
        if (pf && j + PFD < w32)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(pf + (int64_t)(j + PFD) * pf_stride));
      }
      const int m = m_nx;
      double v[4] = {v_nx[0], v_nx[1], v_nx[2], v_nx[3]};
      XV<KL> X;
      load_x<K, KL>(x, m, kc, X);
      if (j + 1 < w32) {
        m_nx = ldg_i(A.col + sbase + 32 * (j + 1));
        ld4s(mine + 4 * 32 * (int64_t)(j + 1), v_nx);
      }
      double p[3][4];
#pragma unroll
      for (int pl = 0; pl < 3; ++pl)
#pragma unroll
        for (int e = 0; e < 4; ++e) p[pl][e] = __shfl_sync(0xffffffffu, v[e], lbase | pl);
      Blk b;
      b.B[0][0] = p[0][0]; b.B[0][1] = p[0][1]; b.B[0][2] = p[0][2];
      b.B[1][0] = p[0][3]; b.B[1][1] = p[1][0]; b.B[1][2] = p[1][1];
      b.B[2][0] = p[1][2]; b.B[2][1] = p[1][3]; b.B[2][2] = p[2][0];
      b.Im[0] = p[2][1]; b.Im[1] = p[2][2]; b.Im[2] = p[2][3];
      fma_block<KL>(b, X, acc);
    }
    if (i < A.n_nodes) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double2* yr = y + (3 * i + c) * K + kc;
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(yr), "d"(acc[c][0].x),
                     "d"(acc[c][0].y), "d"(acc[c][1].x), "d"(acc[c][1].y)
                     : "memory");
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k_dsplit<KL>: lanes = (node, RHS group h of KL columns, block column d).
// Lane d < 3 owns column d of every block of its node: one 256-bit load of the
// column plane (B[d][d], B[d+1][d], B[d+2][d], Im[d]) (rows rotated so that the
// diagonal comes first), the KL values of x component d, and partial sums of
// rows d, d+1, d+2 (mod 3). Nothing is loaded twice; the three column lanes
// are summed once per node with two shuffles per value. Lane d = 3 idles.
template <int KL, int BLOCK, int MINB, int PIPE, int PFD>
__global__ void __launch_bounds__(BLOCK, MINB)
k_dsplit(View A /* blk = column planes */, const double2* __restrict__ x, double2* __restrict__ y) {
  constexpr int K = 8, H = K / KL, G = 4 * H, NPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int d = lane & 3, h = (lane >> 2) % H, kc = h * KL;
  const bool act = d < 3;
  const int dd = act ? d : 2;
  const int64_t warp = (blockIdx.x * (int64_t)BLOCK + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * BLOCK) >> 5;
  const int64_t n_groups = (A.n_nodes + NPW - 1) / NPW;
  for (int64_t gidx = warp; gidx < n_groups; gidx += n_warps) {
    const int64_t wn = gidx * NPW;
    const int64_t i = wn + lane / G;
    const int c32 = (int)(wn >> 5);
    const int o32 = A.off[c32];
    const int w32 = (A.off[c32 + 1] - o32) >> 5;
    const int sbase = o32 + (int)(i & 31);
    double2 acc[3][KL];  // rows d, d + 1, d + 2 (mod 3)
#pragma unroll
    for (int k = 0; k < KL; ++k) acc[0][k] = acc[1][k] = acc[2][k] = make_double2(0.0, 0.0);
    constexpr int LINES = NPW >= 4 ? NPW / 4 : 1;
    const char* pf = nullptr;
    int pf_stride = 0;
    if constexpr (PFD > 0) {
      if (lane < 3 * LINES) {
        pf = reinterpret_cast<const char*>(A.blk + 4 * ((int64_t)(lane / LINES) * A.nslots + o32 +
                                                        (int)(wn & 31))) + 128 * (lane % LINES);
        pf_stride = 32 * 32;
      } else if (lane == 3 * LINES) {
        pf = reinterpret_cast<const char*>(A.col + o32 + (int)(wn & 31));
        pf_stride = 32 * 4;
      }
    }
    const double* mine = A.blk + 4 * ((int64_t)dd * A.nslots + sbase);
    auto step = [&](const double (&v)[4], const double2 (&xv)[KL]) {
#pragma unroll
      for (int k = 0; k < KL; ++k) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          acc[r][k].x += v[r] * xv[k].x;
          acc[r][k].y += v[r] * xv[k].y;
        }
        acc[0][k].x -= v[3] * xv[k].y;
        acc[0][k].y += v[3] * xv[k].x;
      }
    };
    auto loadx = [&](int m, double2 (&xv)[KL]) {
      const double2* xm = x + ((int64_t)3 * m + dd) * K + kc;
#pragma unroll
      for (int k = 0; k < KL; k += 2) ld4x(xm + k, xv[k], xv[k + 1]);
    };
    if constexpr (PIPE == 0) {
      int m = ldg_i(A.col + sbase);
      for (int j = 0; j < w32; ++j) {
        if constexpr (PFD > 0) {
          if (pf && j + PFD < w32)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pf + (int64_t)(j + PFD) * pf_stride));
        }
        double v[4];
        double2 xv[KL];
        if (act) {
          ld4s(mine + 4 * 32 * (int64_t)j, v);
          loadx(m, xv);
        }
        if (j + 1 < w32) m = ldg_i(A.col + sbase + 32 * (j + 1));
        if (act) step(v, xv);
      }
    } else {
      int m_nx = ldg_i(A.col + sbase);
      double v_nx[4] = {0, 0, 0, 0};
      if (act) ld4s(mine, v_nx);
      for (int j = 0; j < w32; ++j) {
        if constexpr (PFD > 0) {
          if (pf && j + PFD < w32)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pf + (int64_t)(j + PFD) * pf_stride));
        }
        const int m = m_nx;
        const double v[4] = {v_nx[0], v_nx[1], v_nx[2], v_nx[3]};
        double2 xv[KL];
        if (act) loadx(m, xv);
        if (j + 1 < w32) {
          m_nx = ldg_i(A.col + sbase + 32 * (j + 1));
          if (act) ld4s(mine + 4 * 32 * (int64_t)(j + 1), v_nx);
        }
        if (act) step(v, xv);
      }
    }
    // row d total = own acc[0] + acc[1] of lane (d + 2) % 3 + acc[2] of lane (d + 1) % 3
    const int lb = lane & ~3;
    const int src1 = lb | ((d + 2) % 3), src2 = lb | ((d + 1) % 3);
#pragma unroll
    for (int k = 0; k < KL; ++k) {
      const double a1x = __shfl_sync(0xffffffffu, acc[1][k].x, src1);
      const double a1y = __shfl_sync(0xffffffffu, acc[1][k].y, src1);
      const double a2x = __shfl_sync(0xffffffffu, acc[2][k].x, src2);
      const double a2y = __shfl_sync(0xffffffffu, acc[2][k].y, src2);
      acc[0][k].x += a1x + a2x;
      acc[0][k].y += a1y + a2y;
    }
    if (act && i < A.n_nodes) {
      double2* yr = y + (3 * i + d) * K + kc;
#pragma unroll
      for (int k = 0; k < KL; k += 2)
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(yr + k), "d"(acc[0][k].x),
                     "d"(acc[0][k].y), "d"(acc[0][k + 1].x), "d"(acc[0][k + 1].y)
                     : "memory");
    }
  }
}

// ---------------------------------------------------------------------------
// the library's current k = 8 kernel (G = 4, CL = 4, KL = 2, one block ahead,
// predicated loop), kPlain mode — the calibration point (0.435 ms on configs[1])
template <int PFD>
__global__ void __launch_bounds__(256, 2)
k_cur(View A, const double2* __restrict__ x, double2* __restrict__ y) {
  constexpr int G = 4, K = 8, CL = 4, GB = 1, KL = 2, NPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int g = lane & (G - 1);
  const int bl = g / CL, cl = g % CL;
  const int kc = cl * KL;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t wn = warp * NPW; wn < A.n_nodes; wn += n_warps * NPW) {
    const int64_t i = wn + lane / G;
    const bool valid = i < A.n_nodes;
    double2 acc[3][KL];
#pragma unroll
    for (int k = 0; k < KL; ++k) acc[0][k] = acc[1][k] = acc[2][k] = make_double2(0.0, 0.0);
    if (valid) {
      const int c32 = (int)(i >> 5);
      const int o32 = A.off[c32];
      const int w32 = (A.off[c32 + 1] - o32) >> 5;
      const int sbase = o32 + (int)(i & 31);
      const int be = sbase + 32 * w32;
      constexpr int GS = 32 * GB;
      int q = sbase + 32 * bl;
      int m_nx = 0;
      Blk b_nx;
      if (q < be) {
        m_nx = ldg_i(A.col + q);
        load_block(A, q, b_nx);
      }
      constexpr int LINES = NPW >= 4 ? NPW / 4 : 1;
      const char* pf = nullptr;
      int pf_stride = 0;
      if constexpr (PFD > 0) {
        if (lane < 3 * LINES) {
          pf = reinterpret_cast<const char*>(A.blk + 4 * ((int64_t)(lane / LINES) * A.nslots + o32 +
                                                          (int)(wn & 31)) + 16 * (lane % LINES));
          pf_stride = 32 * 32;
        } else if (lane == 3 * LINES) {
          pf = reinterpret_cast<const char*>(A.col + o32 + (int)(wn & 31));
          pf_stride = 32 * 4;
        }
      }
      for (; q < be; q += GS) {
        if constexpr (PFD > 0) {
          const int row0 = ((q - sbase) >> 5) - bl + PFD * GB;
          if (pf && row0 < w32)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pf + (int64_t)row0 * pf_stride));
        }
        const int m = m_nx;
        Blk b = b_nx;
        if (q + GS < be) {
          m_nx = ldg_i(A.col + q + GS);
          load_block(A, q + GS, b_nx);
        }
        XV<KL> X;
        load_x<K, KL>(x, m, kc, X);
        fma_block<KL>(b, X, acc);
      }
    }
    if (valid) {
#pragma unroll
      for (int k = 0; k < KL; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) y[(3 * i + c) * K + kc + k] = acc[c][k];
    }
  }
}

// ---------------------------------------------------------------------------
// fp32 smoothing SpMV (matrix and x in fp32), same lane structure as k_wide.
template <int KL>
struct XV32 {
  float2 v[3][KL];
};
template <int K, int KL>
__device__ __forceinline__ void load_x32(const float2* x, int m, int kc, XV32<KL>& X) {
  const float2* xm = x + (int64_t)3 * m * K + kc;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if constexpr (KL % 4 == 0) {
#pragma unroll
      for (int k = 0; k < KL; k += 4) {
        float2 t[4];
        ld8xf(xm + d * K + k, t);
        X.v[d][k] = t[0]; X.v[d][k + 1] = t[1]; X.v[d][k + 2] = t[2]; X.v[d][k + 3] = t[3];
      }
    } else {
#pragma unroll
      for (int k = 0; k < KL; k += 2) ld4xf(xm + d * K + k, X.v[d][k], X.v[d][k + 1]);
    }
  }
}
template <int KL>
__device__ __forceinline__ void fma_block32(const Blk32& b, const XV32<KL>& X,
                                            float2 (&acc)[3][KL]) {
#pragma unroll
  for (int k = 0; k < KL; ++k)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float2 s = acc[c][k];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        s.x = fmaf(b.B[c][d], X.v[d][k].x, s.x);
        s.y = fmaf(b.B[c][d], X.v[d][k].y, s.y);
      }
      s.x = fmaf(-b.Im[c], X.v[c][k].y, s.x);
      s.y = fmaf(b.Im[c], X.v[c][k].x, s.y);
      acc[c][k] = s;
    }
}
template <int KL, int BLOCK, int MINB, int PIPE, int PFD>
__global__ void __launch_bounds__(BLOCK, MINB)
k_wide32(View32 A, const float2* __restrict__ x, float2* __restrict__ y) {
  constexpr int K = 8, CL = K / KL, NPW = 32 / CL;
  const int lane = threadIdx.x & 31;
  const int cl = lane % CL, kc = cl * KL;
  const int64_t warp = (blockIdx.x * (int64_t)BLOCK + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * BLOCK) >> 5;
  const int64_t n_groups = (A.n_nodes + NPW - 1) / NPW;
  for (int64_t gidx = warp; gidx < n_groups; gidx += n_warps) {
    const int64_t wn = gidx * NPW;
    const int64_t i = wn + lane / CL;
    const int c32 = (int)(wn >> 5);
    const int o32 = A.off[c32];
    const int w32 = (A.off[c32 + 1] - o32) >> 5;
    const int sbase = o32 + (int)(i & 31);
    float2 acc[3][KL];
#pragma unroll
    for (int k = 0; k < KL; ++k) acc[0][k] = acc[1][k] = acc[2][k] = make_float2(0.f, 0.f);
    constexpr int LINES = NPW >= 8 ? NPW / 8 : 1;  // 128-B lines per fp32 plane row of the warp
    const char* pf = nullptr;
    int pf_stride = 0;
    if constexpr (PFD > 0) {
      if (lane < 3 * LINES) {
        pf = reinterpret_cast<const char*>(A.blk + 4 * ((int64_t)(lane / LINES) * A.nslots + o32 +
                                                        (int)(wn & 31))) + 128 * (lane % LINES);
        pf_stride = 32 * 16;
      } else if (lane == 3 * LINES) {
        pf = reinterpret_cast<const char*>(A.col + o32 + (int)(wn & 31));
        pf_stride = 32 * 4;
      }
    }
    auto prefetch = [&](int row) {
      if constexpr (PFD > 0) {
        if (pf && row < w32)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(pf + (int64_t)row * pf_stride));
      }
    };
    if constexpr (PIPE == 0) {
      int m = ldg_i(A.col + sbase);
      for (int j = 0; j < w32; ++j) {
        prefetch(j + PFD);
        const int q = sbase + 32 * j;
        Blk32 b;
        load_block32(A, q, b);
        XV32<KL> X;
        load_x32<K, KL>(x, m, kc, X);
        if (j + 1 < w32) m = ldg_i(A.col + q + 32);
        fma_block32<KL>(b, X, acc);
      }
    } else if constexpr (PIPE == 1) {
      int m_nx = ldg_i(A.col + sbase);
      Blk32 b_nx;
      load_block32(A, sbase, b_nx);
      for (int j = 0; j < w32; ++j) {
        prefetch(j + PFD);
        const int q = sbase + 32 * j;
        const int m = m_nx;
        Blk32 b = b_nx;
        XV32<KL> X;
        load_x32<K, KL>(x, m, kc, X);
        if (j + 1 < w32) {
          m_nx = ldg_i(A.col + q + 32);
          load_block32(A, q + 32, b_nx);
        }
        fma_block32<KL>(b, X, acc);
      }
    } else {
      Blk32 b0, b1;
      XV32<KL> X0, X1;
      int m1 = 0, m2 = 0;
      {
        const int m0 = ldg_i(A.col + sbase);
        if (w32 > 1) m1 = ldg_i(A.col + sbase + 32);
        load_block32(A, sbase, b0);
        load_x32<K, KL>(x, m0, kc, X0);
      }
      int j = 0;
      for (; j + 1 < w32; j += 2) {
        prefetch(j + PFD);
        prefetch(j + 1 + PFD);
        const int q = sbase + 32 * j;
        load_block32(A, q + 32, b1);
        load_x32<K, KL>(x, m1, kc, X1);
        if (j + 2 < w32) m2 = ldg_i(A.col + q + 64);
        fma_block32<KL>(b0, X0, acc);
        if (j + 2 < w32) {
          load_block32(A, q + 64, b0);
          load_x32<K, KL>(x, m2, kc, X0);
          if (j + 3 < w32) m1 = ldg_i(A.col + q + 96);
        }
        fma_block32<KL>(b1, X1, acc);
      }
      if (j < w32) fma_block32<KL>(b0, X0, acc);
    }
    if (i < A.n_nodes) {
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int k = 0; k < KL; ++k) y[(3 * i + c) * K + kc + k] = acc[c][k];
    }
  }
}

// the library's current fp32 kernel structure: G = 8 (GB = 2 block lanes x CL = 4), KL = 2
__global__ void __launch_bounds__(256, 2)
k_cur32(View32 A, const float2* __restrict__ x, float2* __restrict__ y) {
  constexpr int G = 8, K = 8, CL = 4, GB = 2, KL = 2, NPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int g = lane & (G - 1);
  const int bl = g / CL, cl = g % CL;
  const int kc = cl * KL;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t wn = warp * NPW; wn < A.n_nodes; wn += n_warps * NPW) {
    const int64_t i = wn + lane / G;
    const bool valid = i < A.n_nodes;
    float2 acc[3][KL];
#pragma unroll
    for (int k = 0; k < KL; ++k) acc[0][k] = acc[1][k] = acc[2][k] = make_float2(0.f, 0.f);
    if (valid) {
      const int c32 = (int)(i >> 5);
      const int o32 = A.off[c32];
      const int w32 = (A.off[c32 + 1] - o32) >> 5;
      const int sbase = o32 + (int)(i & 31), be = sbase + 32 * w32;
      constexpr int GS = 32 * GB;
      int q = sbase + 32 * bl;
      int m_nx = 0;
      Blk32 b_nx;
      if (q < be) {
        m_nx = ldg_i(A.col + q);
        load_block32(A, q, b_nx);
      }
      for (; q < be; q += GS) {
        const int m = m_nx;
        Blk32 b = b_nx;
        if (q + GS < be) {
          m_nx = ldg_i(A.col + q + GS);
          load_block32(A, q + GS, b_nx);
        }
        XV32<KL> X;
        load_x32<K, KL>(x, m, kc, X);
        fma_block32<KL>(b, X, acc);
      }
    }
#pragma unroll
    for (int k = 0; k < KL; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        acc[c][k].x += __shfl_xor_sync(0xffffffffu, acc[c][k].x, CL, G);
        acc[c][k].y += __shfl_xor_sync(0xffffffffu, acc[c][k].y, CL, G);
      }
    if (bl == 0 && valid) {
#pragma unroll
      for (int k = 0; k < KL; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) y[(3 * i + c) * K + kc + k] = acc[c][k];
    }
  }
}

// ---------------------------------------------------------------------------
struct Variant {
  std::string name;
  const void* fn;
  int block;
  bool f32;
  bool colplanes = false;
};

template <typename T>
T* dev(const std::vector<T>& h) {
  T* p;
  CK(cudaMalloc(&p, h.size() * sizeof(T)));
  CK(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

int main(int argc, char** argv) {
  const int nx = 65, ny = 65, nz = 129;
  const int64_t n = (int64_t)nx * ny * nz;
  const int K = 8;
  const std::string only = argc > 1 ? argv[1] : "";
  // Kuhn 15-point stencil: 0 and +-(1,0,0) (0,1,0) (0,0,1) (1,1,0) (0,1,1) (1,0,1) (1,1,1)
  const int st[7][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 0}, {0, 1, 1}, {1, 0, 1}, {1, 1, 1}};
  std::vector<std::vector<int>> nb(n);
  auto id = [&](int i, int j, int k) { return ((int64_t)i * ny + j) * nz + k; };
  for (int i = 0; i < nx; ++i)
    for (int j = 0; j < ny; ++j)
      for (int k = 0; k < nz; ++k) {
        auto& v = nb[id(i, j, k)];
        for (int s = -1; s <= 1; ++s) {
          if (s == 0) {
            v.push_back((int)id(i, j, k));
            continue;
          }
          for (auto& o : st) {
            const int a = i + s * o[0], b = j + s * o[1], c = k + s * o[2];
            if (a < 0 || b < 0 || c < 0 || a >= nx || b >= ny || c >= nz) continue;
            v.push_back((int)id(a, b, c));
          }
        }
        std::sort(v.begin(), v.end());
      }
  const int64_t n_chunks = (n + 31) / 32;
  std::vector<int> off(n_chunks + 1, 0);
  int64_t nblocks = 0;
  for (int64_t c = 0; c < n_chunks; ++c) {
    size_t w = 0;
    for (int64_t i = 32 * c; i < std::min<int64_t>(n, 32 * c + 32); ++i) {
      w = std::max(w, nb[i].size());
      nblocks += (int64_t)nb[i].size();
    }
    off[c + 1] = off[c] + 32 * (int)w;
  }
  const int64_t nslots = off[n_chunks];
  std::vector<int> col(nslots);
  std::vector<double> blk(12 * nslots, 0.0);
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> U(-1, 1);
  for (int64_t c = 0; c < n_chunks; ++c) {
    const int w = (off[c + 1] - off[c]) / 32;
    for (int l = 0; l < 32; ++l) {
      const int64_t i = 32 * c + l;
      for (int j = 0; j < w; ++j) {
        const int64_t sl = off[c] + 32 * (int64_t)j + l;
        const bool real = i < n && j < (int)nb[i].size();
        col[sl] = real ? nb[i][j] : (i < n ? (int)i : 0);
        if (real)
          for (int pl = 0; pl < 3; ++pl)
            for (int e = 0; e < 4; ++e) blk[4 * (pl * nslots + sl) + e] = U(rng);
      }
    }
  }
  // column planes for k_dsplit: plane d = (B[d][d], B[d+1][d], B[d+2][d], Im[d]), rows mod 3
  std::vector<double> blkc(blk.size());
  for (int64_t sl = 0; sl < nslots; ++sl) {
    double f[12];
    for (int pl = 0; pl < 3; ++pl)
      for (int e = 0; e < 4; ++e) f[4 * pl + e] = blk[4 * (pl * nslots + sl) + e];
    for (int d = 0; d < 3; ++d) {
      for (int r = 0; r < 3; ++r) blkc[4 * (d * nslots + sl) + r] = f[3 * ((d + r) % 3) + d];
      blkc[4 * (d * nslots + sl) + 3] = f[9 + d];
    }
  }
  std::vector<float> blk32(blk.size());
  for (size_t q = 0; q < blk.size(); ++q) blk32[q] = (float)blk[q];
  std::vector<double2> x(3 * n * K);
  std::vector<float2> x32(3 * n * K);
  for (size_t q = 0; q < x.size(); ++q) {
    x[q] = make_double2(U(rng), U(rng));
    x32[q] = make_float2((float)x[q].x, (float)x[q].y);
  }
  int* d_off = dev(off);
  int* d_col = dev(col);
  double* d_blk = dev(blk);
  double* d_blkc = dev(blkc);
  float* d_blk32 = dev(blk32);
  double2* d_x = dev(x);
  float2* d_x32 = dev(x32);
  double2 *d_y, *d_ref;
  float2 *d_y32, *d_ref32;
  CK(cudaMalloc(&d_y, x.size() * sizeof(double2)));
  CK(cudaMalloc(&d_ref, x.size() * sizeof(double2)));
  CK(cudaMalloc(&d_y32, x.size() * sizeof(float2)));
  CK(cudaMalloc(&d_ref32, x.size() * sizeof(float2)));
  View A{d_off, d_col, d_blk, nslots, n};
  View32 A32{d_off, d_col, d_blk32, nslots, n};
  View AC{d_off, d_col, d_blkc, nslots, n};
  const double fmt64 = 100.0 * nslots + 4.0 * (n_chunks + 1) + 2.0 * 16.0 * 3 * n * K;
  const double fmt32 = 52.0 * nslots + 4.0 * (n_chunks + 1) + 2.0 * 8.0 * 3 * n * K;
  std::printf("nodes %lld blocks %lld slots %lld (padding %.1f%%)  fp64 format bytes %.3f GB, fp32 %.3f GB\n",
              (long long)n, (long long)nblocks, (long long)nslots,
              100.0 * (nslots - nblocks) / nblocks, fmt64 / 1e9, fmt32 / 1e9);

  std::vector<Variant> vs;
#define V64(name, ...) vs.push_back({name, (const void*)__VA_ARGS__, 0, false})
#define ADD(KL, BLOCK, MINB, PIPE, PFD)                                                    \
  vs.push_back({"wide KL=" #KL " blk=" #BLOCK " minb=" #MINB " pipe=" #PIPE " pfd=" #PFD, \
                (const void*)k_wide<KL, BLOCK, MINB, PIPE, PFD>, BLOCK, false})
#define ADD32(KL, BLOCK, MINB, PIPE, PFD)                                                    \
  vs.push_back({"wide32 KL=" #KL " blk=" #BLOCK " minb=" #MINB " pipe=" #PIPE " pfd=" #PFD, \
                (const void*)k_wide32<KL, BLOCK, MINB, PIPE, PFD>, BLOCK, true})
  vs.push_back({"cur pfd=4 (library)", (const void*)k_cur<4>, 256, false});
  vs.push_back({"cur pfd=0", (const void*)k_cur<0>, 256, false});
  ADD(2, 256, 2, 1, 4);
  ADD(2, 256, 2, 0, 4);
  ADD(2, 128, 5, 0, 4);
  ADD(2, 128, 4, 1, 4);
  ADD(2, 128, 3, 2, 4);
  ADD(2, 128, 3, 2, 0);
  ADD(2, 128, 4, 2, 4);
  ADD(4, 128, 3, 0, 4);
  ADD(4, 128, 3, 1, 4);
  ADD(4, 128, 2, 2, 4);
  ADD(4, 128, 2, 1, 4);
  ADD(4, 256, 1, 2, 4);
  ADD(8, 128, 2, 0, 4);
  ADD(8, 128, 2, 1, 4);
  ADD(8, 128, 1, 2, 4);
#define ADDS(BLOCK, MINB, PFD) \
  vs.push_back({"shfl blk=" #BLOCK " minb=" #MINB " pfd=" #PFD, (const void*)k_shfl<BLOCK, MINB, PFD>, BLOCK, false})
#define ADDD(KL, BLOCK, MINB, PIPE, PFD)                                                    \
  vs.push_back({"dsplit KL=" #KL " blk=" #BLOCK " minb=" #MINB " pipe=" #PIPE " pfd=" #PFD, \
                (const void*)k_dsplit<KL, BLOCK, MINB, PIPE, PFD>, BLOCK, false, true})
  ADD(2, 256, 3, 0, 4);
  ADD(2, 128, 6, 0, 4);
  ADD(2, 128, 7, 0, 4);
  ADD(2, 256, 2, 0, 2);
  ADD(2, 256, 2, 0, 6);
  ADD(2, 256, 2, 0, 8);
  ADDS(256, 2, 4);
  ADDS(128, 5, 4);
  ADDS(128, 6, 4);
  ADDS(128, 8, 4);
  ADDD(8, 128, 3, 0, 4);
  ADDD(8, 128, 3, 1, 4);
  ADDD(8, 128, 4, 0, 4);
  ADDD(8, 256, 2, 1, 4);
  ADDD(4, 128, 4, 0, 4);
  ADDD(4, 128, 5, 0, 4);
  ADDD(4, 128, 5, 1, 4);
  ADDD(4, 128, 6, 0, 4);
  ADDD(4, 128, 6, 1, 4);
  ADDD(4, 256, 3, 1, 4);
  ADDD(2, 128, 8, 0, 4);
  ADDD(2, 128, 8, 1, 4);
  vs.push_back({"cur32 (library)", (const void*)k_cur32, 256, true});
  ADD32(2, 256, 2, 1, 4);
  ADD32(2, 256, 3, 1, 4);
  ADD32(2, 128, 8, 0, 4);
  ADD32(2, 128, 6, 1, 4);
  ADD32(2, 128, 5, 2, 4);
  ADD32(4, 128, 6, 0, 4);
  ADD32(4, 128, 4, 1, 4);
  ADD32(4, 128, 4, 2, 4);
  ADD32(4, 128, 3, 2, 4);
  ADD32(4, 128, 3, 2, 0);
  ADD32(8, 128, 3, 0, 4);
  ADD32(8, 128, 3, 1, 4);
  ADD32(8, 128, 2, 2, 4);
  ADD32(2, 256, 4, 0, 4);
  ADD32(2, 128, 8, 0, 2);
  ADD32(2, 128, 8, 0, 8);
  ADD32(2, 128, 8, 0, 0);
  ADD32(2, 64, 16, 0, 4);
  ADD32(4, 128, 8, 0, 4);

  int dev_id = 0, sms = 0;
  CK(cudaGetDevice(&dev_id));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev_id));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<double2> href(x.size()), hy(x.size());
  std::vector<float2> href32(x.size()), hy32(x.size());
  bool have64 = false, have32 = false;
  for (auto& v : vs) {
    if (!only.empty() && v.name.find(only) == std::string::npos && v.name.find("library") == std::string::npos)
      continue;
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, v.fn));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, v.fn, v.block, 0));
    const int grid = per_sm * sms;
    void* y = v.f32 ? (void*)d_y32 : (void*)d_y;
    void* xx = v.f32 ? (void*)d_x32 : (void*)d_x;
    void* args64[] = {v.colplanes ? (void*)&AC : (void*)&A, &xx, &y};
    void* args32[] = {&A32, &xx, &y};
    void** args = v.f32 ? args32 : args64;
    CK(cudaMemset(y, 0xff, x.size() * (v.f32 ? sizeof(float2) : sizeof(double2))));
    for (int r = 0; r < 3; ++r) CK(cudaLaunchKernel(v.fn, dim3(grid), dim3(v.block), args, 0, 0));
    CK(cudaDeviceSynchronize());
    const int reps = 20;
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) CK(cudaLaunchKernel(v.fn, dim3(grid), dim3(v.block), args, 0, 0));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    double err = 0.0;
    if (!v.f32) {
      CK(cudaMemcpy(hy.data(), d_y, hy.size() * sizeof(double2), cudaMemcpyDeviceToHost));
      if (!have64) { href = hy; have64 = true; }
      for (size_t q = 0; q < hy.size(); ++q)
        err = std::max(err, std::max(std::abs(hy[q].x - href[q].x), std::abs(hy[q].y - href[q].y)));
    } else {
      CK(cudaMemcpy(hy32.data(), d_y32, hy32.size() * sizeof(float2), cudaMemcpyDeviceToHost));
      if (!have32) { href32 = hy32; have32 = true; }
      for (size_t q = 0; q < hy32.size(); ++q)
        err = std::max(err, (double)std::max(std::abs(hy32[q].x - href32[q].x),
                                             std::abs(hy32[q].y - href32[q].y)));
    }
    const double fb = v.f32 ? fmt32 : fmt64;
    std::printf("%-46s regs %3d spill %3zu  ctas/sm %d warps/sm %2d  %.4f ms  %6.0f GB/s  err %.1e\n",
                v.name.c_str(), fa.numRegs, (size_t)fa.localSizeBytes, per_sm,
                per_sm * v.block / 32, ms, fb / ms / 1e6, err);
    std::fflush(stdout);
  }
  return 0;
}
