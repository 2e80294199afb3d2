// Mesh-side device preparation: node->tet incidence, conductor DOF map,
// essential-BC pins, DEFECT tet list.
//
// Reference semantics restated:
//   conductor_map      mesh.cpp:267-284  V-dof = rank of the node among
//                      conductor-incident nodes, ascending node id.
//   classify_boundary  mesh.cpp:145-182  exterior faces (one incident tet)
//                      labelled OUTER_TOP / OUTER_BOTTOM by z-extremes with
//                      tol = 1e-9 * max(1, z_hi - z_lo), else OUTER_LATERAL.
//   apply_essential_bc assembly.cpp:285-312  TOP/BOTTOM pin the z-dof,
//                      LATERAL pins the x- and y-dofs of every face node.
// All outputs are deterministic (integer work; idempotent flag writes).
#include <cub/cub.cuh>

#include "ect_internal.h"

namespace ect {
namespace {

__global__ void k_count_incidence(const int4* __restrict__ tets, int64_t n_tets, int* count) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tets;
       t += (int64_t)gridDim.x * blockDim.x) {
    int4 k = tets[t];
    atomicAdd(&count[k.x], 1);
    atomicAdd(&count[k.y], 1);
    atomicAdd(&count[k.z], 1);
    atomicAdd(&count[k.w], 1);
  }
}

__global__ void k_fill_incidence(const int4* __restrict__ tets, int64_t n_tets,
                                 const int* __restrict__ off, int* cursor, int* inc) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tets;
       t += (int64_t)gridDim.x * blockDim.x) {
    int4 k = tets[t];
    int nodes[4] = {k.x, k.y, k.z, k.w};
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      int pos = atomicAdd(&cursor[nodes[a]], 1);
      inc[off[nodes[a]] + pos] = (int)(4 * t + a);
    }
  }
}

// Insertion sort of each node's incidence list (ascending tet id). Degrees
// are small (24 on a Kuhn mesh), so one thread per node is enough.
__global__ void k_sort_incidence(const int* __restrict__ off, int* inc, int64_t n_nodes,
                                 int* max_deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_nodes;
       i += (int64_t)gridDim.x * blockDim.x) {
    int b = off[i], e = off[i + 1];
    for (int p = b + 1; p < e; ++p) {
      int v = inc[p];
      int q = p - 1;
      while (q >= b && inc[q] > v) {
        inc[q + 1] = inc[q];
        --q;
      }
      inc[q + 1] = v;
    }
    atomicMax(max_deg, e - b);
  }
}

__device__ __forceinline__ bool is_conductor(uint8_t r) {
  // is_conductor_region (types.hpp:46-48): TUBE, TSP, DEFECT
  return r == ECT_REGION_TUBE || r == ECT_REGION_TSP || r == ECT_REGION_DEFECT;
}

__global__ void k_mark_conductor_nodes(const int4* __restrict__ tets,
                                       const uint8_t* __restrict__ region, int64_t n_tets,
                                       int* flag) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tets;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (!is_conductor(region[t])) continue;
    int4 k = tets[t];
    flag[k.x] = 1;
    flag[k.y] = 1;
    flag[k.z] = 1;
    flag[k.w] = 1;
  }
}

__global__ void k_cond_forward(const int* __restrict__ flag, const int* __restrict__ scan,
                               int64_t n, int* fwd) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    fwd[i] = flag[i] ? scan[i] : -1;
  }
}

// One thread per (tet, face). Face f omits local node f (mesh.cpp:107,
// kFaceOf). A face is exterior when no other tet incident to its first node
// contains the two others (build_face_incidence, mesh.cpp:122-143).
__global__ void k_boundary_pins(const int4* __restrict__ tets, int64_t n_tets,
                                const int* __restrict__ off, const int* __restrict__ inc,
                                const double* __restrict__ xyz, double z_lo, double z_hi,
                                double tol, uint8_t* pinned) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < 4 * n_tets;
       g += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = g >> 2;
    int f = (int)(g & 3);
    int4 k4 = tets[t];
    int k[4] = {k4.x, k4.y, k4.z, k4.w};
    int u[3];
    int q = 0;
#pragma unroll
    for (int a = 0; a < 4; ++a)
      if (a != f) u[q++] = k[a];
    bool shared = false;
    for (int p = off[u[0]]; p < off[u[0] + 1] && !shared; ++p) {
      int64_t t2 = inc[p] >> 2;
      if (t2 == t) continue;
      int4 o = tets[t2];
      bool h1 = o.x == u[1] || o.y == u[1] || o.z == u[1] || o.w == u[1];
      bool h2 = o.x == u[2] || o.y == u[2] || o.z == u[2] || o.w == u[2];
      shared = h1 && h2;
    }
    if (shared) continue;
    bool top = true, bottom = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double z = xyz[3 * (int64_t)u[a] + 2];
      top = top && fabs(z - z_hi) <= tol;
      bottom = bottom && fabs(z - z_lo) <= tol;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      int64_t n = u[a];
      if (top || bottom) {
        pinned[3 * n + 2] = 1;
      } else {
        pinned[3 * n] = 1;
        pinned[3 * n + 1] = 1;
      }
    }
  }
}

__global__ void k_mark_defect(const uint8_t* __restrict__ region, int64_t n_tets, int* flag) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tets;
       t += (int64_t)gridDim.x * blockDim.x) {
    flag[t] = region[t] == ECT_REGION_DEFECT ? 1 : 0;
  }
}

__global__ void k_scatter_defect(const int* __restrict__ flag, const int* __restrict__ scan,
                                 int64_t n_tets, int* out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tets;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (flag[t]) out[scan[t]] = (int)t;
  }
}

__global__ void k_count_flags(const uint8_t* __restrict__ f, int64_t n, int* out) {
  int c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += f[i] != 0;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

int blocks_for(ect_ctx* ctx, int64_t n, int block = 256) {
  int64_t b = (n + block - 1) / block;
  int64_t cap = (int64_t)ctx->num_sms * 16;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace

void build_mesh_topology(ect_mesh* m) {
  ect_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  const int64_t nn = m->n_nodes, nt = m->n_tets;
  if (nn >= (1ll << 30) || 4 * nt >= (1ll << 31)) fail(ECT_ERR_MESH, "mesh too large for int32 ids");

  // ---- node -> tet incidence -------------------------------------------
  DevBuf<int> count(nn + 1), cursor(nn);
  m->inc_off.alloc(nn + 1);
  m->inc.alloc(4 * nt);
  CK(cudaMemsetAsync(count.p, 0, count.bytes(), s));
  CK(cudaMemsetAsync(cursor.p, 0, cursor.bytes(), s));
  k_count_incidence<<<blocks_for(ctx, nt), 256, 0, s>>>(m->tets.p, nt, count.p);
  CK_LAUNCH();
  size_t tmp = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, count.p, m->inc_off.p, nn + 1, s));
  CK(cub::DeviceScan::ExclusiveSum(cub_scratch(ctx, tmp), tmp, count.p, m->inc_off.p, nn + 1, s));
  k_fill_incidence<<<blocks_for(ctx, nt), 256, 0, s>>>(m->tets.p, nt, m->inc_off.p, cursor.p,
                                                      m->inc.p);
  CK_LAUNCH();
  DevBuf<int> maxdeg(1);
  CK(cudaMemsetAsync(maxdeg.p, 0, sizeof(int), s));
  k_sort_incidence<<<blocks_for(ctx, nn), 256, 0, s>>>(m->inc_off.p, m->inc.p, nn, maxdeg.p);
  CK_LAUNCH();
  note_launch(ctx, 4);

  // ---- conductor map (mesh.cpp:267-284) ---------------------------------
  DevBuf<int> flag(nn + 1), scan(nn + 1);
  CK(cudaMemsetAsync(flag.p, 0, flag.bytes(), s));
  k_mark_conductor_nodes<<<blocks_for(ctx, nt), 256, 0, s>>>(m->tets.p, m->region.p, nt, flag.p);
  CK_LAUNCH();
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flag.p, scan.p, nn + 1, s));
  CK(cub::DeviceScan::ExclusiveSum(cub_scratch(ctx, tmp), tmp, flag.p, scan.p, nn + 1, s));
  m->cond_fwd.alloc(nn);
  k_cond_forward<<<blocks_for(ctx, nn), 256, 0, s>>>(flag.p, scan.p, nn, m->cond_fwd.p);
  CK_LAUNCH();
  note_launch(ctx, 3);

  // ---- essential-BC pins (mesh.cpp:145-182, assembly.cpp:285-312) -------
  m->pinned.alloc(3 * nn);
  CK(cudaMemsetAsync(m->pinned.p, 0, m->pinned.bytes(), s));
  const double tol = 1e-9 * std::max(1.0, m->z_hi - m->z_lo);
  k_boundary_pins<<<blocks_for(ctx, 4 * nt), 256, 0, s>>>(m->tets.p, nt, m->inc_off.p, m->inc.p,
                                                         m->xyz.p, m->z_lo, m->z_hi, tol,
                                                         m->pinned.p);
  CK_LAUNCH();
  note_launch(ctx, 1);

  // ---- DEFECT tets ascending ---------------------------------------------
  DevBuf<int> dflag(nt + 1), dscan(nt + 1);
  CK(cudaMemsetAsync(dflag.p, 0, dflag.bytes(), s));
  k_mark_defect<<<blocks_for(ctx, nt), 256, 0, s>>>(m->region.p, nt, dflag.p);
  CK_LAUNCH();
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, dflag.p, dscan.p, nt + 1, s));
  CK(cub::DeviceScan::ExclusiveSum(cub_scratch(ctx, tmp), tmp, dflag.p, dscan.p, nt + 1, s));
  note_launch(ctx, 2);

  // ---- counts back to host ------------------------------------------------
  int h_ncond = 0, h_ndef = 0, h_maxdeg = 0;
  CK(cudaMemcpyAsync(&h_ncond, scan.p + nn, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&h_ndef, dscan.p + nt, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&h_maxdeg, maxdeg.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  m->n_cond = h_ncond;
  m->n_defect = h_ndef;
  m->max_inc = h_maxdeg;
  if (m->n_cond == 0) {
    fail(ECT_ERR_MESH, "mesh has no conductor region: scalar potential space is empty");
  }
  m->defect_tets.alloc(std::max<int64_t>(1, h_ndef));
  if (h_ndef > 0) {
    k_scatter_defect<<<blocks_for(ctx, nt), 256, 0, s>>>(dflag.p, dscan.p, nt, m->defect_tets.p);
    CK_LAUNCH();
    note_launch(ctx, 1);
  }
  // pinned-dof count
  DevBuf<int> npins(1);
  CK(cudaMemsetAsync(npins.p, 0, sizeof(int), s));
  k_count_flags<<<blocks_for(ctx, 3 * nn), 256, 0, s>>>(m->pinned.p, 3 * nn, npins.p);
  CK_LAUNCH();
  int h_npins = 0;
  CK(cudaMemcpyAsync(&h_npins, npins.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  m->n_pins = h_npins;
}

}  // namespace ect
