// K1: symbolic pattern of the global A–V matrix.
//
// The reference builds it implicitly: assemble_block pushes a triplet for
// every local entry (assembly.cpp:101-180), reduce_blocks/canonicalize merge
// duplicates keeping explicit zeros (sparse.cpp:13-57), build_global offsets
// the V block by na = 3 n_nodes and CscMatrix::from_triplets sorts by
// (col, row) (assembly.cpp:386-419, sparse.cpp:83-113). Hence:
//   A-row 3i+c : cols {3m+d : m shares any tet with i} ascending, then
//                {na + cond(m) : m shares a CONDUCTOR tet with i} ascending;
//   V-row na+cond(i): cols {3m+d : m shares a conductor tet} then
//                {na + cond(m)} over the same set.
// The pattern is structurally symmetric, so these CSR arrays equal the
// reference CSC col_ptr/row_idx bit for bit.
//
// B200 design: integer-only work; one thread per incidence entry writes the
// candidate neighbours of a node (node<<1 | conductor), a CUB segmented sort
// orders each node's candidates, then a dedupe pass and a warp-per-node fill
// write the column indices coalesced per row. Deterministic by construction.
#include <cub/cub.cuh>

#include "ect_internal.h"

namespace ect {
namespace {

__device__ __forceinline__ bool is_conductor(uint8_t r) {
  return r == ECT_REGION_TUBE || r == ECT_REGION_TSP || r == ECT_REGION_DEFECT;
}

int blocks_for(ect_ctx* ctx, int64_t n, int block = 256) {
  int64_t b = (n + block - 1) / block;
  int64_t cap = (int64_t)ctx->num_sms * 16;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

__global__ void k_candidates(const int4* __restrict__ tets, const uint8_t* __restrict__ region,
                             const int* __restrict__ inc, int64_t n_inc, int* cand) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n_inc;
       p += (int64_t)gridDim.x * blockDim.x) {
    int t = inc[p] >> 2;
    int c = is_conductor(region[t]) ? 1 : 0;
    int4 k = tets[t];
    int4 o = make_int4((k.x << 1) | c, (k.y << 1) | c, (k.z << 1) | c, (k.w << 1) | c);
    reinterpret_cast<int4*>(cand)[p] = o;
  }
}

__global__ void k_times4(const int* __restrict__ in, int64_t n, int* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = 4 * in[i];
}

// Per node: number of distinct neighbours (the group's last key carries the
// OR of its conductor bits).
__global__ void k_count_neighbours(const int* __restrict__ inc_off, const int* __restrict__ cand,
                                   int64_t n_nodes, int* nbr_cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_nodes;
       i += (int64_t)gridDim.x * blockDim.x) {
    int b = 4 * inc_off[i], e = 4 * inc_off[i + 1];
    int u = 0;
    for (int p = b; p < e; ++p) {
      const int v = cand[p];
      u += (p + 1 == e) || ((cand[p + 1] >> 1) != (v >> 1));
    }
    nbr_cnt[i] = u;
  }
}

// Row lengths: A-rows 3u + cc, V-row 4 cc (u neighbours, cc via conductor tets).
__global__ void k_row_lengths(const int* __restrict__ nbr_off, const uint8_t* __restrict__ nbr_cond,
                              const int* __restrict__ cond_fwd, int64_t n_nodes, int* row_len) {
  const int64_t na = 3 * n_nodes;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_nodes;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int b = nbr_off[i], u = nbr_off[i + 1] - b;
    int cc = 0;
    for (int p = b; p < b + u; ++p) cc += nbr_cond[p];
    const int la = 3 * u + cc;
    row_len[3 * i] = la;
    row_len[3 * i + 1] = la;
    row_len[3 * i + 2] = la;
    const int cf = cond_fwd[i];
    if (cf >= 0) row_len[na + cf] = 4 * cc;
  }
}

__global__ void k_write_neighbours(const int* __restrict__ inc_off, const int* __restrict__ cand,
                                   const int* __restrict__ nbr_off, int64_t n_nodes, int* nbr,
                                   uint8_t* nbr_cond) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_nodes;
       i += (int64_t)gridDim.x * blockDim.x) {
    int b = 4 * inc_off[i], e = 4 * inc_off[i + 1];
    int w = nbr_off[i];
    for (int p = b; p < e; ++p) {
      int v = cand[p];
      bool last = (p + 1 == e) || ((cand[p + 1] >> 1) != (v >> 1));
      if (last) {
        nbr[w] = v >> 1;
        nbr_cond[w] = (uint8_t)(v & 1);
        ++w;
      }
    }
  }
}

__global__ void k_narrow_row_ptr(const long long* __restrict__ in, int64_t n, int* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int)in[i];
}

// Warp per node: lane r owns neighbour r (chunks of 32).
__global__ void k_fill_columns(const int* __restrict__ nbr_off, const int* __restrict__ nbr,
                               const uint8_t* __restrict__ nbr_cond,
                               const int* __restrict__ cond_fwd, const int* __restrict__ row_ptr,
                               int64_t n_nodes, int* col) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int na = (int)(3 * n_nodes);
  for (int64_t i = warp; i < n_nodes; i += n_warps) {
    const int b = nbr_off[i], u = nbr_off[i + 1] - b;
    // total conductor neighbours
    int cc = 0;
    for (int r0 = 0; r0 < u; r0 += 32) {
      bool c = (r0 + lane < u) && nbr_cond[b + r0 + lane];
      cc += __popc(__ballot_sync(0xffffffffu, c));
    }
    const int cf_i = cond_fwd[i];
    const int base0 = row_ptr[3 * i], base1 = row_ptr[3 * i + 1], base2 = row_ptr[3 * i + 2];
    const int basev = cf_i >= 0 ? row_ptr[na + cf_i] : 0;
    int rc0 = 0;  // conductor rank offset of this chunk
    for (int r0 = 0; r0 < u; r0 += 32) {
      const int r = r0 + lane;
      const bool valid = r < u;
      const int m = valid ? nbr[b + r] : 0;
      const bool c = valid && nbr_cond[b + r];
      const unsigned mask = __ballot_sync(0xffffffffu, c);
      const int rc = rc0 + __popc(mask & ((1u << lane) - 1u));
      if (valid) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          col[base0 + 3 * r + d] = 3 * m + d;
          col[base1 + 3 * r + d] = 3 * m + d;
          col[base2 + 3 * r + d] = 3 * m + d;
        }
        if (c) {
          const int vcol = na + cond_fwd[m];
          col[base0 + 3 * u + rc] = vcol;
          col[base1 + 3 * u + rc] = vcol;
          col[base2 + 3 * u + rc] = vcol;
          if (cf_i >= 0) {
#pragma unroll
            for (int d = 0; d < 3; ++d) col[basev + 3 * rc + d] = 3 * m + d;
            col[basev + 3 * cc + rc] = vcol;
          }
        }
      }
      rc0 += __popc(mask);
    }
  }
}

// CSR value order -> the reference's CSC value order. The pattern is
// symmetric, so the CSC slot of A(i, j) is the position of column i inside
// row j. Warp per row, binary search per entry; a pure permutation.
__global__ void k_csr_to_csc(const int* __restrict__ row_ptr, const int* __restrict__ col,
                             const double2* __restrict__ val, int64_t n, double2* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += n_warps) {
    for (int p = row_ptr[i] + lane; p < row_ptr[i + 1]; p += 32) {
      const int j = col[p];
      int lo = row_ptr[j], hi = row_ptr[j + 1] - 1;
      while (lo < hi) {
        const int mid = lo + ((hi - lo) >> 1);
        if (col[mid] < (int)i) lo = mid + 1; else hi = mid;
      }
      out[lo] = val[p];
    }
  }
}

}  // namespace

void export_csc_values(ect_matrix* a, double2* out) {
  ect_ctx* ctx = a->ctx;
  k_csr_to_csc<<<blocks_for(ctx, 32 * a->n), 256, 0, ctx->stream>>>(a->row_ptr.p, a->col.p,
                                                                   a->val.p, a->n, out);
  CK_LAUNCH();
  note_launch(ctx, 1);
}

// Mesh-level neighbour structure (once per mesh; matrices borrow it).
static void build_neighbours(ect_mesh* m) {
  ect_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  const int64_t nn = m->n_nodes, n_inc = 4 * m->n_tets, n_cand = 4 * n_inc;
  if (n_cand >= (1ll << 31)) fail(ECT_ERR_MESH, "pattern build: candidate count exceeds int32");
  DevBuf<int> cand(n_cand), cand_sorted(n_cand), seg(nn + 1);
  k_candidates<<<blocks_for(ctx, n_inc), 256, 0, s>>>(m->tets.p, m->region.p, m->inc.p, n_inc,
                                                     cand.p);
  CK_LAUNCH();
  k_times4<<<blocks_for(ctx, nn + 1), 256, 0, s>>>(m->inc_off.p, nn + 1, seg.p);
  CK_LAUNCH();
  size_t tmp = 0;
  CK(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp, cand.p, cand_sorted.p, (int)n_cand, (int)nn,
                                        seg.p, seg.p + 1, s));
  CK(cub::DeviceSegmentedSort::SortKeys(cub_scratch(ctx, tmp), tmp, cand.p, cand_sorted.p,
                                        (int)n_cand, (int)nn, seg.p, seg.p + 1, s));
  DevBuf<int> nbr_cnt(nn + 1);
  CK(cudaMemsetAsync(nbr_cnt.p, 0, nbr_cnt.bytes(), s));
  k_count_neighbours<<<blocks_for(ctx, nn), 256, 0, s>>>(m->inc_off.p, cand_sorted.p, nn,
                                                        nbr_cnt.p);
  CK_LAUNCH();
  m->nbr_off.alloc(nn + 1);
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, nbr_cnt.p, m->nbr_off.p, nn + 1, s));
  CK(cub::DeviceScan::ExclusiveSum(cub_scratch(ctx, tmp), tmp, nbr_cnt.p, m->nbr_off.p, nn + 1, s));
  int total_nbr = 0, max_nbr = 0;
  CK(cudaMemcpyAsync(&total_nbr, m->nbr_off.p + nn, sizeof(int), cudaMemcpyDeviceToHost, s));
  {
    DevBuf<int> mx(1);
    CK(cub::DeviceReduce::Max(nullptr, tmp, nbr_cnt.p, mx.p, nn, s));
    CK(cub::DeviceReduce::Max(cub_scratch(ctx, tmp), tmp, nbr_cnt.p, mx.p, nn, s));
    CK(cudaMemcpyAsync(&max_nbr, mx.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  m->nbr.alloc(std::max(1, total_nbr) + 4);  // staged NB SpMV copies 16-B aligned ranges
  m->nbr_cond.alloc(std::max(1, total_nbr));
  k_write_neighbours<<<blocks_for(ctx, nn), 256, 0, s>>>(m->inc_off.p, cand_sorted.p,
                                                        m->nbr_off.p, nn, m->nbr.p,
                                                        m->nbr_cond.p);
  CK_LAUNCH();
  note_launch(ctx, 5);
  CK(cudaStreamSynchronize(s));
  m->have_nbr = true;
  m->max_nbr = max_nbr;
}

void build_pattern(ect_mesh* m, ect_matrix* a) {
  ect_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  if (!m->have_nbr) build_neighbours(m);
  const int64_t nn = m->n_nodes;
  const int64_t N = 3 * nn + m->n_cond;
  DevBuf<int> row_len(N + 1);
  CK(cudaMemsetAsync(row_len.p, 0, row_len.bytes(), s));
  k_row_lengths<<<blocks_for(ctx, nn), 256, 0, s>>>(m->nbr_off.p, m->nbr_cond.p, m->cond_fwd.p,
                                                   nn, row_len.p);
  CK_LAUNCH();
  size_t tmp = 0;
  DevBuf<long long> rp64(N + 1);
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, row_len.p, rp64.p, N + 1, s));
  CK(cub::DeviceScan::ExclusiveSum(cub_scratch(ctx, tmp), tmp, row_len.p, rp64.p, N + 1, s));
  long long nnz = 0;
  CK(cudaMemcpyAsync(&nnz, rp64.p + N, sizeof(long long), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (nnz >= (1ll << 31)) fail(ECT_ERR_MESH, "pattern build: nnz exceeds int32 row pointers");
  a->n = N;
  a->nnz = nnz;
  a->n_nodes = nn;
  a->n_cond = m->n_cond;
  a->from_mesh = true;
  a->row_ptr.alloc(N + 1);
  a->col.alloc(std::max<long long>(1, nnz));
  a->val.alloc(std::max<long long>(1, nnz));
  k_narrow_row_ptr<<<blocks_for(ctx, N + 1), 256, 0, s>>>(rp64.p, N + 1, a->row_ptr.p);
  CK_LAUNCH();
  k_fill_columns<<<blocks_for(ctx, 32 * nn), 256, 0, s>>>(m->nbr_off.p, m->nbr.p, m->nbr_cond.p,
                                                         m->cond_fwd.p, a->row_ptr.p, nn,
                                                         a->col.p);
  CK_LAUNCH();
  note_launch(ctx, 4);
  CK(cudaStreamSynchronize(s));
}

}  // namespace ect
