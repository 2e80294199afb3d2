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
                              const int* __restrict__ cond_fwd, int64_t n_nodes, int* row_len,
                              int64_t lo, int64_t hi) {
  const int64_t na = 3 * n_nodes;
  for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi;
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
                               int64_t n_nodes, int* col, int64_t lo, int64_t hi) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int na = (int)(3 * n_nodes);
  for (int64_t i = lo + warp; i < hi; i += n_warps) {
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

// Compressed-major -> the other major (CSC -> CSR or CSR -> CSC): expand
// the major index of every entry; a stable radix sort by minor index then
// yields the transposed order (ties keep the input order = ascending major).
__global__ void k_expand_major(const int* __restrict__ ptr, int64_t n, int* __restrict__ major) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < n; j += n_warps)
    for (int p = ptr[j] + lane; p < ptr[j + 1]; p += 32) major[p] = (int)j;
}

__global__ void k_iota(int* v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int)i;
}

__global__ void k_gather_entries(const int* __restrict__ perm, const int* __restrict__ major,
                                 const double2* __restrict__ val, int64_t nnz,
                                 int* __restrict__ out_idx, double2* __restrict__ out_val) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int p = perm[q];
    out_idx[q] = major[p];
    out_val[q] = val[p];
  }
}

__global__ void k_count_minor(const int* __restrict__ minor, int64_t nnz, int* __restrict__ cnt) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz;
       q += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + minor[q], 1);
}

__global__ void k_check_index(const int* __restrict__ ptr, const int* __restrict__ idx, int64_t n,
                              int64_t nnz, int* bad) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz;
       q += (int64_t)gridDim.x * blockDim.x)
    if (idx[q] < 0 || idx[q] >= n) atomicOr(bad, 1);
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    if (ptr[j + 1] < ptr[j]) atomicOr(bad, 2);
}

__device__ __forceinline__ double cabs2(double2 v) { return sqrt(v.x * v.x + v.y * v.y); }

// Symmetry probe: the transposed arrays (CSR of A^T) against the CSR of A.
// Pattern mismatch -> flag 1; value mismatch beyond 1e-12 sqrt(|a_ii a_jj|)
// (SURVEY D10's scale; A is symmetric only up to rounding) -> flag 2.
__global__ void k_symmetry(const int* __restrict__ rp, const int* __restrict__ col,
                           const double2* __restrict__ val, const int* __restrict__ trp,
                           const int* __restrict__ tcol, const double2* __restrict__ tval,
                           const double* __restrict__ dabs, int64_t n, int* flag) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += n_warps) {
    if (rp[i] != trp[i] || rp[i + 1] != trp[i + 1]) {
      if (lane == 0) atomicOr(flag, 1);
      continue;
    }
    for (int p = rp[i] + lane; p < rp[i + 1]; p += 32) {
      const int j = col[p];
      if (tcol[p] != j) {
        atomicOr(flag, 1);
        continue;
      }
      const double2 a = val[p], b = tval[p];
      const double d = hypot(a.x - b.x, a.y - b.y);
      const double scale = sqrt(dabs[i] * dabs[j]);
      if (d > 1e-12 * scale && d > 1e-14 * fmax(cabs2(a), cabs2(b))) atomicOr(flag, 2);
    }
  }
}

__global__ void k_diag_abs(const int* __restrict__ rp, const int* __restrict__ col,
                           const double2* __restrict__ val, int64_t n, double* dabs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double d = 0.0;
    for (int p = rp[i]; p < rp[i + 1]; ++p)
      if (col[p] == (int)i) d = cabs2(val[p]);
    dabs[i] = d;
  }
}

// Transpose (ptr, idx, val) of an n x n compressed matrix into (tptr, tidx, tval).
void transpose_compressed(ect_ctx* ctx, int64_t n, int64_t nnz, const int* ptr, const int* idx,
                          const double2* val, int* tptr, int* tidx, double2* tval) {
  cudaStream_t s = ctx->stream;
  DevBuf<int> major(nnz), perm_in(nnz), perm(nnz), keys_out(nnz), cnt(n + 1);
  k_expand_major<<<blocks_for(ctx, 32 * n), 256, 0, s>>>(ptr, n, major.p);
  CK_LAUNCH();
  k_iota<<<blocks_for(ctx, nnz), 256, 0, s>>>(perm_in.p, nnz);
  CK_LAUNCH();
  int bits = 1;
  while (bits < 31 && (1ll << bits) < n) ++bits;
  size_t tmp = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, idx, keys_out.p, perm_in.p, perm.p, (int)nnz,
                                     0, bits, s));
  CK(cub::DeviceRadixSort::SortPairs(cub_scratch(ctx, tmp), tmp, idx, keys_out.p, perm_in.p,
                                     perm.p, (int)nnz, 0, bits, s));
  k_gather_entries<<<blocks_for(ctx, nnz), 256, 0, s>>>(perm.p, major.p, val, nnz, tidx, tval);
  CK_LAUNCH();
  CK(cudaMemsetAsync(cnt.p, 0, cnt.bytes(), s));
  k_count_minor<<<blocks_for(ctx, nnz), 256, 0, s>>>(idx, nnz, cnt.p);
  CK_LAUNCH();
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.p, tptr, n + 1, s));
  CK(cub::DeviceScan::ExclusiveSum(cub_scratch(ctx, tmp), tmp, cnt.p, tptr, n + 1, s));
  note_launch(ctx, 6);
  CK(cudaStreamSynchronize(s));
}

}  // namespace

void matrix_from_compressed(ect_ctx* ctx, int64_t n, int64_t nnz, const int* ptr, const int* idx,
                            const double2* val, bool csc, ect_matrix* a) {
  cudaStream_t s = ctx->stream;
  {
    DevBuf<int> bad(1);
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    k_check_index<<<blocks_for(ctx, std::max(n, nnz)), 256, 0, s>>>(ptr, idx, n, nnz, bad.p);
    CK_LAUNCH();
    int h = 0;
    CK(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (h) fail(ECT_ERR_SOLVER, "matrix: index out of range or decreasing pointer array");
  }
  a->n = n;
  a->nnz = nnz;
  a->row_ptr.alloc(n + 1);
  a->col.alloc(nnz);
  a->val.alloc(nnz);
  DevBuf<int> tp(n + 1), ti(nnz);
  DevBuf<double2> tv(nnz);
  transpose_compressed(ctx, n, nnz, ptr, idx, val, tp.p, ti.p, tv.p);
  // csc: the transpose IS the CSR of A; csr: the input is, the transpose is A^T
  const int* rp = csc ? tp.p : ptr;
  const int* cl = csc ? ti.p : idx;
  const double2* vl = csc ? tv.p : val;
  const int* trp = csc ? ptr : tp.p;
  const int* tcl = csc ? idx : ti.p;
  const double2* tvl = csc ? val : tv.p;
  DevBuf<double> dabs(n);
  DevBuf<int> flag(1);
  CK(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
  k_diag_abs<<<blocks_for(ctx, n), 256, 0, s>>>(rp, cl, vl, n, dabs.p);
  CK_LAUNCH();
  k_symmetry<<<blocks_for(ctx, 32 * n), 256, 0, s>>>(rp, cl, vl, trp, tcl, tvl, dabs.p, n, flag.p);
  CK_LAUNCH();
  CK(cudaMemcpyAsync(a->row_ptr.p, rp, (n + 1) * sizeof(int), cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(a->col.p, cl, nnz * sizeof(int), cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(a->val.p, vl, nnz * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  int h = 0;
  CK(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  note_launch(ctx, 3);
  a->symmetric = h == 0;
  a->assembled = true;
  a->precond = ctx->precond;
}

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

void build_pattern(ect_mesh* m, ect_matrix* a, int64_t lo, int64_t hi) {
  ect_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  if (!m->have_nbr) build_neighbours(m);
  const int64_t nn = m->n_nodes;
  if (hi < 0) hi = nn;
  // rows of nodes [lo, hi) only (a slab of a row partition): the other rows
  // stay empty, indices stay global
  a->node_lo = lo;
  a->node_hi = hi;
  const int64_t N = 3 * nn + m->n_cond;
  DevBuf<int> row_len(N + 1);
  CK(cudaMemsetAsync(row_len.p, 0, row_len.bytes(), s));
  k_row_lengths<<<blocks_for(ctx, hi - lo), 256, 0, s>>>(m->nbr_off.p, m->nbr_cond.p,
                                                        m->cond_fwd.p, nn, row_len.p, lo, hi);
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
  a->mesh = m;
  a->precond = ctx->precond;
  a->row_ptr.alloc(N + 1);
  a->col.alloc(std::max<long long>(1, nnz));
  a->val.alloc(std::max<long long>(1, nnz));
  k_narrow_row_ptr<<<blocks_for(ctx, N + 1), 256, 0, s>>>(rp64.p, N + 1, a->row_ptr.p);
  CK_LAUNCH();
  k_fill_columns<<<blocks_for(ctx, 32 * (hi - lo)), 256, 0, s>>>(
      m->nbr_off.p, m->nbr.p, m->nbr_cond.p, m->cond_fwd.p, a->row_ptr.p, nn, a->col.p, lo, hi);
  CK_LAUNCH();
  note_launch(ctx, 4);
  CK(cudaStreamSynchronize(s));
}

}  // namespace ect
