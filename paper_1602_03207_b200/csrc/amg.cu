// Aggregation-multigrid setup: the GPU replacement for the reference's ILU(0)
// preconditioner (Ilu0, iterative.cpp:59-105, rebuilt on every
// solve_iterative call at :126). ILU(0) is a sequential triangular sweep; on
// B200 the preconditioner has to be bandwidth-parallel, so the hierarchy is
//
//   * node aggregation (host, greedy three phase, deterministic) of the
//     node graph: mesh nodes on the finest level (the 3 A-dofs and the V-dof
//     of a node move together), aggregates on coarser ones;
//   * plain-aggregation prolongator P_l: dof i -> coarse dof (agg(node(i)),
//     kind(i)), kind = A component 0..2 or V; Dirichlet-pinned dofs (penalty
//     rows, |a_ii| >> sum_j |a_ij|: apply_essential_bc, assembly.cpp:285-327)
//     stay on the fine level only;
//   * Galerkin coarse operators A_{l+1} = P_l^T A_l P_l on the GPU: one
//     (coarse row, coarse col) key per fine entry, a radix sort, a
//     sequential per-key sum in sorted order (deterministic, no atomics);
//     with the plain transpose the hierarchy and the cycle stay complex
//     symmetric, so COCG applies;
//   * the coarsest level (<= kDenseMax dofs) inverted densely on the host.
//
// The cycle (damped-Jacobi smoothing, W-cycle, over-weighted coarse
// correction) runs in krylov.cu next to the COCG kernels it feeds.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <complex>
#include <cstdlib>
#include <numeric>

#include "ect_internal.h"

namespace ect {
namespace {

constexpr int64_t kDenseMaxDefault = 1200;  // coarsest level solved by a dense inverse
constexpr int kMaxLevels = 12;
constexpr double kPinRatio = 1e6;     // |a_ii| > kPinRatio * sum_{j != i} |a_ij| -> pinned

int blocks_for(ect_ctx* ctx, int64_t n, int block = 256) {
  int64_t b = (n + block - 1) / block;
  int64_t cap = (int64_t)ctx->num_sms * 16;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

__device__ __forceinline__ double cabs_d(double2 v) { return sqrt(v.x * v.x + v.y * v.y); }

// free[i] = 1 unless row i is a penalty (Dirichlet) row
__global__ void k_free_rows(const int* __restrict__ rp, const int* __restrict__ col,
                            const double2* __restrict__ val, int64_t n, uint8_t* free_) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double d = 0.0, off = 0.0;
    for (int p = rp[i]; p < rp[i + 1]; ++p) {
      const double a = cabs_d(val[p]);
      if (col[p] == (int)i) d += a; else off += a;
    }
    free_[i] = !(d > kPinRatio * off) && d > 0.0;
  }
}

// Galerkin keys: one per stored entry, (cmap[i], cmap[j]) or the sentinel nc^2.
__global__ void k_galerkin_keys(const int* __restrict__ rp, const int* __restrict__ col,
                                const int* __restrict__ cmap, int64_t n, int64_t nc,
                                unsigned long long* __restrict__ keys, int* __restrict__ idx) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned long long sentinel = (unsigned long long)nc * (unsigned long long)nc;
  for (int64_t i = warp; i < n; i += n_warps) {
    const int ci = cmap[i];
    for (int p = rp[i] + lane; p < rp[i + 1]; p += 32) {
      const int cj = cmap[col[p]];
      keys[p] = (ci >= 0 && cj >= 0) ? (unsigned long long)ci * nc + (unsigned long long)cj
                                     : sentinel;
      idx[p] = p;
    }
  }
}

__global__ void k_segment_heads(const unsigned long long* __restrict__ keys, int64_t nnz,
                                unsigned long long sentinel, int* __restrict__ head) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz;
       q += (int64_t)gridDim.x * blockDim.x)
    head[q] = keys[q] != sentinel && (q == 0 || keys[q] != keys[q - 1]);
}

// segment s = sorted positions [start_s, start_{s+1}); its sum in sorted
// (= fine CSR) order, its coarse column, and a row count
__global__ void k_segment_sums(const unsigned long long* __restrict__ keys,
                               const int* __restrict__ perm, const double2* __restrict__ val,
                               const int* __restrict__ head, const int* __restrict__ seg_of,
                               int64_t nnz, int64_t nc, int64_t n_seg, int* __restrict__ ccol,
                               double2* __restrict__ cval, int* __restrict__ row_cnt) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz;
       q += (int64_t)gridDim.x * blockDim.x) {
    if (!head[q]) continue;
    const unsigned long long key = keys[q];
    double2 s = make_double2(0.0, 0.0);
    for (int64_t e = q; e < nnz && keys[e] == key; ++e) {
      const double2 v = val[perm[e]];
      s.x += v.x;
      s.y += v.y;
    }
    const int sg = seg_of[q];
    ccol[sg] = (int)(key % (unsigned long long)nc);
    cval[sg] = s;
    atomicAdd(row_cnt + (key / (unsigned long long)nc), 1);
  }
}

__global__ void k_dinv(const int* __restrict__ rp, const int* __restrict__ col,
                       const double2* __restrict__ val, int64_t n, double2* dinv, int* missing) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 d = make_double2(0.0, 0.0);
    for (int p = rp[i]; p < rp[i + 1]; ++p)
      if (col[p] == (int)i) d = val[p];
    if (d.x == 0.0 && d.y == 0.0) {
      atomicAdd(missing, 1);
      dinv[i] = make_double2(0.0, 0.0);
    } else {
      const double den = d.x * d.x + d.y * d.y;
      dinv[i] = make_double2(d.x / den, -d.y / den);
    }
  }
}

// Greedy aggregation (deterministic, ascending node order):
//  1. a node whose whole neighbourhood is unaggregated seeds an aggregate
//     with all its neighbours;
//  2. leftovers join the aggregate of their first aggregated neighbour;
//  3. what remains seeds aggregates with its unaggregated neighbours.
int64_t aggregate(int64_t n, const std::vector<int64_t>& ptr, const std::vector<int>& adj,
                  std::vector<int>& agg) {
  agg.assign(n, -1);
  int64_t na = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (agg[i] >= 0) continue;
    bool free_nb = true;
    for (int64_t p = ptr[i]; p < ptr[i + 1] && free_nb; ++p) free_nb = agg[adj[p]] < 0;
    if (!free_nb) continue;
    agg[i] = (int)na;
    for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p) agg[adj[p]] = (int)na;
    ++na;
  }
  std::vector<int> join(n, -1);
  for (int64_t i = 0; i < n; ++i) {
    if (agg[i] >= 0) continue;
    for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p)
      if (agg[adj[p]] >= 0) {
        join[i] = agg[adj[p]];
        break;
      }
  }
  for (int64_t i = 0; i < n; ++i)
    if (join[i] >= 0) agg[i] = join[i];
  for (int64_t i = 0; i < n; ++i) {
    if (agg[i] >= 0) continue;
    agg[i] = (int)na;
    for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p)
      if (agg[adj[p]] < 0) agg[adj[p]] = (int)na;
    ++na;
  }
  return na;
}

// Dense complex inverse (Gauss-Jordan, partial pivoting), row-major.
void dense_inverse(int64_t n, std::vector<std::complex<double>>& a,
                   std::vector<std::complex<double>>& inv) {
  inv.assign(n * n, 0.0);
  for (int64_t i = 0; i < n; ++i) inv[i * n + i] = 1.0;
  for (int64_t c = 0; c < n; ++c) {
    int64_t piv = c;
    double best = std::abs(a[c * n + c]);
    for (int64_t r = c + 1; r < n; ++r)
      if (std::abs(a[r * n + c]) > best) {
        best = std::abs(a[r * n + c]);
        piv = r;
      }
    if (!(best > 0.0)) fail(ECT_ERR_SOLVER, "multigrid: singular coarsest operator");
    if (piv != c) {
      for (int64_t j = 0; j < n; ++j) {
        std::swap(a[c * n + j], a[piv * n + j]);
        std::swap(inv[c * n + j], inv[piv * n + j]);
      }
    }
    const std::complex<double> d = 1.0 / a[c * n + c];
    for (int64_t j = 0; j < n; ++j) {
      a[c * n + j] *= d;
      inv[c * n + j] *= d;
    }
    for (int64_t r = 0; r < n; ++r) {
      if (r == c) continue;
      const std::complex<double> f = a[r * n + c];
      if (f == 0.0) continue;
      for (int64_t j = 0; j < n; ++j) {
        a[r * n + j] -= f * a[c * n + j];
        inv[r * n + j] -= f * inv[c * n + j];
      }
    }
  }
}

// One level's matrix view (level 0 borrows the ect_matrix arrays).
struct Csr {
  int64_t n, nnz;
  const int* rp;
  const int* col;
  const double2* val;
};

template <typename T>
std::vector<T> download(ect_ctx* ctx, const T* p, size_t n) {
  std::vector<T> h(n);
  if (n) CK(cudaMemcpyAsync(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return h;
}

template <typename T>
void upload(ect_ctx* ctx, DevBuf<T>& d, const std::vector<T>& h) {
  d.alloc(std::max<size_t>(1, h.size()));
  if (!h.empty())
    CK(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
}

// A_c = P^T A P for the plain-aggregation P given by cmap (device).
void galerkin(ect_ctx* ctx, const Csr& A, const int* cmap, int64_t nc, AmgLevel& out) {
  cudaStream_t s = ctx->stream;
  const int64_t nnz = A.nnz;
  DevBuf<unsigned long long> keys(nnz), keys_s(nnz);
  DevBuf<int> idx(nnz), perm(nnz), head(nnz), seg_of(nnz);
  k_galerkin_keys<<<blocks_for(ctx, 32 * A.n), 256, 0, s>>>(A.rp, A.col, cmap, A.n, nc, keys.p,
                                                           idx.p);
  CK_LAUNCH();
  const unsigned long long sentinel = (unsigned long long)nc * (unsigned long long)nc;
  int bits = 1;
  while (bits < 64 && (1ull << bits) <= sentinel) ++bits;
  size_t tmp = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys.p, keys_s.p, idx.p, perm.p, nnz, 0, bits,
                                     s));
  CK(cub::DeviceRadixSort::SortPairs(cub_scratch(ctx, tmp), tmp, keys.p, keys_s.p, idx.p, perm.p,
                                     nnz, 0, bits, s));
  k_segment_heads<<<blocks_for(ctx, nnz), 256, 0, s>>>(keys_s.p, nnz, sentinel, head.p);
  CK_LAUNCH();
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, head.p, seg_of.p, nnz, s));
  CK(cub::DeviceScan::ExclusiveSum(cub_scratch(ctx, tmp), tmp, head.p, seg_of.p, nnz, s));
  int last_seg = 0, last_head = 0;
  CK(cudaMemcpyAsync(&last_seg, seg_of.p + nnz - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&last_head, head.p + nnz - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const int64_t n_seg = (int64_t)last_seg + last_head;
  if (n_seg >= (1ll << 31)) fail(ECT_ERR_SOLVER, "multigrid: coarse operator too large");
  out.n = nc;
  out.nnz = n_seg;
  out.col.alloc(std::max<int64_t>(1, n_seg));
  out.val.alloc(std::max<int64_t>(1, n_seg));
  DevBuf<int> cnt(nc + 1);
  CK(cudaMemsetAsync(cnt.p, 0, cnt.bytes(), s));
  k_segment_sums<<<blocks_for(ctx, nnz), 256, 0, s>>>(keys_s.p, perm.p, A.val, head.p, seg_of.p,
                                                     nnz, nc, n_seg, out.col.p, out.val.p, cnt.p);
  CK_LAUNCH();
  out.row_ptr.alloc(nc + 1);
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.p, out.row_ptr.p, nc + 1, s));
  CK(cub::DeviceScan::ExclusiveSum(cub_scratch(ctx, tmp), tmp, cnt.p, out.row_ptr.p, nc + 1, s));
  note_launch(ctx, 6);
  CK(cudaStreamSynchronize(s));
}

}  // namespace

void amg_setup(ect_matrix* a) {
  ect_ctx* ctx = a->ctx;
  cudaStream_t s = ctx->stream;
  const auto t0 = std::chrono::steady_clock::now();
  if (!a->symmetric) fail(ECT_ERR_SOLVER, "multigrid preconditioner needs a symmetric matrix");
  auto H = std::make_unique<Amg>();
  const int64_t N = a->n;
  // tuning overrides (experiments; the defaults are the measured choice)
  auto env_d = [](const char* k, double d) {
    const char* v = std::getenv(k);
    return v ? std::atof(v) : d;
  };
  const int64_t kDenseMax = (int64_t)env_d("ECT_AMG_DENSE_MAX", (double)kDenseMaxDefault);
  const double theta = env_d("ECT_AMG_THETA", 0.05);
  H->omega = env_d("ECT_AMG_OMEGA", H->omega);
  H->oc = env_d("ECT_AMG_OC", H->oc);
  H->wcycle = (int)env_d("ECT_AMG_WCYCLE", H->wcycle);
  H->f32 = env_d("ECT_AMG_F32", 1.0) != 0.0;

  // ---- level structure: A dofs [0, nA) grouped by node (3 components move
  // together), scalar V dofs [nA, n) aggregated on their own strength graph:
  // the V-V couplings are sigma-weighted (element_l22, element_forms.cpp:
  // 101-114), so a weak conductor between strong ones (the reference
  // configuration's sigma_eps deposit) separates V aggregates while the A
  // aggregates (curl-curl + div-div, material-uniform up to mu) cross it.
  // Matrices without mesh structure: every dof is a scalar A "node".
  int64_t nA = N, n_anode = N;
  std::vector<int> a_node, a_kind;  // per A dof
  std::vector<int64_t> gptr;        // A-node graph
  std::vector<int> gadj;
  if (a->from_mesh && a->mesh && a->mesh->have_nbr) {
    ect_mesh* m = a->mesh;
    n_anode = m->n_nodes;
    nA = 3 * n_anode;
    auto off = download(ctx, m->nbr_off.p, n_anode + 1);
    auto nbr = download(ctx, m->nbr.p, (size_t)off[n_anode]);
    a_node.resize(nA);
    a_kind.resize(nA);
    for (int64_t i = 0; i < nA; ++i) {
      a_node[i] = (int)(i / 3);
      a_kind[i] = (int)(i % 3);
    }
    gptr.assign(n_anode + 1, 0);
    gadj.reserve(off[n_anode]);
    for (int64_t i = 0; i < n_anode; ++i) {
      for (int p = off[i]; p < off[i + 1]; ++p)
        if (nbr[p] != (int)i) gadj.push_back(nbr[p]);
      gptr[i + 1] = (int64_t)gadj.size();
    }
  } else {
    auto rp = download(ctx, a->row_ptr.p, N + 1);
    auto cl = download(ctx, a->col.p, (size_t)a->nnz);
    a_node.resize(N);
    std::iota(a_node.begin(), a_node.end(), 0);
    a_kind.assign(N, 0);
    gptr.assign(N + 1, 0);
    gadj.reserve(a->nnz);
    for (int64_t i = 0; i < N; ++i) {
      for (int p = rp[i]; p < rp[i + 1]; ++p)
        if (cl[p] != (int)i) gadj.push_back(cl[p]);
      gptr[i + 1] = (int64_t)gadj.size();
    }
  }

  Csr A{N, a->nnz, a->row_ptr.p, a->col.p, a->val.p};
  H->lv.emplace_back();
  double nnz_sum = (double)a->nnz;
  for (int level = 0;; ++level) {
    AmgLevel& L = H->lv.back();
    L.n = A.n;
    L.nnz = A.nnz;
    if (A.n <= kDenseMax || level + 1 >= kMaxLevels) break;
    const int64_t nV = A.n - nA;
    // free (non-penalty) dofs
    DevBuf<uint8_t> free_d(A.n);
    k_free_rows<<<blocks_for(ctx, A.n), 256, 0, s>>>(A.rp, A.col, A.val, A.n, free_d.p);
    CK_LAUNCH();
    auto free_h = download(ctx, free_d.p, A.n);
    // A aggregation on the node graph
    std::vector<int> agg;
    const int64_t n_agg = aggregate(n_anode, gptr, gadj, agg);
    // V aggregation on the strong V-V couplings |a_ij| >= theta sqrt(|a_ii a_jj|)
    std::vector<int> aggv;
    int64_t n_aggv = 0;
    if (nV > 0) {
      auto vrp = download(ctx, A.rp + nA, nV + 1);
      const int base = vrp[0];
      auto vcl = download(ctx, A.col + base, (size_t)(vrp[nV] - base));
      auto vvl = download(ctx, A.val + base, (size_t)(vrp[nV] - base));
      std::vector<double> dv(nV, 0.0);
      for (int64_t r = 0; r < nV; ++r)
        for (int p = vrp[r] - base; p < vrp[r + 1] - base; ++p)
          if (vcl[p] == (int)(nA + r)) dv[r] = std::hypot(vvl[p].x, vvl[p].y);
      std::vector<int64_t> vptr(nV + 1, 0);
      std::vector<int> vadj;
      for (int64_t r = 0; r < nV; ++r) {
        for (int p = vrp[r] - base; p < vrp[r + 1] - base; ++p) {
          const int64_t c = (int64_t)vcl[p] - nA;
          if (c < 0 || c == r) continue;
          if (std::hypot(vvl[p].x, vvl[p].y) >= theta * std::sqrt(dv[r] * dv[c]))
            vadj.push_back((int)c);
        }
        vptr[r + 1] = (int64_t)vadj.size();
      }
      n_aggv = aggregate(nV, vptr, vadj, aggv);
    }
    // coarse dofs: A keys (agg, kind) ranked, then V aggregates
    std::vector<int> key_idx(3 * n_agg, -1);
    for (int64_t i = 0; i < nA; ++i)
      if (free_h[i]) key_idx[3 * (int64_t)agg[a_node[i]] + a_kind[i]] = 0;
    int64_t ncA = 0;
    for (auto& v : key_idx)
      if (v == 0) v = (int)ncA++;
    std::vector<int> vidx(n_aggv, -1);
    for (int64_t r = 0; r < nV; ++r)
      if (free_h[nA + r]) vidx[aggv[r]] = 0;
    int64_t nc = ncA;
    for (auto& v : vidx)
      if (v == 0) v = (int)nc++;
    if (nc == 0 || nc * 5 > A.n * 4) break;  // no useful coarsening: current level is coarsest
    std::vector<int> cmap(A.n, -1), r_ptr(nc + 1, 0), r_idx;
    for (int64_t i = 0; i < A.n; ++i) {
      if (!free_h[i]) continue;
      cmap[i] = i < nA ? key_idx[3 * (int64_t)agg[a_node[i]] + a_kind[i]] : vidx[aggv[i - nA]];
      ++r_ptr[cmap[i] + 1];
    }
    for (int64_t c = 0; c < nc; ++c) r_ptr[c + 1] += r_ptr[c];
    r_idx.resize(r_ptr[nc]);
    {
      std::vector<int> fill(r_ptr.begin(), r_ptr.end() - 1);
      for (int64_t i = 0; i < A.n; ++i)
        if (cmap[i] >= 0) r_idx[fill[cmap[i]]++] = (int)i;
    }
    upload(ctx, L.cmap, cmap);
    upload(ctx, L.r_ptr, r_ptr);
    upload(ctx, L.r_idx, r_idx);
    L.n_next = nc;
    // coarse operator
    H->lv.emplace_back();
    AmgLevel& C = H->lv.back();
    galerkin(ctx, A, H->lv[H->lv.size() - 2].cmap.p, nc, C);
    nnz_sum += (double)C.nnz;
    A = Csr{C.n, C.nnz, C.row_ptr.p, C.col.p, C.val.p};
    // coarse A-node structure: node = aggregate, kind kept; graph from the
    // coarse A-A couplings
    std::vector<int> cnode(ncA), ckind(ncA);
    for (int64_t k = 0; k < 3 * n_agg; ++k)
      if (key_idx[k] >= 0) {
        cnode[key_idx[k]] = (int)(k / 3);
        ckind[key_idx[k]] = (int)(k % 3);
      }
    auto crp = download(ctx, C.row_ptr.p, ncA + 1);
    auto ccl = download(ctx, C.col.p, (size_t)crp[ncA]);
    std::vector<std::vector<int>> nb(n_agg);
    for (int64_t r = 0; r < ncA; ++r)
      for (int p = crp[r]; p < crp[r + 1]; ++p)
        if (ccl[p] < ncA && cnode[ccl[p]] != cnode[r]) nb[cnode[r]].push_back(cnode[ccl[p]]);
    gptr.assign(n_agg + 1, 0);
    gadj.clear();
    for (int64_t g = 0; g < n_agg; ++g) {
      auto& v = nb[g];
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
      gadj.insert(gadj.end(), v.begin(), v.end());
      gptr[g + 1] = (int64_t)gadj.size();
    }
    n_anode = n_agg;
    nA = ncA;
    a_node = std::move(cnode);
    a_kind = std::move(ckind);
  }
  // Jacobi diagonals of every level (level 0: the matrix's own dinv)
  for (size_t l = 1; l < H->lv.size(); ++l) {
    AmgLevel& L = H->lv[l];
    L.dinv.alloc(L.n);
    DevBuf<int> missing(1);
    CK(cudaMemsetAsync(missing.p, 0, sizeof(int), s));
    k_dinv<<<blocks_for(ctx, L.n), 256, 0, s>>>(L.row_ptr.p, L.col.p, L.val.p, L.n, L.dinv.p,
                                               missing.p);
    CK_LAUNCH();
  }
  // coarsest: dense inverse
  {
    AmgLevel& L = H->lv.back();
    const int64_t n = L.n;
    if (n > 4 * kDenseMax) fail(ECT_ERR_SOLVER, "multigrid: coarsest level too large");
    std::vector<int> rp, cl;
    std::vector<double2> vl;
    if (H->lv.size() == 1) {
      rp = download(ctx, a->row_ptr.p, n + 1);
      cl = download(ctx, a->col.p, (size_t)a->nnz);
      vl = download(ctx, a->val.p, (size_t)a->nnz);
    } else {
      rp = download(ctx, L.row_ptr.p, n + 1);
      cl = download(ctx, L.col.p, (size_t)L.nnz);
      vl = download(ctx, L.val.p, (size_t)L.nnz);
    }
    std::vector<std::complex<double>> dense(n * n, 0.0), inv;
    for (int64_t r = 0; r < n; ++r)
      for (int p = rp[r]; p < rp[r + 1]; ++p) dense[r * n + cl[p]] = {vl[p].x, vl[p].y};
    // The constant-V mode of each conductor component is lifted only by the
    // delta_gauge mass (element_forms.cpp:101-114; ~1e-14 relative)
    // and survives aggregation, so the coarsest operator is singular to
    // working precision (cond ~ 1e16 on configs[1]-like meshes). A relative
    // diagonal shift (1 + reg) keeps its inverse bounded; M stays symmetric.
    const double reg = env_d("ECT_AMG_REG", 1e-8);
    for (int64_t r = 0; r < n; ++r) dense[r * n + r] *= 1.0 + reg;
    dense_inverse(n, dense, inv);
    std::vector<double2> h(n * n);
    for (int64_t q = 0; q < n * n; ++q) h[q] = make_double2(inv[q].real(), inv[q].imag());
    upload(ctx, H->minv, h);
  }
  CK(cudaStreamSynchronize(s));
  H->op_complexity = nnz_sum / (double)a->nnz;
  H->setup_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  a->amg = std::move(H);
}

}  // namespace ect
