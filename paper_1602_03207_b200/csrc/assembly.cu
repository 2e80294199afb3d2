// K2: numeric assembly of the A–V matrix, fused with the essential-BC pins.
//
// Replaces assemble_system (assembly.cpp:243-276) -> assemble_block
// (assembly.cpp:74-235) -> reduce_blocks/canonicalize (sparse.cpp:13-57) ->
// apply_essential_bc/apply_pins_to_matrix (assembly.cpp:285-327) ->
// build_global/from_triplets (assembly.cpp:386-419, sparse.cpp:83-113).
//
// B200 design — row-owner gather, no fp64 atomics, no triplets:
//   * one warp per mesh node i owns the 3 A-rows of i and its V-row;
//   * lane r owns neighbour m_r (from K1's neighbour list), i.e. the 3x3
//     A-A block (3i+c, 3m_r+d), the A-V column, the V-A row and the V-V entry;
//   * the warp walks i's incident tets in ascending tet id (the reference's
//     insertion order with one partition), each lane computing one tet frame
//     per 32-tet chunk into shared memory; every lane then adds the local
//     entry (a_i, b_{m_r}) of each tet containing m_r — so every CSR slot is
//     a left fold over tets in exactly the reference's order, written once.
//   * compiled with -fmad=false: element arithmetic is the reference's IEEE
//     sequence (elements.cuh), making the values bit-identical to the oracle.
// Bytes: coords/connectivity gathers (L2-resident) + one write of each value.
#include <cub/cub.cuh>

#include <algorithm>
#include <array>
#include <complex>

#include "elements.cuh"
#include "ect_internal.h"

namespace ect {
namespace {

constexpr int kWarps = 8;  // warps per block

__device__ __forceinline__ bool is_conductor(uint8_t r) {
  return r == ECT_REGION_TUBE || r == ECT_REGION_TSP || r == ECT_REGION_DEFECT;
}

struct AsmParams {
  RegionCoef coef[ECT_REGION_COUNT];
  double bc_penalty;
  int l22_eps;  // MaterialTable::l22_use_sigma_eps
  // impedance surface terms (element_ibc, element_forms.cpp:116-151), with the
  // complex prefactors formed on the host exactly as the reference does:
  // k1 = -iw * inv_z (aa, va), k2 = -inv_z (av, vv), inv_z = 1.0 / z_surface
  double2 k1, k2;
  const int* ibc_off;      // node -> incident GAMMA_P faces (4 * face + position)
  const int* ibc_inc;
  const int* ibc_nodes;    // [face][3] ascending node ids
  const double* ibc_frame; // [face][13] TriFrame: area, normal, grad_tau
};

// TriFrame::from (element_forms.cpp:32-44) with the shim's cross/norm order.
__global__ void k_tri_frames(int64_t n_faces, const int* __restrict__ fnodes,
                             const double* __restrict__ xyz, double* __restrict__ frame,
                             int* err) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n_faces;
       f += (int64_t)gridDim.x * blockDim.x) {
    double p[3][3];
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int c = 0; c < 3; ++c) p[q][c] = xyz[3 * (int64_t)fnodes[3 * f + q] + c];
    double e1[3], e2[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      e1[c] = p[1][c] - p[0][c];
      e2[c] = p[2][c] - p[0][c];
    }
    const double cr[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                          e1[0] * e2[1] - e1[1] * e2[0]};
    const double two_area = sqrt((cr[0] * cr[0] + cr[1] * cr[1]) + cr[2] * cr[2]);
    if (!(two_area > 0.0)) atomicOr(err, 2);
    double* F = frame + 13 * f;
    F[0] = 0.5 * two_area;
    double n[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) F[1 + c] = n[c] = cr[c] / two_area;
    double opp[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      opp[0][c] = p[2][c] - p[1][c];
      opp[1][c] = p[0][c] - p[2][c];
      opp[2][c] = p[1][c] - p[0][c];
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double* o = opp[a];
      const double g[3] = {n[1] * o[2] - n[2] * o[1], n[2] * o[0] - n[0] * o[2],
                           n[0] * o[1] - n[1] * o[0]};
#pragma unroll
      for (int c = 0; c < 3; ++c) F[4 + 3 * a + c] = g[c] / two_area;
    }
  }
}

struct TetSlot {
  double g[4][3];
  double vol;
  int nodes[4];
  int region;
  int a;  // local index of the owning node
};

template <bool IBC>
__global__ void __launch_bounds__(kWarps * 32)
k_assemble(const int4* __restrict__ tets, const uint8_t* __restrict__ region,
           const double* __restrict__ xyz, const int* __restrict__ inc_off,
           const int* __restrict__ inc, const int* __restrict__ nbr_off,
           const int* __restrict__ nbr, const uint8_t* __restrict__ nbr_cond,
           const int* __restrict__ cond_fwd, const uint8_t* __restrict__ pinned,
           const int* __restrict__ row_ptr, int64_t n_nodes, AsmParams P, double2* val,
           int* err, int64_t lo, int64_t hi) {
  __shared__ TetSlot slots[kWarps][32];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  TetSlot* my = slots[wib];
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int na = (int)(3 * n_nodes);

  for (int64_t i = lo + warp; i < hi; i += n_warps) {
    const int ib = inc_off[i], deg = inc_off[i + 1] - ib;
    const int nb = nbr_off[i], u = nbr_off[i + 1] - nb;
    int ncc = 0;
    for (int r0 = 0; r0 < u; r0 += 32) {
      bool c = (r0 + lane < u) && nbr_cond[nb + r0 + lane];
      ncc += __popc(__ballot_sync(0xffffffffu, c));
    }
    const int cf_i = cond_fwd[i];
    int rc0 = 0;
    for (int r0 = 0; r0 < u; r0 += 32) {
      const int r = r0 + lane;
      const bool valid = r < u;
      const int m = valid ? nbr[nb + r] : -1;
      const bool mc = valid && nbr_cond[nb + r];
      const unsigned cmask = __ballot_sync(0xffffffffu, mc);
      const int rc = rc0 + __popc(cmask & ((1u << lane) - 1u));
      rc0 += __popc(cmask);

      double aa[3][3];     // A-A real parts
      double aa_im[3];     // imaginary parts live on c == d only (volume terms)
      double av[3], va[3];  // couplings are real (element_forms.cpp:75-99)
      double vv_re = 0.0, vv_im = 0.0;
      // IBC: complex surface terms everywhere (aa off-diagonal, couplings)
      double aa_oim[3][3], av_im[3], va_im[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        av_im[c] = va_im[c] = 0.0;
#pragma unroll
        for (int d = 0; d < 3; ++d) aa_oim[c][d] = 0.0;
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        aa_im[c] = 0.0;
        av[c] = 0.0;
        va[c] = 0.0;
#pragma unroll
        for (int d = 0; d < 3; ++d) aa[c][d] = 0.0;
      }
      bool seen = false, seen_c = false;

      for (int t0 = 0; t0 < deg; t0 += 32) {
        const int cnt = min(32, deg - t0);
        __syncwarp();
        if (lane < cnt) {
          const int e = inc[ib + t0 + lane];
          const int t = e >> 2;
          const int4 k = tets[t];
          TetSlot& S = my[lane];
          S.nodes[0] = k.x;
          S.nodes[1] = k.y;
          S.nodes[2] = k.z;
          S.nodes[3] = k.w;
          S.region = region[t];
          S.a = e & 3;
          double p[4][3];
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int c = 0; c < 3; ++c) p[q][c] = xyz[3 * (int64_t)S.nodes[q] + c];
          TetGeom f;
          tet_frame(p, f);
          if (!f.ok) atomicOr(err, 1);
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int c = 0; c < 3; ++c) S.g[q][c] = f.g[q][c];
          S.vol = f.vol;
        }
        __syncwarp();
        if (valid) {
          for (int q = 0; q < cnt; ++q) {
            const TetSlot& S = my[q];
            const int b = S.nodes[0] == m ? 0 : S.nodes[1] == m ? 1 : S.nodes[2] == m ? 2
                                                                : S.nodes[3] == m ? 3 : -1;
            if (b < 0) continue;
            const int a = S.a;
            const RegionCoef& C = P.coef[S.region];
            const double vol = S.vol;
            double ga[3], gb[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              ga[c] = S.g[a][c];
              gb[c] = S.g[b][c];
            }
            // element_l11 (element_forms.cpp:49-73)
            const double dot = dot3(ga, gb);
            const double mass = (vol * (a == b ? 2.0 : 1.0)) / 20.0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
#pragma unroll
              for (int d = 0; d < 3; ++d) {
                const double curl = (c == d ? dot : 0.0) - ga[d] * gb[c];
                double value = vol * (C.mu_inv * curl + (C.mt_inv * ga[c]) * gb[d]);
                if (c == d) value = value + 0.0;  // complexd += (0*mass, ...)
                aa[c][d] = seen ? aa[c][d] + value : value;
              }
              const double im = 0.0 + C.mass_im * mass;
              aa_im[c] = seen ? aa_im[c] + im : im;
            }
            seen = true;
            if (is_conductor((uint8_t)S.region)) {
              const double w = vol / 4.0;
              // element_l12 (3a+c, b) and element_l21 (a, 3b+d)
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                const double x12 = (C.neg_sigma * gb[c]) * w;
                const double x21 = (C.neg_sigma * ga[c]) * w;
                av[c] = seen_c ? av[c] + x12 : x12;
                va[c] = seen_c ? va[c] + x21 : x21;
              }
              // element_l22 (element_forms.cpp:101-114) [+ l22_use_sigma_eps branch,
              // assembly.cpp:147-158]
              const double s = vol * dot;
              double re, imv;
              if (!P.l22_eps) {
                re = (0.0 * s) + C.gauge * mass;
                imv = C.stiff_im * s;
              } else {
                const double g_re = ((0.0 * s) + C.gauge * mass) - ((0.0 * s) + 0.0 * mass);
                const double g_im = C.stiff_im * s - C.stiff_im * s;
                re = ((0.0 * s) + 0.0 * mass) + g_re;
                imv = C.stiff_im_eps * s + g_im;
              }
              vv_re = seen_c ? vv_re + re : re;
              vv_im = seen_c ? vv_im + imv : imv;
              seen_c = true;
            }
          }
        }
      }

      if (IBC && valid) {
        // surface terms of the impedance condition, after every volume term of
        // the entry (assembly.cpp:182-233), faces in boundary_faces order
        for (int e = P.ibc_off[i]; e < P.ibc_off[i + 1]; ++e) {
          const int ent = P.ibc_inc[e], f = ent >> 2, a = ent & 3;
          const int* fn = P.ibc_nodes + 3 * (int64_t)f;
          const int b = fn[0] == m ? 0 : fn[1] == m ? 1 : fn[2] == m ? 2 : -1;
          if (b < 0) continue;
          const double* F = P.ibc_frame + 13 * (int64_t)f;
          const double area = F[0];
          const double* nrm = F + 1;
          const double* gt = F + 4;  // grad_tau[p][c] = gt[3 p + c]
          const double mass = (area * (a == b ? 2.0 : 1.0)) / 12.0;
          const double2 km = make_double2(P.k1.x * mass, P.k1.y * mass);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              const double proj = (c == d ? 1.0 : 0.0) - nrm[c] * nrm[d];
              aa[c][d] = aa[c][d] + km.x * proj;
              if (c == d) aa_im[c] = aa_im[c] + km.y * proj;
              else aa_oim[c][d] = aa_oim[c][d] + km.y * proj;
            }
          }
          if (mc) {
            const double third = area / 3.0;
            const double2 k2t = make_double2(P.k2.x * third, P.k2.y * third);
            const double2 k1t = make_double2(P.k1.x * third, P.k1.y * third);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              av[c] = av[c] + k2t.x * gt[3 * b + c];
              av_im[c] = av_im[c] + k2t.y * gt[3 * b + c];
              va[c] = va[c] + k1t.x * gt[3 * a + c];
              va_im[c] = va_im[c] + k1t.y * gt[3 * a + c];
            }
            const double dot = (gt[3 * a] * gt[3 * b] + gt[3 * a + 1] * gt[3 * b + 1]) +
                               gt[3 * a + 2] * gt[3 * b + 2];
            const double2 ka = make_double2(P.k2.x * area, P.k2.y * area);
            vv_re = vv_re + ka.x * dot;
            vv_im = vv_im + ka.y * dot;
          }
        }
      }

      if (valid) {
        // apply_pins_to_matrix: overwrite the pinned diagonal (assembly.cpp:314-327)
        if (m == (int)i) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            if (pinned[3 * i + c]) {
              aa[c][c] = P.bc_penalty;
              aa_im[c] = 0.0;
            }
          }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int base = row_ptr[3 * i + c];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            val[base + 3 * r + d] = make_double2(aa[c][d], c == d ? aa_im[c] : aa_oim[c][d]);
          }
          if (mc) val[base + 3 * u + rc] = make_double2(av[c], av_im[c]);
        }
        if (mc && cf_i >= 0) {
          const int basev = row_ptr[na + cf_i];
#pragma unroll
          for (int d = 0; d < 3; ++d) val[basev + 3 * rc + d] = make_double2(va[d], va_im[d]);
          val[basev + 3 * ncc + rc] = make_double2(vv_re, vv_im);
        }
      }
    }
  }
}

}  // namespace

// GAMMA_P faces (classify_boundary, mesh.cpp:145-182: interior faces between a
// TSP tet and a non-conductor tet) as sorted node triples in ascending order —
// the order of mesh.boundary_faces, hence of AssemblyPlan::part_ibc_faces with
// one partition (assembly.cpp:28-53) — plus their frames and node incidence.
void build_ibc_faces(ect_mesh* m) {
  if (m->have_ibc) return;
  ect_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  const int64_t nt = m->n_tets;
  std::vector<std::array<int, 4>> recs;  // sorted face nodes + tet
  recs.reserve(4 * nt);
  static const int fl[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
  for (int64_t t = 0; t < nt; ++t) {
    const int* k = &m->h_tets[4 * t];
    for (const auto& q : fl) {
      std::array<int, 3> f{k[q[0]], k[q[1]], k[q[2]]};
      std::sort(f.begin(), f.end());
      recs.push_back({f[0], f[1], f[2], (int)t});
    }
  }
  std::sort(recs.begin(), recs.end());
  auto cond = [](uint8_t r) {
    return r == ECT_REGION_TUBE || r == ECT_REGION_TSP || r == ECT_REGION_DEFECT;
  };
  std::vector<int> faces;
  for (size_t i = 0; i + 1 < recs.size();) {
    size_t j = i + 1;
    while (j < recs.size() && recs[j][0] == recs[i][0] && recs[j][1] == recs[i][1] &&
           recs[j][2] == recs[i][2])
      ++j;
    if (j - i == 2) {
      const uint8_t r0 = m->h_region[recs[i][3]], r1 = m->h_region[recs[i + 1][3]];
      if (cond(r0) != cond(r1) && (cond(r0) ? r0 : r1) == ECT_REGION_TSP)
        faces.insert(faces.end(), {recs[i][0], recs[i][1], recs[i][2]});
    }
    i = j;
  }
  const int64_t nf = (int64_t)faces.size() / 3, nn = m->n_nodes;
  std::vector<int> off(nn + 1, 0), inc(3 * nf);
  for (int64_t f = 0; f < nf; ++f)
    for (int q = 0; q < 3; ++q) ++off[faces[3 * f + q] + 1];
  for (int64_t i = 0; i < nn; ++i) off[i + 1] += off[i];
  std::vector<int> fill(off.begin(), off.end() - 1);
  for (int64_t f = 0; f < nf; ++f)
    for (int q = 0; q < 3; ++q) inc[fill[faces[3 * f + q]]++] = (int)(4 * f + q);
  m->ibc_nodes.alloc(std::max<int64_t>(1, 3 * nf));
  m->ibc_frame.alloc(std::max<int64_t>(1, 13 * nf));
  m->ibc_off.alloc(nn + 1);
  m->ibc_inc.alloc(std::max<int64_t>(1, 3 * nf));
  if (nf) {
    CK(cudaMemcpy(m->ibc_nodes.p, faces.data(), faces.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(m->ibc_inc.p, inc.data(), inc.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  CK(cudaMemcpy(m->ibc_off.p, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice));
  if (nf) {
    DevBuf<int> err(1);
    CK(cudaMemsetAsync(err.p, 0, sizeof(int), s));
    const int grid = (int)std::min<int64_t>((nf + 255) / 256, (int64_t)ctx->num_sms * 8);
    k_tri_frames<<<std::max(grid, 1), 256, 0, s>>>(nf, m->ibc_nodes.p, m->xyz.p, m->ibc_frame.p,
                                                    err.p);
    CK_LAUNCH();
    note_launch(ctx, 1);
    int h = 0;
    CK(cudaMemcpyAsync(&h, err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (h) fail(ECT_ERR_MESH, "element frame on a zero-area triangle");
  }
  m->n_ibc = nf;
  m->have_ibc = true;
}

void assemble_values(ect_mesh* m, const ect_materials& mats, ect_matrix* a) {
  ect_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  if (!a->from_mesh || a->n_nodes != m->n_nodes) {
    fail(ECT_ERR_SOLVER, "assemble: matrix pattern was not built from this mesh");
  }
  AsmParams P{};
  for (int r = 0; r < ECT_REGION_COUNT; ++r) {
    RegionCoef& C = P.coef[r];
    const double sigma = mats.sigma[r], mu = mats.mu[r];
    C.mu_inv = 1.0 / mu;
    C.mt_inv = 1.0 / mats.mu_tilde;
    C.mass_im = (-1.0 * mats.omega) * sigma;
    C.sigma = sigma;
    C.neg_sigma = -sigma;
    C.stiff_im = sigma / mats.omega;
    C.gauge = (mats.delta_gauge * mu) * sigma;
    C.stiff_im_eps = mats.sigma_eps / mats.omega;
  }
  P.bc_penalty = mats.bc_penalty;
  P.l22_eps = mats.l22_use_sigma_eps;
  const bool ibc = mats.ibc_enabled != 0;
  if (ibc) {
    build_ibc_faces(m);
    // element_ibc's prefactors, formed on the host with the reference's
    // std::complex arithmetic (1.0 / z, complex product)
    const std::complex<double> z(mats.z_surface[0], mats.z_surface[1]);
    if (z == std::complex<double>(0.0, 0.0))
      fail(ECT_ERR_SOLVER, "impedance surface term with zero surface impedance");
    const std::complex<double> inv_z = 1.0 / z;
    const std::complex<double> iw(0.0, mats.omega);
    const std::complex<double> k1 = -iw * inv_z, k2 = -inv_z;
    P.k1 = make_double2(k1.real(), k1.imag());
    P.k2 = make_double2(k2.real(), k2.imag());
    P.ibc_off = m->ibc_off.p;
    P.ibc_inc = m->ibc_inc.p;
    P.ibc_nodes = m->ibc_nodes.p;
    P.ibc_frame = m->ibc_frame.p;
  }
  DevBuf<int> err(1);
  CK(cudaMemsetAsync(err.p, 0, sizeof(int), s));
  const int64_t lo = a->node_lo, hi = a->node_hi < 0 ? m->n_nodes : a->node_hi;
  int64_t blocks = (hi - lo + kWarps - 1) / kWarps;
  int64_t cap = (int64_t)ctx->num_sms * 8;
  if (blocks > cap) blocks = cap;
  auto kern = ibc ? k_assemble<true> : k_assemble<false>;
  kern<<<(int)blocks, kWarps * 32, 0, s>>>(m->tets.p, m->region.p, m->xyz.p, m->inc_off.p,
                                          m->inc.p, m->nbr_off.p, m->nbr.p, m->nbr_cond.p,
                                          m->cond_fwd.p, m->pinned.p, a->row_ptr.p, m->n_nodes, P,
                                          a->val.p, err.p, lo, hi);
  CK_LAUNCH();
  note_launch(ctx, 1);
  int h_err = 0;
  CK(cudaMemcpyAsync(&h_err, err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (h_err) fail(ECT_ERR_MESH, "element frame on a degenerate or inverted tet");
  a->assembled = true;
  a->symmetric = !ibc;  // element_ibc: va = i omega av^T
  compute_jacobi(a);
  if (a->node_lo > 0 || (a->node_hi >= 0 && a->node_hi < m->n_nodes)) return;  // slab: see create_part_assembled
  if (ctx->use_sell) build_sell(a, ctx->sell_sigma);
  else if (!ctx->force_csr) build_nb(m, a);
}

}  // namespace ect
