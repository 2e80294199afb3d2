// K3: coil right-hand sides, and K7: impedance variation over DEFECT tets.
//
// K3 replaces ScanSession::position_rhs (scan.cpp:87-93):
//   coil_support      tube_mesh.cpp:272-288  tets whose centroid has
//                     r = hypot(x, y) in [r_inner, r_outer] and z in the coil
//                     window (coil 1 below the probe plane, coil 2 above);
//   assemble_rhs      assembly.cpp:335-378   J = amp (-y/r, x/r, 0) at support
//                     nodes, then b[3k_a+c] += sum_b |K|(1+d_ab)/20 J_{k_b,c}
//                     over every tet touching a support node, in tet order;
//   apply_pins_to_rhs assembly.cpp:329-333   pinned entries = penalty * 0.
// Errors as the reference: empty support, support touching a conductor.
// The per-node accumulation is a row-owner gather over the node's incident
// tets in ascending order (deterministic; -fmad=false keeps the reference's
// operation sequence; hypot may differ from glibc by an ulp).
//
// K7 replaces delta_impedance (signals.cpp:67-99) with curl_on_tet /
// electric_field_on_tet (signals.cpp:22-56): per-tet contributions into a
// buffer, then one fixed-order reduction (deterministic).
#include "elements.cuh"
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

__device__ __forceinline__ void load_tet(const double* __restrict__ xyz, int4 k, double p[4][3]) {
  const int n[4] = {k.x, k.y, k.z, k.w};
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c) p[a][c] = xyz[3 * (int64_t)n[a] + c];
}

__global__ void k_support(const int4* __restrict__ tets, const uint8_t* __restrict__ region,
                          const double* __restrict__ xyz, int64_t n_tets, double r_in,
                          double r_out, double lo, double hi, uint8_t* node_flag, int* count,
                          int* conductor_hit) {
  int local = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tets;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int4 k = tets[t];
    double p[4][3];
    load_tet(xyz, k, p);
    double c[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) c[d] = 0.25 * (((p[0][d] + p[1][d]) + p[2][d]) + p[3][d]);
    const double r = hypot(c[0], c[1]);
    if (r >= r_in && r <= r_out && c[2] >= lo && c[2] <= hi) {
      ++local;
      if (is_conductor(region[t])) atomicMin(conductor_hit, (int)t);
      node_flag[k.x] = 1;
      node_flag[k.y] = 1;
      node_flag[k.z] = 1;
      node_flag[k.w] = 1;
    }
  }
  if (local) atomicAdd(count, local);
}

// assemble_rhs(mesh, support_tets, ...) (assembly.cpp:335-349): flag the
// support nodes of a caller-supplied tet list (or of every tet of a region
// when list == nullptr), report the first conductor tet like the reference.
__global__ void k_support_list(const int4* __restrict__ tets, const uint8_t* __restrict__ region,
                               const int* __restrict__ list, int64_t n_list, int tag,
                               int64_t n_tets, uint8_t* node_flag, int* count, int* conductor_hit,
                               int* bad_index) {
  int local = 0;
  const int64_t n = list ? n_list : n_tets;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = list ? (int64_t)list[q] : q;
    if (t < 0 || t >= n_tets) {
      atomicMin(bad_index, (int)q);
      continue;
    }
    if (!list && region[t] != tag) continue;
    ++local;
    if (is_conductor(region[t])) atomicMin(conductor_hit, (int)t);
    const int4 k = tets[t];
    node_flag[k.x] = 1;
    node_flag[k.y] = 1;
    node_flag[k.z] = 1;
    node_flag[k.w] = 1;
  }
  if (local) atomicAdd(count, local);
}

// apply_pins_to_rhs (assembly.cpp:329-333): pinned entries = penalty * 0.
__global__ void k_pin_rhs(const uint8_t* __restrict__ pinned, int64_t na, int stride,
                          double2* rhs) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < na * stride;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (pinned[e / stride]) rhs[e] = make_double2(0.0, 0.0);
  }
}

__global__ void k_nodal_current(const double* __restrict__ xyz, const uint8_t* __restrict__ flag,
                                int64_t n_nodes, double amplitude, double* j) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_nodes;
       i += (int64_t)gridDim.x * blockDim.x) {
    double jx = 0.0, jy = 0.0, jz = 0.0;
    if (flag[i]) {
      const double x = xyz[3 * i], y = xyz[3 * i + 1];
      const double r = hypot(x, y);
      if (r > 0.0) {
        jx = amplitude * (-y / r);
        jy = amplitude * (x / r);
        jz = amplitude * 0.0;
      }
    }
    j[3 * i] = jx;
    j[3 * i + 1] = jy;
    j[3 * i + 2] = jz;
  }
}

__global__ void k_rhs_gather(const int4* __restrict__ tets, const double* __restrict__ xyz,
                             const int* __restrict__ inc_off, const int* __restrict__ inc,
                             const uint8_t* __restrict__ flag, const double* __restrict__ j,
                             const uint8_t* __restrict__ pinned, int64_t n_nodes, int stride,
                             int column, double2* rhs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_nodes;
       i += (int64_t)gridDim.x * blockDim.x) {
    double out[3] = {0.0, 0.0, 0.0};
    bool any = false;
    for (int q = inc_off[i]; q < inc_off[i + 1]; ++q) {
      const int e = inc[q];
      const int4 k = tets[e >> 2];
      const int a = e & 3;
      const int n[4] = {k.x, k.y, k.z, k.w};
      if (!(flag[n[0]] | flag[n[1]] | flag[n[2]] | flag[n[3]])) continue;
      double p[4][3];
      load_tet(xyz, k, p);
      const double vol = signed_volume(p);
      double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const double s = (vol * (a == b ? 2.0 : 1.0)) / 20.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] = acc[c] + s * j[3 * (int64_t)n[b] + c];
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) out[c] = out[c] + acc[c];
      any = true;
    }
    if (!any) continue;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double v = (pinned && pinned[3 * i + c]) ? 0.0 : out[c];
      rhs[(3 * i + c) * (int64_t)stride + column] = make_double2(v, 0.0);
    }
  }
}

// ---- K7 --------------------------------------------------------------------
struct Cplx {
  double re, im;
};
__device__ __forceinline__ Cplx cm(Cplx a, Cplx b) {
  return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
__device__ __forceinline__ Cplx rc(double r, Cplx a) { return {r * a.re, r * a.im}; }
__device__ __forceinline__ Cplx ca(Cplx a, Cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ Cplx cs(Cplx a, Cplx b) { return {a.re - b.re, a.im - b.im}; }

struct DzParams {
  double omega;
  double mu_d[ECT_REGION_COUNT], mu_eps[ECT_REGION_COUNT];
  double sigma_d[ECT_REGION_COUNT], sigma_eps[ECT_REGION_COUNT];
};

__device__ void curl_and_field(const double2* __restrict__ x, int stride, const int n[4],
                               const TetGeom& f, const int* __restrict__ cond_fwd, int64_t na,
                               double omega, Cplx curl[3], Cplx e[3]) {
  Cplx mean[3] = {{0, 0}, {0, 0}, {0, 0}};
  Cplx gv[3] = {{0, 0}, {0, 0}, {0, 0}};
#pragma unroll
  for (int c = 0; c < 3; ++c) curl[c] = {0.0, 0.0};
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    Cplx A[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double2 v = x[(3 * (int64_t)n[a] + c) * stride];
      A[c] = {v.x, v.y};
    }
    const double* g = f.g[a];
    // curl(lam_a A_a) = grad(lam_a) x A_a   (signals.cpp:22-35)
    curl[0] = ca(curl[0], cs(rc(g[1], A[2]), rc(g[2], A[1])));
    curl[1] = ca(curl[1], cs(rc(g[2], A[0]), rc(g[0], A[2])));
    curl[2] = ca(curl[2], cs(rc(g[0], A[1]), rc(g[1], A[0])));
#pragma unroll
    for (int c = 0; c < 3; ++c) mean[c] = ca(mean[c], A[c]);
    const int dof = cond_fwd[n[a]];
    const double2 vv = x[(na + dof) * stride];
    const Cplx V = {vv.x, vv.y};
#pragma unroll
    for (int c = 0; c < 3; ++c) gv[c] = ca(gv[c], rc(g[c], V));
  }
  const Cplx iw = {0.0, omega};
#pragma unroll
  for (int c = 0; c < 3; ++c) e[c] = ca(cm(iw, rc(0.25, mean[c])), gv[c]);
}

__global__ void k_dz_contrib(const int4* __restrict__ tets, const uint8_t* __restrict__ region,
                             const double* __restrict__ xyz, const int* __restrict__ defect,
                             int64_t n_defect, const int* __restrict__ cond_fwd, int64_t na,
                             const double2* x0, const double2* x1, const double2* x2,
                             const double2* x3, int stride, DzParams P, double* contrib) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_defect;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int t = defect[q];
    const int4 k = tets[t];
    const int n[4] = {k.x, k.y, k.z, k.w};
    double p[4][3];
    load_tet(xyz, k, p);
    TetGeom f;
    tet_frame(p, f);
    const double vol = signed_volume(p);
    const int tag = region[t];
    const double mu_d = P.mu_d[tag], mu_eps = P.mu_eps[tag];
    const double sig_d = P.sigma_d[tag], sig_eps = P.sigma_eps[tag];
    const Cplx inv_iw = {0.0, -1.0 / P.omega};
    const Cplx cmu = rc(((mu_eps - mu_d) / (mu_d * mu_eps)) * vol, inv_iw);
    const double csig = (sig_d - sig_eps) * vol;
    Cplx curl[4][3], e[4][3];
    const double2* xs[4] = {x0, x1, x2, x3};
#pragma unroll
    for (int s = 0; s < 4; ++s) curl_and_field(xs[s], stride, n, f, cond_fwd, na, P.omega, curl[s], e[s]);
    // pairings (k, l) = (1,1), (1,2), (2,1), (2,2): sol_k in {0,1}, ref_l in {2,3}
#pragma unroll
    for (int kk = 0; kk < 2; ++kk)
#pragma unroll
      for (int ll = 0; ll < 2; ++ll) {
        const Cplx* ck = curl[kk];
        const Cplx* cl = curl[2 + ll];
        const Cplx* ek = e[kk];
        const Cplx* el = e[2 + ll];
        const Cplx cp = ca(ca(cm(ck[0], cl[0]), cm(ck[1], cl[1])), cm(ck[2], cl[2]));
        const Cplx fp = ca(ca(cm(ek[0], el[0]), cm(ek[1], el[1])), cm(ek[2], el[2]));
        const Cplx tot = ca(cm(cmu, cp), rc(csig, fp));
        const int slot = 2 * kk + ll;
        contrib[q * 8 + 2 * slot] = tot.re;
        contrib[q * 8 + 2 * slot + 1] = tot.im;
      }
  }
}

__global__ void k_dz_reduce(const double* __restrict__ contrib, int64_t n, double* out) {
  // one block, fixed order: thread j sums rows j, j+B, ...; then a tree.
  __shared__ double sm[256][8];
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t q = threadIdx.x; q < n; q += blockDim.x)
#pragma unroll
    for (int s = 0; s < 8; ++s) acc[s] += contrib[q * 8 + s];
#pragma unroll
  for (int s = 0; s < 8; ++s) sm[threadIdx.x][s] = acc[s];
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w)
#pragma unroll
      for (int s = 0; s < 8; ++s) sm[threadIdx.x][s] += sm[threadIdx.x + w][s];
    __syncthreads();
  }
  if (threadIdx.x == 0)
#pragma unroll
    for (int s = 0; s < 8; ++s) out[s] = sm[0][s];
}

}  // namespace

void build_rhs(ect_mesh* m, const ect_coil& coil, const double* z, const int* which, int n_rhs,
               double amplitude, double2* rhs) {
  ect_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  const int64_t nn = m->n_nodes, N = 3 * nn + m->n_cond;
  CK(cudaMemsetAsync(rhs, 0, (size_t)N * n_rhs * sizeof(double2), s));
  m->rhs_flag.ensure(nn);
  m->rhs_j.ensure(3 * nn);
  m->rhs_stat.ensure(4);
  struct { uint8_t* p; size_t n; size_t bytes() const { return n; } } flag{m->rhs_flag.p, (size_t)nn};
  struct { double* p; } j{m->rhs_j.p};
  struct { int* p; } stat{m->rhs_stat.p};
  for (int col = 0; col < n_rhs; ++col) {
    if (which[col] != 1 && which[col] != 2) fail(ECT_ERR_MESH, "coil_support: coil index must be 1 or 2");
    const double lo = which[col] == 1 ? z[col] - 0.5 * coil.gap - coil.height : z[col] + 0.5 * coil.gap;
    const double hi = lo + coil.height;
    CK(cudaMemsetAsync(flag.p, 0, flag.bytes(), s));
    int init[2] = {0, 0x7fffffff};
    CK(cudaMemcpyAsync(stat.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
    k_support<<<blocks_for(ctx, m->n_tets), 256, 0, s>>>(m->tets.p, m->region.p, m->xyz.p,
                                                        m->n_tets, coil.r_inner, coil.r_outer, lo,
                                                        hi, flag.p, stat.p, stat.p + 1);
    CK_LAUNCH();
    int h[2];
    CK(cudaMemcpyAsync(h, stat.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (h[0] == 0) fail(ECT_ERR_MESH, "coil support is empty");
    if (h[1] != 0x7fffffff) {
      fail(ECT_ERR_MESH, "coil support intersects a conductor region (tet " + std::to_string(h[1]) +
                             "); the source must be divergence-free in the insulator");
    }
    k_nodal_current<<<blocks_for(ctx, nn), 256, 0, s>>>(m->xyz.p, flag.p, nn, amplitude, j.p);
    CK_LAUNCH();
    k_rhs_gather<<<blocks_for(ctx, nn), 256, 0, s>>>(m->tets.p, m->xyz.p, m->inc_off.p, m->inc.p,
                                                    flag.p, j.p, m->pinned.p, nn, n_rhs, col, rhs);
    CK_LAUNCH();
    note_launch(ctx, 3);
  }
  CK(cudaStreamSynchronize(s));
}

void build_rhs_support(ect_mesh* m, const int* support, int64_t n_support, int region_tag,
                       double amplitude, double2* rhs) {
  ect_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  const int64_t nn = m->n_nodes, N = 3 * nn + m->n_cond;
  CK(cudaMemsetAsync(rhs, 0, (size_t)N * sizeof(double2), s));
  m->rhs_flag.ensure(nn);
  m->rhs_j.ensure(3 * nn);
  m->rhs_stat.ensure(4);
  struct { uint8_t* p; size_t n; size_t bytes() const { return n; } } flag{m->rhs_flag.p, (size_t)nn};
  struct { double* p; } j{m->rhs_j.p};
  struct { int* p; } stat{m->rhs_stat.p};
  CK(cudaMemsetAsync(flag.p, 0, flag.bytes(), s));
  int init[3] = {0, 0x7fffffff, 0x7fffffff};
  CK(cudaMemcpyAsync(stat.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
  const int64_t n = support ? n_support : m->n_tets;
  if (n > 0) {
    k_support_list<<<blocks_for(ctx, n), 256, 0, s>>>(m->tets.p, m->region.p, support, n_support,
                                                      region_tag, m->n_tets, flag.p, stat.p,
                                                      stat.p + 1, stat.p + 2);
    CK_LAUNCH();
  }
  int h[3];
  CK(cudaMemcpyAsync(h, stat.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (h[2] != 0x7fffffff) fail(ECT_ERR_MESH, "coil support: tet index out of range");
  if (h[0] == 0) fail(ECT_ERR_MESH, "coil support is empty");
  if (h[1] != 0x7fffffff) {
    fail(ECT_ERR_MESH, "coil support intersects a conductor region (tet " + std::to_string(h[1]) +
                           "); the source must be divergence-free in the insulator");
  }
  k_nodal_current<<<blocks_for(ctx, nn), 256, 0, s>>>(m->xyz.p, flag.p, nn, amplitude, j.p);
  CK_LAUNCH();
  // assemble_rhs itself does not pin (position_rhs applies the pins afterwards)
  k_rhs_gather<<<blocks_for(ctx, nn), 256, 0, s>>>(m->tets.p, m->xyz.p, m->inc_off.p, m->inc.p,
                                                  flag.p, j.p, nullptr, nn, 1, 0, rhs);
  CK_LAUNCH();
  note_launch(ctx, 3);
  CK(cudaStreamSynchronize(s));
}

void apply_pins_rhs(ect_mesh* m, double2* rhs, int n_rhs) {
  ect_ctx* ctx = m->ctx;
  const int64_t na = 3 * m->n_nodes;
  k_pin_rhs<<<blocks_for(ctx, na * n_rhs), 256, 0, ctx->stream>>>(m->pinned.p, na, n_rhs, rhs);
  CK_LAUNCH();
  note_launch(ctx, 1);
  CK(cudaStreamSynchronize(ctx->stream));
}

void delta_impedance(ect_mesh* m, const ect_materials& pm, const ect_materials& rm,
                     const double2* xk1, const double2* xk2, const double2* xl1,
                     const double2* xl2, int stride, double2 out[4]) {
  ect_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  for (int q = 0; q < 4; ++q) out[q] = make_double2(0.0, 0.0);
  if (m->n_defect == 0) return;
  DzParams P{};
  P.omega = pm.omega;
  for (int r = 0; r < ECT_REGION_COUNT; ++r) {
    P.mu_d[r] = pm.mu[r];
    P.mu_eps[r] = rm.mu[r];
    P.sigma_d[r] = pm.sigma[r];
    P.sigma_eps[r] = rm.sigma[r];
  }
  m->dz_contrib.ensure(8 * (size_t)std::max<int64_t>(1, m->n_defect));
  m->dz_res.ensure(8);
  struct { double* p; } contrib{m->dz_contrib.p}, res{m->dz_res.p};
  k_dz_contrib<<<blocks_for(ctx, m->n_defect, 128), 128, 0, s>>>(
      m->tets.p, m->region.p, m->xyz.p, m->defect_tets.p, m->n_defect, m->cond_fwd.p,
      3 * m->n_nodes, xk1, xk2, xl1, xl2, stride, P, contrib.p);
  CK_LAUNCH();
  k_dz_reduce<<<1, 256, 0, s>>>(contrib.p, m->n_defect, res.p);
  CK_LAUNCH();
  note_launch(ctx, 2);
  double h[8];
  CK(cudaMemcpyAsync(h, res.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int q = 0; q < 4; ++q) out[q] = make_double2(h[2 * q], h[2 * q + 1]);
}

}  // namespace ect
