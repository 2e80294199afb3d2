// ectgpu C ABI (include/ectgpu.h) and the host-side mirror of the reference
// API around it: mesh preparation, MaterialTable construction, ScanSession.
//
// Host arithmetic that defines matrix values (mu_tilde, material
// coefficients) follows the reference sequentially and is compiled with
// -ffp-contract=off, exactly like the reference on x86-64.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numbers>
#include <string>
#include <vector>

#include "ect_internal.h"
#include "mesh_io.h"

namespace {

thread_local std::string g_last_error;
constexpr double kMu0 = 1.25663706212e-6;  // types.hpp:18

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return ECT_OK;
  } catch (const ect::Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return ECT_ERR_OTHER;
  }
}

void require(bool ok, int code, const char* what) {
  if (!ok) ect::fail(code, what);
}

// Host <-> device copies of caller buffers. Page-locked host memory (the
// caller's cudaHostAlloc / cudaHostRegister / torch pin_memory) is copied
// directly and asynchronously; pageable memory goes through the context's
// two pinned staging halves (kStageHalf bytes each, allocated once), the
// memcpy into one half overlapping the DMA out of the other.
constexpr size_t kStageHalf = 16u << 20;

bool is_pinned_host(const void* p) {
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeHost;
}

char* stage_buffer(ect_ctx* ctx) {
  if (!ctx->pinned) {
    CK(cudaHostAlloc(&ctx->pinned, 2 * kStageHalf, cudaHostAllocDefault));
    ctx->pinned_bytes = 2 * kStageHalf;
    CK(cudaEventCreateWithFlags(&ctx->stage_ev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->stage_ev[1], cudaEventDisableTiming));
  }
  return static_cast<char*>(ctx->pinned);
}

void copy_h2d(ect_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  if (is_pinned_host(src)) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    return;
  }
  char* st = stage_buffer(ctx);
  bool used[2] = {false, false};
  for (size_t off = 0, q = 0; off < bytes; off += kStageHalf, ++q) {
    const int h = (int)(q & 1);
    const size_t len = std::min(kStageHalf, bytes - off);
    if (used[h]) CK(cudaEventSynchronize(ctx->stage_ev[h]));  // DMA out of this half done
    std::memcpy(st + h * kStageHalf, static_cast<const char*>(src) + off, len);
    CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, st + h * kStageHalf, len,
                       cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaEventRecord(ctx->stage_ev[h], ctx->stream));
    used[h] = true;
  }
  // the staging halves are reused by the next call: wait for the last DMAs
  for (int h = 0; h < 2; ++h)
    if (used[h]) CK(cudaEventSynchronize(ctx->stage_ev[h]));
}

void copy_d2h(ect_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  if (is_pinned_host(dst)) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return;
  }
  char* st = stage_buffer(ctx);
  const size_t n_chunks = (bytes + kStageHalf - 1) / kStageHalf;
  auto issue = [&](size_t q) {
    const size_t off = q * kStageHalf, len = std::min(kStageHalf, bytes - off);
    const int h = (int)(q & 1);
    CK(cudaMemcpyAsync(st + h * kStageHalf, static_cast<const char*>(src) + off, len,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaEventRecord(ctx->stage_ev[h], ctx->stream));
  };
  issue(0);
  for (size_t q = 0; q < n_chunks; ++q) {
    const int h = (int)(q & 1);
    CK(cudaEventSynchronize(ctx->stage_ev[h]));
    if (q + 1 < n_chunks) issue(q + 1);  // next DMA into the other half overlaps this memcpy
    const size_t off = q * kStageHalf, len = std::min(kStageHalf, bytes - off);
    std::memcpy(static_cast<char*>(dst) + off, st + h * kStageHalf, len);
  }
}

// Input buffer that may live on the host or on the context's device.
template <typename T>
struct In {
  const T* dev = nullptr;
  ect::DevBuf<T> tmp;
  In(ect_ctx* ctx, const T* p, size_t count) {
    if (count == 0 || ect::is_device_ptr(p)) {
      dev = p;
      return;
    }
    tmp.alloc(count);
    copy_h2d(ctx, tmp.p, p, count * sizeof(T));
    dev = tmp.p;
  }
};

// Output buffer that may live on the host or on the device.
template <typename T>
struct Out {
  T* dev = nullptr;
  T* host = nullptr;
  size_t count = 0;
  ect::DevBuf<T> tmp;
  ect_ctx* ctx;
  Out(ect_ctx* c, T* p, size_t n) : count(n), ctx(c) {
    if (n == 0 || ect::is_device_ptr(p)) {
      dev = p;
      return;
    }
    host = p;
    tmp.alloc(n);
    dev = tmp.p;
  }
  void finish() {
    if (host) copy_d2h(ctx, host, dev, count * sizeof(T));
    CK(cudaStreamSynchronize(ctx->stream));
  }
};

// In-place buffer (read and written).
template <typename T>
struct InOut : Out<T> {
  InOut(ect_ctx* c, T* p, size_t n) : Out<T>(c, p, n) {
    if (this->host) copy_h2d(c, this->dev, p, n * sizeof(T));
  }
};

struct ScopedDevice {
  int prev = 0;
  explicit ScopedDevice(int d) {
    cudaGetDevice(&prev);
    if (prev != d) CK(cudaSetDevice(d));
  }
  ~ScopedDevice() {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != prev) cudaSetDevice(prev);
  }
};

// Device-time accounting of one phase with its own event pair.
struct EventTimer {  // events come from a per-context pool (created once, reused)
  ect_ctx* ctx;
  double* slot;
  cudaEvent_t a = nullptr, b = nullptr;
  EventTimer(ect_ctx* c, double* s) : ctx(c), slot(s) {
    auto& pool = ctx->timer_events;
    const size_t at = 2 * (size_t)ctx->timer_depth++;
    while (pool.size() < at + 2) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      pool.push_back(e);
    }
    a = pool[at];
    b = pool[at + 1];
    CK(cudaEventRecord(a, ctx->stream));
  }
  ~EventTimer() {
    if (cudaEventRecord(b, ctx->stream) == cudaSuccess && cudaEventSynchronize(b) == cudaSuccess) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, a, b) == cudaSuccess) *slot += ms;
    }
    --ctx->timer_depth;
  }
};

// signed_tet_volume (mesh.cpp:36-38) with the shim's cross/dot order.
double signed_volume_host(const double* a, const double* b, const double* c, const double* d) {
  const double u0 = b[0] - a[0], u1 = b[1] - a[1], u2 = b[2] - a[2];
  const double v0 = c[0] - a[0], v1 = c[1] - a[1], v2 = c[2] - a[2];
  const double w0 = d[0] - a[0], w1 = d[1] - a[1], w2 = d[2] - a[2];
  const double cx = u1 * v2 - u2 * v1, cy = u2 * v0 - u0 * v2, cz = u0 * v1 - u1 * v0;
  return ((cx * w0 + cy * w1) + cz * w2) / 6.0;
}

bool same_coefficients(const ect_materials& a, const ect_materials& b) {
  // MaterialTable::same_coefficients (materials.cpp:24-30)
  if (a.omega != b.omega || a.mu_tilde != b.mu_tilde || a.delta_gauge != b.delta_gauge ||
      a.bc_penalty != b.bc_penalty || a.sigma_eps != b.sigma_eps ||
      a.ibc_enabled != b.ibc_enabled || a.l22_use_sigma_eps != b.l22_use_sigma_eps ||
      a.z_surface[0] != b.z_surface[0] || a.z_surface[1] != b.z_surface[1])
    return false;
  for (int r = 0; r < ECT_REGION_COUNT; ++r)
    if (a.sigma[r] != b.sigma[r] || a.mu[r] != b.mu[r]) return false;
  return true;
}

void check_materials(const ect_materials& m) {
  if (m.ibc_enabled && m.z_surface[0] == 0.0 && m.z_surface[1] == 0.0) {
    // element_ibc (element_forms.cpp:117-119)
    ect::fail(ECT_ERR_SOLVER, "impedance surface term with zero surface impedance");
  }
  require(m.omega > 0.0, ECT_ERR_CONFIG, "materials: omega must be positive");
  require(m.mu_tilde > 0.0, ECT_ERR_CONFIG, "materials: mu_tilde must be positive");
}

}  // namespace

namespace ect {

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes attr{};
  cudaError_t e = cudaPointerGetAttributes(&attr, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

void* cub_scratch(ect_ctx* ctx, size_t bytes) {
  ctx->cub_tmp.ensure(std::max<size_t>(bytes, 1));
  return ctx->cub_tmp.p;
}

int grid_for(ect_ctx* ctx, const void* kernel, int block, size_t smem) {
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem));
  return std::max(1, per_sm) * ctx->num_sms;
}

void note_launch(ect_ctx* ctx, int n) { ctx->timings.kernel_launches += n; }

}  // namespace ect

// ============================================================================
extern "C" {

const char* ect_last_error(void) { return g_last_error.c_str(); }

int ect_ctx_create(int device, ect_ctx** out) {
  return guarded([&] {
    require(out != nullptr, ECT_ERR_OTHER, "ect_ctx_create: null output");
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    require(device >= 0 && device < count, ECT_ERR_CUDA, "ect_ctx_create: no such CUDA device");
    auto ctx = std::make_unique<ect_ctx>();
    ctx->device = device;
    ScopedDevice sd(device);
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) {
      ect::fail(ECT_ERR_CUDA, std::string("ectgpu is built for sm_100a (B200); device is ") +
                                  prop.name);
    }
    ctx->num_sms = prop.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&ctx->ev_a));
    CK(cudaEventCreate(&ctx->ev_b));
    for (auto& e : ctx->marks) CK(cudaEventCreate(&e));
    CK(cudaHostAlloc(reinterpret_cast<void**>(&ctx->pinned_flag), 64, cudaHostAllocDefault));
    *out = ctx.release();
  });
}

int ect_ctx_destroy(ect_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    ScopedDevice sd(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto e : ctx->prof.pool) cudaEventDestroy(e);
    for (auto e : ctx->timer_events) cudaEventDestroy(e);
    if (ctx->pinned_flag) cudaFreeHost(ctx->pinned_flag);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    for (auto e : ctx->stage_ev)
      if (e) cudaEventDestroy(e);
    cudaEventDestroy(ctx->ev_a);
    cudaEventDestroy(ctx->ev_b);
    for (auto e : ctx->marks) cudaEventDestroy(e);
    if (ctx->ev_h1) cudaEventDestroy(ctx->ev_h1);
    if (ctx->ev_h2) cudaEventDestroy(ctx->ev_h2);
    if (ctx->halo_stream) cudaStreamDestroy(ctx->halo_stream);
    ctx->cub_tmp.release();
    cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

int ect_ctx_timings(ect_ctx* ctx, ect_timings* out, int reset) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    if (out) *out = ctx->timings;
    if (reset) ctx->timings = ect_timings{};
  });
}

int ect_ctx_set_profiling(ect_ctx* ctx, int enabled) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ctx->prof.enabled = enabled != 0;
  });
}

int ect_ctx_set_format(ect_ctx* ctx, int format) {
  return guarded([&] {
    require(format == ECT_FORMAT_NB || format == ECT_FORMAT_CSR || format == ECT_FORMAT_SELL,
            ECT_ERR_CONFIG, "ect_ctx_set_format: unknown format");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ctx->force_csr = format == ECT_FORMAT_CSR || format == ECT_FORMAT_SELL;
    ctx->use_sell = format == ECT_FORMAT_SELL;
  });
}

int ect_matrix_format(ect_matrix* m, int32_t* nb) {
  return guarded([&] { *nb = m->has_nb ? 1 : (m->has_sell ? 3 : 0); });
}

int ect_matrix_nb_counts(ect_matrix* m, int64_t* blocks, int64_t* couplings) {
  return guarded([&] {
    *blocks = m->has_nb ? m->nb_blocks : 0;
    *couplings = m->has_nb ? m->nb_ncpl : 0;
  });
}

int ect_ctx_mark(ect_ctx* ctx, int slot) {
  return guarded([&] {
    require(slot >= 0 && slot < 8, ECT_ERR_OTHER, "ect_ctx_mark: slot must be in 0..7");
    ScopedDevice sd(ctx->device);
    CK(cudaEventRecord(ctx->marks[slot], ctx->stream));
  });
}

int ect_ctx_elapsed_ms(ect_ctx* ctx, int a, int b, double* ms) {
  return guarded([&] {
    require(a >= 0 && a < 8 && b >= 0 && b < 8, ECT_ERR_OTHER, "ect_ctx_elapsed_ms: bad slot");
    ScopedDevice sd(ctx->device);
    CK(cudaEventSynchronize(ctx->marks[b]));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, ctx->marks[a], ctx->marks[b]));
    *ms = f;
  });
}

int ect_ctx_synchronize(ect_ctx* ctx) {
  return guarded([&] {
    ScopedDevice sd(ctx->device);
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

// ---- mesh ------------------------------------------------------------------
int ect_mesh_create(ect_ctx* ctx, const double* xyz, int64_t n_nodes, const int32_t* tets,
                    const uint8_t* region, int64_t n_tets, ect_mesh** out) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    require(n_nodes > 0 && n_tets > 0, ECT_ERR_MESH, "mesh: empty node or tet set");
    auto m = std::make_unique<ect_mesh>();
    m->ctx = ctx;
    m->n_nodes = n_nodes;
    m->n_tets = n_tets;
    // Host copies; they also define mu_tilde and the z extremes exactly as
    // the reference computes them. Pointers may be device memory.
    m->h_xyz.resize(3 * n_nodes);
    m->h_tets.resize(4 * n_tets);
    m->h_region.resize(n_tets);
    CK(cudaMemcpy(m->h_xyz.data(), xyz, 3 * n_nodes * sizeof(double), cudaMemcpyDefault));
    CK(cudaMemcpy(m->h_tets.data(), tets, 4 * n_tets * sizeof(int32_t), cudaMemcpyDefault));
    CK(cudaMemcpy(m->h_region.data(), region, n_tets, cudaMemcpyDefault));
    for (int64_t t = 0; t < n_tets; ++t) {
      int32_t* k = &m->h_tets[4 * t];
      for (int a = 0; a < 4; ++a) {
        if (k[a] < 0 || k[a] >= n_nodes) {
          ect::fail(ECT_ERR_MESH, "tet " + std::to_string(t) + " references invalid node " +
                                      std::to_string(k[a]));
        }
      }
      if (m->h_region[t] >= ECT_REGION_COUNT) {
        ect::fail(ECT_ERR_MESH, "tet " + std::to_string(t) + " carries unknown region tag");
      }
      // Mesh::canonicalize_orientation (mesh.cpp:50-61)
      double vol = signed_volume_host(&m->h_xyz[3 * k[0]], &m->h_xyz[3 * k[1]],
                                      &m->h_xyz[3 * k[2]], &m->h_xyz[3 * k[3]]);
      if (vol < 0.0) {
        std::swap(k[2], k[3]);
        vol = -vol;
      }
      if (!(vol > 0.0)) {
        ect::fail(ECT_ERR_MESH, "degenerate tet " + std::to_string(t) + " (zero volume)");
      }
    }
    // classify_boundary's z extremes (mesh.cpp:146-153)
    m->z_lo = m->z_hi = m->h_xyz[2];
    for (int64_t i = 0; i < n_nodes; ++i) {
      m->z_lo = std::min(m->z_lo, m->h_xyz[3 * i + 2]);
      m->z_hi = std::max(m->z_hi, m->h_xyz[3 * i + 2]);
    }
    m->xyz.alloc(3 * n_nodes);
    m->tets.alloc(n_tets);
    m->region.alloc(n_tets);
    CK(cudaMemcpyAsync(m->xyz.p, m->h_xyz.data(), m->xyz.bytes(), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(m->tets.p, m->h_tets.data(), m->tets.bytes(), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(m->region.p, m->h_region.data(), m->region.bytes(), cudaMemcpyHostToDevice,
                       ctx->stream));
    ect::build_mesh_topology(m.get());
    *out = m.release();
  });
}

int ect_mesh_destroy(ect_mesh* mesh) {
  return guarded([&] {
    if (!mesh) return;
    ScopedDevice sd(mesh->ctx->device);
    delete mesh;
  });
}

int ect_mesh_counts(ect_mesh* m, int64_t counts[6]) {
  return guarded([&] {
    counts[0] = m->n_nodes;
    counts[1] = m->n_tets;
    counts[2] = m->n_cond;
    counts[3] = 3 * m->n_nodes + m->n_cond;
    counts[4] = m->n_pins;
    counts[5] = m->n_defect;
  });
}

int ect_mesh_export(ect_mesh* m, int32_t* cond_forward, int32_t* pinned_dofs, int32_t* tets) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(m->ctx->mu);
    ScopedDevice sd(m->ctx->device);
    cudaStream_t s = m->ctx->stream;
    if (cond_forward) {
      Out<int32_t> o(m->ctx, cond_forward, m->n_nodes);
      CK(cudaMemcpyAsync(o.dev, m->cond_fwd.p, m->n_nodes * sizeof(int), cudaMemcpyDeviceToDevice, s));
      o.finish();
    }
    if (pinned_dofs) {
      std::vector<uint8_t> f(3 * m->n_nodes);
      CK(cudaMemcpyAsync(f.data(), m->pinned.p, f.size(), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      std::vector<int32_t> list;
      list.reserve(m->n_pins);
      for (size_t i = 0; i < f.size(); ++i)
        if (f[i]) list.push_back((int32_t)i);
      CK(cudaMemcpy(pinned_dofs, list.data(), list.size() * sizeof(int32_t), cudaMemcpyDefault));
    }
    if (tets) CK(cudaMemcpy(tets, m->h_tets.data(), m->h_tets.size() * sizeof(int32_t), cudaMemcpyDefault));
  });
}

// ---- materials ------------------------------------------------------------
int ect_harmonic_mu_tilde(ect_mesh* m, const ect_materials* mats, double* out) {
  return guarded([&] {
    // harmonic_mu_tilde (materials.cpp:32-42): sequential fold in tet order
    double vol = 0.0, weighted = 0.0;
    for (int64_t t = 0; t < m->n_tets; ++t) {
      const int32_t* k = &m->h_tets[4 * t];
      const double v = signed_volume_host(&m->h_xyz[3 * k[0]], &m->h_xyz[3 * k[1]],
                                          &m->h_xyz[3 * k[2]], &m->h_xyz[3 * k[3]]);
      vol += v;
      weighted += v / mats->mu[m->h_region[t]];
    }
    require(weighted > 0.0, ECT_ERR_CONFIG, "harmonic_mu_tilde: mesh has no volume");
    *out = vol / weighted;
  });
}

void ect_physics_init(ect_physics* ph) {
  // RunConfig's [materials] defaults (config.hpp:25-39)
  if (!ph) return;
  *ph = ect_physics{};
  ph->frequency = 100e3;
  ph->sigma_tube = 1e6;
  ph->mu_r_tube = 1.0;
  ph->sigma_defect = std::nan("");  // std::optional: unset
  ph->mu_r_defect = std::nan("");
  ph->sigma_eps_ratio = 1e-6;
  ph->delta_gauge = 1e-6;
  ph->bc_penalty = 1e13;
  ph->mu_tilde_harmonic = 1;
  ph->mu_tilde_fixed = kMu0;
  ph->sigma_tsp = 5e6;
  ph->mu_r_tsp = 50.0;
  ph->ibc_tsp = 0;
  ph->l22_sigma_eps = 0;
}

int ect_materials_from_physics(ect_mesh* mesh, const ect_physics* ph, ect_materials* primary,
                               ect_materials* reference, int32_t* two_configs) {
  return guarded([&] {
    require(ph != nullptr, ECT_ERR_CONFIG, "physics: null");
    // RunConfig validation (config.cpp:218-236)
    auto need = [](bool ok, const char* key, const char* what) {
      if (!ok) ect::fail(ECT_ERR_CONFIG, std::string(key) + ": " + what);
    };
    need(ph->frequency > 0.0, "materials.frequency", "must be positive");
    need(ph->sigma_tube > 0.0, "materials.sigma_tube", "must be positive");
    need(ph->mu_r_tube > 0.0, "materials.mu_r_tube", "must be positive");
    need(ph->sigma_tsp > 0.0, "materials.sigma_tsp", "must be positive");
    need(ph->mu_r_tsp > 0.0, "materials.mu_r_tsp", "must be positive");
    const bool has_sd = !std::isnan(ph->sigma_defect), has_md = !std::isnan(ph->mu_r_defect);
    if (has_sd) need(ph->sigma_defect > 0.0, "materials.sigma_defect", "must be positive");
    if (has_md) need(ph->mu_r_defect > 0.0, "materials.mu_r_defect", "must be positive");
    need(ph->sigma_eps_ratio > 0.0, "materials.sigma_eps_ratio", "must be positive");
    need(ph->delta_gauge > 0.0 && ph->delta_gauge < 1.0, "materials.delta_gauge",
         "must lie in (0, 1)");
    need(ph->bc_penalty > 0.0, "materials.bc_penalty", "must be positive");
    if (!ph->mu_tilde_harmonic) need(ph->mu_tilde_fixed > 0.0, "materials.mu_tilde", "must be positive");
    // RunConfig::material_table (config.cpp:325-347)
    ect_materials m{};
    m.omega = 2.0 * std::numbers::pi * ph->frequency;
    m.sigma_eps = ph->sigma_eps_ratio * ph->sigma_tube;
    m.delta_gauge = ph->delta_gauge;
    m.bc_penalty = ph->bc_penalty;
    m.l22_use_sigma_eps = ph->l22_sigma_eps ? 1 : 0;
    m.ibc_enabled = 0;
    auto set = [&m](int r, double s, double mu) {
      m.sigma[r] = s;
      m.mu[r] = mu;
    };
    set(ECT_REGION_TUBE, ph->sigma_tube, kMu0 * ph->mu_r_tube);
    set(ECT_REGION_TSP, ph->sigma_tsp, kMu0 * ph->mu_r_tsp);
    set(ECT_REGION_DEFECT, has_sd ? ph->sigma_defect : ph->sigma_tube,
        kMu0 * (has_md ? ph->mu_r_defect : ph->mu_r_tube));
    set(ECT_REGION_COIL1, 0.0, kMu0);
    set(ECT_REGION_COIL2, 0.0, kMu0);
    set(ECT_REGION_VACUUM, 0.0, kMu0);
    if (ph->ibc_tsp) {
      // config.cpp:339-345: the plate volume is assembled as vacuum and
      // represented by the surface impedance of its material (materials.cpp:12-22)
      const double s_tsp = ph->sigma_tsp;
      const double mu_tsp = kMu0 * ph->mu_r_tsp;
      const double delta = std::sqrt(2.0 / (m.omega * mu_tsp * s_tsp));
      const std::complex<double> z = std::complex<double>(1.0, -1.0) / (delta * s_tsp);
      m.ibc_enabled = 1;
      m.z_surface[0] = z.real();
      m.z_surface[1] = z.imag();
      set(ECT_REGION_TSP, m.sigma_eps, kMu0);
    }
    // resolve_mu_tilde (config.cpp:349-352)
    if (ph->mu_tilde_harmonic) {
      int rc = ect_harmonic_mu_tilde(mesh, &m, &m.mu_tilde);
      if (rc) ect::fail(rc, g_last_error);
    } else {
      m.mu_tilde = ph->mu_tilde_fixed;
    }
    // reference_variant (materials.cpp:44-53)
    ect_materials r = m;
    r.sigma[ECT_REGION_DEFECT] = m.sigma_eps;
    r.mu[ECT_REGION_DEFECT] = kMu0;
    r.sigma[ECT_REGION_VACUUM] = m.sigma_eps;
    r.sigma[ECT_REGION_COIL1] = m.sigma_eps;
    r.sigma[ECT_REGION_COIL2] = m.sigma_eps;
    if (primary) *primary = m;
    if (reference) *reference = r;
    // scan.cpp:46-49
    if (two_configs) *two_configs = mesh->n_defect > 0 && !same_coefficients(m, r);
  });
}

// ---- matrix -----------------------------------------------------------------
int ect_matrix_create(ect_ctx* ctx, ect_mesh* mesh, ect_matrix** out) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    auto a = std::make_unique<ect_matrix>();
    a->ctx = ctx;
    EventTimer t(ctx, &ctx->timings.pattern_ms);
    ect::build_pattern(mesh, a.get());
    *out = a.release();
  });
}

static int matrix_from_external(ect_ctx* ctx, int64_t n, int64_t nnz, const int32_t* ptr,
                                const int32_t* idx, const double* values, bool csc,
                                ect_matrix** out) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    require(n > 0 && nnz > 0 && nnz < (1ll << 31) && n < (1ll << 31), ECT_ERR_SOLVER,
            csc ? "from_csc: bad dimensions" : "from_csr: bad dimensions");
    require(ptr && idx && values, ECT_ERR_SOLVER, "matrix: null array");
    auto a = std::make_unique<ect_matrix>();
    a->ctx = ctx;
    In<int> pi(ctx, ptr, n + 1);
    In<int> ii(ctx, idx, nnz);
    In<double2> vi(ctx, reinterpret_cast<const double2*>(values), nnz);
    ect::matrix_from_compressed(ctx, n, nnz, pi.dev, ii.dev, vi.dev, csc, a.get());
    ect::compute_jacobi(a.get());
    if (ctx->use_sell) ect::build_sell(a.get(), ctx->sell_sigma);
    *out = a.release();
  });
}

int ect_matrix_from_csr(ect_ctx* ctx, int64_t n, int64_t nnz, const int32_t* row_ptr,
                        const int32_t* col_idx, const double* values, ect_matrix** out) {
  return matrix_from_external(ctx, n, nnz, row_ptr, col_idx, values, false, out);
}

int ect_matrix_from_csc(ect_ctx* ctx, int64_t n, int64_t nnz, const int32_t* col_ptr,
                        const int32_t* row_idx, const double* values, ect_matrix** out) {
  return matrix_from_external(ctx, n, nnz, col_ptr, row_idx, values, true, out);
}

int ect_ctx_set_preconditioner(ect_ctx* ctx, int32_t precond) {
  return guarded([&] {
    require(precond == ECT_PRECOND_JACOBI || precond == ECT_PRECOND_AMG, ECT_ERR_CONFIG,
            "unknown preconditioner");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ctx->precond = precond;
  });
}

int ect_matrix_set_preconditioner(ect_matrix* m, int32_t precond) {
  return guarded([&] {
    require(precond == ECT_PRECOND_JACOBI || precond == ECT_PRECOND_AMG, ECT_ERR_CONFIG,
            "unknown preconditioner");
    std::lock_guard<std::recursive_mutex> lk(m->ctx->mu);
    m->precond = precond;
  });
}

int ect_matrix_precond_info(ect_matrix* m, double info[4]) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(m->ctx->mu);
    ScopedDevice sd(m->ctx->device);
    if (m->precond == ECT_PRECOND_AMG && m->symmetric && m->assembled && !m->amg)
      ect::amg_setup(m);
    if (m->precond != ECT_PRECOND_AMG || !m->amg) {
      info[0] = 0.0;
      info[1] = info[2] = info[3] = 0.0;
      return;
    }
    info[0] = (double)m->amg->lv.size();
    info[1] = m->amg->setup_ms;
    info[2] = m->amg->op_complexity;
    info[3] = (double)m->amg->lv.back().n;
  });
}

int ect_matrix_symmetric(ect_matrix* m, int32_t* symmetric) {
  return guarded([&] { *symmetric = m->symmetric ? 1 : 0; });
}

int ect_matrix_destroy(ect_matrix* a) {
  return guarded([&] {
    if (!a) return;
    ScopedDevice sd(a->ctx->device);
    delete a;
  });
}

int ect_matrix_counts(ect_matrix* a, int64_t* n, int64_t* nnz) {
  return guarded([&] {
    if (n) *n = a->n;
    if (nnz) *nnz = a->nnz;
  });
}

int ect_matrix_assemble(ect_ctx* ctx, ect_mesh* mesh, const ect_materials* mats, ect_matrix* a) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    check_materials(*mats);
    EventTimer t(ctx, &ctx->timings.assemble_ms);
    a->amg.reset();  // the multigrid hierarchy belongs to the old values
    ect::assemble_values(mesh, *mats, a);
  });
}

int ect_matrix_export(ect_matrix* a, int32_t* row_ptr, int32_t* col_idx, double* values) {
  return guarded([&] {
    ect_ctx* ctx = a->ctx;
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    if (row_ptr) CK(cudaMemcpyAsync(row_ptr, a->row_ptr.p, (a->n + 1) * sizeof(int), cudaMemcpyDefault, ctx->stream));
    if (col_idx) CK(cudaMemcpyAsync(col_idx, a->col.p, a->nnz * sizeof(int), cudaMemcpyDefault, ctx->stream));
    if (values) {
      require(a->assembled, ECT_ERR_SOLVER, "export: matrix values not assembled");
      CK(cudaMemcpyAsync(values, a->val.p, a->nnz * sizeof(double2), cudaMemcpyDefault, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

int ect_matrix_export_csc(ect_matrix* a, int32_t* col_ptr, int32_t* row_idx, double* values) {
  return guarded([&] {
    ect_ctx* ctx = a->ctx;
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    require(a->from_mesh, ECT_ERR_SOLVER,
            "export_csc: only matrices built from a mesh carry the symmetric pattern");
    if (col_ptr) CK(cudaMemcpyAsync(col_ptr, a->row_ptr.p, (a->n + 1) * sizeof(int), cudaMemcpyDefault, ctx->stream));
    if (row_idx) CK(cudaMemcpyAsync(row_idx, a->col.p, a->nnz * sizeof(int), cudaMemcpyDefault, ctx->stream));
    if (values) {
      require(a->assembled, ECT_ERR_SOLVER, "export: matrix values not assembled");
      Out<double2> o(ctx, reinterpret_cast<double2*>(values), a->nnz);
      ect::export_csc_values(a, o.dev);
      o.finish();
    }
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

// ---- rhs / spmv / solve ------------------------------------------------------
int ect_rhs_coil(ect_ctx* ctx, ect_mesh* mesh, const ect_coil* coil, const double* probe_z,
                 const int32_t* which_coil, int32_t n_rhs, double amplitude, double* rhs) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    require(n_rhs >= 1, ECT_ERR_CONFIG, "rhs: n_rhs must be >= 1");
    const size_t N = 3 * mesh->n_nodes + mesh->n_cond;
    std::vector<double> z(probe_z, probe_z + n_rhs);
    std::vector<int> w(which_coil, which_coil + n_rhs);
    Out<double2> o(ctx, reinterpret_cast<double2*>(rhs), N * n_rhs);
    EventTimer t(ctx, &ctx->timings.rhs_ms);
    ect::build_rhs(mesh, *coil, z.data(), w.data(), n_rhs, amplitude, o.dev);
    o.finish();
  });
}

int ect_rhs_support(ect_ctx* ctx, ect_mesh* mesh, const int32_t* support_tets,
                    int64_t n_support, double amplitude, double* rhs) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    require(n_support >= 0 && (n_support == 0 || support_tets), ECT_ERR_MESH,
            "rhs: bad support list");
    if (n_support == 0) ect::fail(ECT_ERR_MESH, "coil support is empty");
    const size_t N = 3 * mesh->n_nodes + mesh->n_cond;
    In<int> sup(ctx, support_tets, (size_t)n_support);
    Out<double2> o(ctx, reinterpret_cast<double2*>(rhs), N);
    EventTimer t(ctx, &ctx->timings.rhs_ms);
    ect::build_rhs_support(mesh, sup.dev, n_support, -1, amplitude, o.dev);
    o.finish();
  });
}

int ect_rhs_region(ect_ctx* ctx, ect_mesh* mesh, int32_t coil_tag, double amplitude, double* rhs) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    require(coil_tag >= 0 && coil_tag < ECT_REGION_COUNT, ECT_ERR_MESH, "rhs: unknown region tag");
    const size_t N = 3 * mesh->n_nodes + mesh->n_cond;
    Out<double2> o(ctx, reinterpret_cast<double2*>(rhs), N);
    EventTimer t(ctx, &ctx->timings.rhs_ms);
    ect::build_rhs_support(mesh, nullptr, 0, coil_tag, amplitude, o.dev);
    o.finish();
  });
}

int ect_apply_pins_to_rhs(ect_ctx* ctx, ect_mesh* mesh, double* rhs, int32_t n_rhs) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    require(n_rhs >= 1, ECT_ERR_CONFIG, "apply_pins_to_rhs: n_rhs must be >= 1");
    const size_t cnt = (size_t)(3 * mesh->n_nodes + mesh->n_cond) * n_rhs;
    InOut<double2> io(ctx, reinterpret_cast<double2*>(rhs), cnt);
    ect::apply_pins_rhs(mesh, io.dev, n_rhs);
    io.finish();
  });
}

int ect_spmv(ect_ctx* ctx, ect_matrix* a, const double* x, double* y, int32_t n_rhs) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    require(a->assembled, ECT_ERR_SOLVER, "spmv: matrix values not assembled");
    const size_t cnt = (size_t)a->n * n_rhs;
    In<double2> xi(ctx, reinterpret_cast<const double2*>(x), cnt);
    Out<double2> yo(ctx, reinterpret_cast<double2*>(y), cnt);
    ect::spmv(ctx, a, xi.dev, yo.dev, n_rhs);
    yo.finish();
  });
}

int ect_solve(ect_ctx* ctx, ect_matrix* a, const double* b, double* x, int32_t n_rhs,
              const ect_iter_options* opts, ect_iter_result* results) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    require(a->assembled, ECT_ERR_SOLVER, "solve: matrix values not assembled");
    ect_iter_options o = opts ? *opts : ect_iter_options{1e-8, 500, 80};
    const size_t cnt = (size_t)a->n * n_rhs;
    In<double2> bi(ctx, reinterpret_cast<const double2*>(b), cnt);
    Out<double2> xo(ctx, reinterpret_cast<double2*>(x), cnt);
    ect::SolveOut so;
    {
      EventTimer t(ctx, &ctx->timings.solve_ms);
      ect::cocg_solve(ctx, a, bi.dev, xo.dev, n_rhs, o, &so);
    }
    ect::throw_on_breakdown(so);
    xo.finish();
    for (int c = 0; c < n_rhs; ++c) {
      results[c].iterations = so.iters[c];
      results[c].residual = so.residual[c];
      results[c].converged = so.converged[c];
    }
  });
}

int ect_delta_impedance(ect_ctx* ctx, ect_mesh* mesh, const ect_materials* primary,
                        const ect_materials* reference, const double* x_k1, const double* x_k2,
                        const double* x_l1, const double* x_l2, double* dz) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    const size_t N = 3 * mesh->n_nodes + mesh->n_cond;
    In<double2> a(ctx, reinterpret_cast<const double2*>(x_k1), N);
    In<double2> b(ctx, reinterpret_cast<const double2*>(x_k2), N);
    In<double2> c(ctx, reinterpret_cast<const double2*>(x_l1), N);
    In<double2> d(ctx, reinterpret_cast<const double2*>(x_l2), N);
    double2 out[4];
    ect::delta_impedance(mesh, *primary, *reference, a.dev, b.dev, c.dev, d.dev, 1, out);
    for (int q = 0; q < 4; ++q) {
      dz[2 * q] = out[q].x;
      dz[2 * q + 1] = out[q].y;
    }
  });
}

}  // extern "C"

// ---- Gmsh files ------------------------------------------------------------------
struct ect_gmsh {
  ect::GmshMesh m;
};

extern "C" {

int ect_gmsh_read(const char* path, ect_gmsh** out) {
  return guarded([&] {
    require(path != nullptr, ECT_ERR_IO, "ect_gmsh_read: null path");
    auto g = std::make_unique<ect_gmsh>();
    g->m = ect::read_gmsh(path);
    *out = g.release();
  });
}

int ect_gmsh_counts(ect_gmsh* g, int64_t counts[3]) {
  return guarded([&] {
    counts[0] = (int64_t)g->m.xyz.size() / 3;
    counts[1] = (int64_t)g->m.region.size();
    counts[2] = (int64_t)g->m.labels.size();
  });
}

int ect_gmsh_arrays(ect_gmsh* g, double* xyz, int32_t* tets, uint8_t* region, int32_t* faces,
                    int32_t* labels) {
  return guarded([&] {
    const auto& m = g->m;
    if (xyz) std::copy(m.xyz.begin(), m.xyz.end(), xyz);
    if (tets) std::copy(m.tets.begin(), m.tets.end(), tets);
    if (region) std::copy(m.region.begin(), m.region.end(), region);
    if (faces) std::copy(m.faces.begin(), m.faces.end(), faces);
    if (labels) std::copy(m.labels.begin(), m.labels.end(), labels);
  });
}

int ect_gmsh_destroy(ect_gmsh* g) {
  return guarded([&] { delete g; });
}

int ect_gmsh_write(const char* path, const double* xyz, int64_t n_nodes, const int32_t* tets,
                   const uint8_t* region, int64_t n_tets, const int32_t* faces,
                   const int32_t* labels, int64_t n_faces) {
  return guarded([&] {
    require(path != nullptr, ECT_ERR_IO, "ect_gmsh_write: null path");
    ect::GmshMesh m;
    m.xyz.assign(xyz, xyz + 3 * n_nodes);
    m.tets.assign(tets, tets + 4 * n_tets);
    m.region.assign(region, region + n_tets);
    for (int64_t t = 0; t < n_tets; ++t)
      require(m.region[t] < ECT_REGION_COUNT, ECT_ERR_MESH, "ect_gmsh_write: unknown region tag");
    if (n_faces) {
      m.faces.assign(faces, faces + 3 * n_faces);
      m.labels.assign(labels, labels + n_faces);
      for (int64_t f = 0; f < n_faces; ++f)
        require(m.labels[f] >= 0 && m.labels[f] < 5, ECT_ERR_MESH,
                "ect_gmsh_write: unknown boundary label");
    }
    ect::write_gmsh(path, m);
  });
}

}  // extern "C"

// ---- ScanSession --------------------------------------------------------------
struct ect_session {
  ect_ctx* ctx = nullptr;
  ect_mesh* mesh = nullptr;
  ect_materials primary{}, reference{};
  bool two_configs = false;
  ect_coil coil{};
  double amplitude = 1.0;
  ect_iter_options opts{};
  ect_matrix* a_primary = nullptr;
  ect_matrix* a_reference = nullptr;
  // right-hand sides and solutions of one batch, kept across calls
  ect::DevBuf<double2> rhs, xp, xr, sol;
  ~ect_session() {
    delete a_primary;
    delete a_reference;
  }
};

extern "C" {

int ect_session_create(ect_ctx* ctx, ect_mesh* mesh, const ect_physics* physics,
                       const ect_coil* coil, double amplitude, const ect_iter_options* opts,
                       ect_session** out) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    auto s = std::make_unique<ect_session>();
    s->ctx = ctx;
    s->mesh = mesh;
    s->coil = *coil;
    s->amplitude = amplitude;
    s->opts = opts ? *opts : ect_iter_options{1e-8, 500, 80};
    int32_t two = 0;
    int rc = ect_materials_from_physics(mesh, physics, &s->primary, &s->reference, &two);
    if (rc) ect::fail(rc, g_last_error);
    s->two_configs = two != 0;
    // ScanSession ctor (scan.cpp:27-85): assemble once per configuration.
    rc = ect_matrix_create(ctx, mesh, &s->a_primary);
    if (rc) ect::fail(rc, g_last_error);
    rc = ect_matrix_assemble(ctx, mesh, &s->primary, s->a_primary);
    if (rc) ect::fail(rc, g_last_error);
    if (s->two_configs) {
      rc = ect_matrix_create(ctx, mesh, &s->a_reference);
      if (rc) ect::fail(rc, g_last_error);
      rc = ect_matrix_assemble(ctx, mesh, &s->reference, s->a_reference);
      if (rc) ect::fail(rc, g_last_error);
    }
    *out = s.release();
  });
}

int ect_session_destroy(ect_session* s) {
  return guarded([&] {
    if (!s) return;
    ScopedDevice sd(s->ctx->device);
    delete s;
  });
}

int ect_session_matrix(ect_session* s, int reference, ect_matrix** out) {
  return guarded([&] {
    *out = reference ? s->a_reference : s->a_primary;
    require(*out != nullptr, ECT_ERR_CONFIG, "session has no reference configuration");
  });
}

int ect_session_solve_positions(ect_session* s, const double* z, int32_t n_pos,
                                int32_t positions_per_batch, ect_signal_point* out,
                                double* solutions) {
  return guarded([&] {
    ect_ctx* ctx = s->ctx;
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    require(positions_per_batch >= 1 && positions_per_batch <= 8, ECT_ERR_CONFIG,
            "positions_per_batch must be in 1..8");
    const int64_t N = 3 * s->mesh->n_nodes + s->mesh->n_cond;
    const int P = positions_per_batch;
    const int kmax = 2 * P;
    s->rhs.ensure((size_t)N * kmax);
    s->xp.ensure((size_t)N * kmax);
    if (s->two_configs) s->xr.ensure((size_t)N * kmax);
    auto &rhs = s->rhs, &xp = s->xp, &xr = s->xr;
    for (int p0 = 0; p0 < n_pos; p0 += P) {
      const int np = std::min(P, n_pos - p0);
      const int k = 2 * np;
      // solve_position (scan.cpp:95-143): coil 1 and coil 2 right-hand sides
      std::vector<double> zz(k);
      std::vector<int> ww(k);
      for (int q = 0; q < np; ++q) {
        zz[2 * q] = zz[2 * q + 1] = z[p0 + q];
        ww[2 * q] = 1;
        ww[2 * q + 1] = 2;
      }
      std::vector<ect_signal_point> pts(np);
      for (int q = 0; q < np; ++q) {
        std::memset(&pts[q], 0, sizeof(ect_signal_point));
        pts[q].z = z[p0 + q];
      }
      try {
        {
          EventTimer t(ctx, &ctx->timings.rhs_ms);
          ect::build_rhs(s->mesh, s->coil, zz.data(), ww.data(), k, s->amplitude, rhs.p);
        }
        ect::SolveOut sp, sr;
        {
          EventTimer t(ctx, &ctx->timings.solve_ms);
          ect::cocg_solve(ctx, s->a_primary, rhs.p, xp.p, k, s->opts, &sp);
          if (s->two_configs) ect::cocg_solve(ctx, s->a_reference, rhs.p, xr.p, k, s->opts, &sr);
        }
        // a failed solve (non-convergence or breakdown) fails its own position
        // only (scan.cpp:111-114,139-141)
        for (int q = 0; q < np; ++q) {
          ect_signal_point& pt = pts[q];
          bool ok = sp.converged[2 * q] && sp.converged[2 * q + 1];
          pt.iterations[0] = sp.iters[2 * q];
          pt.iterations[1] = sp.iters[2 * q + 1];
          if (s->two_configs) {
            ok = ok && sr.converged[2 * q] && sr.converged[2 * q + 1];
            pt.iterations[2] = sr.iters[2 * q];
            pt.iterations[3] = sr.iters[2 * q + 1];
          }
          if (!ok) {
            pt.failed = 1;  // scan.cpp:111-114,139-141
            continue;
          }
          double2 dz[4] = {};
          if (s->two_configs) {
            ect::delta_impedance(s->mesh, s->primary, s->reference, xp.p + 2 * q,
                                 xp.p + 2 * q + 1, xr.p + 2 * q, xr.p + 2 * q + 1, k, dz);
          }
          for (int j = 0; j < 4; ++j) {
            pt.dz[2 * j] = dz[j].x;
            pt.dz[2 * j + 1] = dz[j].y;
          }
          // signal_modes (signals.cpp:101-107): Z_FA = (i/2)(Z11 + Z12), Z_F3 = (i/2)(Z11 - Z22)
          const double s_re = dz[0].x + dz[1].x, s_im = dz[0].y + dz[1].y;
          const double d_re = dz[0].x - dz[3].x, d_im = dz[0].y - dz[3].y;
          pt.z_fa[0] = 0.0 * s_re - 0.5 * s_im;
          pt.z_fa[1] = 0.0 * s_im + 0.5 * s_re;
          pt.z_f3[0] = 0.0 * d_re - 0.5 * d_im;
          pt.z_f3[1] = 0.0 * d_im + 0.5 * d_re;
        }
        if (solutions && p0 + np == n_pos) {
          // 4 solution vectors of the last position: primary c1, c2, reference c1, c2
          const int q = np - 1;
          // columns gathered into contiguous vectors on the device, then ONE
          // contiguous copy (a strided 16-byte-row copy to the host costs ~10 ms
          // per vector over PCIe)
          double2* dst = reinterpret_cast<double2*>(solutions);
          const bool dev = ect::is_device_ptr(solutions);
          double2* stage = dst;
          if (!dev) {
            s->sol.ensure((size_t)4 * N);
            stage = s->sol.p;
          }
          const int cols[2] = {2 * q, 2 * q + 1};
          ect::gather_columns(ctx, xp.p, k, cols, 2, N, stage);
          ect::gather_columns(ctx, s->two_configs ? xr.p : xp.p, k, cols, 2, N, stage + 2 * N);
          if (!dev) copy_d2h(ctx, dst, stage, (size_t)4 * N * sizeof(double2));
          CK(cudaStreamSynchronize(ctx->stream));
        }
      } catch (const ect::Error& e) {
        if (e.code != ECT_ERR_SOLVER) throw;
        for (auto& pt : pts) pt.failed = 1;  // SolverError marks the points failed
      }
      for (int q = 0; q < np; ++q) out[p0 + q] = pts[q];
    }
  });
}

}  // extern "C"

// ============================================================================
// Distributed solve: halo plans (host only), parts, NCCL transport.
#include <dlfcn.h>
#include <nccl.h>

struct ect_halo_plan {
  ect::HaloPlan plan;
};

namespace ect {

struct NcclApi {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};

// NCCL is resolved at run time (dlopen of libnccl.so.2, which reuses the copy
// torch.distributed already loaded), so libectgpu.so has no link dependency.
const NcclApi* nccl_api() {
  static NcclApi api;
  static bool loaded = [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
    api.send = reinterpret_cast<decltype(api.send)>(dlsym(h, "ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(h, "ncclRecv"));
    api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(h, "ncclGroupStart"));
    api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(h, "ncclGroupEnd"));
    api.errorString = reinterpret_cast<decltype(api.errorString)>(dlsym(h, "ncclGetErrorString"));
    return api.getUniqueId && api.commInitRank && api.allReduce && api.send && api.recv &&
           api.groupStart && api.groupEnd;
  }();
  if (!loaded) fail(ECT_ERR_CUDA, "NCCL (libnccl.so.2) could not be loaded");
  return &api;
}

static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const NcclApi* a = nccl_api();
    fail(ECT_ERR_CUDA, std::string(what) + ": " + (a->errorString ? a->errorString(r) : "nccl error"));
  }
}

void nccl_allreduce_sum(ect_comm* c, double* buf, size_t n, cudaStream_t s) {
  nccl_check(nccl_api()->allReduce(buf, buf, n, ncclFloat64, ncclSum,
                                   static_cast<ncclComm_t>(c->comm), s), "ncclAllReduce");
}
void nccl_group_start() { nccl_check(nccl_api()->groupStart(), "ncclGroupStart"); }
void nccl_group_end() { nccl_check(nccl_api()->groupEnd(), "ncclGroupEnd"); }
void nccl_send(ect_comm* c, const void* buf, size_t n_doubles, int peer, cudaStream_t s) {
  nccl_check(nccl_api()->send(buf, n_doubles, ncclFloat64, peer, static_cast<ncclComm_t>(c->comm), s),
             "ncclSend");
}
void nccl_recv(ect_comm* c, void* buf, size_t n_doubles, int peer, cudaStream_t s) {
  nccl_check(nccl_api()->recv(buf, n_doubles, ncclFloat64, peer, static_cast<ncclComm_t>(c->comm), s),
             "ncclRecv");
}

}  // namespace ect

extern "C" {

int ect_halo_plan_create(int64_t n_nodes, const int32_t* nbr_off, const int32_t* nbr,
                         const int32_t* cond_fwd, const int64_t* splits, int32_t n_parts,
                         int32_t part, ect_halo_plan** out) {
  return guarded([&] {
    auto p = std::make_unique<ect_halo_plan>();
    try {
      p->plan = ect::build_halo_plan(n_nodes, nbr_off, nbr, cond_fwd, splits, n_parts, part);
    } catch (const std::invalid_argument& e) {
      ect::fail(ECT_ERR_CONFIG, e.what());
    }
    *out = p.release();
  });
}

int ect_halo_plan_destroy(ect_halo_plan* p) {
  return guarded([&] { delete p; });
}

int ect_halo_plan_info(ect_halo_plan* p, int64_t info[8]) {
  return guarded([&] {
    const auto& H = p->plan;
    const int64_t v[8] = {H.n0, H.n1, H.L, H.G, H.c0, H.Vo, H.Vg, (int64_t)H.peers.size()};
    for (int i = 0; i < 8; ++i) info[i] = v[i];
  });
}

int ect_halo_plan_arrays(ect_halo_plan* p, int32_t* ghost_nodes, int32_t* local_vdof) {
  return guarded([&] {
    const auto& H = p->plan;
    if (ghost_nodes) std::memcpy(ghost_nodes, H.ghost_nodes.data(), H.G * sizeof(int32_t));
    if (local_vdof) std::memcpy(local_vdof, H.local_vdof.data(), (H.L + H.G) * sizeof(int32_t));
  });
}

int ect_halo_plan_peer(ect_halo_plan* p, int32_t i, int64_t info[7], int32_t* send_nodes,
                       int32_t* send_cond_nodes) {
  return guarded([&] {
    const auto& H = p->plan;
    require(i >= 0 && i < (int)H.peers.size(), ECT_ERR_CONFIG, "halo plan: peer index out of range");
    const auto& q = H.peers[i];
    const int64_t v[7] = {q.part, q.recv_node_begin, q.recv_node_count, q.recv_v_begin,
                          q.recv_v_count, (int64_t)q.send_nodes.size(),
                          (int64_t)q.send_cond_nodes.size()};
    for (int j = 0; j < 7; ++j) info[j] = v[j];
    if (send_nodes) std::memcpy(send_nodes, q.send_nodes.data(), q.send_nodes.size() * 4);
    if (send_cond_nodes)
      std::memcpy(send_cond_nodes, q.send_cond_nodes.data(), q.send_cond_nodes.size() * 4);
  });
}

int ect_comm_unique_id(void* out128) {
  return guarded([&] {
    ncclUniqueId id;
    ect::nccl_check(ect::nccl_api()->getUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
  });
}

int ect_comm_create(ect_ctx* ctx, int32_t rank, int32_t world, const void* id128, ect_comm** out) {
  return guarded([&] {
    ScopedDevice sd(ctx->device);
    auto c = std::make_unique<ect_comm>();
    c->rank = rank;
    c->world = world;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm = nullptr;
    ect::nccl_check(ect::nccl_api()->commInitRank(&comm, world, id, rank), "ncclCommInitRank");
    c->comm = comm;
    *out = c.release();
  });
}

int ect_comm_destroy(ect_comm* c) {
  return guarded([&] {
    if (!c) return;
    if (c->comm) ect::nccl_api()->commDestroy(static_cast<ncclComm_t>(c->comm));
    delete c;
  });
}

int ect_part_create(ect_ctx* ctx, ect_mesh* mesh, ect_matrix* a, const int64_t* splits,
                    int32_t n_parts, int32_t part, ect_part** out) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    require(a->assembled, ECT_ERR_SOLVER, "part: matrix values not assembled");
    try {
      *out = ect::create_part(mesh, a, splits, n_parts, part);
    } catch (const std::invalid_argument& e) {
      ect::fail(ECT_ERR_CONFIG, e.what());
    }
  });
}

int ect_part_create_assembled(ect_ctx* ctx, ect_mesh* mesh, const ect_materials* mats,
                              const int64_t* splits, int32_t n_parts, int32_t part,
                              ect_part** out) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    check_materials(*mats);
    try {
      EventTimer t(ctx, &ctx->timings.assemble_ms);
      *out = ect::create_part_assembled(mesh, *mats, splits, n_parts, part);
    } catch (const std::invalid_argument& e) {
      ect::fail(ECT_ERR_CONFIG, e.what());
    }
  });
}

int ect_part_destroy(ect_part* p) {
  return guarded([&] {
    if (!p) return;
    ScopedDevice sd(p->ctx->device);
    delete p;
  });
}

int ect_part_info(ect_part* p, int64_t info[8]) {
  return guarded([&] {
    const auto& H = p->plan;
    const int64_t v[8] = {H.n0, H.n1, H.L, H.G, H.Vo, H.Vg, (int64_t)H.peers.size(), p->nblk};
    for (int i = 0; i < 8; ++i) info[i] = v[i];
  });
}

int ect_dist_solve(ect_part** parts, int32_t n_parts, ect_comm* comm, const double* b, double* x,
                   int32_t n_rhs, const ect_iter_options* opts, ect_iter_result* results) {
  return guarded([&] {
    require(n_parts >= 1 && parts && parts[0], ECT_ERR_SOLVER, "dist_solve: no parts");
    ect_ctx* ctx = parts[0]->ctx;
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ScopedDevice sd(ctx->device);
    ect_iter_options o = opts ? *opts : ect_iter_options{1e-8, 500, 80};
    const size_t cnt = (size_t)parts[0]->n_global * n_rhs;
    In<double2> bi(ctx, reinterpret_cast<const double2*>(b), cnt);
    // x is written only on the rows the given parts own: stage the caller's
    // buffer so untouched rows keep their values
    Out<double2> xo(ctx, reinterpret_cast<double2*>(x), cnt);
    if (xo.host) CK(cudaMemcpyAsync(xo.dev, x, cnt * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
    ect::SolveOut so;
    {
      EventTimer t(ctx, &ctx->timings.solve_ms);
      ect::dist_solve(parts, n_parts, comm, bi.dev, xo.dev, n_rhs, o, &so);
    }
    xo.finish();
    for (int c = 0; c < n_rhs; ++c) {
      results[c].iterations = so.iters[c];
      results[c].residual = so.residual[c];
      results[c].converged = so.converged[c];
    }
  });
}

}  // extern "C"
