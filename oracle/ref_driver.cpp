// C driver around the UNMODIFIED ectsim reference core — TEST INFRASTRUCTURE.
//
// Built by oracle/Makefile from the reference sources where they lie
// (/root/reference/proj/core/src/*.cpp, never copied) plus the Eigen-subset
// shim in oracle/shim/, into oracle/_ref/libectref.so. Only tests/,
// __graft_entry__.smoke() and bench.py's reference/cpu_baseline legs may load
// it, and only as the checker / CPU baseline. Nothing in the product links it.
//
// Every entry point below calls the reference's own public API:
//   mesh:      Mesh::canonicalize_orientation, classify_boundary, conductor_map
//              (mesh.hpp:26-89)
//   materials: RunConfig::material_table / resolve_mu_tilde (config.cpp:325-352),
//              reference_variant (materials.cpp:44-53)
//   assembly:  partition_tets, assemble_system, apply_essential_bc, build_global
//              (assembly.hpp:64-95)
//   rhs:       coil_support (tube_mesh.cpp:272-288), assemble_rhs,
//              apply_pins_to_rhs (assembly.cpp:329-378)
//   solve:     CscMatrix::multiply (sparse.cpp:115-124), solve_iterative
//              (iterative.cpp:109-228), Factorization (solver.cpp:197-376)
//   signals:   split_solution, delta_impedance, signal_modes (signals.cpp:10-107)
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "ectsim/assembly.hpp"
#include "ectsim/config.hpp"
#include "ectsim/element_forms.hpp"
#include "ectsim/materials.hpp"
#include "ectsim/mesh.hpp"
#include "ectsim/mesh_io.hpp"
#include "ectsim/partition.hpp"
#include "ectsim/scan.hpp"
#include "ectsim/signals.hpp"
#include "ectsim/solver.hpp"
#include "ectsim/sparse.hpp"
#include "ectsim/tube_mesh.hpp"
#include "ectsim/worker_pool.hpp"

using namespace ectsim;

namespace {

thread_local std::string g_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const MeshError& e) {
    g_error = e.what();
    return 3;
  } catch (const ConfigError& e) {
    g_error = e.what();
    return 2;
  } catch (const SolverError& e) {
    g_error = e.what();
    return 4;
  } catch (const IoError& e) {
    g_error = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 1;
  }
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

struct RefMesh {
  Mesh mesh;
  ConductorIndexMap cmap;
};

struct RefSystem {
  BlockSystem block;
  CscMatrix matrix;
  std::vector<int> dof_node;
};

}  // namespace

// Packed MaterialTable (materials.hpp:21-48); identical layout to the
// product's ect_materials (include/ectgpu.h).
struct ref_materials {
  double omega;
  double sigma[6];
  double mu[6];
  double mu_tilde;
  double delta_gauge;
  double bc_penalty;
  double sigma_eps;
  int32_t ibc_enabled;
  int32_t l22_use_sigma_eps;
  double z_surface[2];  // surface impedance of the plate (IBC), re / im
};

// The subset of RunConfig [materials] keys (config.hpp:25-39).
struct ref_physics {
  double frequency;
  double sigma_tube;
  double mu_r_tube;
  double sigma_defect;  // < 0: unset (defaults to tube)
  double mu_r_defect;   // < 0: unset
  double sigma_eps_ratio;
  double delta_gauge;
  double bc_penalty;
  int32_t mu_tilde_harmonic;
  double mu_tilde_fixed;
  double sigma_tsp;  // < 0: default (config.hpp:29)
  double mu_r_tsp;   // < 0: default (config.hpp:30)
  int32_t ibc_tsp;   // materials.ibc_tsp (config.hpp:38)
};

static MaterialTable unpack(const ref_materials* m) {
  MaterialTable t;
  t.omega = m->omega;
  for (int r = 0; r < kRegionCount; ++r) {
    t.sigma[r] = m->sigma[r];
    t.mu[r] = m->mu[r];
  }
  t.mu_tilde = m->mu_tilde;
  t.delta_gauge = m->delta_gauge;
  t.bc_penalty = m->bc_penalty;
  t.sigma_eps = m->sigma_eps;
  t.ibc_enabled = m->ibc_enabled != 0;
  t.l22_use_sigma_eps = m->l22_use_sigma_eps != 0;
  t.z_surface = complexd(m->z_surface[0], m->z_surface[1]);
  return t;
}

static void pack(const MaterialTable& t, ref_materials* m) {
  std::memset(m, 0, sizeof(*m));
  m->omega = t.omega;
  for (int r = 0; r < kRegionCount; ++r) {
    m->sigma[r] = t.sigma[r];
    m->mu[r] = t.mu[r];
  }
  m->mu_tilde = t.mu_tilde;
  m->delta_gauge = t.delta_gauge;
  m->bc_penalty = t.bc_penalty;
  m->sigma_eps = t.sigma_eps;
  m->ibc_enabled = t.ibc_enabled;
  m->l22_use_sigma_eps = t.l22_use_sigma_eps;
  m->z_surface[0] = t.z_surface.real();
  m->z_surface[1] = t.z_surface.imag();
}

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

int ref_sizeof_materials() { return static_cast<int>(sizeof(ref_materials)); }

// Mesh from flat arrays, built exactly as tests/support/test_meshes.hpp:15-54
// builds its fixture: nodes + tets, canonicalize_orientation, then
// boundary faces from classify_boundary.
int ref_mesh_create(int64_t n_nodes, const double* xyz, int64_t n_tets, const int32_t* tets,
                    const uint8_t* region, void** out) {
  return guarded([&] {
    auto m = std::make_unique<RefMesh>();
    m->mesh.nodes.reserve(n_nodes);
    for (int64_t i = 0; i < n_nodes; ++i) {
      m->mesh.nodes.emplace_back(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
    }
    m->mesh.tets.reserve(n_tets);
    for (int64_t t = 0; t < n_tets; ++t) {
      Tet tet;
      for (int a = 0; a < 4; ++a) tet.nodes[a] = tets[4 * t + a];
      tet.region = static_cast<RegionTag>(region[t]);
      m->mesh.tets.push_back(tet);
    }
    m->mesh.canonicalize_orientation();
    for (const auto& fc : classify_boundary(m->mesh)) {
      m->mesh.boundary_faces.push_back({fc.nodes, fc.label});
    }
    m->cmap = conductor_map(m->mesh);
    *out = m.release();
  });
}

void ref_mesh_destroy(void* h) { delete static_cast<RefMesh*>(h); }

// generate_tube_mesh (tube_mesh.cpp:85-270) from a packed TubeMeshSpec:
// [domain_radius, z_min, z_max, tube_r_inner, tube_r_outer, tube_z_min,
//  tube_z_max, tsp(r_in, r_out, z_min, z_max), defect(4), coil(r_in, r_out,
//  height, gap), coil_ref_z, resolution, outer_radial_grading]; NaN = unset.
int ref_tube_mesh_create(const double* p, const double* scan_z, int32_t n_scan, void** out) {
  return guarded([&] {
    TubeMeshSpec spec;
    spec.domain_radius = p[0];
    spec.z_min = p[1];
    spec.z_max = p[2];
    spec.tube_r_inner = p[3];
    spec.tube_r_outer = p[4];
    if (p[5] == p[5]) spec.tube_z_min = p[5];
    if (p[6] == p[6]) spec.tube_z_max = p[6];
    if (p[7] == p[7]) spec.tsp = AnnularBox{p[7], p[8], p[9], p[10]};
    if (p[11] == p[11]) spec.defect = AnnularBox{p[11], p[12], p[13], p[14]};
    spec.coil = CoilPair{p[15], p[16], p[17], p[18]};
    spec.coil_ref_z = p[19];
    spec.resolution = static_cast<int>(p[20]);
    spec.outer_radial_grading = p[21];
    spec.scan_z.assign(scan_z, scan_z + n_scan);
    auto m = std::make_unique<RefMesh>();
    m->mesh = generate_tube_mesh(spec);
    m->cmap = conductor_map(m->mesh);
    *out = m.release();
  });
}

// ScanSession (scan.cpp:27-143) with solver.method = "iterative" on a
// generated tube mesh (TubeMeshSpec packed as in ref_tube_mesh_create): the
// reference's own per-position chain with RunConfig defaults otherwise
// (parts = 1). solve_iterative is the reference's GMRES(restart)+ILU(0) in
// libectref.so and the ectgpu drop-in (binding/iterative_gpu.cpp) in
// libectref_gpu.so. out per position: z, dz (8), z_fa (2), z_f3 (2), failed.
int ref_scan_session_tube(const double* p, const double* scan_z, int32_t n_scan,
                          const ref_physics* ph, double amplitude, double tol, int32_t max_iter,
                          int32_t restart, double* out) {
  return guarded([&] {
    RunConfig cfg;
    cfg.mesh_source = "generate";
    TubeMeshSpec& spec = cfg.geometry;
    spec.domain_radius = p[0];
    spec.z_min = p[1];
    spec.z_max = p[2];
    spec.tube_r_inner = p[3];
    spec.tube_r_outer = p[4];
    if (p[5] == p[5]) spec.tube_z_min = p[5];
    if (p[6] == p[6]) spec.tube_z_max = p[6];
    if (p[7] == p[7]) spec.tsp = AnnularBox{p[7], p[8], p[9], p[10]};
    if (p[11] == p[11]) spec.defect = AnnularBox{p[11], p[12], p[13], p[14]};
    spec.coil = CoilPair{p[15], p[16], p[17], p[18]};
    spec.coil_ref_z = p[19];
    spec.resolution = static_cast<int>(p[20]);
    spec.outer_radial_grading = p[21];
    spec.scan_z.assign(scan_z, scan_z + n_scan);
    cfg.frequency = ph->frequency;
    cfg.sigma_tube = ph->sigma_tube;
    cfg.mu_r_tube = ph->mu_r_tube;
    if (ph->sigma_defect >= 0) cfg.sigma_defect = ph->sigma_defect;
    if (ph->mu_r_defect >= 0) cfg.mu_r_defect = ph->mu_r_defect;
    cfg.sigma_eps_ratio = ph->sigma_eps_ratio;
    cfg.delta_gauge = ph->delta_gauge;
    cfg.bc_penalty = ph->bc_penalty;
    cfg.mu_tilde_policy = ph->mu_tilde_harmonic ? "harmonic" : "fixed";
    cfg.mu_tilde_fixed = ph->mu_tilde_fixed;
    if (ph->sigma_tsp >= 0) cfg.sigma_tsp = ph->sigma_tsp;
    if (ph->mu_r_tsp >= 0) cfg.mu_r_tsp = ph->mu_r_tsp;
    cfg.ibc_tsp = ph->ibc_tsp != 0;
    cfg.coil_amplitude = amplitude;
    cfg.parts = 1;
    cfg.workers = 1;
    cfg.solver_method = "iterative";
    cfg.solver_tol = tol;
    cfg.solver_max_iter = max_iter;
    cfg.solver_restart = restart;
    ScanSession session(cfg);
    for (int32_t i = 0; i < n_scan; ++i) {
      SignalPoint pt = session.solve_position(scan_z[i]);
      double* o = out + 14 * i;
      o[0] = pt.z;
      for (int k = 0; k < 2; ++k)
        for (int l = 0; l < 2; ++l) {
          o[1 + 2 * (2 * k + l)] = pt.delta_z.z[k][l].real();
          o[2 + 2 * (2 * k + l)] = pt.delta_z.z[k][l].imag();
        }
      o[9] = pt.z_fa.real();
      o[10] = pt.z_fa.imag();
      o[11] = pt.z_f3.real();
      o[12] = pt.z_f3.imag();
      o[13] = pt.failed ? 1.0 : 0.0;
    }
  });
}

// load_mesh / write_mesh (mesh_io.cpp), canonical tag map
int ref_mesh_load(const char* path, void** out) {
  return guarded([&] {
    auto m = std::make_unique<RefMesh>();
    m->mesh = load_mesh(path);
    m->cmap = conductor_map(m->mesh);
    *out = m.release();
  });
}
int ref_mesh_write(void* h, const char* path) {
  return guarded([&] { write_mesh(static_cast<RefMesh*>(h)->mesh, path); });
}

// node coordinates and tet regions of a mesh (after canonicalization)
int ref_mesh_geometry(void* h, double* xyz, uint8_t* region) {
  return guarded([&] {
    auto* m = static_cast<RefMesh*>(h);
    for (int n = 0; n < m->mesh.node_count(); ++n)
      for (int a = 0; a < 3; ++a) xyz[3 * n + a] = m->mesh.nodes[n][a];
    for (int t = 0; t < m->mesh.tet_count(); ++t)
      region[t] = static_cast<uint8_t>(m->mesh.tets[t].region);
  });
}

int ref_mesh_counts(void* h, int64_t* n_nodes, int64_t* n_tets, int64_t* n_cond,
                    int64_t* n_boundary_faces) {
  return guarded([&] {
    auto* m = static_cast<RefMesh*>(h);
    *n_nodes = m->mesh.node_count();
    *n_tets = m->mesh.tet_count();
    *n_cond = m->cmap.count();
    *n_boundary_faces = static_cast<int64_t>(m->mesh.boundary_faces.size());
  });
}

int ref_mesh_export(void* h, int32_t* tets, int32_t* cond_forward, int32_t* faces,
                    int32_t* face_labels) {
  return guarded([&] {
    auto* m = static_cast<RefMesh*>(h);
    if (tets) {
      for (int t = 0; t < m->mesh.tet_count(); ++t)
        for (int a = 0; a < 4; ++a) tets[4 * t + a] = m->mesh.tets[t].nodes[a];
    }
    if (cond_forward) {
      for (int n = 0; n < m->mesh.node_count(); ++n) cond_forward[n] = m->cmap.forward[n];
    }
    if (faces) {
      for (size_t f = 0; f < m->mesh.boundary_faces.size(); ++f) {
        for (int a = 0; a < 3; ++a) faces[3 * f + a] = m->mesh.boundary_faces[f].nodes[a];
        if (face_labels) face_labels[f] = static_cast<int32_t>(m->mesh.boundary_faces[f].label);
      }
    }
  });
}

// RunConfig::material_table + resolve_mu_tilde (config.cpp:325-352).
int ref_materials_from_physics(void* h, const ref_physics* p, ref_materials* primary,
                               ref_materials* reference, int32_t* two_configs) {
  return guarded([&] {
    auto* m = static_cast<RefMesh*>(h);
    RunConfig cfg;
    cfg.frequency = p->frequency;
    cfg.sigma_tube = p->sigma_tube;
    cfg.mu_r_tube = p->mu_r_tube;
    if (p->sigma_defect >= 0) cfg.sigma_defect = p->sigma_defect;
    if (p->mu_r_defect >= 0) cfg.mu_r_defect = p->mu_r_defect;
    cfg.sigma_eps_ratio = p->sigma_eps_ratio;
    cfg.delta_gauge = p->delta_gauge;
    cfg.bc_penalty = p->bc_penalty;
    cfg.mu_tilde_policy = p->mu_tilde_harmonic ? "harmonic" : "fixed";
    cfg.mu_tilde_fixed = p->mu_tilde_fixed;
    if (p->sigma_tsp >= 0) cfg.sigma_tsp = p->sigma_tsp;
    if (p->mu_r_tsp >= 0) cfg.mu_r_tsp = p->mu_r_tsp;
    cfg.ibc_tsp = p->ibc_tsp != 0;
    MaterialTable mats = cfg.material_table();
    cfg.resolve_mu_tilde(mats, m->mesh);
    MaterialTable ref = reference_variant(mats);
    pack(mats, primary);
    pack(ref, reference);
    // scan.cpp:49: a second configuration only with defect tets.
    *two_configs = !m->mesh.region_tets(RegionTag::kDefect).empty() && !ref.same_coefficients(mats);
  });
}

// assemble_system -> apply_essential_bc -> build_global, as ScanSession does
// (scan.cpp:52-59). timings[0..3] = assemble, reduce, bc, build_global (s).
int ref_assemble(void* h, const ref_materials* mats, int32_t parts, int32_t workers,
                 uint32_t seed, void** out, double* timings) {
  return guarded([&] {
    auto* m = static_cast<RefMesh*>(h);
    auto s = std::make_unique<RefSystem>();
    PartitionMap pmap = partition_tets(m->mesh, parts, seed);
    AssembleTimings at;
    MaterialTable t = unpack(mats);
    s->block = assemble_system(m->mesh, m->cmap, t, pmap, workers, &at);
    auto t0 = std::chrono::steady_clock::now();
    apply_essential_bc(s->block, m->mesh);
    double t_bc = seconds_since(t0);
    t0 = std::chrono::steady_clock::now();
    GlobalSystem g = build_global(s->block);
    double t_global = seconds_since(t0);
    s->matrix = std::move(g.matrix);
    s->dof_node = std::move(g.dof_node);
    if (timings) {
      timings[0] = at.assemble;
      timings[1] = at.reduce;
      timings[2] = t_bc;
      timings[3] = t_global;
    }
    *out = s.release();
  });
}

void ref_system_destroy(void* h) { delete static_cast<RefSystem*>(h); }

// A RefSystem around externally supplied CSC arrays (used to hand the
// reference's solve_iterative a matrix that tests have shown bit-identical
// to its own assembly, without re-running the minutes-long reference
// assembly inside a bounded CPU-baseline sample). pins: optional.
int ref_system_from_csc(int64_t n, int64_t nnz, const int32_t* col_ptr, const int32_t* row_idx,
                        const double* values, void** out) {
  return guarded([&] {
    auto s = std::make_unique<RefSystem>();
    s->matrix.n_rows = static_cast<int>(n);
    s->matrix.n_cols = static_cast<int>(n);
    s->matrix.col_ptr.assign(col_ptr, col_ptr + n + 1);
    s->matrix.row_idx.assign(row_idx, row_idx + nnz);
    const complexd* v = reinterpret_cast<const complexd*>(values);
    s->matrix.values.assign(v, v + nnz);
    *out = s.release();
  });
}

int ref_system_counts(void* h, int64_t* n, int64_t* nnz, int64_t* n_pins) {
  return guarded([&] {
    auto* s = static_cast<RefSystem*>(h);
    *n = s->matrix.n_rows;
    *nnz = static_cast<int64_t>(s->matrix.nnz());
    *n_pins = static_cast<int64_t>(s->block.pins.size());
  });
}

// CSC arrays (sparse.hpp:55-66). values interleaved (re, im).
int ref_system_export(void* h, int32_t* col_ptr, int32_t* row_idx, double* values,
                      int32_t* pins) {
  return guarded([&] {
    auto* s = static_cast<RefSystem*>(h);
    const CscMatrix& a = s->matrix;
    if (col_ptr) std::memcpy(col_ptr, a.col_ptr.data(), sizeof(int) * a.col_ptr.size());
    if (row_idx) std::memcpy(row_idx, a.row_idx.data(), sizeof(int) * a.row_idx.size());
    if (values) std::memcpy(values, a.values.data(), sizeof(complexd) * a.values.size());
    if (pins) {
      for (size_t i = 0; i < s->block.pins.size(); ++i) pins[i] = s->block.pins[i].first;
    }
  });
}

// CscMatrix::multiply (sparse.cpp:115-124); repeat times, returns seconds.
int ref_multiply(void* h, const double* x, double* y, int32_t repeat, double* seconds) {
  return guarded([&] {
    auto* s = static_cast<RefSystem*>(h);
    const size_t n = s->matrix.n_rows;
    std::span<const complexd> xs(reinterpret_cast<const complexd*>(x), n);
    std::span<complexd> ys(reinterpret_cast<complexd*>(y), n);
    auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < std::max(1, repeat); ++r) s->matrix.multiply(xs, ys);
    if (seconds) *seconds = seconds_since(t0);
  });
}

// coil_support for a CoilPair {r_inner, r_outer, height, gap}.
int ref_coil_support(void* h, const double* coil, double probe_z, int32_t which, int32_t* out,
                     int64_t* count) {
  return guarded([&] {
    auto* m = static_cast<RefMesh*>(h);
    CoilPair c{coil[0], coil[1], coil[2], coil[3]};
    std::vector<int> sup = coil_support(m->mesh, c, probe_z, which);
    if (out) std::memcpy(out, sup.data(), sizeof(int) * sup.size());
    *count = static_cast<int64_t>(sup.size());
  });
}

// ScanSession::position_rhs (scan.cpp:87-93).
int ref_position_rhs(void* hm, void* hs, const double* coil, double probe_z, int32_t which,
                     double amplitude, double* rhs) {
  return guarded([&] {
    auto* m = static_cast<RefMesh*>(hm);
    auto* s = static_cast<RefSystem*>(hs);
    CoilPair c{coil[0], coil[1], coil[2], coil[3]};
    std::vector<int> sup = coil_support(m->mesh, c, probe_z, which);
    std::vector<complexd> b = assemble_rhs(m->mesh, sup, amplitude, s->block.total_dofs());
    apply_pins_to_rhs(s->block, b);
    std::memcpy(rhs, b.data(), sizeof(complexd) * b.size());
  });
}

// solve_iterative (iterative.cpp:109-228).
int ref_solve_iterative(void* h, const double* b, double tol, int32_t max_iter, int32_t restart,
                        double* x, int32_t* iterations, double* residual, int32_t* converged,
                        double* seconds) {
  return guarded([&] {
    auto* s = static_cast<RefSystem*>(h);
    const size_t n = s->matrix.n_rows;
    std::span<const complexd> bs(reinterpret_cast<const complexd*>(b), n);
    IterativeOptions opt{tol, max_iter, restart};
    auto t0 = std::chrono::steady_clock::now();
    IterativeResult r = solve_iterative(s->matrix, bs, opt);
    if (seconds) *seconds = seconds_since(t0);
    std::memcpy(x, r.x.data(), sizeof(complexd) * n);
    *iterations = r.iterations;
    *residual = r.residual;
    *converged = r.converged;
  });
}

// Parallel solve_iterative over n_rhs right-hand sides on `threads` workers,
// via the reference's parallel_for (worker_pool.hpp:15-28) as run_scan does
// with positions (scan.cpp:155-156). x may be null. Returns wall seconds.
int ref_solve_iterative_batch(void* h, const double* b, int32_t n_rhs, double tol,
                              int32_t max_iter, int32_t restart, int32_t threads, double* x,
                              int32_t* iterations, double* residual, double* seconds) {
  return guarded([&] {
    auto* s = static_cast<RefSystem*>(h);
    const size_t n = s->matrix.n_rows;
    std::vector<std::string> errors(n_rhs);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<IterativeResult> res(n_rhs);
    parallel_for(n_rhs, threads, [&](int i) {
      try {
        std::span<const complexd> bs(reinterpret_cast<const complexd*>(b) + i * n, n);
        res[i] = solve_iterative(s->matrix, bs, IterativeOptions{tol, max_iter, restart});
      } catch (const std::exception& e) {
        errors[i] = e.what();
      }
    });
    *seconds = seconds_since(t0);
    for (int i = 0; i < n_rhs; ++i) {
      if (!errors[i].empty()) throw SolverError(errors[i]);
      if (x) std::memcpy(x + 2 * i * n, res[i].x.data(), sizeof(complexd) * n);
      iterations[i] = res[i].iterations;
      residual[i] = res[i].residual;
    }
  });
}

// Factorization::compute + solve (solver.cpp:197-376): the reference's
// default direct path; feasible on small meshes only.
int ref_solve_direct(void* h, const double* b, int32_t n_rhs, double* x, double* residual) {
  return guarded([&] {
    auto* s = static_cast<RefSystem*>(h);
    const size_t n = s->matrix.n_rows;
    Factorization f = Factorization::compute(s->matrix, s->dof_node);
    for (int i = 0; i < n_rhs; ++i) {
      std::span<const complexd> bs(reinterpret_cast<const complexd*>(b) + i * n, n);
      SolveResult r = f.solve(bs);
      std::memcpy(x + 2 * i * n, r.x.data(), sizeof(complexd) * n);
      residual[i] = r.residual;
    }
  });
}

// relative_residual (sparse.cpp:135-145).
int ref_relative_residual(void* h, const double* x, const double* b, double* out) {
  return guarded([&] {
    auto* s = static_cast<RefSystem*>(h);
    const size_t n = s->matrix.n_rows;
    *out = relative_residual(s->matrix, std::span<const complexd>(reinterpret_cast<const complexd*>(x), n),
                             std::span<const complexd>(reinterpret_cast<const complexd*>(b), n));
  });
}

// delta_impedance over the mesh's DEFECT tets (signals.cpp:67-99, scan.cpp:123-135).
int ref_delta_impedance(void* hm, const ref_materials* primary, const ref_materials* reference,
                        const double* x_k, const double* x_l, double* out) {
  return guarded([&] {
    auto* m = static_cast<RefMesh*>(hm);
    MaterialTable p = unpack(primary), r = unpack(reference);
    const int nn = m->mesh.node_count(), nc = m->cmap.count();
    const size_t n = 3 * static_cast<size_t>(nn) + nc;
    PotentialSolution sk = split_solution(
        std::span<const complexd>(reinterpret_cast<const complexd*>(x_k), n), nn, nc, p.omega);
    PotentialSolution sl = split_solution(
        std::span<const complexd>(reinterpret_cast<const complexd*>(x_l), n), nn, nc, p.omega);
    std::vector<int> defect = m->mesh.region_tets(RegionTag::kDefect);
    complexd z = delta_impedance(m->mesh, m->cmap, defect, p, r, sk, sl);
    out[0] = z.real();
    out[1] = z.imag();
  });
}

// signal_modes (signals.cpp:101-107): dz = 4 complex (11, 12, 21, 22) -> z_fa, z_f3.
void ref_signal_modes(const double* dz, double* out) {
  DeltaZ d;
  d.z[0][0] = complexd(dz[0], dz[1]);
  d.z[0][1] = complexd(dz[2], dz[3]);
  d.z[1][0] = complexd(dz[4], dz[5]);
  d.z[1][1] = complexd(dz[6], dz[7]);
  SignalModes s = signal_modes(d);
  out[0] = s.z_fa.real();
  out[1] = s.z_fa.imag();
  out[2] = s.z_f3.real();
  out[3] = s.z_f3.imag();
}

// write_trace_csv (scan.cpp:170-207) of n points: dz = 8 doubles per point,
// modes = 4 doubles per point (z_fa, z_f3).
int ref_trace_write(const char* path, int32_t n, const double* z, const double* dz,
                    const double* modes, const int32_t* failed, const char* config_hash) {
  return guarded([&] {
    ImpedanceTrace tr;
    tr.config_hash = config_hash ? config_hash : "";
    for (int i = 0; i < n; ++i) {
      SignalPoint p;
      p.z = z[i];
      for (int q = 0; q < 4; ++q) p.delta_z.z[q / 2][q % 2] = complexd(dz[8 * i + 2 * q], dz[8 * i + 2 * q + 1]);
      p.z_fa = complexd(modes[4 * i], modes[4 * i + 1]);
      p.z_f3 = complexd(modes[4 * i + 2], modes[4 * i + 3]);
      p.failed = failed && failed[i];
      tr.points.push_back(p);
    }
    write_trace_csv(tr, path);
  });
}

// read_trace_csv x2 + max_relative_deviation (scan.cpp:209-272).
int ref_trace_max_relative_deviation(const char* a, const char* b, double* out) {
  return guarded([&] { *out = max_relative_deviation(read_trace_csv(a), read_trace_csv(b)); });
}

// Element forms for known-answer checks (element_forms.cpp:8-114).
// grad: 12 doubles, vol: 1; l11: 12x12 complex col-major (288 doubles).
int ref_tet_frame(const double* p, double* grad, double* vol) {
  return guarded([&] {
    TetFrame f = TetFrame::from(Vec3(p[0], p[1], p[2]), Vec3(p[3], p[4], p[5]),
                                Vec3(p[6], p[7], p[8]), Vec3(p[9], p[10], p[11]));
    for (int a = 0; a < 4; ++a)
      for (int c = 0; c < 3; ++c) grad[3 * a + c] = f.grad[a][c];
    *vol = f.volume;
  });
}

int ref_element_blocks(const double* p, double mu, double mu_tilde, double sigma, double omega,
                       double delta_gauge, double* l11, double* l12, double* l21, double* l22) {
  return guarded([&] {
    TetFrame f = TetFrame::from(Vec3(p[0], p[1], p[2]), Vec3(p[3], p[4], p[5]),
                                Vec3(p[6], p[7], p[8]), Vec3(p[9], p[10], p[11]));
    Mat12c a = element_l11(f, mu, mu_tilde, sigma, omega);
    Mat12x4c b = element_l12(f, sigma);
    Mat4x12c c = element_l21(f, sigma);
    Mat4c d = element_l22(f, sigma, omega, delta_gauge, mu);
    // row-major output
    for (int i = 0; i < 12; ++i)
      for (int j = 0; j < 12; ++j) {
        l11[2 * (12 * i + j)] = a(i, j).real();
        l11[2 * (12 * i + j) + 1] = a(i, j).imag();
      }
    for (int i = 0; i < 12; ++i)
      for (int j = 0; j < 4; ++j) {
        l12[2 * (4 * i + j)] = b(i, j).real();
        l12[2 * (4 * i + j) + 1] = b(i, j).imag();
        l21[2 * (12 * j + i)] = c(j, i).real();
        l21[2 * (12 * j + i) + 1] = c(j, i).imag();
      }
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) {
        l22[2 * (4 * i + j)] = d(i, j).real();
        l22[2 * (4 * i + j) + 1] = d(i, j).imag();
      }
  });
}

}  // extern "C"
