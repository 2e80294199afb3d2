// Reference-side binding of the ectgpu drop-in: the
// definition of ectsim::solve_iterative (solver.hpp:69-70) a maintainer links
// INSTEAD OF proj/core/src/iterative.cpp. Everything above it — ScanSession's
// per-position chain (scan.cpp:95-143), run_scan, the CLI — is the unmodified
// reference. Built by oracle/Makefile into _ref/libectref_gpu.so with the
// other twelve reference translation units (compiled where they lie) so the
// tests can run the reference's own ScanSession on the GPU solver.
//
// The reference hands over its CscMatrix (sparse.hpp:56-66) as is:
// ect_matrix_from_csc uploads it, probes symmetry (COCG, else BiCGStab) and the
// matrix is cached for the session's later calls (ScanSession keeps its
// matrices immutable for its lifetime, scan.hpp:36-38). The contract of
// iterative.cpp is kept: non-convergence clears `converged`, breakdown and bad
// options raise SolverError (iterative.cpp:112-118, 176).
#include <map>
#include <mutex>
#include <stdexcept>
#include <tuple>

#include "ectsim/solver.hpp"
#include "ectgpu.h"

namespace ectsim {
namespace {

void check(int rc) {
  if (rc == ECT_OK) return;
  const std::string msg = ect_last_error();
  if (rc == ECT_ERR_SOLVER) throw SolverError(msg);
  if (rc == ECT_ERR_MESH) throw MeshError(msg);
  if (rc == ECT_ERR_CONFIG) throw ConfigError(msg);
  if (rc == ECT_ERR_IO) throw IoError(msg);
  throw std::runtime_error(msg);
}

struct GpuState {
  std::mutex mu;
  ect_ctx* ctx = nullptr;
  // (matrix object, values buffer, nnz) -> uploaded device matrix
  std::map<std::tuple<const CscMatrix*, const complexd*, size_t>, ect_matrix*> cache;
};

GpuState& state() {
  static GpuState s;
  return s;
}

ect_matrix* device_matrix(const CscMatrix& a) {
  GpuState& s = state();
  std::lock_guard<std::mutex> lk(s.mu);
  if (!s.ctx) check(ect_ctx_create(0, &s.ctx));
  const auto key = std::make_tuple(&a, a.values.data(), a.nnz());
  auto it = s.cache.find(key);
  if (it != s.cache.end()) return it->second;
  ect_matrix* m = nullptr;
  check(ect_matrix_from_csc(s.ctx, a.n_rows, static_cast<int64_t>(a.nnz()), a.col_ptr.data(),
                            a.row_idx.data(), reinterpret_cast<const double*>(a.values.data()),
                            &m));
  s.cache.emplace(key, m);
  return m;
}

}  // namespace

IterativeResult solve_iterative(const CscMatrix& a, std::span<const complexd> b,
                                const IterativeOptions& options) {
  // argument checks as iterative.cpp:111-115
  if (a.n_rows != a.n_cols) throw SolverError("solve_iterative: matrix must be square");
  if (static_cast<int>(b.size()) != a.n_rows) {
    throw SolverError("solve_iterative: rhs dimension mismatch");
  }
  if (!(options.tol > 0.0)) throw SolverError("solve_iterative: tolerance must be positive");
  ect_matrix* m = device_matrix(a);
  IterativeResult r;
  r.x.assign(b.size(), complexd(0.0, 0.0));
  const ect_iter_options opt{options.tol, options.max_iter, options.restart};
  ect_iter_result res{};
  check(ect_solve(state().ctx, m, reinterpret_cast<const double*>(b.data()),
                  reinterpret_cast<double*>(r.x.data()), 1, &opt, &res));
  r.iterations = res.iterations;
  r.residual = res.residual;  // true ||b - A x|| / ||b|| (iterative.cpp:208-216)
  r.converged = res.converged != 0;
  return r;
}

}  // namespace ectsim
