// Internal types shared by the ectgpu translation units (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ectgpu.h"

namespace ect {

// Error carrying an ABI status code; thrown inside the library, converted to
// a status at the C boundary (mirrors the reference's exception classes,
// types.hpp:53-64).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& what) { throw Error(code, what); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    fail(ECT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                           std::to_string(line) + ")");
  }
}
#define CK(x) ::ect::cuda_check((x), #x, __FILE__, __LINE__)
#define CK_LAUNCH() ::ect::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// Owning device buffer.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) CK(cudaMalloc(&p, count * sizeof(T)));
  }
  void ensure(size_t count) {
    if (count > n) alloc(count);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// Device-side per-right-hand-side Krylov state (see krylov.cu).
struct RhsState {
  double2 rho;    // r^T z (unconjugated, COCG); (r_hat, r) in BiCGStab
  double2 alpha;
  double2 beta;
  double2 omega;  // BiCGStab stabilisation step
  double bnorm;
  double rnorm;
  int iters;
  int status;     // kActive / kConverged / kBreakdown / kMaxIter / kZeroRhs
  int xpend;      // COCG: x += alpha p still owed (applied by the next p-update)
  int restart_dir;  // COCG: stalled, the next direction is p = z (beta = 0)
  double rbest;     // smallest recurrence residual since the last (re)start
  double best_iter; // iteration that set rbest
};
enum RhsStatus : int { kActive = 0, kConverged = 1, kBreakdown = 2, kMaxIter = 3, kZeroRhs = 4 };

// Per-context kernel accounting and optional SpMV event profiling.
struct Profile {
  bool enabled = false;
  std::vector<cudaEvent_t> pool;  // pairs (start, stop)
  std::vector<int> kinds;          // kind of the pair starting at index i
  // solver samples: the batch width and the slot of `snaps` holding the
  // device-side active-column count at the sampled iteration (-1: none)
  std::vector<int> widths, snap_of;
  DevBuf<int> snaps;
  size_t n_snaps = 0;
  size_t used = 0;
  int64_t launches = 0;
};

// Aggregation multigrid hierarchy (amg.cu setup, krylov.cu cycle). Level 0
// is the matrix itself; level l+1 = P_l^T A_l P_l with the plain-aggregation
// prolongator P_l (0/1 entries: dof i -> coarse dof cmap[i], -1 for
// Dirichlet-pinned dofs), coarsest level inverted densely.
struct AmgLevel {
  int64_t n = 0, nnz = 0;
  DevBuf<int> row_ptr, col;          // levels >= 1 (level 0 streams the ect_matrix)
  DevBuf<double2> val, dinv;
  int64_t n_next = 0;
  DevBuf<int> cmap;                  // [n] coarse dof of each dof (-1: not aggregated)
  DevBuf<int> r_ptr, r_idx;          // coarse dof -> its dofs, ascending
  DevBuf<double2> xt, t, b, out, b2, out2;  // cycle work vectors [n][kcap]
};
// One solver iteration captured as a CUDA graph, kept with the hierarchy it
// replays; valid while the batch width, the solver workspace and the stopping
// parameters baked into the kernel arguments are unchanged.
struct IterGraph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int launches = 0, k = 0, max_iter = 0;
  double tol = 0.0;
  const void* tag[3] = {nullptr, nullptr, nullptr};
  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
  }
  ~IterGraph() { reset(); }
};
struct Amg {
  IterGraph iter;
  std::vector<AmgLevel> lv;          // lv.back() is the dense coarsest level
  DevBuf<double2> minv;              // [n][n] row-major inverse of the coarsest matrix
  double omega = 0.6;                // damped-Jacobi weight
  double oc = 1.5;                   // coarse-correction over-weighting
  int wcycle = 1;                    // 1: W-cycle (two coarse visits per level), 0: V
  int kcap = 0;                      // batch width the work vectors hold
  double setup_ms = 0.0;
  double op_complexity = 0.0;        // sum of level nnz / fine nnz
  // finest-level smoothing in fp32 (krylov.cu k_nbe32): NB-E block / coupling
  // copies and the level's iterate and residual
  bool f32 = true;
  DevBuf<float> blk32, cpl32;
  DevBuf<float2> xt32, t32;
};

}  // namespace ect

struct ect_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  std::recursive_mutex mu;
  ect::DevBuf<char> cub_tmp;
  ect_timings timings{};
  ect::Profile prof;
  // pinned staging for host<->device copies
  void* pinned = nullptr;                      // two staging halves (ectgpu.cpp copy_h2d/d2h)
  size_t pinned_bytes = 0;
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  int* pinned_flag = nullptr;  // small pinned word for convergence polling
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;  // convergence polling (krylov.cu)
  cudaEvent_t marks[8] = {};                    // ect_ctx_mark / ect_ctx_elapsed_ms
  std::vector<cudaEvent_t> timer_events;        // EventTimer pool (2 per nesting level)
  int timer_depth = 0;
  cudaStream_t halo_stream = nullptr;           // distributed solve: halo exchange
  cudaEvent_t ev_h1 = nullptr, ev_h2 = nullptr;
  bool force_csr = false;                       // ect_ctx_set_format(ctx, ECT_FORMAT_CSR)
  bool use_sell = false;                        // ect_ctx_set_format(ctx, ECT_FORMAT_SELL)
  int precond = ECT_PRECOND_AMG;                // default for matrices created afterwards
  int sell_sigma = 256;
  struct SolverWorkspace {                      // cocg_solve buffers, reused across solves
    ect::DevBuf<double2> bb, xx, r, p, q, z;
    ect::DevBuf<double2> rh, ph, sh, t;         // BiCGStab extras
    ect::DevBuf<ect::RhsState> st;
    ect::DevBuf<int> n_active;
    ect::DevBuf<unsigned> counter;
    ect::DevBuf<double> partial;
  } ws;
};

struct ect_mesh {
  ect_ctx* ctx = nullptr;
  int64_t n_nodes = 0, n_tets = 0, n_cond = 0, n_pins = 0, n_defect = 0;
  ect::DevBuf<double> xyz;         // [n_nodes][3]
  ect::DevBuf<int4> tets;          // canonical connectivity
  ect::DevBuf<uint8_t> region;     // RegionTag per tet
  ect::DevBuf<int> cond_fwd;       // node -> conductor dof or -1
  ect::DevBuf<int> inc_off;        // node -> incident tet range (n_nodes + 1)
  ect::DevBuf<int> inc;            // 4 * tet + local index, ascending tet per node
  ect::DevBuf<uint8_t> pinned;     // per A-dof (3 n_nodes) essential-BC flag
  ect::DevBuf<int> defect_tets;    // DEFECT tets ascending (signals.cpp:67-99)
  // node-neighbour structure produced by the pattern build (K1)
  ect::DevBuf<int> nbr_off;        // n_nodes + 1
  ect::DevBuf<int> nbr;            // neighbour node ids ascending, incl. self
  ect::DevBuf<uint8_t> nbr_cond;   // neighbour shares a conductor tet
  bool have_nbr = false;
  // scratch of the per-position kernels (right-hand sides, impedance), kept
  // across calls: cudaMalloc / cudaFree take driver-wide locks and synchronise
  // the device, which showed up as sporadic 0.3-1.3 s stalls per sweep step
  ect::DevBuf<uint8_t> rhs_flag;
  ect::DevBuf<double> rhs_j, dz_contrib, dz_res;
  ect::DevBuf<int> rhs_stat;
  // host copies (host-side reference semantics: mu_tilde, z extremes)
  std::vector<double> h_xyz;
  std::vector<int32_t> h_tets;
  std::vector<uint8_t> h_region;
  double z_lo = 0.0, z_hi = 0.0;
  int max_inc = 0, max_nbr = 0;
  // impedance (GAMMA_P) faces, built on first IBC assembly (assembly.cu):
  // sorted node triples in classify_boundary's order, their TriFrames, and
  // per node the incident faces ascending (entry = 4 * face + position)
  bool have_ibc = false;
  int64_t n_ibc = 0;
  ect::DevBuf<int> ibc_nodes;      // [n_ibc][3]
  ect::DevBuf<double> ibc_frame;   // [n_ibc][13]: area, normal[3], grad_tau[3][3]
  ect::DevBuf<int> ibc_off;        // n_nodes + 1
  ect::DevBuf<int> ibc_inc;
};

#include <memory>

struct ect_matrix {
  ect_ctx* ctx = nullptr;
  ect_mesh* mesh = nullptr;         // the mesh a from-mesh pattern was built on (borrowed)
  int precond = ECT_PRECOND_JACOBI;  // ECT_PRECOND_* used by ect_solve / the session
  std::unique_ptr<ect::Amg> amg;    // built on first use of ECT_PRECOND_AMG
  int64_t n_zero_diag = 0;          // Jacobi: rows without a usable diagonal
  int64_t node_lo = 0, node_hi = -1;  // rows of these nodes only (slab), -1: all
  int64_t n = 0, nnz = 0;
  int64_t n_nodes = 0, n_cond = 0;  // DOF structure when built from a mesh
  bool from_mesh = false;
  bool assembled = false;
  bool symmetric = true;  // false with impedance surface terms (va = i omega av^T)
  ect::DevBuf<int> row_ptr;
  ect::DevBuf<int> col;
  ect::DevBuf<double2> val;
  ect::DevBuf<double2> dinv;       // Jacobi preconditioner 1/diag
  // Node-block (NB) streaming format for the SpMV (krylov.cu, build_nb):
  // per node i, 3x3 A-A blocks (real parts + the 3 diagonal imaginary parts,
  // 6 double2 planes) over the neighbour list, and conductor couplings
  // (A-V column, V-A row, V-V entry: 4 double2 planes).
  bool has_nb = false;
  int64_t nb_blocks = 0, nb_ncpl = 0;
  const int* nb_blk_ptr = nullptr;  // = mesh->nbr_off (borrowed)
  const int* nb_blk_col = nullptr;  // = mesh->nbr (borrowed)
  const int* nb_cond_fwd = nullptr; // = mesh->cond_fwd (borrowed)
  ect::DevBuf<double2> nb_blk;      // [6][nb_blocks] (released once NB-E is built)
  ect::DevBuf<int> nb_cpl_ptr;      // n_nodes + 1
  ect::DevBuf<int2> nb_cpl_idx;     // (node m, cond dof of m)
  ect::DevBuf<double2> nb_cpl;      // [4][nb_cpl]
  // NB-E: sliced-ELL copy of the NB blocks (chunks of 32 nodes, slot-major)
  bool has_nbe = false;
  int64_t nbe_slots = 0;
  ect::DevBuf<int> nbe_off, nbe_col;
  ect::DevBuf<double2> nbe_blk;
  // SELL-C-sigma (ECT_FORMAT_SELL): chunk offsets, slot -> row, padded entries
  bool has_sell = false;
  int64_t sell_chunks = 0, sell_stored = 0;
  ect::DevBuf<int> sell_off, sell_perm, sell_col;
  ect::DevBuf<double2> sell_val;
};

#include "dist_plan.h"

// One row partition of the global matrix on one GPU (distributed solve).
struct ect_part {
  ect_ctx* ctx = nullptr;
  ect::HaloPlan plan;
  int64_t n_global = 0, na_global = 0, n_nodes_global = 0;
  int64_t nblk = 0, ncpl = 0;
  ect::DevBuf<int> blk_ptr, cpl_ptr, cond_local;
  ect::DevBuf<int2> cpl_idx;
  ect::DevBuf<double2> cpl, dinv;  // coupling planes (2 x 4 doubles), local dinv
  int64_t int_lo = 0, int_hi = 0;        // interior owned nodes (no ghost columns)
  bool has_nbe = false;                  // sliced-ELL copy of blk (default SpMV layout)
  int64_t nbe_slots = 0;
  ect::DevBuf<int> nbe_off, nbe_col;
  ect::DevBuf<double2> nbe_blk;
  struct Peer {
    ect::DevBuf<int> send_nodes, send_cond;
    ect::DevBuf<double2> sendbuf;
    int64_t ns = 0, nsc = 0;
  };
  std::vector<Peer> peers;  // parallel to plan.peers
};

// NCCL communicator for the distributed solve (loaded with dlopen).
struct ect_comm {
  int rank = 0, world = 1;
  void* comm = nullptr;  // ncclComm_t
};

namespace ect {

// Buffer argument that may be host or device memory.
bool is_device_ptr(const void* p);

// Kernel entry points implemented in the .cu files.
void build_mesh_topology(ect_mesh* m);                         // mesh.cu
// K1 pattern; rows of nodes [lo, hi) only when a range is given (slab of a
// row partition: the other rows stay empty, indices stay global)
void build_pattern(ect_mesh* m, ect_matrix* a, int64_t lo = 0, int64_t hi = -1);  // pattern.cu
void export_csc_values(ect_matrix* a, double2* out);           // pattern.cu (symmetric pattern)
// External CSC (csc = true) or CSR arrays on the device -> a's CSR + symmetry probe
void matrix_from_compressed(ect_ctx* ctx, int64_t n, int64_t nnz, const int* ptr, const int* idx,
                            const double2* val, bool csc, ect_matrix* a);  // pattern.cu
void assemble_values(ect_mesh* m, const ect_materials& mats, ect_matrix* a);  // assembly.cu
void compute_jacobi(ect_matrix* a);                            // krylov.cu
void build_nb(ect_mesh* m, ect_matrix* a);                     // krylov.cu (NB format)
void build_sell(ect_matrix* a, int sigma);                     // krylov.cu (SELL-C-sigma)
void spmv(ect_ctx* ctx, ect_matrix* a, const double2* x, double2* y, int k);  // spmv.cu
// dst[c * n + i] = src[i * k + cols[c]] for c < n_cols <= 4 (columns of an
// interleaved [n][k] batch as contiguous vectors, on the context stream)
void gather_columns(ect_ctx* ctx, const double2* src, int k, const int* cols, int n_cols,
                    int64_t n, double2* dst);
void build_rhs(ect_mesh* m, const ect_coil& coil, const double* z, const int* which, int n_rhs,
               double amplitude, double2* rhs);                // rhs.cu
void build_rhs_support(ect_mesh* m, const int* support, int64_t n_support, int region_tag,
                       double amplitude, double2* rhs);  // rhs.cu (support == nullptr: region)
void apply_pins_rhs(ect_mesh* m, double2* rhs, int n_rhs);  // rhs.cu
void delta_impedance(ect_mesh* m, const ect_materials& p, const ect_materials& r,
                     const double2* xk1, const double2* xk2, const double2* xl1,
                     const double2* xl2, int stride, double2 out[4]);  // signals.cu
struct SolveOut {
  std::vector<int> iters;
  std::vector<double> residual;
  std::vector<int> converged;
  std::vector<int> breakdown;  // per column: the Krylov recurrence broke down
};
// ect_solve's contract (iterative.cpp:176): a breakdown is a SolverError
void throw_on_breakdown(const SolveOut& out);
void cocg_solve(ect_ctx* ctx, ect_matrix* a, const double2* b, double2* x, int k,
                const ect_iter_options& opt, SolveOut* out);  // krylov.cu
void amg_setup(ect_matrix* a);                                  // amg.cu

// distributed solve (krylov.cu)
ect_part* create_part(ect_mesh* m, ect_matrix* a, const int64_t* splits, int n_parts, int part);
// the same part assembled directly: only the slab's rows are ever built
ect_part* create_part_assembled(ect_mesh* m, const ect_materials& mats, const int64_t* splits,
                                int n_parts, int part);
void dist_solve(ect_part** parts, int n_parts, ect_comm* comm, const double2* b_global,
                double2* x_global, int k, const ect_iter_options& opt, SolveOut* out);
// NCCL entry points resolved at runtime (ectgpu.cpp)
struct NcclApi;
const NcclApi* nccl_api();
void nccl_allreduce_sum(ect_comm* c, double* buf, size_t n, cudaStream_t s);
void nccl_group_start();
void nccl_group_end();
void nccl_send(ect_comm* c, const void* buf, size_t n_doubles, int peer, cudaStream_t s);
void nccl_recv(ect_comm* c, void* buf, size_t n_doubles, int peer, cudaStream_t s);

// cub temporary storage helper
void* cub_scratch(ect_ctx* ctx, size_t bytes);
int grid_for(ect_ctx* ctx, const void* kernel, int block, size_t smem = 0);
void note_launch(ect_ctx* ctx, int n = 1);

}  // namespace ect
