/*
 * ectgpu — B200 (sm_100a) drop-in for the ectsim A–V assembly + Krylov hot path.
 *
 * C ABI only: plain pointers and sizes, no C++/torch types cross it. Complex
 * arrays are interleaved (re, im) doubles = std::complex<double> /
 * cuDoubleComplex layout. Every buffer argument may be HOST memory (copied
 * through pinned staging) or DEVICE memory of the context's GPU (used in
 * place); the library detects which with cudaPointerGetAttributes.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/proj/core/...). Status codes mirror the reference's
 * exception classes (types.hpp:53-64, exit codes ect_main.cpp:18-22):
 *   0 ok, 2 ConfigError, 3 MeshError, 4 SolverError, 5 IoError,
 *   6 CUDA/device error, 1 other. ect_last_error() returns the message of the
 *   calling thread's last failure.
 *
 * Thread safety: a context owns one CUDA stream; calls on one context are
 * serialised internally, so ScanSession-style concurrent callers
 * (scan.cpp:155-156) are safe. Use one context per host thread for overlap.
 */
#ifndef ECTGPU_H_
#define ECTGPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ECT_OK 0
#define ECT_ERR_OTHER 1
#define ECT_ERR_CONFIG 2
#define ECT_ERR_MESH 3
#define ECT_ERR_SOLVER 4
#define ECT_ERR_IO 5
#define ECT_ERR_CUDA 6

/* RegionTag (types.hpp:22-29). */
#define ECT_REGION_TUBE 0
#define ECT_REGION_TSP 1
#define ECT_REGION_DEFECT 2
#define ECT_REGION_COIL1 3
#define ECT_REGION_COIL2 4
#define ECT_REGION_VACUUM 5
#define ECT_REGION_COUNT 6

typedef struct ect_ctx ect_ctx;
typedef struct ect_mesh ect_mesh;
typedef struct ect_matrix ect_matrix;
typedef struct ect_session ect_session;

/* MaterialTable (materials.hpp:21-48), same field order. */
typedef struct ect_materials {
  double omega;
  double sigma[ECT_REGION_COUNT];
  double mu[ECT_REGION_COUNT];
  double mu_tilde;
  double delta_gauge;
  double bc_penalty;
  double sigma_eps;
  int32_t ibc_enabled;       /* impedance condition on the GAMMA_P (plate) faces */
  int32_t l22_use_sigma_eps;
  double z_surface[2];       /* surface impedance (re, im) used when ibc_enabled */
} ect_materials;

/* RunConfig [materials] keys (config.hpp:25-39), same defaults. Fill with
 * ect_physics_init() and override fields; the values are validated as
 * RunConfig's parser does (config.cpp:218-236: positive frequency, sigmas,
 * mu_r, sigma_eps_ratio, bc_penalty, 0 < delta_gauge < 1) -> ECT_ERR_CONFIG.
 * sigma_defect / mu_r_defect are std::optional in the reference: NaN means
 * unset (defaults to the tube values, config.cpp:334-335). */
typedef struct ect_physics {
  double frequency;        /* 100e3 */
  double sigma_tube;       /* 1e6 */
  double mu_r_tube;        /* 1 */
  double sigma_defect;     /* NaN = unset */
  double mu_r_defect;      /* NaN = unset */
  double sigma_eps_ratio;  /* 1e-6 */
  double delta_gauge;      /* 1e-6 */
  double bc_penalty;       /* 1e13 */
  int32_t mu_tilde_harmonic; /* 1: mu_tilde_policy = harmonic, 0: fixed */
  double mu_tilde_fixed;   /* kMu0 */
  double sigma_tsp;        /* 5e6 (config.hpp:29) */
  double mu_r_tsp;         /* 50 (config.hpp:30) */
  int32_t ibc_tsp;         /* materials.ibc_tsp (config.hpp:38): plate as surface impedance */
  int32_t l22_sigma_eps;   /* materials.l22_sigma_eps (config.hpp:39) */
} ect_physics;

/* RunConfig's [materials] defaults (config.hpp:25-39). */
void ect_physics_init(ect_physics* physics);

/* CoilPair (tube_mesh.hpp:13-21). */
typedef struct ect_coil {
  double r_inner;
  double r_outer;
  double height;
  double gap;
} ect_coil;

/* IterativeOptions (solver.hpp:54-58). max_iter counts Krylov iterations per
 * right-hand side; restart is accepted for signature parity (COCG has none). */
typedef struct ect_iter_options {
  double tol;
  int32_t max_iter;
  int32_t restart;
} ect_iter_options;

/* IterativeResult (solver.hpp:60-65) minus x (written to the caller's buffer). */
typedef struct ect_iter_result {
  double residual;     /* true ||b - A x|| / ||b|| at exit */
  int32_t iterations;
  int32_t converged;
} ect_iter_result;

/* SignalPoint (signals.hpp:63-69). dz = {Z11, Z12, Z21, Z22} complex. */
typedef struct ect_signal_point {
  double z;
  double dz[8];
  double z_fa[2];
  double z_f3[2];
  int32_t failed;
  int32_t iterations[4]; /* primary coil1, coil2, reference coil1, coil2 */
} ect_signal_point;

/* Per-phase device timings (ms, CUDA events) of the last call on a context. */
typedef struct ect_timings {
  double pattern_ms;
  double assemble_ms;
  double rhs_ms;
  double solve_ms;
  /* Sampled solver kernels (ect_ctx_set_profiling): only iterations in which
   * EVERY column of the batch was still active are summed here, so that a
   * duration matches the full-width algorithmic bytes; samples taken after some
   * columns converged (cheaper launches) are counted in *_partial_launches. */
  double spmv_ms_total;   /* sum of SpMV kernel durations inside the solve */
  int64_t spmv_launches;
  int64_t kernel_launches;
  double vec_ms_total;    /* fused vector-update kernels (update + p-update) */
  int64_t vec_launches;
  int64_t spmv_partial_launches;
  int64_t vec_partial_launches;
  double precond_ms_total;  /* multigrid cycles inside the solve (sampled as the SpMV) */
  int64_t precond_launches;
} ect_timings;

/* ---- context --------------------------------------------------------- */
int ect_ctx_create(int device, ect_ctx** out);
int ect_ctx_destroy(ect_ctx* ctx);
const char* ect_last_error(void);
int ect_ctx_timings(ect_ctx* ctx, ect_timings* out, int reset);
/* Record per-launch SpMV events inside solves (adds two event records per
 * iteration; used by bench.py for the roofline figure). */
int ect_ctx_set_profiling(ect_ctx* ctx, int enabled);
int ect_ctx_synchronize(ect_ctx* ctx);
/* SpMV storage for matrices assembled on this context afterwards:
 * ECT_FORMAT_NB (default: node-block, 3x3 real blocks + diagonal imaginary
 * parts + real couplings) or ECT_FORMAT_CSR (plain complex CSR). Both give
 * the same matrix; NB moves ~40% fewer bytes per SpMV (configs[2]'s
 * storage comparison). */
#define ECT_FORMAT_NB 0
#define ECT_FORMAT_CSR 1
#define ECT_FORMAT_SELL 3     /* SELL-32-sigma (sigma = 256), configs[2]'s comparison */
int ect_ctx_set_format(ect_ctx* ctx, int format);
/* 0: CSR, 1: NB (sliced-ELL node blocks), 3: SELL-C-sigma. */
int ect_matrix_format(ect_matrix* m, int32_t* nb);
/* NB storage counts: 3x3 node blocks and conductor couplings (0 for CSR). */
int ect_matrix_nb_counts(ect_matrix* m, int64_t* blocks, int64_t* couplings);
/* Device-side timing on the context stream: record event `slot` (0..7), and
 * the elapsed ms between two recorded slots (waits for the later one). */
int ect_ctx_mark(ect_ctx* ctx, int slot);
int ect_ctx_elapsed_ms(ect_ctx* ctx, int a, int b, double* ms);

/* ---- mesh --------------------------------------------------------------
 * Replaces Mesh construction + canonicalize_orientation (mesh.cpp:50-61),
 * conductor_map (mesh.cpp:267-284) and the boundary classification that
 * apply_essential_bc pins (mesh.cpp:145-182, assembly.cpp:285-312).
 * tets: int32[n_tets*4] (reoriented in the device copy if negative),
 * region: uint8 RegionTag per tet, xyz: double[n_nodes*3]. */
int ect_mesh_create(ect_ctx* ctx, const double* xyz, int64_t n_nodes, const int32_t* tets,
                    const uint8_t* region, int64_t n_tets, ect_mesh** out);
int ect_mesh_destroy(ect_mesh* mesh);
/* counts: n_nodes, n_tets, n_cond, n_dofs (3 n_nodes + n_cond), n_pins, n_defect_tets */
int ect_mesh_counts(ect_mesh* mesh, int64_t counts[6]);
/* ConductorIndexMap::forward (mesh.hpp:81-86), pinned A-dofs ascending
 * (the std::set order of apply_essential_bc), canonical connectivity. */
int ect_mesh_export(ect_mesh* mesh, int32_t* cond_forward, int32_t* pinned_dofs, int32_t* tets);

/* ---- Gmsh ASCII v2.2 files (host only, no GPU needed) ----------------------
 * load_mesh / write_mesh (mesh_io.hpp:30-38, mesh_io.cpp:68-213) with the
 * canonical tag map (regions 1..6, boundary labels 11..15): the reader
 * canonicalises tet orientation and validates like the reference (conformity,
 * boundary labels equal to classify_boundary) -> ECT_ERR_MESH / ECT_ERR_IO with
 * "path:line: ..." messages. Feed the arrays to ect_mesh_create. */
typedef struct ect_gmsh ect_gmsh;
int ect_gmsh_read(const char* path, ect_gmsh** out);
/* counts: n_nodes, n_tets, n_boundary_faces */
int ect_gmsh_counts(ect_gmsh* g, int64_t counts[3]);
/* any pointer may be NULL; faces/labels in file order (BoundaryLabel values) */
int ect_gmsh_arrays(ect_gmsh* g, double* xyz, int32_t* tets, uint8_t* region, int32_t* faces,
                    int32_t* labels);
int ect_gmsh_destroy(ect_gmsh* g);
int ect_gmsh_write(const char* path, const double* xyz, int64_t n_nodes, const int32_t* tets,
                   const uint8_t* region, int64_t n_tets, const int32_t* faces,
                   const int32_t* labels, int64_t n_faces);

/* ---- materials (host) ---------------------------------------------------
 * RunConfig::material_table + resolve_mu_tilde (config.cpp:325-352),
 * reference_variant (materials.cpp:44-53), and ScanSession's two-config rule
 * (scan.cpp:46-49). */
int ect_materials_from_physics(ect_mesh* mesh, const ect_physics* physics, ect_materials* primary,
                               ect_materials* reference, int32_t* two_configs);
/* harmonic_mu_tilde (materials.cpp:32-42), sequential in tet order. */
int ect_harmonic_mu_tilde(ect_mesh* mesh, const ect_materials* mats, double* out);

/* ---- matrix ------------------------------------------------------------
 * K1: symbolic pattern == the CSC arrays CscMatrix::from_triplets produces
 * for build_global (sparse.cpp:83-113, assembly.cpp:386-419). The pattern is
 * structurally symmetric, so the CSR row_ptr/col_idx returned here are
 * bit-identical to the reference's col_ptr/row_idx. */
int ect_matrix_create(ect_ctx* ctx, ect_mesh* mesh, ect_matrix** out);
/* The reference's own matrix type as the input: CscMatrix {n_rows = n_cols = n,
 * col_ptr[n+1], row_idx[nnz], values[nnz]} (sparse.hpp:56-66) exactly as
 * build_global / from_triplets produce it, e.g. a GlobalSystem::matrix handed
 * to solve_iterative (solver.hpp:69-70). Transposed on the device into the
 * CSR the kernels stream (no assumption that the pattern is symmetric). A
 * value-symmetry probe (max |a_ij - a_ji| <= 1e-12 sqrt(|a_ii a_jj|) over the
 * stored pattern) decides the Krylov method: COCG for A = A^T, BiCGStab
 * otherwise (impedance surface terms make A non-symmetric). */
int ect_matrix_from_csc(ect_ctx* ctx, int64_t n, int64_t nnz, const int32_t* col_ptr,
                        const int32_t* row_idx, const double* values, ect_matrix** out);
/* Same for an external CSR (row_ptr, col_idx, values). */
int ect_matrix_from_csr(ect_ctx* ctx, int64_t n, int64_t nnz, const int32_t* row_ptr,
                        const int32_t* col_idx, const double* values, ect_matrix** out);
/* 1 if the matrix is complex symmetric (COCG), 0 if not (BiCGStab). */
int ect_matrix_symmetric(ect_matrix* m, int32_t* symmetric);
int ect_matrix_destroy(ect_matrix* m);
int ect_matrix_counts(ect_matrix* m, int64_t* n, int64_t* nnz);
/* K2: assemble_system + apply_essential_bc + build_global values
 * (assembly.cpp:74-276, 285-327, 386-419). Deterministic, no fp64 atomics. */
int ect_matrix_assemble(ect_ctx* ctx, ect_mesh* mesh, const ect_materials* mats, ect_matrix* m);
int ect_matrix_export(ect_matrix* m, int32_t* row_ptr, int32_t* col_idx, double* values);
/* The reference's own storage: CscMatrix {col_ptr, row_idx, values}
 * (sparse.hpp:55-66) of build_global. Pattern arrays equal the CSR ones;
 * values are A(row_idx[p], col) in column order — bit-identical to the
 * reference's (A is symmetric only up to rounding, so the CSR and CSC value
 * arrays are different permutations). */
int ect_matrix_export_csc(ect_matrix* m, int32_t* col_ptr, int32_t* row_idx, double* values);

/* ---- right-hand sides ----------------------------------------------------
 * K3: coil_support + assemble_rhs + apply_pins_to_rhs for n_rhs (probe z,
 * coil) pairs (tube_mesh.cpp:272-288, assembly.cpp:329-378, scan.cpp:87-93 =
 * ScanSession::position_rhs). Output column r of an interleaved
 * [n_dofs][n_rhs] complex array. */
int ect_rhs_coil(ect_ctx* ctx, ect_mesh* mesh, const ect_coil* coil, const double* probe_z,
                 const int32_t* which_coil, int32_t n_rhs, double amplitude, double* rhs);
/* assemble_rhs(mesh, support_tets, amplitude, total_dofs) (assembly.hpp:84-85,
 * assembly.cpp:335-378): caller-supplied support tets (any order, duplicates
 * allowed); NOT pinned, as the reference (use ect_apply_pins_to_rhs).
 * Errors as the reference: empty support, support in a conductor (ECT_ERR_MESH). */
int ect_rhs_support(ect_ctx* ctx, ect_mesh* mesh, const int32_t* support_tets,
                    int64_t n_support, double amplitude, double* rhs);
/* assemble_rhs(mesh, coil_tag, amplitude, total_dofs) (assembly.hpp:86-87,
 * assembly.cpp:380-384): the support is every tet of region coil_tag. */
int ect_rhs_region(ect_ctx* ctx, ect_mesh* mesh, int32_t coil_tag, double amplitude, double* rhs);
/* apply_pins_to_rhs (assembly.hpp:79, assembly.cpp:329-333) on n_rhs
 * interleaved vectors: every pinned A-dof entry = bc_penalty * 0. */
int ect_apply_pins_to_rhs(ect_ctx* ctx, ect_mesh* mesh, double* rhs, int32_t n_rhs);

/* ---- SpMV / solve --------------------------------------------------------
 * K4: y = A x (CscMatrix::multiply, sparse.cpp:115-124) for n_rhs vectors in
 * interleaved [n][n_rhs] layout. */
int ect_spmv(ect_ctx* ctx, ect_matrix* m, const double* x, double* y, int32_t n_rhs);
/* Preconditioner of the Krylov solve. ECT_PRECOND_JACOBI: point Jacobi.
 * ECT_PRECOND_AMG (default): one aggregation-multigrid W-cycle per iteration
 * (greedy node aggregation, Galerkin coarse operators with the plain transpose
 * so the preconditioner stays complex symmetric for COCG, damped-Jacobi
 * smoothing, dense coarsest solve) — the GPU replacement for the reference's
 * ILU(0) (iterative.cpp:59-105), built once per matrix. The context default
 * applies to matrices created afterwards (sessions included). */
#define ECT_PRECOND_JACOBI 0
#define ECT_PRECOND_AMG 1
int ect_ctx_set_preconditioner(ect_ctx* ctx, int32_t precond);
int ect_matrix_set_preconditioner(ect_matrix* m, int32_t precond);
/* info: levels, setup ms, operator complexity (sum nnz / fine nnz), coarsest n */
int ect_matrix_precond_info(ect_matrix* m, double info[4]);
/* K5/K6: solve_iterative (iterative.cpp:109-228) replacement: preconditioned
 * COCG (A complex symmetric; BiCGStab when it is not) for n_rhs right-hand
 * sides sharing one matrix pass per iteration; true-residual confirmation as
 * iterative.cpp:208-216. b, x interleaved [n][n_rhs]. Non-convergence is
 * reported in results (not an error), breakdown returns ECT_ERR_SOLVER. */
int ect_solve(ect_ctx* ctx, ect_matrix* m, const double* b, double* x, int32_t n_rhs,
              const ect_iter_options* opts, ect_iter_result* results);

/* ---- impedance ----------------------------------------------------------
 * K7: delta_impedance over DEFECT tets for the four (k, l) pairings of
 * primary solutions x_k (k=1,2) and reference solutions x_l (l=1,2)
 * (signals.cpp:67-99, scan.cpp:123-135). xs: 4 device-or-host vectors
 * [x_k1, x_k2, x_l1, x_l2], each n_dofs complex. dz: 8 doubles. */
int ect_delta_impedance(ect_ctx* ctx, ect_mesh* mesh, const ect_materials* primary,
                        const ect_materials* reference, const double* x_k1, const double* x_k2,
                        const double* x_l1, const double* x_l2, double* dz);

/* ---- scan session (ScanSession, scan.hpp:39-72) ---------------------------
 * Assembles the primary (+ reference) matrix once; solve_positions runs
 * solve_position (scan.cpp:95-143) for each z with the coil pair's two
 * right-hand sides batched into one COCG per material configuration. */
int ect_session_create(ect_ctx* ctx, ect_mesh* mesh, const ect_physics* physics,
                       const ect_coil* coil, double amplitude, const ect_iter_options* opts,
                       ect_session** out);
int ect_session_destroy(ect_session* s);
int ect_session_matrix(ect_session* s, int reference, ect_matrix** out);
/* positions_per_batch: probe positions whose 2*P right-hand sides share one
 * matrix pass (1..8). solutions: optional host/device buffer receiving the
 * 4 solution vectors of the LAST position ([4][n_dofs] complex) or NULL. */
int ect_session_solve_positions(ect_session* s, const double* z, int32_t n_pos,
                                int32_t positions_per_batch, ect_signal_point* out,
                                double* solutions);

/* ---- distributed solve: row partition over GPUs (SURVEY §8(e), configs[4]) --
 * A part owns a contiguous node range [splits[part], splits[part+1]) — with
 * the reference node numbering a slab of i-planes — i.e. its A-rows and the
 * V-rows of its conductor nodes. Per SpMV the ghost values are exchanged with
 * the neighbour parts (NCCL send/recv over NVLink) and each iteration's dot
 * products are summed across parts (ncclAllReduce of <= 4 n_rhs doubles).
 * Replaces nothing in the reference (its solve is serial); the paper's
 * mpiAllReduce of matrices is the closest analogue. */
typedef struct ect_halo_plan ect_halo_plan;
typedef struct ect_part ect_part;
typedef struct ect_comm ect_comm;
/* Host-only halo plan from the node neighbour lists (no GPU needed).
 * info: n0, n1, L (owned nodes), G (ghost nodes), c0 (first owned V-dof),
 * Vo, Vg (owned / ghost V-dofs), n_peers. */
int ect_halo_plan_create(int64_t n_nodes, const int32_t* nbr_off, const int32_t* nbr,
                         const int32_t* cond_fwd, const int64_t* splits, int32_t n_parts,
                         int32_t part, ect_halo_plan** out);
int ect_halo_plan_destroy(ect_halo_plan* p);
int ect_halo_plan_info(ect_halo_plan* p, int64_t info[8]);
int ect_halo_plan_arrays(ect_halo_plan* p, int32_t* ghost_nodes, int32_t* local_vdof);
/* peer info: part, recv_node_begin, recv_node_count, recv_v_begin, recv_v_count,
 * n_send_nodes, n_send_cond_nodes (+ the send lists, local node ids). */
int ect_halo_plan_peer(ect_halo_plan* p, int32_t i, int64_t info[7], int32_t* send_nodes,
                       int32_t* send_cond_nodes);
/* NCCL communicator (libnccl.so.2 loaded at run time). */
int ect_comm_unique_id(void* out128);
int ect_comm_create(ect_ctx* ctx, int32_t rank, int32_t world, const void* id128, ect_comm** out);
int ect_comm_destroy(ect_comm* c);
/* One part of an assembled (NB) global matrix on ctx's GPU. info: n0, n1, L,
 * G, Vo, Vg, n_peers, n_blocks. */
int ect_part_create(ect_ctx* ctx, ect_mesh* mesh, ect_matrix* m, const int64_t* splits,
                    int32_t n_parts, int32_t part, ect_part** out);
/* The same part without a global matrix: only the slab's rows are patterned
 * and assembled on this GPU (K1 + K2 over nodes [splits[part], splits[part+1]),
 * the reference's per-partition assembly, assembly.cpp:246-258), so device
 * memory per rank is the slab's share of the matrix. Bit-identical blocks to
 * ect_part_create on the assembled global matrix. */
int ect_part_create_assembled(ect_ctx* ctx, ect_mesh* mesh, const ect_materials* mats,
                              const int64_t* splits, int32_t n_parts, int32_t part,
                              ect_part** out);
int ect_part_destroy(ect_part* p);
int ect_part_info(ect_part* p, int64_t info[8]);
/* Partitioned Jacobi-COCG on GLOBAL b/x ([n][n_rhs]); each part reads and
 * writes its owned rows. comm == NULL: all n_parts parts live in this
 * process on one context (halo = device copies); else n_parts == 1 and the
 * halo / reductions go through NCCL. */
int ect_dist_solve(ect_part** parts, int32_t n_parts, ect_comm* comm, const double* b, double* x,
                   int32_t n_rhs, const ect_iter_options* opts, ect_iter_result* results);

#ifdef __cplusplus
}
#endif

#endif /* ECTGPU_H_ */
