/* stmg_b200 — B200-native space-time multigrid (STMG) solve, C ABI.
 *
 * This is the drop-in boundary for the reference's solver path
 * (/root/reference/proj, namespace stmg).  Each entry point names the
 * reference interface it replaces.  Plain pointers and sizes only; no C++ or
 * torch types cross this boundary.  All arithmetic is IEEE fp64.
 *
 * Errors: every int-returning function returns STMG_OK (0) or one of the
 * codes below; stmg_last_error() (thread-local) describes the last failure.
 * The three exception classes the reference throws map to
 *   std::invalid_argument -> STMG_EINVAL, std::runtime_error -> STMG_ERUNTIME,
 *   std::out_of_range -> STMG_ERANGE.
 * Non-convergence is data, not an error (stmg_solve_report.status), exactly
 * as SolveStatus in proj/include/stmg/multigrid.hpp:79.
 *
 * Threading: one hierarchy handle must not be used from two threads at once;
 * distinct handles are independent (proj/src/multigrid.cpp:228-239).
 *
 * Memory: b/u arguments of stmg_mg_solve may be host (pageable or pinned) or
 * device pointers; the kind is detected.  Level-kernel entry points take
 * device pointers to full level vectors in the reference's time-major layout
 * flat = n * (n_el + 1) + i (proj/include/stmg/mesh.hpp:46-48).
 */
#ifndef STMG_B200_H
#define STMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STMG_ABI_VERSION 4

enum stmg_status_code {
  STMG_OK = 0,
  STMG_EINVAL = 1,   /* std::invalid_argument */
  STMG_ERUNTIME = 2, /* std::runtime_error */
  STMG_ERANGE = 3,   /* std::out_of_range */
  STMG_ECUDA = 4,    /* CUDA runtime / driver failure */
  STMG_ENOMEM = 5    /* host or device allocation failure */
};

/* CoarseningDirection, proj/include/stmg/mesh.hpp:23 */
enum stmg_direction { STMG_DIR_X = 0, STMG_DIR_T = 1, STMG_DIR_XT = 2 };
/* ReassemblyMethod, proj/include/stmg/rediscretisation.hpp:36 */
enum stmg_reassembly { STMG_REASM_K = 0, STMG_REASM_D = 1, STMG_REASM_R = 2, STMG_REASM_P = 3 };
/* PlanStrategy, proj/include/stmg/strategy.hpp:74 */
enum stmg_strategy {
  STMG_PLAN_UNIFORM = 0,
  STMG_PLAN_CONTRAST = 1,
  STMG_PLAN_RESOLUTION = 2,
  STMG_PLAN_DESIGN_INDEPENDENT = 3
};
/* SolveStatus, proj/include/stmg/multigrid.hpp:79 */
enum stmg_solve_status { STMG_CONVERGED = 0, STMG_MAX_CYCLES = 1, STMG_DIVERGED = 2 };

/* SpaceTimeGrid geometry, proj/include/stmg/mesh.hpp:27-37 (dx, dt derived). */
typedef struct stmg_grid {
  double L;
  double t_T;
  int64_t n_el;
  int64_t n_t;
} stmg_grid;

/* MaterialPair, proj/include/stmg/materials.hpp:16-23 */
typedef struct stmg_material_pair {
  double k_ins, k_con, c_ins, c_con, p_k, p_c;
} stmg_material_pair;

/* PlanRequest, proj/include/stmg/strategy.hpp:76-86 (chi/mat passed separately). */
typedef struct stmg_plan_request {
  int32_t n_levels;
  double lambda_crit;
  int32_t strategy;   /* stmg_strategy */
  int32_t reassembly; /* stmg_reassembly */
  int64_t min_elements;
} stmg_plan_request;

/* SolveOptions, proj/include/stmg/multigrid.hpp:83-89 */
typedef struct stmg_solve_options {
  int32_t nu;
  double omega;
  double tol;
  double div_tol;
  int32_t max_cycles;
} stmg_solve_options;

/* SolveReport, proj/include/stmg/multigrid.hpp:91-102 (history is caller-allocated). */
typedef struct stmg_solve_report {
  int32_t status; /* stmg_solve_status */
  int32_t cycles;
  double factor;
  int32_t absolute_norms;
  int32_t n_history;           /* entries written to history (cycles + 1) */
  double seconds;              /* wall time of the solve, as SolveReport.seconds */
  double device_seconds;       /* device time between the first and last kernel (CUDA events) */
  double smoother_dof_updates; /* sum over levels and cycles of Jacobi DOF updates */
  int64_t kernel_launches;     /* kernels this solve launched (graph nodes counted) */
  /* Filled only when profiling is on (stmg_hierarchy_set_profiling): device time
   * of the finest level's kernels, measured by CUDA events inside the graph. */
  int64_t fine_sweeps;         /* plain fine-level Jacobi sweep launches timed */
  double fine_sweep_seconds;   /* their summed device time */
  int64_t fine_restricts;      /* fine-level residual+restriction launches timed */
  double fine_restrict_seconds;
  int64_t fine_prolong_sweeps; /* fused prolongation + first post-sweep launches */
  double fine_prolong_sweep_seconds;
  int64_t fine_sweep_pairs;    /* fused two-sweep (temporally blocked) launches */
  double fine_sweep_pair_seconds;
  /* the level-0 pass closing each cycle: residual norm + speculative first sweep
   * (+ the next cycle's level-0 restriction under STMG_FUSE_FINE_DOWN) */
  int64_t fine_norm_passes;
  double fine_norm_pass_seconds;
  /* the level-0 up-pass closing each cycle under STMG_FUSE_FINE_UP: prolongation +
   * post-sweep + residual norm + the next cycle's first sweep */
  int64_t fine_ups;
  double fine_up_seconds;
} stmg_solve_report;

typedef struct stmg_hierarchy stmg_hierarchy;

const char* stmg_last_error(void);
int stmg_abi_version(void);

/* ---- host-side setup (proj/src/{materials,assembly,strategy}.cpp) ---------------- */

/* apply_design, proj/include/stmg/materials.hpp:48-49 */
int stmg_apply_design(const double* chi, int64_t n, const stmg_material_pair* mat, double* k_out,
                      double* c_out);

/* load_vector(g, q), proj/include/stmg/assembly.hpp:54-56, for the preset sources
 * (kind 0 uniform, 1 mirrored box, 2 modulated mirrored box, 3 heat_load_value; see
 * paper_2505_10168_b200/configs.py); masked != 0 zeroes fixed DOFs as
 * assemble_system does (proj/src/assembly.cpp:128-130).  b is a host array of
 * (n_t+1)(n_el+1) doubles. */
int stmg_load_vector(const stmg_grid* g, int32_t kind, const double* params, int32_t masked,
                     double* b);

/* The same on the device: b is device memory of
 * (n_t+1)(n_el+1) doubles on any GPU, filled by a kernel on cuda_stream (a
 * cudaStream_t; NULL = legacy default stream), which is synchronised unless it is
 * being captured.  Kinds 0 and 1 are bit-identical to stmg_load_vector; kinds 2 and
 * 3 use the device sin / cos and agree to a few ulp. */
int stmg_load_vector_device(const stmg_grid* g, int32_t kind, const double* params, int32_t masked,
                            double* b, void* cuda_stream);

/* load_vector with a caller callback q(x, t, ctx) (the std::function overload). */
typedef double (*stmg_source_fn)(double x, double t, void* ctx);
int stmg_load_vector_cb(const stmg_grid* g, stmg_source_fn q, void* ctx, int32_t masked,
                        double* b);

/* plan_coarsening, proj/include/stmg/strategy.hpp:104-105.  k/c (n_el each) may be
 * NULL only for DesignIndependent; chi/mat are needed by D reassembly and
 * DesignIndependent.  dirs_out/indicator_out hold n_levels-1 entries. */
int stmg_plan_coarsening(const stmg_grid* g, const double* k, const double* c, const double* chi,
                         const stmg_material_pair* mat, const stmg_plan_request* req,
                         int32_t* dirs_out, double* indicator_out);

/* ---- hierarchy (proj/src/multigrid.cpp:86-160) ------------------------------------- */

/* build_hierarchy, proj/include/stmg/multigrid.hpp:70-74.  method is the reference's
 * two-letter name (parse_method, proj/src/rediscretisation.cpp:19-38): interpolation
 * C (causal) or B (bilinear, proj/src/transfer.cpp:64-68) and reassembly K, D, R or
 * P (Galerkin R J P, proj/src/rediscretisation.cpp:112-115).  dirs: n_dirs coarsening
 * directions (STMG_DIR_X / STMG_DIR_T / STMG_DIR_XT; XT is causal-only, as in
 * proj/src/transfer.cpp:44-47).  device: CUDA ordinal.  Level operators, transfers
 * and the coarsest exact solver all live on the device; no CSR matrix is formed
 * (Galerkin levels are stored as per-DOF 9-point stencils, and a Galerkin coarsest
 * level is solved by a block-tridiagonal march over dense host-factored blocks,
 * which fails with STMG_ERUNTIME beyond 4 GB of factors). */
int stmg_hierarchy_create(const stmg_grid* g, const double* k, const double* c,
                          const double* chi, const stmg_material_pair* mat, const char* method,
                          int32_t n_dirs, const int32_t* dirs, int32_t device,
                          stmg_hierarchy** out);

/* transposed_hierarchy, proj/include/stmg/multigrid.hpp:77: same levels/transfers,
 * every operator transposed (the adjoint solve). */
int stmg_hierarchy_transposed(const stmg_hierarchy* h, stmg_hierarchy** out);

void stmg_hierarchy_destroy(stmg_hierarchy* h);

int stmg_hierarchy_n_levels(const stmg_hierarchy* h, int32_t* n_levels);
int stmg_hierarchy_level_info(const stmg_hierarchy* h, int32_t level, int64_t* n_el,
                              int64_t* n_t, double* w_diri);
/* Per-node stencil coefficients of a level (host arrays of n_el+1): the row's
 * same-time (i-1, i, i+1) and other-time (i-1, i, i+1) entries and 1/diag, in the
 * hierarchy's orientation (J for primal, J^T for transposed). */
int stmg_hierarchy_level_coeffs(const stmg_hierarchy* h, int32_t level, double* cur_m,
                                double* cur_0, double* cur_p, double* oth_m, double* oth_0,
                                double* oth_p, double* inv_diag);
/* Any level's operator as a 9-point stencil in the hierarchy's orientation (host
 * arrays): v9[k * ndofs + r] is row r's entry at column (n + dn, i + di) with
 * k = 3 (dn + 1) + (di + 1), mask[r] bit k set where the reference's CSR row
 * stores that entry, inv_diag[r] = 1 / diagonal.  ndofs = (n_el + 1)(n_t + 1).
 * stmg_hierarchy_level_coeffs fails with STMG_EINVAL on a Galerkin level. */
int stmg_hierarchy_level_stencil9(const stmg_hierarchy* h, int32_t level, double* v9, uint16_t* mask,
                                  double* inv_diag);
/* Host-only form of the same (no device work): build_hierarchy's host half for
 * the given inputs, then level `level`'s operator (transposed if adjoint != 0).
 * Lets CPU-only hosts pin the Galerkin R J P build against the reference. */
int stmg_level_stencil9_host(const stmg_grid* g, const double* k, const double* c, const double* chi,
                             const stmg_material_pair* mat, const char* method, int32_t n_dirs,
                             const int32_t* dirs, int32_t level, int32_t adjoint, double* v9,
                             uint16_t* mask, double* inv_diag);
/* Run this hierarchy's work on a caller stream (cudaStream_t, NULL restores the
 * hierarchy's own stream).  Graphs are captured on a private stream and launched
 * on this one. */
int stmg_hierarchy_set_stream(stmg_hierarchy* h, void* cuda_stream);
/* Record CUDA events around kernels inside the V-cycle graph: on = 1 the finest
 * level's kernels (timings in stmg_solve_report), on = 2 every kernel of every
 * level (stmg_hierarchy_profile; adds a few us per kernel).  0 = off (default). */
int stmg_hierarchy_set_profiling(stmg_hierarchy* h, int32_t on);
/* Accumulated in-graph device time of one kernel kind on one level over all
 * profiled solves (kind: 0 sweep, 1 residual+restriction, 2 prolongation+sweep,
 * 3 fused two-sweep, 4 first sweep from zero, 5 coarsest exact solve, 6 the
 * coarse-tail cluster kernel, attributed to its first level). */
int stmg_hierarchy_profile(const stmg_hierarchy* h, int32_t level, int32_t kind, int64_t* launches,
                           double* seconds);
/* Bytes of device memory the hierarchy holds. */
int stmg_hierarchy_device_bytes(const stmg_hierarchy* h, int64_t* bytes);

/* ---- solve (proj/src/multigrid.cpp:212-279) ---------------------------------------- */

/* mg_solve, proj/include/stmg/multigrid.hpp:107-108.  u is in/out (warm start).
 * history must hold history_cap >= opts->max_cycles + 1 doubles. */
int stmg_mg_solve(stmg_hierarchy* h, const double* b, double* u, const stmg_solve_options* opts,
                  stmg_solve_report* report, double* history, int32_t history_cap);
/* The same with flags.  STMG_SOLVE_ZERO_GUESS: the initial iterate is zero and u is
 * output only -- what every reference caller outside optimise()'s warm start passes
 * (std::vector<double> u(n, 0.0): proj/tests/acceptance_main.cpp:70, proj/src/
 * experiments.cpp).  u is then neither read nor uploaded (a host u saves one of the two
 * host-to-device copies); the result equals stmg_mg_solve on a zeroed u bit for bit. */
enum { STMG_SOLVE_ZERO_GUESS = 1 };
int stmg_mg_solve_ex(stmg_hierarchy* h, const double* b, double* u, const stmg_solve_options* opts, int32_t flags,
                     stmg_solve_report* report, double* history, int32_t history_cap);

/* Independent solves run concurrently (SURVEY.md §2.2 "data parallel over
 * independent solves", §8(f) item 4 "experiment sweeps as batched replicas"):
 * entry i is mg_solve(hs[i], bs[i], us[i], opts) with reports[i] and
 * histories[i] (history_cap doubles each).  Each hierarchy works on its own
 * stream and device, so the solves overlap on one GPU and spread over several.
 * Entries must not share a workspace (no repeats, not a hierarchy together with
 * its transpose).  On failure the first failing entry's error is returned. */
int stmg_mg_solve_batch(int32_t count, stmg_hierarchy* const* hs, const double* const* bs, double* const* us,
                        const stmg_solve_options* opts, stmg_solve_report* reports, double* const* histories,
                        int32_t history_cap);

/* A stream of solves on ONE hierarchy with HOST vectors (many right-hand sides on one
 * operator: the load cases of an experiment sweep, proj/src/experiments.cpp, whose
 * solves share the hierarchy).  Entry k is stmg_mg_solve_ex(h, bs[k], us[k], opts, flags,
 * &reports[k], histories[k], history_cap), run in order, bit-identical results; the
 * host<->device copies are software-pipelined over two device (b, u) slots: b_{k+1}
 * (and u_{k+1} unless STMG_SOLVE_ZERO_GUESS) uploads and u_{k-1} downloads while solve k
 * runs, so an entry costs max(upload, solve, download) instead of their sum (config 2 on
 * PCIe 5: ~0.16 s instead of ~0.37 s).  The overlap needs page-locked host vectors
 * (cudaHostAlloc / cudaHostRegister); pageable ones work but copy synchronously.  No
 * b may alias a u.  The slots (4 level-0 vectors of device memory) are kept for the next
 * call; stmg_hierarchy_release_staging frees them.  With count == 1 or any device
 * pointer among the entries this is the plain sequence of stmg_mg_solve_ex calls. */
int stmg_mg_solve_stream(stmg_hierarchy* h, int32_t count, const double* const* bs, double* const* us,
                         const stmg_solve_options* opts, int32_t flags, stmg_solve_report* reports,
                         double* const* histories, int32_t history_cap);
int stmg_hierarchy_release_staging(stmg_hierarchy* h);

/* ---- level kernels on device vectors (parity tests, profiling) ------------------- */
/* `sweeps` damped-Jacobi sweeps in place (csr_residual + jacobi_update). */
int stmg_level_sweeps(stmg_hierarchy* h, int32_t level, const double* f, double* x,
                      int32_t sweeps, double omega);
/* Benchmark form: `launches` back-to-back kernel launches ping-ponging between
 * x and y (x -> y -> x ...), each a single sweep (fused_pairs = 0) or a fused
 * two-sweep pass (fused_pairs = 1); asynchronous on the hierarchy's stream, no
 * copies.  The iterate ends in x after an even number of launches. */
int stmg_level_sweep_kernels(stmg_hierarchy* h, int32_t level, const double* f, double* x, double* y,
                             int32_t launches, int32_t fused_pairs, double omega);
/* r = f - J_l x  (csr_residual) */
int stmg_level_residual(stmg_hierarchy* h, int32_t level, const double* f, const double* x,
                        double* r);
/* f_{l+1} = R (f - J_l x), residual recomputed on the fly (csr_residual + csr_spmv) */
int stmg_level_restrict_residual(stmg_hierarchy* h, int32_t level, const double* f,
                                 const double* x, double* f_coarse);
/* Fused V-cycle kernel forms (parity tests of the fusions; S = one damped-Jacobi
 * sweep, S(0) = 0 + omega (f * inv_diag) the first sweep from a zero iterate,
 * recomputed from f, never read from memory):
 *   STMG_FUSED_ZERO_SWEEP          y = S(S(0))
 *   STMG_FUSED_ZERO_PAIR           y = S(S(S(0)))
 *   STMG_FUSED_ZERO_RESTRICT       f_coarse = R (f - J S(0))
 *   STMG_FUSED_ZERO_PROLONG_SWEEP  y = S(S(0) + P x_coarse)
 *   STMG_FUSED_FINE_DOWN           y = S(x), f_coarse = R (f - J y), *norm2 = ||f - J x||^2
 *   STMG_FUSED_NORM_SWEEP          y = S(x), *norm2 = ||f - J x||^2 (the solve loop's norm pass)
 *   STMG_FUSED_PROLONG_SWEEP       y = S(x + P x_coarse) (the first post-smoothing sweep)
 *   STMG_FUSED_FINE_UP             y = S(x + P x_coarse), f_coarse = S(y) (a FINE-level vector here:
 *                                  the next cycle's speculative pre-sweep), *norm2 = ||f - J y||^2
 * Unused pointers may be null. */
enum {
  STMG_FUSED_ZERO_SWEEP = 0,
  STMG_FUSED_ZERO_PAIR = 1,
  STMG_FUSED_ZERO_RESTRICT = 2,
  STMG_FUSED_ZERO_PROLONG_SWEEP = 3,
  STMG_FUSED_FINE_DOWN = 4,
  STMG_FUSED_NORM_SWEEP = 5,
  STMG_FUSED_PROLONG_SWEEP = 6,
  STMG_FUSED_FINE_UP = 7
};
int stmg_level_fused(stmg_hierarchy* h, int32_t level, int32_t kind, const double* f, const double* x,
                     const double* x_coarse, double* y, double* f_coarse, double omega, double* norm2);
/* f_{l+1} = R r  (csr_spmv with R = s P^T) */
int stmg_level_restrict(stmg_hierarchy* h, int32_t level, const double* r, double* f_coarse);
/* x_l += P x_{l+1}  (csr_spmv_add) */
int stmg_level_prolong_add(stmg_hierarchy* h, int32_t level, const double* x_coarse, double* x);
/* exact solve of the coarsest level (DirectSolver::solve) */
int stmg_coarsest_solve(stmg_hierarchy* h, const double* f, double* x);
/* ||f - J_0 x||_2 on level 0 (device reduction, fixed order) */
int stmg_residual_norm(stmg_hierarchy* h, const double* f, const double* x, double* norm);
/* ||x||_2 over n doubles on the hierarchy's device */
int stmg_norm2(stmg_hierarchy* h, const double* x, int64_t n, double* norm);
int stmg_synchronize(stmg_hierarchy* h);

/* ---- topology-optimisation driver (BASELINE config 4) ---------------------------
 * optimise(), proj/src/optimisation.cpp:83-186: per iteration apply_design ->
 * plan_coarsening -> build (here: coefficients refreshed in place when the path
 * is unchanged) -> warm primal mg_solve -> objective -> adjoint mg_solve on the
 * transposed hierarchy -> sensitivities (on the GPU, the reference's
 * arithmetic) -> MMA design update (host, restating proj/src/mma.cpp). */
typedef struct stmg_optimise_options {
  stmg_material_pair mat;
  char method[4];       /* "CR" (OptimisationOptions default), "CK", "CD" */
  int32_t strategy;     /* stmg_strategy */
  int32_t n_levels;
  double lambda_crit;
  int64_t min_elements;
  int32_t warm_start;
  double volume_limit;
  double theta_ref;
  double chi_init;
  int32_t max_iterations;
  double rel_change_tol;
  int32_t stable_iterations;
  stmg_solve_options solve;
  double mma_x_min, mma_x_max, mma_move_limit, mma_asym_init, mma_asym_shrink, mma_asym_grow;
} stmg_optimise_options;

/* IterationRecord, proj/include/stmg/optimisation.hpp:77-92.  path: the coarsening
 * path used this iteration as path_to_string writes it (proj/src/strategy.cpp:118-125,
 * "x,t,..."), NUL-terminated (up to 32 directions). */
typedef struct stmg_iteration_record {
  int32_t iteration;
  double theta, volume, constraint, change;
  int32_t primal_status, adjoint_status, primal_cycles, adjoint_cycles;
  double primal_factor, adjoint_factor, primal_seconds, adjoint_seconds;
  char path[96];
} stmg_iteration_record;

/* Fills chi_out (n_el, the final post-update design), records (max_iterations),
 * and the scalars; design_history (may be NULL; max_iterations x n_el doubles):
 * row i = the design evaluated at iteration i + 1 (OptimisationResult::design_history,
 * proj/include/stmg/optimisation.hpp:100-102).  Returns STMG_OK or an error code. */
int stmg_optimise(const stmg_grid* geom, const stmg_optimise_options* opts, int32_t device,
                  double* chi_out, stmg_iteration_record* records, int32_t* n_records,
                  double* theta, int32_t* converged, double* seconds, double* design_history);

/* objective_sensitivities, proj/src/optimisation.cpp:34-73: d theta / d chi_e (before
 * the dt / theta_ref scaling of optimise) for states u and lambda ((n_t+1)(n_el+1)
 * doubles each, host or device), on `device`; bitwise the reference's arithmetic.
 * sens: host array of n_el. */
int stmg_objective_sensitivities(const stmg_grid* geom, const stmg_material_pair* mat, const double* chi,
                                 const double* u, const double* lam, double* sens, int32_t device);

/* ---- time-slab multi-GPU ------------------------------------
 * A distributed hierarchy splits the time axis of every level that can be cut
 * into `world` equal slabs (>= min_slab levels, even where the next step
 * coarsens in time) and gathers the remaining coarse levels to rank 0.  With
 * nccl_id != NULL this process is rank `rank` of an NCCL job (one GPU per
 * process; get the id with stmg_dist_nccl_unique_id on rank 0 and broadcast
 * it); with nccl_id == NULL this process hosts all `world` ranks on `device`
 * and exchanges through device copies (loopback, for validation).
 * stmg_dist_mg_solve takes full-size b and u (host or device); u receives this
 * process's slab rows of the finest level (loopback: all rows).
 * With STMG_DIST_P2P=1 in the environment at create time the ghost levels are
 * pulled straight from the neighbours' vectors over peer memory (CUDA IPC
 * mappings across processes, local pointers in loopback) behind a
 * neighbour-only epoch barrier instead of NCCL send/recv; stmg_dist_transport
 * names the exchange in use ("nccl", "loopback", "p2p"). */
typedef struct stmg_dist stmg_dist;
int stmg_dist_partition(int32_t n_levels, const int64_t* n_t, const int32_t* dirs, int32_t world,
                        int64_t min_slab, int32_t* n_distributed, int64_t* bounds);
int stmg_dist_nccl_unique_id(void* id_out, int32_t cap);
int stmg_dist_create(const stmg_grid* g, const double* k, const double* c, const double* chi,
                     const stmg_material_pair* mat, const char* method, int32_t n_dirs,
                     const int32_t* dirs, int32_t adjoint, int32_t world, int32_t rank,
                     const void* nccl_id, int32_t device, int64_t min_slab, stmg_dist** out);
int stmg_dist_info(const stmg_dist* d, int32_t* n_distributed, int64_t* row_lo, int64_t* row_hi,
                   int32_t* n_local, int64_t* device_bytes);
int stmg_dist_mg_solve(stmg_dist* d, const double* b, double* u, const stmg_solve_options* opts,
                       stmg_solve_report* report, double* history, int32_t history_cap);
/* The same solve with slab-local vectors: b_local and u_local hold only this
 * process's rows [row_lo, row_hi) of level 0 (stmg_dist_info), (row_hi - row_lo) *
 * (n_el + 1) doubles each, so the caller's memory scales as 1/W like the
 * hierarchy's; ghost rows are exchanged by the library. */
int stmg_dist_mg_solve_local(stmg_dist* d, const double* b_local, double* u_local, const stmg_solve_options* opts,
                             stmg_solve_report* report, double* history, int32_t history_cap);
int stmg_dist_transport(const stmg_dist* d, char* name_out, int32_t cap);
/* *yes = 1 when the last solve's cycle loop ran as ONE device graph (a conditional WHILE
 * node around the distributed V-cycle, the all-reduced norm and the bookkeeping kernel;
 * one launch and one read-back per solve), 0 for the host loop with a norm read-back per
 * cycle.  Default: device loop when every rank is in this process (loopback); across
 * processes (NCCL calls inside the loop body) opt in with STMG_DIST_DEVICE_LOOP=1. */
int stmg_dist_loop_on_device(const stmg_dist* d, int32_t* yes);
/* Passes captured in split form so far: with STMG_DIST_OVERLAP=<minimum slab DOFs> a level's
 * ghost exchange runs on a forked side stream while every rank's kernel runs on the interior
 * rows of its slab (no ghost level read); the first and last 16 rows follow after the join.
 * Opt-in (its benefit needs more than one GPU to measure); results are bit-identical. */
int stmg_dist_split_passes(const stmg_dist* d, int64_t* count);
void stmg_dist_destroy(stmg_dist* d);

/* Per-handle tiling of the stencil kernels (A/B measurements, tests of every
 * tile depth; not part of the reference-facing surface): levels with at most
 * tiny_dofs DOFs use 2-level time tiles, at most small_dofs 4-level tiles, the
 * rest 8-level tiles.  Values <= 0 restore the defaults (5,000,000 / 600,000).
 * Captured V-cycle graphs of the handle are rebuilt on the next solve. */
int stmg_hierarchy_set_tiling(stmg_hierarchy* h, int64_t small_dofs, int64_t tiny_dofs);
/* Per-handle V-cycle fusions (A/B measurements and bitwise tests; default
 * STMG_FUSE_DEFAULT = STMG_FUSE_VIRTUAL_ZERO | STMG_FUSE_FINE_UP, the combination measured fastest).
 * Every combination gives bit-identical iterates.
 *   STMG_FUSE_VIRTUAL_ZERO: a coarse level's first sweep from zero is recomputed
 *     from f by the kernels that read it instead of being stored and re-read;
 *   STMG_FUSE_FINE_DOWN: for nu = 1, level 0's residual norm, pre-smoothing sweep
 *     and residual restriction run as one pass over memory;
 *   STMG_FUSE_FINE_UP: for nu = 1, level 0's prolongation, post-smoothing sweep, the
 *     residual norm closing the cycle and the next cycle's pre-smoothing sweep run as
 *     one pass (36 B/DOF instead of 28 + 24; needs a third level-0 vector); takes
 *     precedence over STMG_FUSE_FINE_DOWN.
 * Captured graphs of the handle are rebuilt on the next solve. */
enum {
  STMG_FUSE_VIRTUAL_ZERO = 1,
  STMG_FUSE_FINE_DOWN = 2,
  STMG_FUSE_FINE_UP = 4,
  STMG_FUSE_ALL = 7,
  STMG_FUSE_DEFAULT = 5
};
int stmg_hierarchy_set_fusion(stmg_hierarchy* h, int32_t flags);

#ifdef __cplusplus
}
#endif
#endif /* STMG_B200_H */
