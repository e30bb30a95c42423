/* TEST INFRASTRUCTURE — CPU oracle for the STMG solve path.
 *
 * A plain-C, matrix-free restatement of the reference algorithm
 * (/root/reference/proj/src/{assembly,transfer,rediscretisation,strategy,
 * multigrid}.cpp and src/kernels/kernels.cpp) with int64 indexing, so that it
 * also covers grids the reference's int32 CSR cannot hold (BASELINE configs
 * 2/3).  Every per-row reduction follows the reference's canonical 4-lane
 * order, so smoother sweeps, residuals and transfers are bit-for-bit the
 * reference's; only the coarsest exact solve (Thomas march here, sparse LU in
 * the reference) and nothing else differs, at rounding level.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load this library.  It is the checker, never the product.
 */
#ifndef STMG_ORACLE_H
#define STMG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Directions, interpolation, reassembly, strategies: same numbering as the
 * product C-ABI (include/stmg_b200.h). */
enum { OR_DIR_X = 0, OR_DIR_T = 1, OR_DIR_XT = 2 };
enum { OR_REASM_K = 0, OR_REASM_D = 1, OR_REASM_R = 2, OR_REASM_P = 3 };
enum { OR_PLAN_UNIFORM = 0, OR_PLAN_CONTRAST = 1, OR_PLAN_RESOLUTION = 2, OR_PLAN_DESIGN_INDEPENDENT = 3 };
enum { OR_OK = 0, OR_EINVAL = 1, OR_ERUNTIME = 2, OR_ERANGE = 3, OR_ENOMEM = 5 };

typedef struct or_material {
  double k_ins, k_con, c_ins, c_con, p_k, p_c;
} or_material;

typedef struct or_hier or_hier;

const char* or_last_error(void);

/* proj/src/strategy.cpp:127-234 */
int or_plan(double L, double t_T, int64_t n_el, int64_t n_t, const double* k, const double* c,
            const double* chi, const or_material* mat, int n_levels, double lambda_crit,
            int strategy, int reassembly, int64_t min_elements, int32_t* dirs_out,
            double* indicator_out);

/* proj/src/multigrid.cpp:86-143 (+ transposed_hierarchy :145-160 when adjoint=1) */
int or_build(double L, double t_T, int64_t n_el, int64_t n_t, const double* k, const double* c,
             const double* chi, const or_material* mat, int reassembly, int n_dirs,
             const int32_t* dirs, int adjoint, or_hier** out);
void or_free(or_hier* h);
int or_n_levels(const or_hier* h);
int or_level_shape(const or_hier* h, int l, int64_t* n_el, int64_t* n_t, double* w_diri);
/* Coefficients of level l (arrays of n_el+1): W, D, E, SW, S, SE, inv_diag. */
int or_level_coeffs(const or_hier* h, int l, double* W, double* D, double* E, double* SW,
                    double* S, double* SE, double* inv_diag);

/* Kernel-level restatements on level l vectors (full, time-major). */
int or_residual(const or_hier* h, int l, const double* f, const double* x, double* r);
int or_jacobi_sweeps(const or_hier* h, int l, const double* f, double* x, int sweeps, double omega);
int or_restrict(const or_hier* h, int l, const double* r_fine, double* f_coarse);
int or_prolong_add(const or_hier* h, int l, const double* x_coarse, double* x_fine);
int or_coarsest_solve(const or_hier* h, const double* f, double* x);
double or_norm2(const double* x, int64_t n);
/* residual norms of or_mg_solve: 0 = the reference's 4-lane order (default), 1 = pairwise */
void or_set_norm_mode(int mode);
double or_dot(const double* x, const double* y, int64_t n);

/* proj/src/multigrid.cpp:212-279.  history must hold max_cycles+1 entries. */
int or_mg_solve(const or_hier* h, const double* b, double* u, int nu, double omega, double tol,
                double div_tol, int max_cycles, int* status, int* cycles, double* factor,
                int* absolute_norms, double* history, int64_t* n_history);

/* proj/src/materials.cpp:27-50 */
int or_apply_design(const double* chi, int64_t n, const or_material* mat, double* k, double* c);

/* proj/src/assembly.cpp:65-83 for the BASELINE sources (kind: see
 * paper_2505_10168_b200/configs.py), b zeroed at masked DOFs
 * (proj/src/assembly.cpp:128-130) when masked=1. */
int or_load_vector(double L, double t_T, int64_t n_el, int64_t n_t, int kind, const double* params,
                   int masked, double* b);

#ifdef __cplusplus
}
#endif
#endif
