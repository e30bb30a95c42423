/* TEST INFRASTRUCTURE — CPU oracle for the STMG solve path (see stmg_oracle.h).
 *
 * Restates, matrix-free and with int64 indices, the reference's
 *   element terms / masking / w_diri ....... proj/src/assembly.cpp:17-32, 52-57, 85-132
 *   canonical 4-lane row reduction ......... proj/src/kernels/kernels.cpp:23-46, 62-73
 *   transfers (x, causal t) ................ proj/src/transfer.cpp:35-104
 *   coarse materials (K, D, R) ............. proj/src/rediscretisation.cpp:53-110
 *   level geometry ......................... proj/src/mesh.cpp:16-42
 *   planner ................................ proj/src/strategy.cpp:9-28, 85-106, 127-234
 *   V-cycle + solve loop ................... proj/src/multigrid.cpp:184-279
 *   transposed hierarchy ................... proj/src/multigrid.cpp:145-160, sparse.cpp:74-96
 *   exact coarsest solve ................... proj/tests/oracle/oracle.cpp:38-97 (Thomas march,
 *                                            replacing Eigen SparseLU, multigrid.cpp:20-57)
 * Parity status: pinned bitwise (sweeps, residuals, transfers, load vectors) and
 * to 1e-12 (whole solves) against the compiled reference in oracle/_ref — see
 * tests/test_oracle_vs_ref.py.
 */
#include "stmg_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static __thread char g_err[512];
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}
const char* or_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ */
/* Canonical reductions (proj/src/kernels/kernels.cpp:23-46)            */
/* ------------------------------------------------------------------ */
double or_dot(const double* x, const double* y, int64_t n) {
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = 0; i < n; ++i) s[i & 3] += x[i] * y[i];
  return (s[0] + s[1]) + (s[2] + s[3]);
}
/* The solve loop's residual norms (or_mg_solve) in one of two summation orders:
 *  0: the reference's own 4-lane sequential order (or_norm2, kernels.cpp:23-31);
 *  1: pairwise -- sequential sums of 1024-entry blocks, then a binary tree over the
 *     blocks -- accurate to ~1e-13 at 1e9 entries, where the sequential order
 *     loses up to ~1e-9 (profiles/round2_norm_order.txt).  A checker mode for
 *     full-size configs; the iterates do not depend on it. */
static int g_norm_mode = 0;
void or_set_norm_mode(int mode) { g_norm_mode = mode; }

static double sumsq_pairwise(const double* x, int64_t n) {
  if (n <= 1024) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += x[i] * x[i];
    return s;
  }
  int64_t half = ((n / 2) + 1023) / 1024 * 1024;
  if (half >= n) half = n / 2;
  return sumsq_pairwise(x, half) + sumsq_pairwise(x + half, n - half);
}

double or_norm2(const double* x, int64_t n) { return sqrt(or_dot(x, x, n)); }
static double solve_norm(const double* x, int64_t n) {
  return g_norm_mode == 1 ? sqrt(sumsq_pairwise(x, n)) : or_norm2(x, n);
}

static inline double rowdot(const double* v, const double* x, int cnt) {
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int p = 0; p < cnt; ++p) s[p & 3] += v[p] * x[p];
  return (s[0] + s[1]) + (s[2] + s[3]);
}

/* ------------------------------------------------------------------ */
/* Levels                                                              */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t n_el, n_t, nn; /* nn = n_el + 1 nodes per time level */
  double L, t_T, dx, dt, w, inv_w;
  double *k, *c, *chi;
  double *W, *D, *E, *SW, *S, *SE, *inv_diag; /* per node i (index 0 unused) */
} or_level;

struct or_hier {
  int n_levels;
  int adjoint;
  int32_t* dirs;
  or_level* lv;
};

static void level_free(or_level* l) {
  free(l->k); free(l->c); free(l->chi);
  free(l->W); free(l->D); free(l->E); free(l->SW); free(l->S); free(l->SE); free(l->inv_diag);
}

/* proj/src/assembly.cpp:17-32 (element terms), :52-57 (w_diri), :99-123
 * (per-row triplets; duplicates are pairs, so summation order is moot) and
 * proj/src/multigrid.cpp:73-82 (1/diag). */
static int level_coeffs(or_level* l) {
  const int64_t ne = l->n_el, nn = ne + 1;
  double kmax = l->k[0], cmax = l->c[0];
  for (int64_t e = 1; e < ne; ++e) {
    if (l->k[e] > kmax) kmax = l->k[e];
    if (l->c[e] > cmax) cmax = l->c[e];
  }
  for (int64_t e = 0; e < ne; ++e)
    if (!(l->k[e] > 0.0) || !(l->c[e] > 0.0) || !(l->dx > 0.0))
      return fail(OR_EINVAL, "element_matrices: non-positive input");
  l->w = cmax * l->dx / l->dt + kmax / l->dx;
  l->inv_w = 1.0 / l->w;
  double** arrs[7] = {&l->W, &l->D, &l->E, &l->SW, &l->S, &l->SE, &l->inv_diag};
  for (int a = 0; a < 7; ++a) {
    *arrs[a] = (double*)calloc((size_t)nn, sizeof(double));
    if (!*arrs[a]) return fail(OR_ENOMEM, "oracle: out of memory");
  }
  for (int64_t i = 1; i <= ne; ++i) {
    /* element i-1 (local node a = 1) */
    const double kdl = l->k[i - 1] / l->dx;
    const double cdl = l->c[i - 1] * l->dx / 6.0;
    const double c11 = (2.0 * cdl) / l->dt, c10 = cdl / l->dt;
    double D = c11 + kdl;
    double S = -c11;
    l->W[i] = c10 + (-kdl);
    l->SW[i] = -c10;
    if (i <= ne - 1) { /* element i (local node a = 0) */
      const double kdr = l->k[i] / l->dx;
      const double cdr = l->c[i] * l->dx / 6.0;
      const double c00 = (2.0 * cdr) / l->dt, c01 = cdr / l->dt;
      D = D + (c00 + kdr);
      S = S + (-c00);
      l->E[i] = c01 + (-kdr);
      l->SE[i] = -c01;
    }
    l->D[i] = D;
    l->S[i] = S;
    if (D == 0.0) return fail(OR_ERUNTIME, "build_hierarchy: level operator has a zero diagonal entry");
    l->inv_diag[i] = 1.0 / D;
  }
  l->inv_diag[0] = l->inv_w;
  return OR_OK;
}

/* Row (n, i) of J (adjoint = 0) or J^T (adjoint = 1) as (values, columns)
 * in ascending-column (CSR) order; returns the entry count. */
static inline int row_entries(const or_level* l, int adjoint, int64_t n, int64_t i, double* v,
                              int64_t* col) {
  const int64_t nn = l->nn, ne = l->n_el;
  if (n == 0 || i == 0) {
    v[0] = l->w;
    col[0] = n * nn + i;
    return 1;
  }
  int p = 0;
  if (!adjoint) {
    /* columns (n-1, i-1), (n-1, i), (n-1, i+1), (n, i-1), (n, i), (n, i+1);
     * masked columns (time 0 or node 0) are dropped (assembly.cpp:115-117). */
    if (n >= 2) {
      if (i >= 2) { v[p] = l->SW[i]; col[p++] = (n - 1) * nn + i - 1; }
      v[p] = l->S[i]; col[p++] = (n - 1) * nn + i;
      if (i <= ne - 1) { v[p] = l->SE[i]; col[p++] = (n - 1) * nn + i + 1; }
    }
    if (i >= 2) { v[p] = l->W[i]; col[p++] = n * nn + i - 1; }
    v[p] = l->D[i]; col[p++] = n * nn + i;
    if (i <= ne - 1) { v[p] = l->E[i]; col[p++] = n * nn + i + 1; }
  } else {
    /* J^T row (n, i) = J column (n, i): (n, i-1) from row (n,i-1)'s E, the
     * diagonal, (n, i+1) from row (n,i+1)'s W, then the next time level's
     * SE / S / SW entries of rows (n+1, i-1), (n+1, i), (n+1, i+1). */
    if (i >= 2) { v[p] = l->E[i - 1]; col[p++] = n * nn + i - 1; }
    v[p] = l->D[i]; col[p++] = n * nn + i;
    if (i <= ne - 1) { v[p] = l->W[i + 1]; col[p++] = n * nn + i + 1; }
    if (n + 1 <= l->n_t) {
      if (i >= 2) { v[p] = l->SE[i - 1]; col[p++] = (n + 1) * nn + i - 1; }
      v[p] = l->S[i]; col[p++] = (n + 1) * nn + i;
      if (i <= ne - 1) { v[p] = l->SW[i + 1]; col[p++] = (n + 1) * nn + i + 1; }
    }
  }
  return p;
}

/* ------------------------------------------------------------------ */
/* Level passes run over time levels on host threads (OR_THREADS, default */
/* every online core, at most 64).  Each entry is computed by one thread   */
/* with the same arithmetic, so results do not depend on the thread count; */
/* reductions (norms, dots) stay sequential in the reference's order.      */
/* ------------------------------------------------------------------ */
typedef void (*range_fn)(void* ctx, int64_t lo, int64_t hi);
typedef struct {
  range_fn fn;
  void* ctx;
  int64_t lo, hi;
} par_job;
static void* par_run(void* a) {
  par_job* j = (par_job*)a;
  j->fn(j->ctx, j->lo, j->hi);
  return NULL;
}
static int n_threads(void) {
  const char* e = getenv("OR_THREADS");
  long t = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
  if (t < 1) t = 1;
  if (t > 64) t = 64;
  return (int)t;
}
static void par_for(int64_t lo, int64_t hi, int64_t work_per_item, range_fn fn, void* ctx) {
  const int64_t total = hi - lo;
  int T = n_threads();
  if (total * work_per_item < (1 << 18)) T = 1; /* small levels: not worth a thread */
  if (T > total) T = (int)(total > 0 ? total : 1);
  if (T <= 1) {
    fn(ctx, lo, hi);
    return;
  }
  pthread_t th[64];
  par_job jobs[64];
  int started[64] = {0};
  for (int t = 0; t < T; ++t) {
    jobs[t].fn = fn;
    jobs[t].ctx = ctx;
    jobs[t].lo = lo + total * t / T;
    jobs[t].hi = lo + total * (t + 1) / T;
    if (t > 0) started[t] = pthread_create(&th[t], NULL, par_run, &jobs[t]) == 0;
  }
  par_run(&jobs[0]);
  for (int t = 1; t < T; ++t) {
    if (started[t]) pthread_join(th[t], NULL);
    else par_run(&jobs[t]); /* thread creation failed: run it here */
  }
}

typedef struct {
  const or_level* l;
  const or_level* c;
  int adjoint, dir;
  double omega;
  const double *f, *x;
  double* out;
} pass_ctx;

/* proj/src/kernels/kernels.cpp:62-68 */
static void residual_rows(void* vc, int64_t lo, int64_t hi) {
  const pass_ctx* q = (const pass_ctx*)vc;
  const or_level* l = q->l;
  const int64_t nn = l->nn;
  double v[6], xv[6];
  int64_t col[6];
  for (int64_t n = lo; n < hi; ++n)
    for (int64_t i = 0; i < nn; ++i) {
      const int cnt = row_entries(l, q->adjoint, n, i, v, col);
      for (int p = 0; p < cnt; ++p) xv[p] = q->x[col[p]];
      q->out[n * nn + i] = q->f[n * nn + i] - rowdot(v, xv, cnt);
    }
}
static void residual_level(const or_level* l, int adjoint, const double* f, const double* x, double* r) {
  pass_ctx q = {l, NULL, adjoint, 0, 0.0, f, x, r};
  par_for(0, l->n_t + 1, l->nn, residual_rows, &q);
}

/* proj/src/kernels/kernels.cpp:70-73 */
static void jacobi_rows(void* vc, int64_t lo, int64_t hi) {
  const pass_ctx* q = (const pass_ctx*)vc;
  const or_level* l = q->l;
  const int64_t nn = l->nn;
  for (int64_t n = lo; n < hi; ++n)
    for (int64_t i = 0; i < nn; ++i) {
      const double id = (n == 0 || i == 0) ? l->inv_w : l->inv_diag[i];
      q->out[n * nn + i] = q->out[n * nn + i] + q->omega * (q->x[n * nn + i] * id);
    }
}
static void jacobi_level(const or_level* l, double omega, const double* r, double* x) {
  pass_ctx q = {l, NULL, 0, 0, omega, NULL, r, x};
  par_for(0, l->n_t + 1, l->nn, jacobi_rows, &q);
}

/* R = s P^T rows in ascending fine-column order (transfer.cpp:74-104). */
static void restrict_rows(void* vc, int64_t lo, int64_t hi) {
  const pass_ctx* q = (const pass_ctx*)vc;
  const or_level *fine = q->l, *coarse = q->c;
  const int dir = q->dir;
  const double* r = q->x;
  double* fc = q->out;
  const int64_t nnf = fine->nn, nnc = coarse->nn;
  double v[3], xv[3];
  for (int64_t N = lo; N < hi; ++N)
    for (int64_t I = 0; I < nnc; ++I) {
      int p = 0;
      if (dir == OR_DIR_X) {
        const int64_t i0 = 2 * I;
        if (i0 - 1 >= 0) { v[p] = 0.5; xv[p++] = r[N * nnf + i0 - 1]; }
        v[p] = 1.0; xv[p++] = r[N * nnf + i0];
        if (i0 + 1 <= fine->n_el) { v[p] = 0.5; xv[p++] = r[N * nnf + i0 + 1]; }
      } else {
        v[p] = 0.5; xv[p++] = r[(2 * N) * nnf + I];
        if (2 * N + 1 <= fine->n_t) { v[p] = 0.5; xv[p++] = r[(2 * N + 1) * nnf + I]; }
      }
      fc[N * nnc + I] = rowdot(v, xv, p);
    }
}
static void restrict_level(const or_level* fine, const or_level* coarse, int dir, const double* r,
                           double* fc) {
  pass_ctx q = {fine, coarse, 0, dir, 0.0, NULL, r, fc};
  par_for(0, coarse->n_t + 1, coarse->nn, restrict_rows, &q);
}

/* P rows (csr_spmv_add, kernels.cpp:55-60). */
static void prolong_rows(void* vc, int64_t lo, int64_t hi) {
  const pass_ctx* q = (const pass_ctx*)vc;
  const or_level *fine = q->l, *coarse = q->c;
  const int dir = q->dir;
  const double* xc = q->x;
  double* x = q->out;
  const int64_t nnf = fine->nn, nnc = coarse->nn;
  double v[2], xv[2];
  for (int64_t n = lo; n < hi; ++n)
    for (int64_t i = 0; i < nnf; ++i) {
      int p = 0;
      if (dir == OR_DIR_X) {
        if ((i & 1) == 0) { v[p] = 1.0; xv[p++] = xc[n * nnc + i / 2]; }
        else {
          v[p] = 0.5; xv[p++] = xc[n * nnc + (i - 1) / 2];
          v[p] = 0.5; xv[p++] = xc[n * nnc + (i + 1) / 2];
        }
      } else {
        v[p] = 1.0; xv[p++] = xc[(n / 2) * nnc + i];
      }
      x[n * nnf + i] = x[n * nnf + i] + rowdot(v, xv, p);
    }
}
static void prolong_add_level(const or_level* fine, const or_level* coarse, int dir, const double* xc,
                              double* x) {
  pass_ctx q = {fine, coarse, 0, dir, 0.0, NULL, xc, x};
  par_for(0, fine->n_t + 1, fine->nn, prolong_rows, &q);
}

/* Exact solve of the coarsest system.  Masked rows: x = f / w.  Unmasked
 * rows: block forward (J) or backward (J^T) march, one tridiagonal system per
 * time level, T = (W, D, E) which is symmetric (W_{i+1} == E_i bitwise); the
 * Thomas elimination follows proj/tests/oracle/oracle.cpp:19-34. */
static int coarsest_level(const or_level* l, int adjoint, const double* f, double* x) {
  const int64_t nn = l->nn, ne = l->n_el, nt = l->n_t;
  for (int64_t n = 0; n <= nt; ++n) x[n * nn] = f[n * nn] / l->w;
  for (int64_t i = 1; i < nn; ++i) x[i] = f[i] / l->w;
  if (ne < 1 || nt < 1) return OR_OK;
  double* cp = (double*)malloc(sizeof(double) * (size_t)nn);
  double* rhs = (double*)malloc(sizeof(double) * (size_t)nn);
  if (!cp || !rhs) { free(cp); free(rhs); return fail(OR_ENOMEM, "oracle: out of memory"); }
  for (int64_t s = 1; s <= nt; ++s) {
    const int64_t n = adjoint ? nt + 1 - s : s;
    const int64_t m = adjoint ? n + 1 : n - 1; /* coupled time level */
    const int coupled = adjoint ? (m <= nt) : (m >= 1);
    for (int64_t i = 1; i <= ne; ++i) {
      double acc = f[n * nn + i];
      if (coupled) {
        if (!adjoint) {
          if (i >= 2) acc -= l->SW[i] * x[m * nn + i - 1];
          acc -= l->S[i] * x[m * nn + i];
          if (i <= ne - 1) acc -= l->SE[i] * x[m * nn + i + 1];
        } else {
          if (i >= 2) acc -= l->SE[i - 1] * x[m * nn + i - 1];
          acc -= l->S[i] * x[m * nn + i];
          if (i <= ne - 1) acc -= l->SW[i + 1] * x[m * nn + i + 1];
        }
      }
      rhs[i] = acc;
    }
    /* Thomas on rows 1..ne: lower_i = W_i (i>=2), diag_i = D_i, upper_i = E_i (i<=ne-1) */
    double piv = l->D[1];
    cp[1] = (ne >= 2 ? l->E[1] : 0.0) / piv;
    x[n * nn + 1] = rhs[1] / piv;
    for (int64_t i = 2; i <= ne; ++i) {
      piv = l->D[i] - l->W[i] * cp[i - 1];
      if (piv == 0.0) { free(cp); free(rhs); return fail(OR_ERUNTIME, "coarsest: zero pivot"); }
      cp[i] = (i <= ne - 1 ? l->E[i] : 0.0) / piv;
      x[n * nn + i] = (rhs[i] - l->W[i] * x[n * nn + i - 1]) / piv;
    }
    for (int64_t i = ne - 1; i >= 1; --i) x[n * nn + i] -= cp[i] * x[n * nn + i + 1];
  }
  free(cp);
  free(rhs);
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Materials, coarsening, planning                                     */
/* ------------------------------------------------------------------ */
static int check_material(const or_material* m) {
  if (m->k_ins <= 0.0 || m->k_con <= 0.0 || m->c_ins <= 0.0 || m->c_con <= 0.0)
    return fail(OR_EINVAL, "material properties must be positive");
  if (m->p_k <= 0.0 || m->p_c <= 0.0) return fail(OR_EINVAL, "penalisation exponents must be positive");
  return OR_OK;
}

/* proj/src/materials.cpp:27-32, 44-50 */
int or_apply_design(const double* chi, int64_t n, const or_material* mat, double* k, double* c) {
  int rc = check_material(mat);
  if (rc) return rc;
  for (int64_t e = 0; e < n; ++e) {
    if (!(chi[e] >= 0.0 && chi[e] <= 1.0)) return fail(OR_EINVAL, "volume fraction outside [0, 1]");
    k[e] = mat->k_ins + (mat->k_con - mat->k_ins) * pow(chi[e], mat->p_k);
    c[e] = mat->c_ins + (mat->c_con - mat->c_ins) * pow(chi[e], mat->p_c);
  }
  return OR_OK;
}

/* proj/src/rediscretisation.cpp:53-110 (x step; t step copies). */
static int coarsen_materials_x(int64_t ne, const double* k, const double* c, const double* chi,
                               const or_material* mat, int reassembly, double* kc, double* cc,
                               double* chic) {
  const int64_t nc = ne / 2;
  if (reassembly == OR_REASM_D) {
    if (!chi || !mat) return fail(OR_EINVAL, "coarsen_materials: D method needs the design field and materials");
    for (int64_t e = 0; e < nc; ++e) chic[e] = 0.5 * (chi[2 * e] + chi[2 * e + 1]);
    return or_apply_design(chic, nc, mat, kc, cc);
  }
  for (int64_t e = 0; e < nc; ++e) {
    const double a = k[2 * e], b = k[2 * e + 1];
    if (reassembly == OR_REASM_R) kc[e] = 2.0 * a * b / (a + b);
    else kc[e] = 0.5 * (a + b);
    cc[e] = 0.5 * (c[2 * e] + c[2 * e + 1]);
  }
  return OR_OK;
}

/* proj/src/strategy.cpp:9-21 (lambda_eff of a level) */
static double lambda_eff(int64_t ne, const double* k, const double* c, double dx, double dt) {
  const double scale = dt / (dx * dx);
  double lo = 0.0, hi = 0.0;
  for (int64_t e = 0; e < ne; ++e) {
    const double le = (k[e] / c[e]) * scale;
    if (e == 0 || le < lo) lo = le;
    if (e == 0 || le > hi) hi = le;
  }
  return sqrt(lo * hi);
}

/* proj/src/strategy.cpp:85-106 */
static int design_independent_diffusivity(const or_material* mat, double* out) {
  const double d0 = mat->k_ins / mat->c_ins, d1 = mat->k_con / mat->c_con;
  const double lo = d0 < d1 ? d0 : d1, hi = d0 < d1 ? d1 : d0;
  for (int i = 0; i < 1001; ++i) {
    const double chi = (double)i / (1001 - 1);
    int rc = check_material(mat);
    if (rc) return rc;
    const double k = mat->k_ins + (mat->k_con - mat->k_ins) * pow(chi, mat->p_k);
    const double c = mat->c_ins + (mat->c_con - mat->c_ins) * pow(chi, mat->p_c);
    const double d = k / c;
    if (d < lo * (1.0 - 1e-9) || d > hi * (1.0 + 1e-9))
      return fail(OR_EINVAL, "design_independent_diffusivity: interpolated diffusivity has an interior extremum");
  }
  *out = sqrt(d0 * d1);
  return OR_OK;
}

int or_plan(double L, double t_T, int64_t n_el, int64_t n_t, const double* k, const double* c,
            const double* chi, const or_material* mat, int n_levels, double lambda_crit,
            int strategy, int reassembly, int64_t min_elements, int32_t* dirs_out,
            double* indicator_out) {
  if (n_levels < 1) return fail(OR_EINVAL, "plan_coarsening: need at least one level");
  if (lambda_crit <= 0.0) return fail(OR_EINVAL, "plan_coarsening: lambda_crit must be positive");
  if (L <= 0.0 || t_T <= 0.0 || n_el <= 0 || n_t <= 0) return fail(OR_EINVAL, "build_fine_grid: bad grid");
  double fixed_d = 0.0;
  int rc;
  if (strategy == OR_PLAN_DESIGN_INDEPENDENT) {
    if (!mat) return fail(OR_EINVAL, "plan_coarsening: design-independent planning needs the material pair");
    if ((rc = design_independent_diffusivity(mat, &fixed_d))) return rc;
  } else if (!k || !c) {
    return fail(OR_EINVAL, "plan_coarsening: grid has no materials");
  }
  const int track_chi = reassembly == OR_REASM_D && strategy != OR_PLAN_DESIGN_INDEPENDENT;
  if (track_chi && (!chi || !mat))
    return fail(OR_EINVAL, "plan_coarsening: D reassembly needs the design field and materials");

  int64_t ne = n_el, nt = n_t;
  double *lk = NULL, *lc = NULL, *lchi = NULL;
  if (strategy != OR_PLAN_DESIGN_INDEPENDENT) {
    lk = (double*)malloc(sizeof(double) * (size_t)ne);
    lc = (double*)malloc(sizeof(double) * (size_t)ne);
    memcpy(lk, k, sizeof(double) * (size_t)ne);
    memcpy(lc, c, sizeof(double) * (size_t)ne);
    if (track_chi) {
      lchi = (double*)malloc(sizeof(double) * (size_t)ne);
      memcpy(lchi, chi, sizeof(double) * (size_t)ne);
    }
  }
  rc = OR_OK;
  for (int l = 1; l < n_levels; ++l) {
    const double dx = L / (double)ne, dt = t_T / (double)nt;
    double lambda = 0.0;
    if (strategy == OR_PLAN_UNIFORM) {
      for (int64_t e = 1; e < ne; ++e)
        if (lk[e] != lk[0] || lc[e] != lc[0]) { rc = fail(OR_EINVAL, "plan_coarsening: uniform strategy on non-uniform materials"); goto done; }
      lambda = (lk[0] / lc[0]) * dt / (dx * dx);
    } else if (strategy == OR_PLAN_CONTRAST || strategy == OR_PLAN_RESOLUTION) {
      lambda = lambda_eff(ne, lk, lc, dx, dt);
    } else {
      lambda = fixed_d * dt / (dx * dx);
    }
    const int guard = strategy == OR_PLAN_RESOLUTION && ne / 2 < min_elements;
    const int want_time = lambda < lambda_crit || guard;
    const int x_ok = ne % 2 == 0 && ne >= 2, t_ok = nt % 2 == 0 && nt >= 2;
    int dir;
    if (want_time) {
      if (t_ok) dir = OR_DIR_T;
      else if (guard) { rc = fail(OR_ERUNTIME, "plan_coarsening: forced time-coarsening impossible and the element floor forbids space-coarsening"); goto done; }
      else if (x_ok) dir = OR_DIR_X;
      else { rc = fail(OR_ERUNTIME, "plan_coarsening: no legal coarsening step"); goto done; }
    } else {
      if (x_ok) dir = OR_DIR_X;
      else if (t_ok) dir = OR_DIR_T;
      else { rc = fail(OR_ERUNTIME, "plan_coarsening: no legal coarsening step"); goto done; }
    }
    dirs_out[l - 1] = dir;
    if (indicator_out) indicator_out[l - 1] = lambda;
    if (dir == OR_DIR_X) {
      if (strategy != OR_PLAN_DESIGN_INDEPENDENT) {
        const int64_t nc = ne / 2;
        double* kc = (double*)malloc(sizeof(double) * (size_t)nc);
        double* cc = (double*)malloc(sizeof(double) * (size_t)nc);
        double* chic = track_chi ? (double*)malloc(sizeof(double) * (size_t)nc) : NULL;
        rc = coarsen_materials_x(ne, lk, lc, lchi, mat, reassembly, kc, cc, chic);
        free(lk); free(lc); free(lchi);
        lk = kc; lc = cc; lchi = chic;
        if (rc) goto done;
      }
      ne /= 2;
    } else {
      nt /= 2;
    }
  }
done:
  free(lk); free(lc); free(lchi);
  return rc;
}

/* ------------------------------------------------------------------ */
/* Hierarchy                                                           */
/* ------------------------------------------------------------------ */
void or_free(or_hier* h) {
  if (!h) return;
  for (int l = 0; l < h->n_levels; ++l) level_free(&h->lv[l]);
  free(h->lv);
  free(h->dirs);
  free(h);
}

int or_build(double L, double t_T, int64_t n_el, int64_t n_t, const double* k, const double* c,
             const double* chi, const or_material* mat, int reassembly, int n_dirs,
             const int32_t* dirs, int adjoint, or_hier** out) {
  *out = NULL;
  if (L <= 0.0 || t_T <= 0.0) return fail(OR_EINVAL, "build_fine_grid: non-positive extent");
  if (n_el <= 0 || n_t <= 0) return fail(OR_EINVAL, "build_fine_grid: non-positive count");
  if (!k || !c) return fail(OR_EINVAL, "build_hierarchy: fine grid has no materials");
  if (reassembly == OR_REASM_P) return fail(OR_EINVAL, "oracle: Galerkin (P) reassembly is out of scope");
  if (reassembly == OR_REASM_D && (!chi || !mat))
    return fail(OR_EINVAL, "build_hierarchy: D reassembly needs the design field and materials");
  or_hier* h = (or_hier*)calloc(1, sizeof(or_hier));
  h->n_levels = n_dirs + 1;
  h->adjoint = adjoint;
  h->dirs = (int32_t*)calloc((size_t)(n_dirs + 1), sizeof(int32_t));
  h->lv = (or_level*)calloc((size_t)h->n_levels, sizeof(or_level));
  if (n_dirs) memcpy(h->dirs, dirs, sizeof(int32_t) * (size_t)n_dirs);
  int rc = OR_OK;
  for (int l = 0; l < h->n_levels; ++l) {
    or_level* lv = &h->lv[l];
    lv->L = L;
    lv->t_T = t_T;
    if (l == 0) {
      lv->n_el = n_el;
      lv->n_t = n_t;
      lv->k = (double*)malloc(sizeof(double) * (size_t)n_el);
      lv->c = (double*)malloc(sizeof(double) * (size_t)n_el);
      memcpy(lv->k, k, sizeof(double) * (size_t)n_el);
      memcpy(lv->c, c, sizeof(double) * (size_t)n_el);
      if (chi) {
        lv->chi = (double*)malloc(sizeof(double) * (size_t)n_el);
        memcpy(lv->chi, chi, sizeof(double) * (size_t)n_el);
      }
    } else {
      const or_level* p = &h->lv[l - 1];
      const int dir = h->dirs[l - 1];
      if (dir != OR_DIR_X && dir != OR_DIR_T) { rc = fail(OR_EINVAL, "oracle: FullST coarsening is out of scope"); break; }
      const int hx = dir == OR_DIR_X;
      if ((hx && p->n_el % 2) || (!hx && p->n_t % 2)) { rc = fail(OR_EINVAL, "coarsen_grid: odd count"); break; }
      if ((hx && p->n_el < 2) || (!hx && p->n_t < 2)) { rc = fail(OR_EINVAL, "coarsen_grid: grid too small to coarsen"); break; }
      lv->n_el = hx ? p->n_el / 2 : p->n_el;
      lv->n_t = hx ? p->n_t : p->n_t / 2;
      lv->k = (double*)malloc(sizeof(double) * (size_t)lv->n_el);
      lv->c = (double*)malloc(sizeof(double) * (size_t)lv->n_el);
      if (p->chi) lv->chi = (double*)malloc(sizeof(double) * (size_t)lv->n_el);
      if (hx) {
        rc = coarsen_materials_x(p->n_el, p->k, p->c, p->chi, mat, reassembly, lv->k, lv->c, lv->chi);
        if (rc) break;
      } else {
        memcpy(lv->k, p->k, sizeof(double) * (size_t)lv->n_el);
        memcpy(lv->c, p->c, sizeof(double) * (size_t)lv->n_el);
        if (p->chi) memcpy(lv->chi, p->chi, sizeof(double) * (size_t)lv->n_el);
      }
    }
    lv->nn = lv->n_el + 1;
    lv->dx = L / (double)lv->n_el;
    lv->dt = t_T / (double)lv->n_t;
    if ((rc = level_coeffs(lv))) break;
  }
  if (rc) { or_free(h); return rc; }
  *out = h;
  return OR_OK;
}

int or_n_levels(const or_hier* h) { return h->n_levels; }

int or_level_shape(const or_hier* h, int l, int64_t* n_el, int64_t* n_t, double* w) {
  if (l < 0 || l >= h->n_levels) return fail(OR_ERANGE, "level out of range");
  *n_el = h->lv[l].n_el;
  *n_t = h->lv[l].n_t;
  if (w) *w = h->lv[l].w;
  return OR_OK;
}

int or_level_coeffs(const or_hier* h, int l, double* W, double* D, double* E, double* SW, double* S,
                    double* SE, double* inv_diag) {
  if (l < 0 || l >= h->n_levels) return fail(OR_ERANGE, "level out of range");
  const or_level* lv = &h->lv[l];
  const size_t bytes = sizeof(double) * (size_t)lv->nn;
  memcpy(W, lv->W, bytes); memcpy(D, lv->D, bytes); memcpy(E, lv->E, bytes);
  memcpy(SW, lv->SW, bytes); memcpy(S, lv->S, bytes); memcpy(SE, lv->SE, bytes);
  memcpy(inv_diag, lv->inv_diag, bytes);
  return OR_OK;
}

static int64_t ndofs(const or_level* l) { return (l->n_t + 1) * l->nn; }

int or_residual(const or_hier* h, int l, const double* f, const double* x, double* r) {
  if (l < 0 || l >= h->n_levels) return fail(OR_ERANGE, "level out of range");
  residual_level(&h->lv[l], h->adjoint, f, x, r);
  return OR_OK;
}

int or_jacobi_sweeps(const or_hier* h, int l, const double* f, double* x, int sweeps, double omega) {
  if (l < 0 || l >= h->n_levels) return fail(OR_ERANGE, "level out of range");
  double* r = (double*)malloc(sizeof(double) * (size_t)ndofs(&h->lv[l]));
  if (!r) return fail(OR_ENOMEM, "oracle: out of memory");
  for (int s = 0; s < sweeps; ++s) {
    residual_level(&h->lv[l], h->adjoint, f, x, r);
    jacobi_level(&h->lv[l], omega, r, x);
  }
  free(r);
  return OR_OK;
}

int or_restrict(const or_hier* h, int l, const double* r_fine, double* f_coarse) {
  if (l < 0 || l + 1 >= h->n_levels) return fail(OR_ERANGE, "level out of range");
  restrict_level(&h->lv[l], &h->lv[l + 1], h->dirs[l], r_fine, f_coarse);
  return OR_OK;
}

int or_prolong_add(const or_hier* h, int l, const double* x_coarse, double* x_fine) {
  if (l < 0 || l + 1 >= h->n_levels) return fail(OR_ERANGE, "level out of range");
  prolong_add_level(&h->lv[l], &h->lv[l + 1], h->dirs[l], x_coarse, x_fine);
  return OR_OK;
}

int or_coarsest_solve(const or_hier* h, const double* f, double* x) {
  return coarsest_level(&h->lv[h->n_levels - 1], h->adjoint, f, x);
}

/* ------------------------------------------------------------------ */
/* V-cycle and solve loop (proj/src/multigrid.cpp:178-279)              */
/* ------------------------------------------------------------------ */
typedef struct {
  double **f, **x, **r;
} workspace;

static int v_cycle(const or_hier* h, int l, const double* f, double* x, workspace* ws, int nu,
                   double omega) {
  if (l == h->n_levels - 1) return coarsest_level(&h->lv[l], h->adjoint, f, x);
  const or_level* lv = &h->lv[l];
  double* r = ws->r[l];
  for (int s = 0; s < nu; ++s) {
    residual_level(lv, h->adjoint, f, x, r);
    jacobi_level(lv, omega, r, x);
  }
  residual_level(lv, h->adjoint, f, x, r);
  restrict_level(lv, &h->lv[l + 1], h->dirs[l], r, ws->f[l + 1]);
  memset(ws->x[l + 1], 0, sizeof(double) * (size_t)ndofs(&h->lv[l + 1]));
  int rc = v_cycle(h, l + 1, ws->f[l + 1], ws->x[l + 1], ws, nu, omega);
  if (rc) return rc;
  prolong_add_level(lv, &h->lv[l + 1], h->dirs[l], ws->x[l + 1], x);
  for (int s = 0; s < nu; ++s) {
    residual_level(lv, h->adjoint, f, x, r);
    jacobi_level(lv, omega, r, x);
  }
  return OR_OK;
}

int or_mg_solve(const or_hier* h, const double* b, double* u, int nu, double omega, double tol,
                double div_tol, int max_cycles, int* status, int* cycles, double* factor,
                int* absolute_norms, double* history, int64_t* n_history) {
  if (nu < 0 || omega <= 0.0 || tol <= 0.0 || div_tol <= tol || max_cycles < 0)
    return fail(OR_EINVAL, "mg_solve: invalid options");
  const int nl = h->n_levels;
  workspace ws;
  ws.f = (double**)calloc((size_t)nl, sizeof(double*));
  ws.x = (double**)calloc((size_t)nl, sizeof(double*));
  ws.r = (double**)calloc((size_t)nl, sizeof(double*));
  int rc = OR_OK;
  for (int l = 0; l < nl; ++l) {
    const size_t nd = (size_t)ndofs(&h->lv[l]);
    ws.r[l] = (double*)malloc(sizeof(double) * nd);
    if (l > 0) {
      ws.f[l] = (double*)malloc(sizeof(double) * nd);
      ws.x[l] = (double*)malloc(sizeof(double) * nd);
    }
    if (!ws.r[l] || (l > 0 && (!ws.f[l] || !ws.x[l]))) { rc = fail(OR_ENOMEM, "oracle: out of memory"); goto out; }
  }
  {
    const int64_t n = ndofs(&h->lv[0]);
    const double norm_b = solve_norm(b, n);
    *absolute_norms = norm_b == 0.0;
    const double denom = *absolute_norms ? 1.0 : norm_b;
    residual_level(&h->lv[0], h->adjoint, b, u, ws.r[0]);
    const double r0 = solve_norm(ws.r[0], n) / denom;
    int64_t nh = 0;
    history[nh++] = r0;
    *cycles = 0;
    *factor = 1.0;
    if (r0 < tol) {
      *status = 0;
      *n_history = nh;
      goto out;
    }
    *status = 1;
    for (int cyc = 1; cyc <= max_cycles; ++cyc) {
      if ((rc = v_cycle(h, 0, b, u, &ws, nu, omega))) goto out;
      residual_level(&h->lv[0], h->adjoint, b, u, ws.r[0]);
      const double rn = solve_norm(ws.r[0], n) / denom;
      history[nh++] = rn;
      *cycles = cyc;
      if (rn < tol) { *status = 0; break; }
      if (!isfinite(rn) || rn > div_tol) { *status = 2; break; }
    }
    if (*cycles > 0) *factor = pow(history[nh - 1] / r0, 1.0 / *cycles);
    *n_history = nh;
  }
out:
  for (int l = 0; l < nl; ++l) { free(ws.f[l]); free(ws.x[l]); free(ws.r[l]); }
  free(ws.f); free(ws.x); free(ws.r);
  return rc;
}

/* ------------------------------------------------------------------ */
/* Load vectors (proj/src/assembly.cpp:59-83, 128-130)                  */
/* ------------------------------------------------------------------ */
static double source_value(int kind, const double* p, double x, double t, double L, double t_T) {
  switch (kind) {
    case 0: return p[0];                                               /* uniform q */
    case 1: return (L - x < p[1]) ? p[0] : 0.0;                        /* mirrored box */
    case 2: return (L - x < p[2]) ? 1.0 + p[0] * sin(2.0 * M_PI * p[1] * t) : 0.0;
    case 3: {                                                          /* heat_load_value */
      const double xs = x / L - 0.5, ts = t / t_T - 0.5;
      return (1.0 + cos(200.0 * (xs * xs + ts * ts))) * 1.0e6;
    }
  }
  return NAN;
}

typedef struct {
  double L, t_T, dx, dt;
  int64_t n_el;
  int kind;
  const double* params;
  double* b;
} load_ctx;
/* time levels [lo, hi) of proj/src/assembly.cpp:65-83 (each level independent) */
static void load_rows(void* vc, int64_t lo, int64_t hi) {
  const load_ctx* q = (const load_ctx*)vc;
  const int64_t nn = q->n_el + 1;
  for (int64_t n = lo; n < hi; ++n) {
    if (n == 0) continue;
    const double t = (double)n * q->dt;
    double* row = q->b + n * nn;
    for (int64_t e = 0; e < q->n_el; ++e) {
      const double qe = source_value(q->kind, q->params, ((double)e + 0.5) * q->dx, t, q->L, q->t_T) * q->dx / 2.0;
      row[e] += qe;
      row[e + 1] += qe;
    }
  }
}

int or_load_vector(double L, double t_T, int64_t n_el, int64_t n_t, int kind, const double* params,
                   int masked, double* b) {
  if (kind < 0 || kind > 3) return fail(OR_EINVAL, "load_vector: unknown source kind");
  const int64_t nn = n_el + 1;
  const double dx = L / (double)n_el, dt = t_T / (double)n_t;
  memset(b, 0, sizeof(double) * (size_t)((n_t + 1) * nn));
  load_ctx q = {L, t_T, dx, dt, n_el, kind, params, b};
  par_for(0, n_t + 1, nn, load_rows, &q);
  if (masked) {
    for (int64_t i = 0; i < nn; ++i) b[i] = 0.0;
    for (int64_t n = 1; n <= n_t; ++n) b[n * nn] = 0.0;
  }
  return OR_OK;
}
