// Internal definitions shared by the sm_100a kernels and the host orchestration.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace stmgb {

// Device view of one level's operator.  The stencil of row (n, i) is stored
// per node i in the row's own orientation (J for a primal hierarchy, J^T for a
// transposed one), so kernels never index i-1/i+1 coefficient arrays:
//   cm, c0, cp : same-time-level entries at columns i-1, i, i+1
//   om, o0, op : other-time-level entries (n-1 for J, n+1 for J^T) at i-1, i, i+1
// Masked rows (n == 0 || i == 0) have the single diagonal w
// (proj/src/assembly.cpp:85-88, 122-123).
struct LevelView {
  int64_t n_el;
  int64_t n_t;
  int64_t nn;  // n_el + 1 nodes per time level
  double w;
  double inv_w;
  const double* coef;  // 7 * nn: cm, c0, cp, om, o0, op, inv_diag
  // Rows (time levels) a launch computes: [n_lo, n_hi).  The full level is
  // [0, n_t + 1); a time slab of a distributed level is a sub-range (vectors
  // stay full-size and globally indexed; only the slab is read and written).
  int64_t n_lo;
  int64_t n_hi;
  // Time levels per tile of the overlapping-warp kernels (8, or 4 / 2 on small,
  // latency-bound levels); fixed when the hierarchy is built.
  int64_t tile_nt = 8;
};

inline bool full_range(const LevelView& L) { return L.n_lo == 0 && L.n_hi == L.n_t + 1; }

enum Coef { kCm = 0, kC0 = 1, kCp = 2, kOm = 3, kO0 = 4, kOp = 5, kInvD = 6, kNumCoef = 7 };

// PCR tables for the exact coarsest solve (per tridiagonal step system of the
// unmasked nodes 1..n_el, identical on every time level).
struct CoarsestView {
  LevelView lv;
  int32_t m;            // n_el unmasked nodes per time level
  int32_t n_steps;      // ceil(log2(m))
  const double* alpha;  // n_steps * m
  const double* gamma;  // n_steps * m
  const double* bfin;   // m, final diagonal after reduction
  // n_el <= 32: dense step inverse T^-1 and propagator A = -T^-1 S (32 x 32,
  // column-major, zero-padded), for the parallel-RHS + propagator march
  const double* tinv;
  const double* prop;
  // chunked (parallel-in-time) march: n_t = n_chunks * chunk_len, A^chunk_len
  int32_t n_chunks;
  int32_t chunk_len;
  const double* prop_chunk;
  // n_el > 32 (wide coarsest levels, e.g. config 4's 256 x 8192): parallel-in-time
  // march over pint_chunks chunks of pint_len steps, one CTA per chunk, linked by
  // a log-depth scan with the powers Q^(2^r), Q = A^pint_len (pint_rounds m x m
  // column-major matrices, contiguous); 0 chunks = sequential march.
  int32_t pint_chunks;
  int32_t pint_len;
  int32_t pint_rounds;
  const double* pint_pow;
};
// Kernel launches one coarsest solve issues (the parallel-in-time march: the
// chunk marches, one launch per scan round, the chunk corrections).
inline int coarsest_launches(const CoarsestView& cv) {
  return cv.m > 32 && cv.pint_chunks > 1 ? 2 + cv.pint_rounds : 1;
}
// Scratch doubles the coarsest solve needs (two buffers of chunk end states).
inline int64_t coarsest_scratch(const CoarsestView& cv) {
  return cv.m > 32 && cv.pint_chunks > 1 ? 2 * (int64_t)cv.pint_chunks * cv.m : 0;
}

// Shared memory of the chunked coarsest march: g (n_t x 32), chunk end and
// start states (2 C + 1) x 32, one 32-double vector slot per warp (<= 16).
inline size_t coarsest_chunked_smem(const CoarsestView& cv) {
  return sizeof(double) * 32 * ((size_t)cv.lv.n_t + 2 * (size_t)cv.n_chunks + 1 + 16);
}

// ---- general coarse discretisations (stmg_general.cu) ------------------------------
// Per-DOF 9-point operator of a Galerkin (R J P) level, in the hierarchy's row
// orientation: slot k = 3 (dn + 1) + (di + 1) holds the entry at column
// (n + dn, i + di); mask bit k is set where the reference's CSR row stores it.
struct Dia9View {
  int64_t n_el;
  int64_t n_t;
  int64_t nn;
  const double* v;         // 9 * ndofs, slot-major: v[k * ndofs + r]
  const uint16_t* mask;    // ndofs
  const double* inv_diag;  // ndofs
};
// One transfer (level l fine, l + 1 coarse), proj/src/transfer.cpp:39-104.
struct XferView {
  int64_t f_nn, f_nt, c_nn, c_nt;
  int dir;       // 0 x, 1 t, 2 x and t (FullST)
  int bilinear;  // temporal stencil: 0 causal, 1 bilinear
};
// Exact block-tridiagonal solve of a Galerkin coarsest level.
struct BlockMarchView {
  int64_t m;    // nodes per time level (n_el + 1)
  int64_t n_t;
  const double* G;  // (n_t + 1) column-major m x m blocks M_n^-1
  const double* H;  // n_t blocks M_n^-1 C_n (null when the operator is causal)
  int has_upper;
  Dia9View A;  // dn = -1 slots
};
int launch_g_sweep(const Dia9View& A, const double* f, const double* x, double* y, double omega,
                   cudaStream_t s);
int launch_g_residual(const Dia9View& A, const double* f, const double* x, double* r, cudaStream_t s);
int launch_g_from_zero(const Dia9View& A, const double* f, double* y, double omega, cudaStream_t s);
int launch_xfer_restrict(const XferView& T, const double* r, double* fc, cudaStream_t s);
// y = x + P xc (y may alias x)
int launch_xfer_prolong_add(const XferView& T, const double* xc, const double* x, double* y,
                            cudaStream_t s);
int launch_block_march(const BlockMarchView& B, const double* f, double* x, cudaStream_t s);
// Device-side state of a solve loop run as a conditional WHILE graph node.
struct SolveLoopCtl {
  double tol;
  double div_tol;
  int32_t max_cycles;
  int32_t cycles;  // V-cycles done
  int32_t status;  // stmg_solve_status
  int32_t pad;
};
// One cycle's bookkeeping (history, status) and the loop's continue flag.
int launch_cycle_check(const double* scalars, SolveLoopCtl* ctl, double* hist,
                       cudaGraphConditionalHandle handle, cudaStream_t s);
// launch_finalize_sum(partials, n, scalars + 1) and launch_cycle_check in one
// kernel (same summation order, so the same bits).
int launch_finalize_check(const double* partials, int64_t n, double* scalars, SolveLoopCtl* ctl, double* hist,
                          cudaGraphConditionalHandle handle, cudaStream_t s);
#ifdef __CUDACC__
// mg_solve's per-cycle bookkeeping (proj/src/multigrid.cpp:260-273) from the
// squared norms ||b||^2 and ||b - J u||^2; sqrt is correctly rounded, so rn
// equals the host loop's value bit for bit.
__device__ __forceinline__ void cycle_check_body(double bb, double rr, SolveLoopCtl* ctl, double* hist,
                                                 cudaGraphConditionalHandle handle) {
  const double norm_b = sqrt(bb);
  const double denom = norm_b == 0.0 ? 1.0 : norm_b;
  const double rn = sqrt(rr) / denom;
  const int c = ctl->cycles + 1;
  ctl->cycles = c;
  hist[c] = rn;
  unsigned go = 1;
  if (rn < ctl->tol) {
    ctl->status = 0;  // STMG_CONVERGED
    go = 0;
  } else if (!isfinite(rn) || rn > ctl->div_tol) {
    ctl->status = 2;  // STMG_DIVERGED
    go = 0;
  } else if (c >= ctl->max_cycles) {
    go = 0;  // STMG_MAX_CYCLES (set by the host)
  }
  cudaGraphSetConditional(handle, go);
}
#endif
// y = x * a (y may alias x)
int launch_scale(const double* x, double a, double* y, int64_t n, cudaStream_t s);
// load_vector(g, q) + masking into device memory (source kinds as stmg_load_vector)
int launch_load_vector(int kind, const double* params, int n_params, double L, double t_T, int64_t n_el,
                       int64_t n_t, int masked, double* b, cudaStream_t s);

// ---- kernel launchers (stmg_kernels.cu); all asynchronous on `s` ------------------
// One damped-Jacobi sweep y = x + omega (f - J x) / diag.  If partials != nullptr,
// the block partial sums of r^2 are written too (deterministic order).  If y ==
// nullptr only the residual norm partials are produced.  x == nullptr: x is the
// first sweep from zero S(0) = 0 + omega (f * inv_diag), recomputed from f (this
// convention holds for launch_sweep2, launch_sweep_prolong and
// launch_restrict_residual too).
int launch_sweep(bool adjoint, const LevelView& L, const double* f, const double* x, double* y,
                 double omega, double* partials, int64_t* n_partials, cudaStream_t s);
// Two sweeps y = S(S(x)) in one pass (temporal blocking); bit-identical to two
// launch_sweep calls.  y must not alias x.
int launch_sweep2(bool adjoint, const LevelView& L, const double* f, const double* x, double* y,
                  double omega, cudaStream_t s);
// Tail padding (doubles) of every level vector and coefficient table.
constexpr int64_t kVecPad = 32;
// First sweep from a zero iterate: y = 0 + omega * (f * inv_diag), bitwise equal
// to the general sweep applied to x = +0.
int launch_sweep_from_zero(const LevelView& L, const double* f, double* y, double omega,
                           cudaStream_t s);
// Jacobi sweep applied to (x + P xc), i.e. prolong-add fused into the first
// post-smoothing sweep.  dir: 0 = x, 1 = t.
int launch_sweep_prolong(bool adjoint, const LevelView& L, const LevelView& C, int dir,
                         const double* f, const double* x, const double* xc, double* y,
                         double omega, cudaStream_t s);
int launch_residual(bool adjoint, const LevelView& L, const double* f, const double* x, double* r,
                    cudaStream_t s);
// fc = R (f - J x).  If xc0 != nullptr, also the coarse level's first sweep
// from a zero iterate, xc0 = 0 + omega (fc * inv_diag_c) (bitwise equal to
// launch_sweep_from_zero on fc).
int launch_restrict_residual(bool adjoint, const LevelView& F, const LevelView& C, int dir,
                             const double* f, const double* x, double* fc, cudaStream_t s,
                             double* xc0 = nullptr, double omega = 0.0, const double* const* x_ind = nullptr);
// y = S(0) = 0 + omega (f * inv_diag) and block partials of sum f^2 in one pass over f
// (the opening pass of a solve from a zero iterate)
int launch_sweep_from_zero_norm(const LevelView& L, const double* f, double* y, double omega, double* partials,
                                int64_t* n_partials, cudaStream_t s);
int64_t zero_norm_partials_needed(const LevelView& L);
// Opening pass of a zero-guess solve fused with cycle 1's level-0 restriction: y = S(0),
// f_c = R (f - A S(0)) (x_c0: the stored coarse first sweep, or null), per-warp partials
// of sum f^2 (20 B/DOF instead of 16 + 20).
int launch_restrict_open(bool adjoint, const LevelView& F, const LevelView& C, int dir, const double* f, double* fc,
                         double* xc0, double* y, double omega, double* partials, int64_t* n_partials,
                         cudaStream_t s);
int64_t restrict_open_partials_needed(const LevelView& F, const LevelView& C, int dir);
// p[0] <-> p[1] (device-resident buffer pointers of the fine up-pass)
int launch_swap_ptrs(double** p, cudaStream_t s);
// dst[0 .. count) = w.v[0 .. count) (values passed as kernel arguments, no copy engine)
constexpr int kPokeWords = 8;
struct PokeWords {
  double v[kPokeWords];
};
int launch_poke(double* dst, const PokeWords& w, int count, cudaStream_t s);
// host_dst[0 .. count) = src[0 .. count): host_dst is page-locked host memory, written by the device
int launch_peek(double* host_dst, const double* src, int count, cudaStream_t s);
// Level-0 down-pass of a V(1,1) cycle in one pass: block partials of
// ||f - J x||^2, y = S(x), fc = R (f - J y) and, if xc0 != nullptr, the coarse
// first sweep from zero (bitwise the separate sweep / restriction kernels).
int launch_down(bool adjoint, const LevelView& F, const LevelView& C, int dir, const double* f, const double* x,
                double* y, double* fc, double* xc0, double omega, double* partials, int64_t* n_partials,
                cudaStream_t s);
int64_t down_partials_needed(const LevelView& F, const LevelView& C, int dir);
// Fine up-pass of a V(1,1) cycle in one pass (k_up): u_out = S(x + P xc) (the cycle's
// result), *w_ind = S(u_out) (the next cycle's speculative pre-sweep), one partial per
// warp of ||f - A u_out||^2.  x_ind: optional device-resident pointer to the input
// iterate (read instead of x).  x, u_out and *w_ind are three distinct buffers.
int launch_up(bool adjoint, const LevelView& L, const LevelView& C, int dir, const double* f, const double* x,
              const double* xc, double* u_out, double* const* w_ind, const double* const* x_ind, double omega,
              double* partials, int64_t* n_partials, cudaStream_t s);
int64_t up_partials_needed(const LevelView& L);
int launch_restrict(const LevelView& F, const LevelView& C, int dir, const double* r, double* fc,
                    cudaStream_t s);
int launch_prolong_add(const LevelView& F, const LevelView& C, int dir, const double* xc, double* x,
                       cudaStream_t s);
int launch_coarsest(bool adjoint, const CoarsestView& cv, const double* f, double* x,
                    double* scratch, cudaStream_t s);
// Q = A^pint_len (column-major m x m) into P by m parallel homogeneous marches,
// then its squares Q^2, Q^4, ... into P + m^2, P + 2 m^2, ... (rounds matrices in all)
int launch_coarsest_pint_prop(const CoarsestView& cv, double* P, int rounds, cudaStream_t s);
// Doubles every partials buffer holds past its largest partial count (the first
// stage of a two-stage sum of many partials writes there).
constexpr int64_t kPartialsScratch = 1184;
// Kernel launches launch_finalize_sum / launch_finalize_check issue for n partials.
inline int finalize_launches(int64_t n) { return n > (int64_t{1} << 16) ? 2 : 1; }
// Sum of n_partials doubles in a fixed order into *out (device scalar).
int launch_finalize_sum(const double* partials, int64_t n, double* out, cudaStream_t s);
// Sum of squares of x[0..n) into partials (fixed grid) then *out.
int launch_sumsq(const double* x, int64_t n, double* partials, int64_t* n_partials, cudaStream_t s);
int64_t sweep_partials_needed(const LevelView& L);
// objective_sensitivities (proj/src/optimisation.cpp:34-73), one thread per element
int launch_sensitivities(int64_t n_el, int64_t n_t, double dt, const double* dk_dx,
                         const double* dc_dx6, const double* u, const double* lam, double* sens,
                         cudaStream_t s);
// sum x*y into fixed-grid partials (then launch_finalize_sum)
int launch_dot(const double* x, const double* y, int64_t n, double* partials, int64_t* n_partials,
               cudaStream_t s);
int kernels_init();  // once per device
int64_t sumsq_partials_needed(int64_t n);

}  // namespace stmgb
