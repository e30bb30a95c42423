// sm_100a kernels for the STMG V-cycle (fp64, memory-bound stencils).
//
// Every per-row reduction reproduces the reference's canonical CSR order
// (proj/src/kernels/kernels.cpp:39-46): the row's stored entries in ascending
// column order go to lanes p & 3, each lane starts at 0.0, the row value is
// (s0 + s1) + (s2 + s3).  The library is compiled with --fmad=false, so no
// product is contracted into an FMA (the reference pins -ffp-contract=off on
// its kernel TUs, proj/CMakeLists.txt:41-57).  Sweeps, residuals and
// transfers are therefore bit-identical to the reference; only norms (parallel
// reduction order) and the coarsest exact solve differ at rounding level.
//
// Layout: level vectors are time-major, flat = n * nn + i (nn = n_el + 1),
// exactly the reference's (proj/include/stmg/mesh.hpp:46-48).  The stencil
// sweep kernels march each thread column (one node i) through NT consecutive
// time levels, keeping the previous level's values in registers, so each
// vector element is read from HBM once per sweep (24 B per DOF update).
#include <cuda_runtime.h>

#include <cstdint>

#include "stmg_internal.h"

namespace stmgb {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kNT = 8;           // time levels per thread column
constexpr int kMaxTW = 256;      // threads per block along x (nodes)
constexpr int kFlatBlock = 256;  // flat kernels
constexpr int kSumGrid = 148 * 8;

// Canonical 4-lane accumulator for rows whose entry pattern is not the
// interior one (boundaries, masked columns).
struct Acc {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int p = 0;
  __device__ __forceinline__ void add(double v) {
    switch (p & 3) {
      case 0: s0 = s0 + v; break;
      case 1: s1 = s1 + v; break;
      case 2: s2 = s2 + v; break;
      default: s3 = s3 + v; break;
    }
    ++p;
  }
  __device__ __forceinline__ double result() const { return (s0 + s1) + (s2 + s3); }
};

struct Coefs {
  double cm, c0, cp, om, o0, op, invd;
};

__device__ __forceinline__ Coefs load_coefs(const LevelView& L, int64_t i) {
  const int64_t nn = L.nn;
  Coefs c;
  c.cm = __ldg(L.coef + kCm * nn + i);
  c.c0 = __ldg(L.coef + kC0 * nn + i);
  c.cp = __ldg(L.coef + kCp * nn + i);
  c.om = __ldg(L.coef + kOm * nn + i);
  c.o0 = __ldg(L.coef + kO0 * nn + i);
  c.op = __ldg(L.coef + kOp * nn + i);
  c.invd = __ldg(L.coef + kInvD * nn + i);
  return c;
}

// Row (n, i) of J (ADJ = false) or J^T (ADJ = true) applied to x, given the
// same-time values (xm, x0, xp) at i-1, i, i+1 and the other-time values
// (ym, y0, yp): time n-1 for J, n+1 for J^T.
//   J   row order: [SW, S, SE, W, D, E]  (other level first)
//   J^T row order: [W, D, E, NW, N, NE]  (same level first)
// Masked columns (node 0 or time 0) and entries past the grid are absent
// (proj/src/assembly.cpp:99-123; proj/src/sparse.cpp:74-96).
template <bool ADJ>
__device__ __forceinline__ double row_sum(const LevelView& L, int64_t n, int64_t i, const Coefs& c,
                                          double xm, double x0, double xp, double ym, double y0,
                                          double yp) {
  if (n == 0 || i == 0) {
    const double s0 = 0.0 + L.w * x0;
    return (s0 + 0.0) + (0.0 + 0.0);
  }
  const bool has_m = i >= 2;
  const bool has_p = i <= L.n_el - 1;
  const bool has_o = ADJ ? (n <= L.n_t - 1) : (n >= 2);
  if (has_m && has_p && has_o) {
    double s0, s1, s2, s3;
    if (!ADJ) {
      s0 = (0.0 + c.om * ym) + c.c0 * x0;
      s1 = (0.0 + c.o0 * y0) + c.cp * xp;
      s2 = 0.0 + c.op * yp;
      s3 = 0.0 + c.cm * xm;
    } else {
      s0 = (0.0 + c.cm * xm) + c.o0 * y0;
      s1 = (0.0 + c.c0 * x0) + c.op * yp;
      s2 = 0.0 + c.cp * xp;
      s3 = 0.0 + c.om * ym;
    }
    return (s0 + s1) + (s2 + s3);
  }
  Acc a;
  if (!ADJ) {
    if (has_o) {
      if (has_m) a.add(c.om * ym);
      a.add(c.o0 * y0);
      if (has_p) a.add(c.op * yp);
    }
    if (has_m) a.add(c.cm * xm);
    a.add(c.c0 * x0);
    if (has_p) a.add(c.cp * xp);
  } else {
    if (has_m) a.add(c.cm * xm);
    a.add(c.c0 * x0);
    if (has_p) a.add(c.cp * xp);
    if (has_o) {
      if (has_m) a.add(c.om * ym);
      a.add(c.o0 * y0);
      if (has_p) a.add(c.op * yp);
    }
  }
  return a.result();
}

// P x_c at fine DOF (n, i) (csr_spmv_add row, proj/src/transfer.cpp:74-88).
template <int DIR>
__device__ __forceinline__ double prolong_row(const double* __restrict__ xc, int64_t nnc, int64_t n,
                                              int64_t i) {
  if (DIR == 0) {
    if ((i & 1) == 0) {
      const double s0 = 0.0 + 1.0 * __ldg(xc + n * nnc + (i >> 1));
      return (s0 + 0.0) + (0.0 + 0.0);
    }
    const double s0 = 0.0 + 0.5 * __ldg(xc + n * nnc + ((i - 1) >> 1));
    const double s1 = 0.0 + 0.5 * __ldg(xc + n * nnc + ((i + 1) >> 1));
    return (s0 + s1) + (0.0 + 0.0);
  } else {
    const double s0 = 0.0 + 1.0 * __ldg(xc + (n >> 1) * nnc + i);
    return (s0 + 0.0) + (0.0 + 0.0);
  }
}

struct PlainLoad {
  const double* __restrict__ x;
  int64_t nn;
  __device__ __forceinline__ double operator()(int64_t n, int64_t i) const { return x[n * nn + i]; }
};

template <int DIR>
struct ProlongLoad {
  const double* __restrict__ x;
  const double* __restrict__ xc;
  int64_t nn, nnc;
  __device__ __forceinline__ double operator()(int64_t n, int64_t i) const {
    return x[n * nn + i] + prolong_row<DIR>(xc, nnc, n, i);
  }
};

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double warp_sums[32];
  for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(kFull, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_warps = (blockDim.x + 31) >> 5;
  if (lane == 0) warp_sums[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = lane < n_warps ? warp_sums[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t = t + __shfl_xor_sync(kFull, t, o);
  }
  return t;  // valid in thread 0
}

enum Mode { kSweep = 0, kResidual = 1, kNormOnly = 2 };

// Thread column march: blockIdx.x = time tile (kNT levels), blockIdx.y = node
// tile (blockDim.x nodes).  Same-level neighbours come from warp shuffles
// (warp-edge lanes load them), the other time level is carried in registers.
template <bool ADJ, int MODE, bool NORM, class Ld>
__global__ void __launch_bounds__(kMaxTW) k_march(LevelView L, Ld ld, const double* __restrict__ f,
                                                  double* __restrict__ y, double omega,
                                                  double* __restrict__ partials) {
  const int lane = threadIdx.x & 31;
  const int64_t nn = L.nn, nt = L.n_t;
  const int64_t i = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  const int64_t n0 = (int64_t)blockIdx.x * kNT;
  const bool valid = i < nn;
  Coefs c{};
  if (valid) c = load_coefs(L, i);

  auto fetch = [&](int64_t n, double& xm, double& x0, double& xp) {
    x0 = valid ? ld(n, i) : 0.0;
    xm = __shfl_up_sync(kFull, x0, 1);
    xp = __shfl_down_sync(kFull, x0, 1);
    if (lane == 0) xm = (valid && i >= 1) ? ld(n, i - 1) : 0.0;
    if (lane == 31) xp = (i + 1 < nn) ? ld(n, i + 1) : 0.0;
  };

  double acc = 0.0;
  double xm = 0.0, x0 = 0.0, xp = 0.0, ym = 0.0, y0 = 0.0, yp = 0.0;
  if (!ADJ) {
    if (n0 >= 1) fetch(n0 - 1, ym, y0, yp);
  } else {
    fetch(n0, xm, x0, xp);
  }
#pragma unroll
  for (int t = 0; t < kNT; ++t) {
    const int64_t n = n0 + t;
    if (n > nt) break;
    if (!ADJ) {
      fetch(n, xm, x0, xp);
    } else {
      if (n + 1 <= nt) {
        fetch(n + 1, ym, y0, yp);
      } else {
        ym = 0.0;
        y0 = 0.0;
        yp = 0.0;
      }
    }
    if (valid) {
      const double row = row_sum<ADJ>(L, n, i, c, xm, x0, xp, ym, y0, yp);
      const double r = f[n * nn + i] - row;
      if (NORM) acc = acc + r * r;
      if (MODE == kSweep) {
        const double id = (n == 0 || i == 0) ? L.inv_w : c.invd;
        y[n * nn + i] = x0 + omega * (r * id);
      } else if (MODE == kResidual) {
        y[n * nn + i] = r;
      }
    }
    if (!ADJ) {
      ym = xm;
      y0 = x0;
      yp = xp;
    } else {
      xm = ym;
      x0 = y0;
      xp = yp;
    }
  }
  if (NORM) {
    const double s = block_sum(acc);
    if (threadIdx.x == 0) partials[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
  }
}

__global__ void k_sweep_from_zero(LevelView L, const double* __restrict__ f, double* __restrict__ y,
                                  double omega, int64_t total) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int64_t n = idx / L.nn, i = idx - n * L.nn;
  const double id = (n == 0 || i == 0) ? L.inv_w : __ldg(L.coef + kInvD * L.nn + i);
  y[idx] = 0.0 + omega * (f[idx] * id);
}

// f_c = R (f - J x), with R = s P^T (proj/src/transfer.cpp:95-104): the fine
// residual is recomputed at the (up to 3) contributing fine rows and never
// written to memory.
template <bool ADJ, int DIR, bool FROM_R>
__global__ void k_restrict(LevelView F, LevelView C, const double* __restrict__ f,
                           const double* __restrict__ x, double* __restrict__ fc, int64_t total) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int64_t nnf = F.nn, nnc = C.nn;
  const int64_t N = idx / nnc, I = idx - N * nnc;
  auto xat = [&](int64_t n, int64_t i) -> double {
    return (n >= 0 && n <= F.n_t && i >= 0 && i < nnf) ? __ldg(x + n * nnf + i) : 0.0;
  };
  auto resid = [&](int64_t n, int64_t i) -> double {
    if (FROM_R) return __ldg(x + n * nnf + i);
    const Coefs c = load_coefs(F, i);
    const int64_t no = ADJ ? n + 1 : n - 1;
    const double row = row_sum<ADJ>(F, n, i, c, xat(n, i - 1), xat(n, i), xat(n, i + 1),
                                    xat(no, i - 1), xat(no, i), xat(no, i + 1));
    return __ldg(f + n * nnf + i) - row;
  };
  Acc a;
  if (DIR == 0) {
    const int64_t i0 = 2 * I;
    if (i0 - 1 >= 0) a.add(0.5 * resid(N, i0 - 1));
    a.add(1.0 * resid(N, i0));
    if (i0 + 1 <= F.n_el) a.add(0.5 * resid(N, i0 + 1));
  } else {
    a.add(0.5 * resid(2 * N, I));
    if (2 * N + 1 <= F.n_t) a.add(0.5 * resid(2 * N + 1, I));
  }
  fc[idx] = a.result();
}

template <int DIR>
__global__ void k_prolong_add(LevelView F, LevelView C, const double* __restrict__ xc,
                              double* __restrict__ x, int64_t total) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int64_t n = idx / F.nn, i = idx - n * F.nn;
  x[idx] = x[idx] + prolong_row<DIR>(xc, C.nn, n, i);
}

// Exact coarsest solve: masked rows x = f / w; unmasked rows by a block
// forward (J) / backward (J^T) march in time, one tridiagonal solve per time
// level by parallel cyclic reduction with host-precomputed elimination
// factors (the step matrix is the same on every level).  Replaces the
// reference's SparseLU (proj/src/multigrid.cpp:20-57); exact up to rounding.
template <bool ADJ>
__global__ void __launch_bounds__(1024) k_coarsest(CoarsestView cv, const double* __restrict__ f,
                                                   double* __restrict__ x, double* gscratch,
                                                   int use_smem) {
  extern __shared__ double smem[];
  const LevelView& L = cv.lv;
  const int m = cv.m;
  const int64_t nn = L.nn, nt = L.n_t;
  const int tid = threadIdx.x, bs = blockDim.x;
  double* d0 = use_smem ? smem : gscratch;
  double* d1 = d0 + m;
  for (int64_t i = tid; i < nn; i += bs) x[i] = f[i] / L.w;
  for (int64_t n = 1 + tid; n <= nt; n += bs) x[n * nn] = f[n * nn] / L.w;
  __syncthreads();
  const double* om = L.coef + kOm * nn;
  const double* o0 = L.coef + kO0 * nn;
  const double* op = L.coef + kOp * nn;
  for (int64_t s = 1; s <= nt; ++s) {
    const int64_t n = ADJ ? nt + 1 - s : s;
    const int64_t no = ADJ ? n + 1 : n - 1;
    const bool coupled = ADJ ? (no <= nt) : (no >= 1);
    for (int j = tid; j < m; j += bs) {
      const int64_t i = j + 1;
      double acc = f[n * nn + i];
      if (coupled) {
        if (i >= 2) acc = acc - om[i] * x[no * nn + i - 1];
        acc = acc - o0[i] * x[no * nn + i];
        if (i <= m - 1) acc = acc - op[i] * x[no * nn + i + 1];
      }
      d0[j] = acc;
    }
    __syncthreads();
    for (int k = 0; k < cv.n_steps; ++k) {
      const int st = 1 << k;
      for (int j = tid; j < m; j += bs) {
        double v = d0[j];
        if (j - st >= 0) v = v + cv.alpha[(int64_t)k * m + j] * d0[j - st];
        if (j + st < m) v = v + cv.gamma[(int64_t)k * m + j] * d0[j + st];
        d1[j] = v;
      }
      __syncthreads();
      double* t = d0;
      d0 = d1;
      d1 = t;
    }
    for (int j = tid; j < m; j += bs) x[n * nn + j + 1] = d0[j] / cv.bfin[j];
    __syncthreads();
  }
}

__global__ void k_sumsq(const double* __restrict__ x, int64_t n, double* __restrict__ partials) {
  double acc = 0.0;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[idx];
    acc = acc + v * v;
  }
  const double s = block_sum(acc);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void k_finalize_sum(const double* __restrict__ partials, int64_t n, double* out) {
  double acc = 0.0;
  for (int64_t idx = threadIdx.x; idx < n; idx += blockDim.x) acc = acc + partials[idx];
  const double s = block_sum(acc);
  if (threadIdx.x == 0) *out = s;
}

// Launchers return the cudaError_t of the launch (0 on success).
inline int check_launch() { return static_cast<int>(cudaGetLastError()); }

inline dim3 march_block(const LevelView& L) {
  int tw = L.nn >= kMaxTW ? kMaxTW : (int)((L.nn + 31) / 32 * 32);
  return dim3(tw);
}
inline dim3 march_grid(const LevelView& L, dim3 blk) {
  return dim3((unsigned)((L.n_t + 1 + kNT - 1) / kNT), (unsigned)((L.nn + blk.x - 1) / blk.x));
}
inline unsigned flat_grid(int64_t total) { return (unsigned)((total + kFlatBlock - 1) / kFlatBlock); }

template <bool ADJ>
int sweep_impl(const LevelView& L, const double* f, const double* x, double* y, double omega,
               double* partials, cudaStream_t s) {
  const dim3 blk = march_block(L), grd = march_grid(L, blk);
  const PlainLoad ld{x, L.nn};
  if (y != nullptr && partials != nullptr)
    k_march<ADJ, kSweep, true><<<grd, blk, 0, s>>>(L, ld, f, y, omega, partials);
  else if (y != nullptr)
    k_march<ADJ, kSweep, false><<<grd, blk, 0, s>>>(L, ld, f, y, omega, partials);
  else
    k_march<ADJ, kNormOnly, true><<<grd, blk, 0, s>>>(L, ld, f, y, omega, partials);
  return check_launch();
}

template <bool ADJ, int DIR>
int sweep_prolong_impl(const LevelView& L, const LevelView& C, const double* f, const double* x,
                       const double* xc, double* y, double omega, cudaStream_t s) {
  const dim3 blk = march_block(L), grd = march_grid(L, blk);
  const ProlongLoad<DIR> ld{x, xc, L.nn, C.nn};
  k_march<ADJ, kSweep, false><<<grd, blk, 0, s>>>(L, ld, f, y, omega, nullptr);
  return check_launch();
}

}  // namespace

int64_t sweep_partials_needed(const LevelView& L) {
  const dim3 blk = march_block(L), grd = march_grid(L, blk);
  return (int64_t)grd.x * grd.y;
}

int64_t sumsq_partials_needed(int64_t) { return kSumGrid; }

int launch_sweep(bool adjoint, const LevelView& L, const double* f, const double* x, double* y,
                 double omega, double* partials, int64_t* n_partials, cudaStream_t s) {
  if (n_partials) *n_partials = sweep_partials_needed(L);
  return adjoint ? sweep_impl<true>(L, f, x, y, omega, partials, s)
                 : sweep_impl<false>(L, f, x, y, omega, partials, s);
}

int launch_sweep_from_zero(const LevelView& L, const double* f, double* y, double omega,
                           cudaStream_t s) {
  const int64_t total = L.nn * (L.n_t + 1);
  k_sweep_from_zero<<<flat_grid(total), kFlatBlock, 0, s>>>(L, f, y, omega, total);
  return check_launch();
}

int launch_sweep_prolong(bool adjoint, const LevelView& L, const LevelView& C, int dir,
                         const double* f, const double* x, const double* xc, double* y,
                         double omega, cudaStream_t s) {
  if (adjoint)
    return dir == 0 ? sweep_prolong_impl<true, 0>(L, C, f, x, xc, y, omega, s)
                    : sweep_prolong_impl<true, 1>(L, C, f, x, xc, y, omega, s);
  return dir == 0 ? sweep_prolong_impl<false, 0>(L, C, f, x, xc, y, omega, s)
                  : sweep_prolong_impl<false, 1>(L, C, f, x, xc, y, omega, s);
}

int launch_residual(bool adjoint, const LevelView& L, const double* f, const double* x, double* r,
                    cudaStream_t s) {
  const dim3 blk = march_block(L), grd = march_grid(L, blk);
  const PlainLoad ld{x, L.nn};
  if (adjoint)
    k_march<true, kResidual, false><<<grd, blk, 0, s>>>(L, ld, f, r, 0.0, nullptr);
  else
    k_march<false, kResidual, false><<<grd, blk, 0, s>>>(L, ld, f, r, 0.0, nullptr);
  return check_launch();
}

int launch_restrict_residual(bool adjoint, const LevelView& F, const LevelView& C, int dir,
                             const double* f, const double* x, double* fc, cudaStream_t s) {
  const int64_t total = C.nn * (C.n_t + 1);
  const unsigned g = flat_grid(total);
  if (adjoint) {
    if (dir == 0) k_restrict<true, 0, false><<<g, kFlatBlock, 0, s>>>(F, C, f, x, fc, total);
    else k_restrict<true, 1, false><<<g, kFlatBlock, 0, s>>>(F, C, f, x, fc, total);
  } else {
    if (dir == 0) k_restrict<false, 0, false><<<g, kFlatBlock, 0, s>>>(F, C, f, x, fc, total);
    else k_restrict<false, 1, false><<<g, kFlatBlock, 0, s>>>(F, C, f, x, fc, total);
  }
  return check_launch();
}

int launch_restrict(const LevelView& F, const LevelView& C, int dir, const double* r, double* fc,
                    cudaStream_t s) {
  const int64_t total = C.nn * (C.n_t + 1);
  const unsigned g = flat_grid(total);
  if (dir == 0) k_restrict<false, 0, true><<<g, kFlatBlock, 0, s>>>(F, C, nullptr, r, fc, total);
  else k_restrict<false, 1, true><<<g, kFlatBlock, 0, s>>>(F, C, nullptr, r, fc, total);
  return check_launch();
}

int launch_prolong_add(const LevelView& F, const LevelView& C, int dir, const double* xc, double* x,
                       cudaStream_t s) {
  const int64_t total = F.nn * (F.n_t + 1);
  if (dir == 0) k_prolong_add<0><<<flat_grid(total), kFlatBlock, 0, s>>>(F, C, xc, x, total);
  else k_prolong_add<1><<<flat_grid(total), kFlatBlock, 0, s>>>(F, C, xc, x, total);
  return check_launch();
}

int launch_coarsest(bool adjoint, const CoarsestView& cv, const double* f, double* x,
                    double* scratch, cudaStream_t s) {
  const size_t smem = sizeof(double) * 2 * (size_t)cv.m;
  const int use_smem = smem <= 160 * 1024 ? 1 : 0;
  int threads = cv.m >= 1024 ? 1024 : (int)((cv.m + 31) / 32 * 32);
  if (threads < 32) threads = 32;
  const size_t dyn = use_smem ? smem : 0;
  if (adjoint) k_coarsest<true><<<1, threads, dyn, s>>>(cv, f, x, scratch, use_smem);
  else k_coarsest<false><<<1, threads, dyn, s>>>(cv, f, x, scratch, use_smem);
  return check_launch();
}

int kernels_init() {
  // The coarsest march keeps its two PCR work vectors in shared memory up to 160 KB.
  cudaError_t e = cudaFuncSetAttribute(k_coarsest<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  if (e != cudaSuccess) return static_cast<int>(e);
  e = cudaFuncSetAttribute(k_coarsest<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           160 * 1024);
  return static_cast<int>(e);
}

int launch_finalize_sum(const double* partials, int64_t n, double* out, cudaStream_t s) {
  k_finalize_sum<<<1, 1024, 0, s>>>(partials, n, out);
  return check_launch();
}

int launch_sumsq(const double* x, int64_t n, double* partials, int64_t* n_partials, cudaStream_t s) {
  k_sumsq<<<kSumGrid, 256, 0, s>>>(x, n, partials);
  if (n_partials) *n_partials = kSumGrid;
  return check_launch();
}

}  // namespace stmgb
