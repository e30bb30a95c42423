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
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "stmg_internal.h"

namespace stmgb {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kNT = 8;           // time levels per thread column
constexpr int kMaxTW = 256;      // threads per block along x (nodes)
constexpr int kFlatBlock = 256;  // flat kernels
constexpr int kSumGrid = 148 * 8;

// Programmatic dependent launch.  Every kernel is launched with programmatic
// stream serialization, so inside a captured V-cycle graph the next kernel's
// launch and CTA rasterisation overlap the tail of the current one.  Each
// kernel therefore begins with griddepcontrol.wait (returns once the preceding
// grid has completed and its writes are visible; a no-op for ordinary
// launches) before touching memory, and then releases its own dependents.
// STMG_PDL=0 turns the attribute off (A/B measurements).
bool g_pdl = true;

__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <class... KArgs, class... Args>
inline void pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// The pointer's value, hidden from the optimiser: a 32-bit element offset from
// it then costs one IMAD.WIDE per access instead of being folded back into
// 64-bit index arithmetic.
template <class T>
__device__ __forceinline__ T* opaque(T* p) {
  asm("mov.b64 %0, %0;" : "+l"(p));
  return p;
}

__device__ __forceinline__ void st_global(double* p, double v) {
  asm volatile("st.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

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

// Interior row (all six entries present): the fixed canonical lane order.
// x*: same-time values at i-1, i, i+1; y*: coupled-level values.
template <bool ADJ>
__device__ __forceinline__ double row_interior(const Coefs& c, double xm, double x0, double xp,
                                               double ym, double y0, double yp) {
  // Canonical lanes: s0 = (0 + a) + b, s1 = (0 + c) + d, s2 = 0 + e, s3 = 0 + g,
  // row = (s0 + s1) + (s2 + s3).  "0 + v" equals v as a real number and only
  // turns an exact -0 into +0, so every intermediate equals the raw sum's in
  // value; and a sum of operands none of which is -0 is never -0.  Hence the
  // canonical row is the raw sum with a final -0 -> +0, i.e. raw + 0.0:
  // bit-identical, 6 additions instead of 10.
  double raw;
  if (!ADJ)
    raw = ((c.om * ym + c.c0 * x0) + (c.o0 * y0 + c.cp * xp)) + (c.op * yp + c.cm * xm);
  else
    raw = ((c.cm * xm + c.o0 * y0) + (c.c0 * x0 + c.op * yp)) + (c.cp * xp + c.om * ym);
  return raw + 0.0;
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
    return 0.0 + L.w * x0;  // = (s0 + 0) + (0 + 0) with s0 = 0 + w x0 (never -0)
  }
  const bool has_m = i >= 2;
  const bool has_p = i <= L.n_el - 1;
  const bool has_o = ADJ ? (n <= L.n_t - 1) : (n >= 2);
  if (has_m && has_p && has_o) return row_interior<ADJ>(c, xm, x0, xp, ym, y0, yp);
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
  // canonical lanes with the "0 +" initialisations folded into one final +0.0
  // (see row_interior): bit-identical to ((0 + a) + (0 + b)) + (0 + 0)
  if (DIR == 0) {
    if ((i & 1) == 0) return 0.0 + 1.0 * __ldg(xc + n * nnc + (i >> 1));
    return (0.5 * __ldg(xc + n * nnc + ((i - 1) >> 1)) + 0.5 * __ldg(xc + n * nnc + ((i + 1) >> 1))) + 0.0;
  } else {
    return 0.0 + 1.0 * __ldg(xc + (n >> 1) * nnc + i);
  }
}

// Staged-row loaders.  operator() is the per-lane form (any lane subset);
// warp_row() is called by all 32 lanes of a warp whose nodes wfirst-1 ..
// wfirst+30 are all inside the grid (interior tiles).
// Interior staging is split in two phases: warp_load issues every global load
// of a row (all rows of a tile first, so the loads are in flight together),
// warp_finish combines them (shuffles) once they are needed.
struct PlainLoad {
  const double* __restrict__ x;
  int64_t nn;
  __device__ __forceinline__ double operator()(int64_t n, int64_t i) const { return x[n * nn + i]; }
  __device__ __forceinline__ double warp_row(int64_t n, int64_t i, int64_t, int) const { return x[n * nn + i]; }
  struct Raw {
    double x;
  };
  __device__ __forceinline__ Raw warp_load(int64_t n, int64_t i, int64_t, int) const { return {x[n * nn + i]}; }
  __device__ __forceinline__ double warp_finish(const Raw& r, int64_t, int64_t, int) const { return r.x; }
};

template <int DIR>
struct ProlongLoad {
  const double* __restrict__ x;
  const double* __restrict__ xc;
  int64_t nn, nnc;
  __device__ __forceinline__ double operator()(int64_t n, int64_t i) const {
    return x[n * nn + i] + prolong_row<DIR>(xc, nnc, n, i);
  }
  // x step: the warp's fine nodes need coarse nodes c0 .. c0+16, c0 = (wfirst-1)/2;
  // lanes 0..17 load them once (coalesced) and every lane takes its one or two
  // values by shuffle; even/odd rows are selected, not branched.  Same
  // arithmetic as prolong_row.
  __device__ __forceinline__ double warp_row(int64_t n, int64_t i, int64_t wfirst, int lane) const {
    return warp_finish(warp_load(n, i, wfirst, lane), i, wfirst, lane);
  }
  struct Raw {
    double x, v;
  };
  __device__ __forceinline__ Raw warp_load(int64_t n, int64_t i, int64_t wfirst, int lane) const {
    Raw r;
    r.x = x[n * nn + i];
    if (DIR == 1) {
      r.v = __ldg(xc + (n >> 1) * nnc + i);
    } else {
      const int64_t c0 = (wfirst - 1) >> 1;
      r.v = (lane <= 17 && c0 + lane < nnc) ? __ldg(xc + n * nnc + c0 + lane) : 0.0;
    }
    return r;
  }
  __device__ __forceinline__ double warp_finish(const Raw& r, int64_t i, int64_t wfirst, int) const {
    if (DIR == 1) return r.x + (0.0 + 1.0 * r.v);  // prolong_row<1>
    const int64_t c0 = (wfirst - 1) >> 1;
    const int k0 = (int)((i >> 1) - c0);
    const double va = __shfl_sync(kFull, r.v, k0);      // xc[i/2] (even), xc[(i-1)/2] (odd)
    const double vb = __shfl_sync(kFull, r.v, k0 + 1);  // xc[(i+1)/2] (odd)
    const double pe = 0.0 + 1.0 * va;
    const double po = (0.5 * va + 0.5 * vb) + 0.0;
    return r.x + ((i & 1) == 0 ? pe : po);
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

// ---------------------------------------------------------------------------
// Lean stencil kernels (production): blockIdx.x = time tile of NT levels,
// blockIdx.y = node tile of blockDim.x nodes, one node column per thread.  No
// shared memory and no block barrier: every global load of the tile (x on the
// NT + 1 staged levels, f on the NT rows, and the strip-edge halo node of
// lanes 0 / 31) is issued up front, same-level neighbours then come from warp
// shuffles.  Tiles whose rows and nodes are all interior (the overwhelming
// majority) take a branch-free path with the fixed interior lane order; the
// rest use the general row evaluation.
// ---------------------------------------------------------------------------
template <bool ADJ, int MODE, bool NORM, int NT, int MINB, class Ld>
__global__ void __launch_bounds__(kMaxTW, MINB) k_lean(LevelView L, Ld ld,
                                                       const double* __restrict__ f,
                                                       double* __restrict__ y, double omega,
                                                       double* __restrict__ partials) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int64_t nn = L.nn, nt = L.n_t;
  const int64_t i = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  const int64_t n0 = (int64_t)blockIdx.x * NT;
  const int64_t nbase = ADJ ? n0 : n0 - 1;  // level of staged row 0
  const int64_t wfirst = i - lane;          // first node of this warp
  const bool valid = i < nn;
  // rows n0..n0+NT-1 all have their coupled level and are unmasked in time
  const bool rows_in = ADJ ? (n0 >= 1 && n0 + NT - 1 <= nt - 1) : (n0 >= 2 && n0 + NT - 1 <= nt);
  const bool nodes_in = wfirst >= 2 && wfirst + 31 <= L.n_el - 1;
  const int64_t ih = lane == 0 ? i - 1 : i + 1;  // halo node of the edge lanes
  const bool edge = lane == 0 || lane == 31;
  double xr[NT + 1], hr[NT + 1], fv[NT];
  Coefs c{};
  double acc = 0.0;
  if (rows_in && nodes_in) {
    // ---- interior fast path: no bounds checks, fixed canonical lane order ----
    const double* fp = f + n0 * nn + i;
#pragma unroll
    for (int k = 0; k < NT; ++k) fv[k] = fp[k * nn];
#pragma unroll
    for (int r = 0; r <= NT; ++r) {
      xr[r] = ld(nbase + r, i);
      hr[r] = edge ? ld(nbase + r, ih) : 0.0;
    }
    c = load_coefs(L, i);
    double pm = 0.0, pp = 0.0;  // neighbours of staged row 0 / the previous row
    {
      pm = __shfl_up_sync(kFull, xr[0], 1);
      pp = __shfl_down_sync(kFull, xr[0], 1);
      if (lane == 0) pm = hr[0];
      if (lane == 31) pp = hr[0];
    }
    double* yp = y + n0 * nn + i;
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const double x1 = xr[k + 1];
      double qm = __shfl_up_sync(kFull, x1, 1);
      double qp = __shfl_down_sync(kFull, x1, 1);
      if (lane == 0) qm = hr[k + 1];
      if (lane == 31) qp = hr[k + 1];
      double s0, s1, s2, s3, x0;
      if (!ADJ) {  // row n0+k: level = staged k+1 (q), coupled = staged k (p)
        x0 = x1;
        s0 = (0.0 + c.om * pm) + c.c0 * x1;
        s1 = (0.0 + c.o0 * xr[k]) + c.cp * qp;
        s2 = 0.0 + c.op * pp;
        s3 = 0.0 + c.cm * qm;
      } else {  // row n0+k: level = staged k (p), coupled = staged k+1 (q)
        x0 = xr[k];
        s0 = (0.0 + c.cm * pm) + c.o0 * x1;
        s1 = (0.0 + c.c0 * x0) + c.op * qp;
        s2 = 0.0 + c.cp * pp;
        s3 = 0.0 + c.om * qm;
      }
      const double r = fv[k] - ((s0 + s1) + (s2 + s3));
      if (NORM) acc = acc + r * r;
      if (MODE == kSweep) yp[k * nn] = x0 + omega * (r * c.invd);
      else if (MODE == kResidual) yp[k * nn] = r;
      pm = qm;
      pp = qp;
    }
  } else {
    // ---- general path (time-boundary tiles, boundary nodes, partial tiles) ----
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const int64_t n = n0 + k;
      fv[k] = (valid && n <= nt) ? f[n * nn + i] : 0.0;
    }
#pragma unroll
    for (int r = 0; r <= NT; ++r) {
      const int64_t n = nbase + r;
      const bool nok = n >= 0 && n <= nt;
      xr[r] = (nok && valid) ? ld(n, i) : 0.0;
      hr[r] = (nok && edge && ih >= 0 && ih < nn) ? ld(n, ih) : 0.0;
    }
    if (valid) c = load_coefs(L, i);
    double pm = __shfl_up_sync(kFull, xr[0], 1);
    double pp = __shfl_down_sync(kFull, xr[0], 1);
    if (lane == 0) pm = hr[0];
    if (lane == 31) pp = hr[0];
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const int64_t n = n0 + k;
      if (n > nt) break;
      const double x1 = xr[k + 1];
      double qm = __shfl_up_sync(kFull, x1, 1);
      double qp = __shfl_down_sync(kFull, x1, 1);
      if (lane == 0) qm = hr[k + 1];
      if (lane == 31) qp = hr[k + 1];
      if (valid) {
        // J: level = staged k+1 (q), coupled = staged k (p); J^T: the reverse
        const double row = ADJ ? row_sum<true>(L, n, i, c, pm, xr[k], pp, qm, x1, qp)
                               : row_sum<false>(L, n, i, c, qm, x1, qp, pm, xr[k], pp);
        const double x0 = ADJ ? xr[k] : x1;
        const double r = fv[k] - row;
        if (NORM) acc = acc + r * r;
        if (MODE == kSweep) {
          const double id = (n == 0 || i == 0) ? L.inv_w : c.invd;
          y[n * nn + i] = x0 + omega * (r * id);
        } else if (MODE == kResidual) {
          y[n * nn + i] = r;
        }
      }
      pm = qm;
      pp = qp;
    }
  }
  if (NORM) {
    const double s = block_sum(acc);
    if (threadIdx.x == 0) partials[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
  }
}

// Lean variant with overlapping warps: each warp covers 32 consecutive nodes
// but only lanes 1..30 compute and store; lanes 0 and 31 load the strip-edge
// nodes, so no separate halo registers are needed (lower register pressure,
// higher occupancy).  Grid: blockIdx.x = node tile (fastest, so the staged
// coupled level of a time tile is usually still in L2), blockIdx.y strides
// over time tiles.  Interior tiles (the overwhelming majority) are detected
// before any load and take a predicate-free path: row pointers computed once,
// unconditional loads, the fixed interior lane order.
// Tile body (callable from the stand-alone kernel and the coarse-tail kernel):
// node tile `tile`, time tile `ttile`, `tw` threads; returns the thread's r^2 sum.
template <bool ADJ, int MODE, bool NORM, int NT, class Ld>
__device__ __forceinline__ double dev_lean2(const LevelView& L, const Ld& ld, const double* __restrict__ f,
                                            double* __restrict__ y, double omega, int64_t tile,
                                            int64_t ttile, int tw) {
  if ((int)threadIdx.x >= tw) return 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nn = L.nn, nt = L.n_t;
  const int64_t wfirst = tile * ((tw >> 5) * 30) + warp * 30;  // first computing node of the warp
  if (wfirst >= nn) return 0.0;                                  // whole warp past the grid
  const int64_t i = wfirst + lane - 1;                           // node of this lane
  const int64_t n0 = L.n_lo + ttile * NT;
  const int64_t nbase = ADJ ? n0 : n0 - 1;
  const bool rows_in = (ADJ ? (n0 >= 1 && n0 + NT - 1 <= nt - 1) : (n0 >= 2 && n0 + NT - 1 <= nt)) &&
                       n0 + NT - 1 < L.n_hi;
  const bool nodes_in = wfirst >= 2 && wfirst + 29 <= L.n_el - 1;
  double xr[NT + 1], fv[NT];
  double acc = 0.0;
  if (rows_in && nodes_in) {
    // every lane's node is inside the grid: lanes 0 / 31 load too (unused values)
    const bool computes = lane >= 1 && lane <= 30;
    const double* fp = f + (n0 * nn + i);
#pragma unroll
    for (int k = 0; k < NT; ++k) fv[k] = fp[k * nn];
    typename Ld::Raw raw[NT + 1];
#pragma unroll
    for (int r = 0; r <= NT; ++r) raw[r] = ld.warp_load(nbase + r, i, wfirst, lane);
    const Coefs c = load_coefs(L, i);
#pragma unroll
    for (int r = 0; r <= NT; ++r) xr[r] = ld.warp_finish(raw[r], i, wfirst, lane);
    double* yp = y + (n0 * nn + i);
    double pm = __shfl_up_sync(kFull, xr[0], 1);
    double pp = __shfl_down_sync(kFull, xr[0], 1);
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const double x1 = xr[k + 1];
      const double qm = __shfl_up_sync(kFull, x1, 1);
      const double qp = __shfl_down_sync(kFull, x1, 1);
      const double x0 = ADJ ? xr[k] : x1;
      const double row = ADJ ? row_interior<true>(c, pm, xr[k], pp, qm, x1, qp)
                             : row_interior<false>(c, qm, x1, qp, pm, xr[k], pp);
      const double r = fv[k] - row;
      if (computes) {
        if (NORM) acc = acc + r * r;
        if (MODE == kSweep) yp[k * nn] = x0 + omega * (r * c.invd);
        else if (MODE == kResidual) yp[k * nn] = r;
      }
      pm = qm;
      pp = qp;
    }
    return acc;
  }
  const bool in_grid = i >= 0 && i < nn;
  const bool computes = lane >= 1 && lane <= 30 && in_grid;
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const int64_t n = n0 + k;
    fv[k] = (computes && n < L.n_hi) ? f[n * nn + i] : 0.0;
  }
#pragma unroll
  for (int r = 0; r <= NT; ++r) {
    const int64_t n = nbase + r;
    xr[r] = (n >= 0 && n <= nt && in_grid) ? ld(n, i) : 0.0;
  }
  Coefs c{};
  if (computes) c = load_coefs(L, i);
  double pm = __shfl_up_sync(kFull, xr[0], 1);
  double pp = __shfl_down_sync(kFull, xr[0], 1);
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const int64_t n = n0 + k;
    if (n >= L.n_hi) break;
    const double x1 = xr[k + 1];
    const double qm = __shfl_up_sync(kFull, x1, 1);
    const double qp = __shfl_down_sync(kFull, x1, 1);
    if (computes) {
      const double row = ADJ ? row_sum<true>(L, n, i, c, pm, xr[k], pp, qm, x1, qp)
                             : row_sum<false>(L, n, i, c, qm, x1, qp, pm, xr[k], pp);
      const double x0 = ADJ ? xr[k] : x1;
      const double r = fv[k] - row;
      if (NORM) acc = acc + r * r;
      if (MODE == kSweep) {
        const double id = (n == 0 || i == 0) ? L.inv_w : c.invd;
        y[n * nn + i] = x0 + omega * (r * id);
      } else if (MODE == kResidual) {
        y[n * nn + i] = r;
      }
    }
    pm = qm;
    pp = qp;
  }
  return acc;
}

inline __host__ __device__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

template <bool ADJ, int MODE, bool NORM, int NT, int MINB, class Ld>
__global__ void __launch_bounds__(kMaxTW, MINB) k_lean2(LevelView L, Ld ld,
                                                        const double* __restrict__ f,
                                                        double* __restrict__ y, double omega,
                                                        double* __restrict__ partials) {
  pdl_entry();
  const int64_t tt = (int64_t)blockIdx.z * gridDim.y + blockIdx.y;  // time tile
  double acc = 0.0;
  if (tt < ceil_div(L.n_hi - L.n_lo, NT))
    acc = dev_lean2<ADJ, MODE, NORM, NT>(L, ld, f, y, omega, blockIdx.x, tt, blockDim.x);
  if (NORM) {
    const double s = block_sum(acc);
    if (threadIdx.x == 0) partials[tt * gridDim.x + blockIdx.x] = s;
  }
}

// Two damped-Jacobi sweeps fused into one pass over memory (temporal
// blocking), bit-identical to two separate sweeps.  Warps overlap by two
// nodes on each side: lanes 1..30 evaluate sweep 1, lanes 2..29 evaluate and
// store sweep 2 (28 nodes per warp).  Sweep 1 is also evaluated on the one
// staged row before the tile (J) / after it (J^T) that sweep 2 couples to.
// Staged: x on NT + 2 levels, f on NT + 1 levels.  Grid as k_lean2.
// W2: omega is an exact power of two (the reference's 1/2), so
// omega * (r * invd) == r * (omega * invd) bit for bit (scaling by 2^k commutes
// with rounding for normal results) and the interior rows save one DMUL each.
template <bool ADJ, int NT, bool W2 = false>
__device__ __forceinline__ void dev_lean2x2(const LevelView& L, const double* __restrict__ f,
                                            const double* __restrict__ x, double* __restrict__ y,
                                            double omega, int64_t tile, int64_t ttile) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nn = L.nn, nt = L.n_t;
  const int64_t node1 = tile * ((int64_t)(blockDim.x >> 5) * 28) + warp * 28 - 1;  // node of lane 1
  if (node1 + 1 >= nn) return;  // no stored node in this warp (whole warp exits)
  const int64_t i = node1 + lane - 1;  // node of this lane
  const int64_t n0 = L.n_lo + ttile * NT;
  // staged rows: J: n0-2 .. n0+NT-1 ; J^T: n0 .. n0+NT+1  (NT + 2 levels)
  const int64_t sbase = ADJ ? n0 : n0 - 2;
  // sweep-1 rows: J: n0-1 .. n0+NT-1 ; J^T: n0 .. n0+NT   (NT + 1 rows)
  const int64_t s1base = ADJ ? n0 : n0 - 1;
  // interior tile: every sweep-1 and sweep-2 row has its coupled level and is
  // unmasked, every sweep-1 node (lanes 1..30) has both neighbours
  const bool rows_in = (ADJ ? (n0 >= 1 && n0 + NT <= nt - 1) : (n0 >= 3 && n0 + NT - 1 <= nt)) &&
                       n0 + NT - 1 < L.n_hi;
  const bool nodes_in = node1 >= 2 && node1 + 29 <= L.n_el - 1;
  double xs[NT + 2], fv[NT + 1], y1[NT + 1];
  if (rows_in && nodes_in) {
    // one 64-bit row base for x, f and y; 32-bit element offsets from it
    // (o[j] = node i on staged row sbase + j), so each access is one IMAD.WIDE
    const int64_t rowbase = sbase * nn;
    const double* __restrict__ xb = opaque(x + rowbase);
    const double* __restrict__ fb = opaque(f + rowbase);
    double* __restrict__ yb = opaque(y + rowbase);
    const uint32_t nn32 = (uint32_t)nn;
    uint32_t o[NT + 2];
    o[0] = (uint32_t)i;
#pragma unroll
    for (int r = 1; r < NT + 2; ++r) o[r] = o[r - 1] + nn32;
#pragma unroll
    for (int r = 0; r < NT + 2; ++r) xs[r] = __ldg(xb + o[r]);
#pragma unroll
    for (int r = 0; r < NT + 1; ++r) fv[r] = __ldg(fb + o[ADJ ? r : r + 1]);  // f rows s1base + r
    const Coefs c = load_coefs(L, i);
    const double sc = c.invd * omega;  // used only when W2
    auto upd = [&](double x0, double fval, double row) {
      return W2 ? x0 + (fval - row) * sc : x0 + omega * ((fval - row) * c.invd);
    };
    double pm = __shfl_up_sync(kFull, xs[0], 1), pp = __shfl_down_sync(kFull, xs[0], 1);
#pragma unroll
    for (int r = 0; r <= NT; ++r) {
      const double x1 = xs[r + 1];
      const double qm = __shfl_up_sync(kFull, x1, 1), qp = __shfl_down_sync(kFull, x1, 1);
      if (ADJ) y1[r] = upd(xs[r], fv[r], row_interior<true>(c, pm, xs[r], pp, qm, x1, qp));
      else y1[r] = upd(x1, fv[r], row_interior<false>(c, qm, x1, qp, pm, xs[r], pp));
      pm = qm;
      pp = qp;
    }
    const bool lane2 = lane >= 2 && lane <= 29;
    double am = __shfl_up_sync(kFull, y1[0], 1), ap = __shfl_down_sync(kFull, y1[0], 1);
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const double z1 = y1[k + 1];
      const double bm = __shfl_up_sync(kFull, z1, 1), bp = __shfl_down_sync(kFull, z1, 1);
      // evaluated on every lane (no divergence around the shuffles); stored on
      // lanes 2..29; row n0 + k is staged row k (J^T) / k + 2 (J)
      const double v = ADJ ? upd(y1[k], fv[k], row_interior<true>(c, am, y1[k], ap, bm, z1, bp))
                           : upd(z1, fv[k + 1], row_interior<false>(c, bm, z1, bp, am, y1[k], ap));
      if (lane2) st_global(yb + o[ADJ ? k : k + 2], v);
      am = bm;
      ap = bp;
    }
    return;
  }
  const bool in_grid = i >= 0 && i < nn;
  const bool lane1 = lane >= 1 && lane <= 30 && in_grid;
  const bool lane2 = lane >= 2 && lane <= 29 && in_grid;
#pragma unroll
  for (int r = 0; r < NT + 2; ++r) {
    const int64_t n = sbase + r;
    xs[r] = (n >= 0 && n <= nt && in_grid) ? x[n * nn + i] : 0.0;
  }
#pragma unroll
  for (int r = 0; r < NT + 1; ++r) {
    const int64_t n = s1base + r;
    fv[r] = (n >= 0 && n <= nt && lane1) ? f[n * nn + i] : 0.0;
  }
  Coefs c{};
  if (lane1) c = load_coefs(L, i);
  // ---- general path: sweep 1 on NT + 1 rows -> y1[r] (row s1base + r)
  double pm = __shfl_up_sync(kFull, xs[0], 1), pp = __shfl_down_sync(kFull, xs[0], 1);
  if (ADJ) {
    // row m uses staged (m, m+1): iterate r = 0..NT, row level xs[r], coupled xs[r+1]
#pragma unroll
    for (int r = 0; r <= NT; ++r) {
      const double x1 = xs[r + 1];
      const double qm = __shfl_up_sync(kFull, x1, 1), qp = __shfl_down_sync(kFull, x1, 1);
      const int64_t n = s1base + r;
      double v = 0.0;
      if (lane1 && n <= nt) {
        const double row = row_sum<true>(L, n, i, c, pm, xs[r], pp, qm, x1, qp);
        const double id = (n == 0 || i == 0) ? L.inv_w : c.invd;
        v = xs[r] + omega * ((fv[r] - row) * id);
      }
      y1[r] = v;
      pm = qm;
      pp = qp;
    }
  } else {
    // row m uses staged (m-1, m): iterate r = 0..NT, row level xs[r+1], coupled xs[r]
#pragma unroll
    for (int r = 0; r <= NT; ++r) {
      const double x1 = xs[r + 1];
      const double qm = __shfl_up_sync(kFull, x1, 1), qp = __shfl_down_sync(kFull, x1, 1);
      const int64_t n = s1base + r;
      double v = 0.0;
      if (lane1 && n >= 0 && n <= nt) {
        const double row = row_sum<false>(L, n, i, c, qm, x1, qp, pm, xs[r], pp);
        const double id = (n == 0 || i == 0) ? L.inv_w : c.invd;
        v = x1 + omega * ((fv[r] - row) * id);
      }
      y1[r] = v;
      pm = qm;
      pp = qp;
    }
  }
  // ---- sweep 2 on rows n0 .. n0+NT-1 from y1
  double am = __shfl_up_sync(kFull, y1[0], 1), ap = __shfl_down_sync(kFull, y1[0], 1);
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const double z1 = y1[k + 1];
    const double bm = __shfl_up_sync(kFull, z1, 1), bp = __shfl_down_sync(kFull, z1, 1);
    const int64_t n = n0 + k;
    if (lane2 && n < L.n_hi) {
      double row, x0, fval;
      if (ADJ) {  // row n = y1[k] level, coupled y1[k+1]
        row = row_sum<true>(L, n, i, c, am, y1[k], ap, bm, z1, bp);
        x0 = y1[k];
        fval = fv[k];
      } else {  // row n = y1[k+1] level, coupled y1[k]
        row = row_sum<false>(L, n, i, c, bm, z1, bp, am, y1[k], ap);
        x0 = z1;
        fval = fv[k + 1];
      }
      const double id = (n == 0 || i == 0) ? L.inv_w : c.invd;
      y[n * nn + i] = x0 + omega * ((fval - row) * id);
    }
    am = bm;
    ap = bp;
  }
}

// Resident blocks per SM the kernels are compiled for: 5 (48 registers) pays on
// mid-sized levels, where the launch fills the GPU and latency is hidden by
// warps; on small levels the few blocks never fill the SMs and the spills of the
// tighter register budget cost latency, so 3 is used there (launch sites).
constexpr int64_t kMinB5Dofs = 200000;
template <int NT>
constexpr int minb_for_nt() { return NT <= 2 ? 5 : NT <= 4 ? 4 : 3; }

template <bool ADJ, int NT, int MINB = minb_for_nt<NT>(), bool W2 = false>
__global__ void __launch_bounds__(kMaxTW, MINB) k_lean2x2(LevelView L, const double* __restrict__ f,
                                                       const double* __restrict__ x,
                                                       double* __restrict__ y, double omega) {
  pdl_entry();
  const int64_t tt = (int64_t)blockIdx.z * gridDim.y + blockIdx.y;  // time tile
  if (tt < ceil_div(L.n_hi - L.n_lo, NT)) dev_lean2x2<ADJ, NT, W2>(L, f, x, y, omega, blockIdx.x, tt);
}

// D damped-Jacobi sweeps fused into one pass (temporal blocking of depth D,
// the generalisation of k_lean2x2), bit-identical to D separate sweeps.  Lane
// l holds node first - D + l; stage s (1..D) is valid on lanes s..31-s, so
// lanes D..31-D (32 - 2D nodes per warp) are stored.  J: staged x rows
// n0-D .. n0+NT-1, stage s produces rows n0-D+s .. n0+NT-1 in place (row j of
// the stage array: own level j+1, coupled level j).  J^T: staged rows n0 ..
// n0+NT+D-1, stage s produces rows n0 .. n0+NT+D-1-s (own j, coupled j+1).
// Used on small, latency-bound levels, where one launch replaces D/2 pair
// launches; full-range levels only (slab solves exchange ghosts every sweep).
template <bool ADJ, int NT, int D, bool EDGE>
__device__ __forceinline__ void leanD_body(const LevelView& L, const double* __restrict__ f,
                                           const double* __restrict__ x, double* __restrict__ y,
                                           double omega, int64_t first, int64_t n0, int lane) {
  constexpr int S = NT + D;      // staged x rows
  constexpr int F = NT + D - 1;  // f rows
  const int64_t nn = L.nn, nt = L.n_t;
  const int64_t i = first + lane - D;
  const int64_t sbase = ADJ ? n0 : n0 - D;
  const int64_t fbase = ADJ ? n0 : n0 - D + 1;
  const bool in_grid = !EDGE || (i >= 0 && i < nn);
  double v[S], fv[F];
  Coefs c{};
  if (!EDGE) {
    const double* xp = x + (sbase * nn + i);
    const double* fp = f + (fbase * nn + i);
#pragma unroll
    for (int j = 0; j < S; ++j) v[j] = xp[j * nn];
#pragma unroll
    for (int j = 0; j < F; ++j) fv[j] = fp[j * nn];
    c = load_coefs(L, i);
  } else {
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const int64_t n = sbase + j;
      v[j] = (n >= 0 && n <= nt && in_grid) ? x[n * nn + i] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < F; ++j) {
      const int64_t n = fbase + j;
      fv[j] = (n >= 0 && n <= nt && in_grid) ? f[n * nn + i] : 0.0;
    }
    if (in_grid) c = load_coefs(L, i);
  }
#pragma unroll
  for (int st = 1; st <= D; ++st) {
    double pm = __shfl_up_sync(kFull, v[0], 1), pp = __shfl_down_sync(kFull, v[0], 1);
#pragma unroll
    for (int j = 0; j < S - st; ++j) {
      const double x1 = v[j + 1];
      const double qm = __shfl_up_sync(kFull, x1, 1), qp = __shfl_down_sync(kFull, x1, 1);
      const int64_t n = ADJ ? sbase + j : sbase + st + j;
      const double fval = ADJ ? fv[j] : fv[st - 1 + j];
      const double own = ADJ ? v[j] : x1;
      double out;
      if (!EDGE) {
        const double row = ADJ ? row_interior<true>(c, pm, v[j], pp, qm, x1, qp)
                               : row_interior<false>(c, qm, x1, qp, pm, v[j], pp);
        out = own + omega * ((fval - row) * c.invd);
      } else {
        out = 0.0;
        if (in_grid && n >= 0 && n <= nt) {
          const double row = ADJ ? row_sum<true>(L, n, i, c, pm, v[j], pp, qm, x1, qp)
                                 : row_sum<false>(L, n, i, c, qm, x1, qp, pm, v[j], pp);
          const double id = (n == 0 || i == 0) ? L.inv_w : c.invd;
          out = own + omega * ((fval - row) * id);
        }
      }
      v[j] = out;
      pm = qm;
      pp = qp;
    }
  }
  if (lane >= D && lane <= 31 - D && in_grid) {
    double* yp = y + (n0 * nn + i);
#pragma unroll
    for (int k = 0; k < NT; ++k)
      if (!EDGE || n0 + k < L.n_hi) yp[k * nn] = v[k];
  }
}

template <bool ADJ, int NT, int D>
__global__ void __launch_bounds__(kMaxTW, 3) k_leanD(LevelView L, const double* __restrict__ f,
                                                     const double* __restrict__ x, double* __restrict__ y,
                                                     double omega) {
  pdl_entry();
  const int64_t tt = (int64_t)blockIdx.z * gridDim.y + blockIdx.y;  // time tile
  if (tt >= ceil_div(L.n_hi - L.n_lo, NT)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t first = ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp) * (32 - 2 * D);  // first stored node
  if (first >= L.nn) return;
  const int64_t n0 = L.n_lo + tt * NT, nt = L.n_t;
  const bool rows_in = (ADJ ? (n0 >= 1 && n0 + NT + D - 1 <= nt) : (n0 >= D + 1 && n0 + NT - 1 <= nt)) &&
                       n0 + NT - 1 < L.n_hi;
  const bool nodes_in = first - D + 1 >= 2 && first - D + 30 <= L.n_el - 1;
  if (rows_in && nodes_in) leanD_body<ADJ, NT, D, false>(L, f, x, y, omega, first, n0, lane);
  else leanD_body<ADJ, NT, D, true>(L, f, x, y, omega, first, n0, lane);
}

// Streaming fused pair: two damped-Jacobi sweeps in one pass, bit-identical to
// k_lean2x2 (same overlapping-warp strips: lane l holds node node1 + l - 1,
// sweep 1 valid on lanes 1..30, lanes 2..29 stored), but each warp marches
// its strip through a whole segment [a, b) of S rows instead of an NT-row tile.
// Both sweeps of row m are evaluated in the step that stages level m: sweep 1
// from (x_m, x_{m-1}) and sweep 2 from (y1_m, y1_{m-1}), the coupled level and
// its shuffled neighbours carried in registers from the previous step (J
// marches up in time; J^T couples to m + 1 and marches down).  x and f of the
// next Q rows are in flight in a register queue.  Per stored row this is
// 2 loads, 1 store, 2 row evaluations and 4 shuffles of 64-bit values, with
// one redundant sweep-1 row per segment (k_lean2x2 with NT = 4 evaluates
// 9 rows and re-stages 2 levels per 4 stored rows).
template <bool ADJ, int Q>
__device__ __forceinline__ void march2_body(const LevelView& L, const double* __restrict__ f,
                                            const double* __restrict__ x, double* __restrict__ y,
                                            double omega, int64_t node1, int64_t a, int S, int lane) {
  const int64_t nn = L.nn;
  const int64_t i = node1 + lane - 1;
  const bool lane2 = lane >= 2 && lane <= 29;
  const int64_t dn = ADJ ? -nn : nn;            // element step between consecutive rows
  const int64_t m0 = ADJ ? a + S : a - 1;       // sweep-1-only row
  const Coefs c = load_coefs(L, i);
  const double* px = x + ((m0 - (ADJ ? -1 : 1)) * nn + i);  // its staged coupled level
  const double* pf = f + (m0 * nn + i);
  double* py = y + (m0 * nn + i);
  double xprev = px[0];
  px += dn;
  double x1 = px[0], fm = pf[0];
  px += dn;
  pf += dn;
  double qx[Q], qf[Q];
#pragma unroll
  for (int k = 0; k < Q; ++k) {
    qx[k] = px[0];
    qf[k] = pf[0];
    px += dn;
    pf += dn;
  }
  // row m0: sweep 1 only
  double pm = __shfl_up_sync(kFull, xprev, 1), pp = __shfl_down_sync(kFull, xprev, 1);
  double qm = __shfl_up_sync(kFull, x1, 1), qp = __shfl_down_sync(kFull, x1, 1);
  double y1prev = x1 + omega * ((fm - row_interior<ADJ>(c, qm, x1, qp, pm, xprev, pp)) * c.invd);
  double am = __shfl_up_sync(kFull, y1prev, 1), ap = __shfl_down_sync(kFull, y1prev, 1);
  xprev = x1;
  pm = qm;
  pp = qp;
  py += dn;
  // one queue group of Q rows; PRE: refill the queue with the next group
  auto group = [&](auto pre) {
#pragma unroll
    for (int k = 0; k < Q; ++k) {
      x1 = qx[k];
      fm = qf[k];
      if (decltype(pre)::value) {
        qx[k] = px[0];
        qf[k] = pf[0];
        px += dn;
        pf += dn;
      }
      qm = __shfl_up_sync(kFull, x1, 1);
      qp = __shfl_down_sync(kFull, x1, 1);
      const double y1 = x1 + omega * ((fm - row_interior<ADJ>(c, qm, x1, qp, pm, xprev, pp)) * c.invd);
      const double bm = __shfl_up_sync(kFull, y1, 1), bp = __shfl_down_sync(kFull, y1, 1);
      if (lane2) *py = y1 + omega * ((fm - row_interior<ADJ>(c, bm, y1, bp, am, y1prev, ap)) * c.invd);
      py += dn;
      xprev = x1;
      pm = qm;
      pp = qp;
      y1prev = y1;
      am = bm;
      ap = bp;
    }
  };
  for (int g = Q; g < S; g += Q) group(std::true_type{});
  group(std::false_type{});
}

// Boundary segments (time 0 / n_t, the first or last nodes, a short last
// segment) stream through the same march with the general row evaluation.
// Not inlined: its registers do not count against the interior march's budget.
template <bool ADJ>
__device__ __noinline__ void march2_edge(const LevelView& L, const double* __restrict__ f,
                                         const double* __restrict__ x, double* __restrict__ y,
                                         double omega, int64_t node1, int64_t a, int64_t b) {
  const int lane = threadIdx.x & 31;
  const int64_t nn = L.nn, nt = L.n_t;
  const int64_t i = node1 + lane - 1;
  const bool in_grid = i >= 0 && i < nn;
  const bool lane1 = lane >= 1 && lane <= 30 && in_grid;
  const bool lane2 = lane >= 2 && lane <= 29 && in_grid;
  const int64_t step = ADJ ? -1 : 1;
  const int64_t m0 = ADJ ? b : a - 1;  // first sweep-1 row
  const int64_t s0 = m0 - step;        // its staged coupled level
  Coefs c{};
  if (lane1) c = load_coefs(L, i);
  double xprev = (s0 >= 0 && s0 <= nt && in_grid) ? x[s0 * nn + i] : 0.0;
  double pm = __shfl_up_sync(kFull, xprev, 1), pp = __shfl_down_sync(kFull, xprev, 1);
  double y1prev = 0.0, am = 0.0, ap = 0.0;
  for (int64_t j = 0, m = m0; j <= b - a; ++j, m += step) {
    const bool ok = m >= 0 && m <= nt;
    const double x1 = (ok && in_grid) ? x[m * nn + i] : 0.0;
    const double fm = (ok && lane1) ? f[m * nn + i] : 0.0;
    const double qm = __shfl_up_sync(kFull, x1, 1), qp = __shfl_down_sync(kFull, x1, 1);
    double y1 = 0.0;
    if (lane1 && ok) {
      const double row = row_sum<ADJ>(L, m, i, c, qm, x1, qp, pm, xprev, pp);
      const double id = (m == 0 || i == 0) ? L.inv_w : c.invd;
      y1 = x1 + omega * ((fm - row) * id);
    }
    const double bm = __shfl_up_sync(kFull, y1, 1), bp = __shfl_down_sync(kFull, y1, 1);
    if (j >= 1 && lane2) {
      const double row = row_sum<ADJ>(L, m, i, c, bm, y1, bp, am, y1prev, ap);
      const double id = (m == 0 || i == 0) ? L.inv_w : c.invd;
      y[m * nn + i] = y1 + omega * ((fm - row) * id);
    }
    xprev = x1;
    pm = qm;
    pp = qp;
    y1prev = y1;
    am = bm;
    ap = bp;
  }
}

// seg is a multiple of Q: a segment that touches a boundary or is cut short by
// the end of the level takes march2_edge.
template <bool ADJ, int Q, int MINB>
__global__ void __launch_bounds__(kMaxTW, MINB) k_march2(LevelView L, const double* __restrict__ f,
                                                      const double* __restrict__ x, double* __restrict__ y,
                                                      double omega, int64_t seg) {
  pdl_entry();
  const int64_t tt = (int64_t)blockIdx.z * gridDim.y + blockIdx.y;  // segment
  const int64_t a = L.n_lo + tt * seg;
  if (a >= L.n_hi) return;
  const int64_t b = a + seg < L.n_hi ? a + seg : L.n_hi;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t node1 = (int64_t)blockIdx.x * ((int64_t)(blockDim.x >> 5) * 28) + warp * 28 - 1;
  if (node1 + 1 >= L.nn) return;  // no stored node in this warp
  const int64_t nt = L.n_t;
  // every sweep-1 row has its coupled level and is unmasked; every sweep-1
  // node (lanes 1..30) has both neighbours
  const bool rows_in = ADJ ? (a >= 1 && b <= nt - 1) : (a >= 3);
  const bool nodes_in = node1 >= 2 && node1 + 29 <= L.n_el - 1;
  if (rows_in && nodes_in && b - a == seg) {
    march2_body<ADJ, Q>(L, f, x, y, omega, node1, a, (int)seg, lane);
  } else {
    march2_edge<ADJ>(L, f, x, y, omega, node1, a, b);
  }
}

// f_c = R (f - J x) over one lean tile, R = s P^T (proj/src/transfer.cpp:95-104);
// the fine residual never reaches memory.  x step (DIR 0): lane l computes the
// residual at its node (lane 0 also at the node before its strip, from an
// extra halo), lanes 0..15 gather nodes 2I-1, 2I, 2I+1 of coarse node
// I = wfirst/2 + l by shuffles.  Causal t step (DIR 1): coarse level N takes
// fine levels 2N, 2N+1 at the same node (NT is even, tiles start even).
template <bool ADJ, int DIR, int NT>
__device__ __forceinline__ void dev_lean_restrict(const LevelView& F, const LevelView& C,
                                                  const double* __restrict__ f,
                                                  const double* __restrict__ x,
                                                  double* __restrict__ fc, int64_t bx, int64_t by,
                                                  int tw) {
  if ((int)threadIdx.x >= tw) return;
  const int lane = threadIdx.x & 31;
  const int64_t nn = F.nn, nt = F.n_t, nnc = C.nn;
  const int64_t i = by * tw + threadIdx.x;
  const int64_t n0 = F.n_lo + bx * NT;
  const int64_t nbase = ADJ ? n0 : n0 - 1;
  const int64_t wfirst = i - lane;
  const bool valid = i < nn;
  const int64_t ih = lane == 0 ? i - 1 : i + 1;
  const bool edge = lane == 0 || lane == 31;
  const bool x2 = DIR == 0 && lane == 0 && i >= 2;   // node i - 2 for the extra residual
  const bool xr1 = DIR == 0 && lane == 0 && i >= 1;  // extra residual at node i - 1
  double xr[NT + 1], hr[NT + 1], h2[NT + 1], fv[NT], f1[NT];
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const int64_t n = n0 + k;
    fv[k] = (valid && n < F.n_hi) ? f[n * nn + i] : 0.0;
    f1[k] = (xr1 && n < F.n_hi) ? f[n * nn + i - 1] : 0.0;
  }
#pragma unroll
  for (int r = 0; r <= NT; ++r) {
    const int64_t n = nbase + r;
    const bool nok = n >= 0 && n <= nt;
    xr[r] = (nok && valid) ? x[n * nn + i] : 0.0;
    hr[r] = (nok && edge && ih >= 0 && ih < nn) ? x[n * nn + ih] : 0.0;
    h2[r] = (nok && x2) ? x[n * nn + i - 2] : 0.0;
  }
  Coefs c{}, ch{};
  if (valid) c = load_coefs(F, i);
  if (xr1) ch = load_coefs(F, i - 1);
  // interior tile: every row has its coupled level, every node (incl. lane 0's
  // extra node i - 1) has both same-level neighbours, every coarse node has
  // all three fine contributions -> fixed canonical orders, no branches.
  const bool rows_in = (ADJ ? (n0 >= 1 && n0 + NT - 1 <= nt - 1) : (n0 >= 2 && n0 + NT - 1 <= nt)) &&
                       n0 + NT - 1 < F.n_hi;
  const bool nodes_in = wfirst >= 32 && wfirst + 31 <= F.n_el - 1;
  double pm = __shfl_up_sync(kFull, xr[0], 1);
  double pp = __shfl_down_sync(kFull, xr[0], 1);
  if (lane == 0) pm = hr[0];
  if (lane == 31) pp = hr[0];
  double r_even = 0.0;
  if (rows_in && nodes_in) {
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const int64_t n = n0 + k;
      const double x1 = xr[k + 1];
      double qm = __shfl_up_sync(kFull, x1, 1);
      double qp = __shfl_down_sync(kFull, x1, 1);
      if (lane == 0) qm = hr[k + 1];
      if (lane == 31) qp = hr[k + 1];
      double r;
      if (!ADJ) {
        const double s0 = (0.0 + c.om * pm) + c.c0 * x1;
        const double s1 = (0.0 + c.o0 * xr[k]) + c.cp * qp;
        const double s2 = 0.0 + c.op * pp;
        const double s3 = 0.0 + c.cm * qm;
        r = fv[k] - ((s0 + s1) + (s2 + s3));
      } else {
        const double s0 = (0.0 + c.cm * pm) + c.o0 * x1;
        const double s1 = (0.0 + c.c0 * xr[k]) + c.op * qp;
        const double s2 = 0.0 + c.cp * pp;
        const double s3 = 0.0 + c.om * qm;
        r = fv[k] - ((s0 + s1) + (s2 + s3));
      }
      if (DIR == 0) {
        double r1 = 0.0;
        if (lane == 0) {  // node i - 1: same-level (h2, hr, x) and coupled-level triples
          double t0, t1, t2, t3;
          if (!ADJ) {
            t0 = (0.0 + ch.om * h2[k]) + ch.c0 * hr[k + 1];
            t1 = (0.0 + ch.o0 * hr[k]) + ch.cp * x1;
            t2 = 0.0 + ch.op * xr[k];
            t3 = 0.0 + ch.cm * h2[k + 1];
          } else {
            t0 = (0.0 + ch.cm * h2[k]) + ch.o0 * hr[k + 1];
            t1 = (0.0 + ch.c0 * hr[k]) + ch.op * x1;
            t2 = 0.0 + ch.cp * xr[k];
            t3 = 0.0 + ch.om * h2[k + 1];
          }
          r1 = f1[k] - ((t0 + t1) + (t2 + t3));
        }
        const int src = 2 * lane;
        const double ra = __shfl_sync(kFull, r, (src - 1) & 31);
        const double rb = __shfl_sync(kFull, r, src & 31);
        const double rc = __shfl_sync(kFull, r, (src + 1) & 31);
        if (lane < 16) {
          const int64_t I = wfirst / 2 + lane;
          const double a0 = 0.0 + 0.5 * (lane == 0 ? r1 : ra);
          const double a1 = 0.0 + 1.0 * rb;
          const double a2 = 0.0 + 0.5 * rc;
          fc[n * nnc + I] = (a0 + a1) + (a2 + 0.0);
        }
      } else {
        if ((k & 1) == 0) {
          r_even = r;
        } else {
          const double a0 = 0.0 + 0.5 * r_even;
          const double a1 = 0.0 + 0.5 * r;
          fc[(n >> 1) * nnc + i] = (a0 + a1) + (0.0 + 0.0);
        }
      }
      pm = qm;
      pp = qp;
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const int64_t n = n0 + k;
    if (n >= F.n_hi) break;
    const double x1 = xr[k + 1];
    double qm = __shfl_up_sync(kFull, x1, 1);
    double qp = __shfl_down_sync(kFull, x1, 1);
    if (lane == 0) qm = hr[k + 1];
    if (lane == 31) qp = hr[k + 1];
    // (cur, oth) triples at nodes (i-1, i, i+1): J uses staged k+1 / k, J^T k / k+1
    double r = 0.0;
    if (valid)
      r = fv[k] - (ADJ ? row_sum<true>(F, n, i, c, pm, xr[k], pp, qm, x1, qp)
                       : row_sum<false>(F, n, i, c, qm, x1, qp, pm, xr[k], pp));
    if (DIR == 0) {
      double r1 = 0.0;  // residual at node i - 1 (lane 0): triples at nodes i-2, i-1, i
      if (xr1)
        r1 = f1[k] - (ADJ ? row_sum<true>(F, n, i - 1, ch, h2[k], hr[k], xr[k], h2[k + 1], hr[k + 1], x1)
                          : row_sum<false>(F, n, i - 1, ch, h2[k + 1], hr[k + 1], x1, h2[k], hr[k], xr[k]));
      const int src = 2 * lane;
      const double ra = __shfl_sync(kFull, r, (src - 1) & 31);
      const double rb = __shfl_sync(kFull, r, src & 31);
      const double rc = __shfl_sync(kFull, r, (src + 1) & 31);
      if (lane < 16) {
        const int64_t I = wfirst / 2 + lane;
        if (I < nnc) {
          Acc a;
          if (I >= 1) a.add(0.5 * (lane == 0 ? r1 : ra));
          a.add(1.0 * rb);
          if (2 * I + 1 <= F.n_el) a.add(0.5 * rc);
          fc[n * nnc + I] = a.result();
        }
      }
    } else if (valid) {
      if ((k & 1) == 0) {
        r_even = r;
        if (n == nt) {  // last coarse level: truncated row, 0.5 * r(2N) only
          Acc a;
          a.add(0.5 * r);
          fc[(n >> 1) * nnc + i] = a.result();
        }
      } else {
        Acc a;
        a.add(0.5 * r_even);
        a.add(0.5 * r);
        fc[(n >> 1) * nnc + i] = a.result();
      }
    }
    pm = qm;
    pp = qp;
  }
}

template <bool ADJ, int DIR, int NT>
__global__ void __launch_bounds__(kMaxTW, 2) k_lean_restrict(LevelView F, LevelView C,
                                                             const double* __restrict__ f,
                                                             const double* __restrict__ x,
                                                             double* __restrict__ fc) {
  pdl_entry();
  dev_lean_restrict<ADJ, DIR, NT>(F, C, f, x, fc, blockIdx.x, blockIdx.y, blockDim.x);
}

// Residual + restriction on the overlapping-warp chassis (production).  Lane l
// of a warp holds node base - 1 + l; lanes 1..30 evaluate the fine residual.
// x step (DIR 0): coarse node I = base/2 + j, j = 1..14, takes fine nodes
// 2I-1, 2I, 2I+1 = lanes 2j, 2j+1, 2j+2 (shuffles); warps advance 28 fine
// nodes (14 coarse), base = 28 w - 2 so that warp 0 owns coarse node 0.
// Causal t step (DIR 1): coarse level N = fine levels 2N, 2N+1 at the same
// node; warps advance 30 nodes (NT even, tiles start even).  Interior tiles
// take a predicate-free path with the folded canonical orders; bitwise equal
// to csr_spmv(R, r) of the stored fine residual (proj/src/multigrid.cpp:199).
// First coarse sweep from a zero iterate, 0 + omega (f * inv_diag), at coarse
// DOF (N, I) -- the dev_sweep_from_zero expression, fused into the restriction
// that produces f.
__device__ __forceinline__ double coarse_from_zero(const LevelView& C, int64_t N, int64_t I, double fv,
                                                   double omega) {
  const double id = (N == 0 || I == 0) ? C.inv_w : __ldg(C.coef + kInvD * C.nn + I);
  return 0.0 + omega * (fv * id);
}

template <bool ADJ, int DIR, int NT>
__device__ __forceinline__ void dev_restrict2(const LevelView& F, const LevelView& C,
                                              const double* __restrict__ f, const double* __restrict__ x,
                                              double* __restrict__ fc, int64_t tile, int64_t ttile, int tw,
                                              double* __restrict__ xc0 = nullptr, double omega = 0.0) {
  if ((int)threadIdx.x >= tw) return;
  constexpr int kAdv = DIR == 0 ? 28 : 30;  // nodes per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nn = F.nn, nt = F.n_t, nnc = C.nn;
  const int64_t base = tile * ((tw >> 5) * kAdv) + warp * kAdv + (DIR == 0 ? -2 : 0);
  if (DIR == 0 ? (base / 2 + 1 >= nnc) : (base >= nn)) return;  // whole warp past the grid
  const int64_t i = base - 1 + lane;
  const int64_t n0 = F.n_lo + ttile * NT;
  const int64_t nbase = ADJ ? n0 : n0 - 1;
  const bool rows_in = (ADJ ? (n0 >= 1 && n0 + NT - 1 <= nt - 1) : (n0 >= 2 && n0 + NT - 1 <= nt)) &&
                       n0 + NT - 1 < F.n_hi;
  const bool nodes_in = base >= 2 && base + 29 <= F.n_el - 1;
  double xr[NT + 1], fv[NT];
  if (rows_in && nodes_in) {
    const double* fp = f + (n0 * nn + i);
    const double* xp = x + (nbase * nn + i);
#pragma unroll
    for (int k = 0; k < NT; ++k) fv[k] = fp[k * nn];
#pragma unroll
    for (int r = 0; r <= NT; ++r) xr[r] = xp[r * nn];
    const Coefs c = load_coefs(F, i);
    // coarse inverse diagonal at this lane's coarse node (first coarse sweep from zero)
    double idc = 0.0;
    if (xc0 != nullptr) {
      const int64_t I = DIR == 0 ? base / 2 + lane : i;
      if (DIR == 1 || (lane >= 1 && lane <= 14)) idc = __ldg(C.coef + kInvD * nnc + I);
    }
    double pm = __shfl_up_sync(kFull, xr[0], 1), pp = __shfl_down_sync(kFull, xr[0], 1);
    double r_even = 0.0;
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const double x1 = xr[k + 1];
      const double qm = __shfl_up_sync(kFull, x1, 1), qp = __shfl_down_sync(kFull, x1, 1);
      const double r = fv[k] - (ADJ ? row_interior<true>(c, pm, xr[k], pp, qm, x1, qp)
                                    : row_interior<false>(c, qm, x1, qp, pm, xr[k], pp));
      if (DIR == 0) {
        const int src = 2 * lane;
        const double ra = __shfl_sync(kFull, r, src & 31);
        const double rb = __shfl_sync(kFull, r, (src + 1) & 31);
        const double rc = __shfl_sync(kFull, r, (src + 2) & 31);
        // canonical ((0 + .5 ra) + (0 + rb)) + ((0 + .5 rc) + 0), folded (see row_interior)
        if (lane >= 1 && lane <= 14) {
          const double v = ((0.5 * ra + 1.0 * rb) + 0.5 * rc) + 0.0;
          fc[(n0 + k) * nnc + base / 2 + lane] = v;
          if (xc0 != nullptr) xc0[(n0 + k) * nnc + base / 2 + lane] = 0.0 + omega * (v * idc);
        }
      } else {
        if ((k & 1) == 0) {
          r_even = r;
        } else if (lane >= 1 && lane <= 30) {
          const double v = (0.5 * r_even + 0.5 * r) + 0.0;
          fc[((n0 + k) >> 1) * nnc + i] = v;
          if (xc0 != nullptr) xc0[((n0 + k) >> 1) * nnc + i] = 0.0 + omega * (v * idc);
        }
      }
      pm = qm;
      pp = qp;
    }
    return;
  }
  const bool in_grid = i >= 0 && i < nn;
  const bool computes = lane >= 1 && lane <= 30 && in_grid;
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const int64_t n = n0 + k;
    fv[k] = (computes && n < F.n_hi) ? f[n * nn + i] : 0.0;
  }
#pragma unroll
  for (int r = 0; r <= NT; ++r) {
    const int64_t n = nbase + r;
    xr[r] = (n >= 0 && n <= nt && in_grid) ? x[n * nn + i] : 0.0;
  }
  Coefs c{};
  if (computes) c = load_coefs(F, i);
  double pm = __shfl_up_sync(kFull, xr[0], 1), pp = __shfl_down_sync(kFull, xr[0], 1);
  double r_even = 0.0;
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const int64_t n = n0 + k;
    if (n >= F.n_hi) break;
    const double x1 = xr[k + 1];
    const double qm = __shfl_up_sync(kFull, x1, 1), qp = __shfl_down_sync(kFull, x1, 1);
    double r = 0.0;
    if (computes)
      r = fv[k] - (ADJ ? row_sum<true>(F, n, i, c, pm, xr[k], pp, qm, x1, qp)
                       : row_sum<false>(F, n, i, c, qm, x1, qp, pm, xr[k], pp));
    if (DIR == 0) {
      const int src = 2 * lane;
      const double ra = __shfl_sync(kFull, r, src & 31);
      const double rb = __shfl_sync(kFull, r, (src + 1) & 31);
      const double rc = __shfl_sync(kFull, r, (src + 2) & 31);
      const int64_t I = base / 2 + lane;
      if (lane >= 1 && lane <= 14 && I >= 0 && I < nnc) {
        Acc a;
        if (I >= 1) a.add(0.5 * ra);
        a.add(1.0 * rb);
        if (2 * I + 1 <= F.n_el) a.add(0.5 * rc);
        const double v = a.result();
        fc[n * nnc + I] = v;
        if (xc0 != nullptr) xc0[n * nnc + I] = coarse_from_zero(C, n, I, v, omega);
      }
    } else if (computes) {
      if ((k & 1) == 0) {
        r_even = r;
        if (n == nt) {  // last coarse level: truncated row, 0.5 * r(2N) only
          Acc a;
          a.add(0.5 * r);
          const double v = a.result();
          fc[(n >> 1) * nnc + i] = v;
          if (xc0 != nullptr) xc0[(n >> 1) * nnc + i] = coarse_from_zero(C, n >> 1, i, v, omega);
        }
      } else {
        Acc a;
        a.add(0.5 * r_even);
        a.add(0.5 * r);
        const double v = a.result();
        fc[(n >> 1) * nnc + i] = v;
        if (xc0 != nullptr) xc0[(n >> 1) * nnc + i] = coarse_from_zero(C, n >> 1, i, v, omega);
      }
    }
    pm = qm;
    pp = qp;
  }
}

template <bool ADJ, int DIR, int NT, int MINB = minb_for_nt<NT>()>
__global__ void __launch_bounds__(kMaxTW, MINB) k_restrict2(LevelView F, LevelView C, const double* __restrict__ f,
                                                         const double* __restrict__ x, double* __restrict__ fc,
                                                         double* __restrict__ xc0, double omega) {
  pdl_entry();
  const int64_t tt = (int64_t)blockIdx.z * gridDim.y + blockIdx.y;
  if (tt < ceil_div(F.n_hi - F.n_lo, NT))
    dev_restrict2<ADJ, DIR, NT>(F, C, f, x, fc, blockIdx.x, tt, blockDim.x, xc0, omega);
}

// Elementwise kernels on a level, 2-D grid (no 64-bit division): blockIdx.x =
// time tile of kFlatNT levels, blockIdx.y = node tile of blockDim.x nodes.
constexpr int kFlatNT = 8;

__device__ __forceinline__ void dev_sweep_from_zero(const LevelView& L, const double* __restrict__ f,
                                                    double* __restrict__ y, double omega, int64_t bx,
                                                    int64_t by, int tw) {
  if ((int)threadIdx.x >= tw) return;
  const int64_t i = by * tw + threadIdx.x;
  if (i >= L.nn) return;
  const int64_t n0 = L.n_lo + bx * kFlatNT;
  const double idv = __ldg(L.coef + kInvD * L.nn + i);
#pragma unroll
  for (int k = 0; k < kFlatNT; ++k) {
    const int64_t n = n0 + k;
    if (n >= L.n_hi) break;
    const double id = (n == 0 || i == 0) ? L.inv_w : idv;
    y[n * L.nn + i] = 0.0 + omega * (f[n * L.nn + i] * id);
  }
}

__global__ void k_sweep_from_zero2(LevelView L, const double* __restrict__ f, double* __restrict__ y,
                                   double omega) {
  pdl_entry();
  dev_sweep_from_zero(L, f, y, omega, blockIdx.x, blockIdx.y, blockDim.x);
}

template <int DIR>
__global__ void k_prolong_add2(LevelView F, LevelView C, const double* __restrict__ xc,
                               double* __restrict__ x) {
  pdl_entry();
  const int64_t i = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= F.nn) return;
  const int64_t n0 = F.n_lo + (int64_t)blockIdx.x * kFlatNT;
#pragma unroll
  for (int k = 0; k < kFlatNT; ++k) {
    const int64_t n = n0 + k;
    if (n >= F.n_hi) break;
    x[n * F.nn + i] = x[n * F.nn + i] + prolong_row<DIR>(xc, C.nn, n, i);
  }
}

// ---------------------------------------------------------------------------
// Tiled stencil kernels: blockIdx.x = time tile of NT levels, blockIdx.y =
// node tile of TW = blockDim.x nodes.  Tile row r holds time level nbase + r
// (nbase = n0 - 1 for J, n0 for J^T), so row pairs (r, r + 1) are a level and
// its coupled level.  Every global load of the tile is issued before the
// shared-memory stores, so each thread has ~2 NT + 1 independent loads in
// flight; then one barrier, then the rows are evaluated from shared memory.
// ---------------------------------------------------------------------------
struct TileGeom {
  int64_t i0, n0, nbase;
};

template <bool ADJ, int NT>
__device__ __forceinline__ TileGeom tile_geom() {
  TileGeom g;
  g.i0 = (int64_t)blockIdx.y * blockDim.x;
  g.n0 = (int64_t)blockIdx.x * NT;
  g.nbase = ADJ ? g.n0 : g.n0 - 1;
  return g;
}

template <int NT, int HL, int HR, class Ld>
__device__ __forceinline__ void stage_x(const LevelView& L, const Ld& ld, const TileGeom& g,
                                        double* tile, double (&own)[NT + 1]) {
  const int t = threadIdx.x, tw = blockDim.x, W = tw + HL + HR;
  const int64_t i = g.i0 + t;
  double halo[NT + 1];
  const bool is_halo = t < HL + HR;
  const int64_t ih = t < HL ? g.i0 - HL + t : g.i0 + tw + (t - HL);
  const int hcol = t < HL ? t : HL + tw + (t - HL);
#pragma unroll
  for (int r = 0; r <= NT; ++r) {
    const int64_t n = g.nbase + r;
    const bool nok = n >= 0 && n <= L.n_t;
    own[r] = (nok && i < L.nn) ? ld(n, i) : 0.0;
    halo[r] = (is_halo && nok && ih >= 0 && ih < L.nn) ? ld(n, ih) : 0.0;
  }
#pragma unroll
  for (int r = 0; r <= NT; ++r) {
    tile[r * W + HL + t] = own[r];
    if (is_halo) tile[r * W + hcol] = halo[r];
  }
}

template <bool ADJ, int MODE, bool NORM, int NT, int MINB, class Ld>
__global__ void __launch_bounds__(kMaxTW, MINB) k_tile(LevelView L, Ld ld,
                                                       const double* __restrict__ f,
                                                       double* __restrict__ y, double omega,
                                                       double* __restrict__ partials) {
  pdl_entry();
  extern __shared__ double tile[];
  const TileGeom g = tile_geom<ADJ, NT>();
  const int t = threadIdx.x, W = blockDim.x + 2;
  const int64_t nn = L.nn, nt = L.n_t;
  const int64_t i = g.i0 + t;
  const bool valid = i < nn;
  double own[NT + 1];
  double fv[NT];
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const int64_t n = g.n0 + k;
    fv[k] = (valid && n <= nt) ? f[n * nn + i] : 0.0;
  }
  Coefs c{};
  if (valid) c = load_coefs(L, i);
  stage_x<NT, 1, 1>(L, ld, g, tile, own);
  __syncthreads();
  double acc = 0.0;
  if (valid) {
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const int64_t n = g.n0 + k;
      if (n > nt) break;
      const int rc = ADJ ? k : k + 1;
      const int ro = ADJ ? k + 1 : k;
      const double* cur = tile + rc * W + t;
      const double* oth = tile + ro * W + t;
      const double x0 = own[rc];
      const double row = row_sum<ADJ>(L, n, i, c, cur[0], x0, cur[2], oth[0], oth[1], oth[2]);
      const double r = fv[k] - row;
      if (NORM) acc = acc + r * r;
      if (MODE == kSweep) {
        const double id = (n == 0 || i == 0) ? L.inv_w : c.invd;
        y[n * nn + i] = x0 + omega * (r * id);
      } else if (MODE == kResidual) {
        y[n * nn + i] = r;
      }
    }
  }
  if (NORM) {
    const double s = block_sum(acc);
    if (threadIdx.x == 0) partials[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
  }
}

template <bool ADJ, int DIR, int NT>
__global__ void __launch_bounds__(kMaxTW) k_restrict_tile(LevelView F, LevelView C,
                                                          const double* __restrict__ f,
                                                          const double* __restrict__ x,
                                                          double* __restrict__ fc) {
  pdl_entry();
  extern __shared__ double smem[];
  const TileGeom g = tile_geom<ADJ, NT>();
  const int t = threadIdx.x, tw = blockDim.x;
  const int64_t nn = F.nn, nt = F.n_t, nnc = C.nn;
  const PlainLoad ld{x, nn};
  constexpr int HL = DIR == 0 ? 2 : 1;
  const int W = tw + HL + 1;
  double* tile = smem;
  double own[NT + 1];
  const int64_t i = g.i0 + t;
  double fv[NT], fh[NT];
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const int64_t n = g.n0 + k;
    fv[k] = (i < nn && n <= nt) ? f[n * nn + i] : 0.0;
    fh[k] = (DIR == 0 && t == 0 && g.i0 >= 1 && n <= nt) ? f[n * nn + g.i0 - 1] : 0.0;
  }
  Coefs c{}, ch{};
  if (i < nn) c = load_coefs(F, i);
  if (DIR == 0 && t == 0 && g.i0 >= 1) ch = load_coefs(F, g.i0 - 1);
  stage_x<NT, HL, 1>(F, ld, g, tile, own);
  __syncthreads();
  auto resid = [&](int k, int col, int64_t node, const Coefs& cc, double fval) -> double {
    const int64_t n = g.n0 + k;
    const int rc = ADJ ? k : k + 1;
    const int ro = ADJ ? k + 1 : k;
    const double* cur = tile + rc * W + col;
    const double* oth = tile + ro * W + col;
    return fval - row_sum<ADJ>(F, n, node, cc, cur[-1], cur[0], cur[1], oth[-1], oth[0], oth[1]);
  };
  if (DIR == 0) {
    double* R = smem + (NT + 1) * W;  // NT rows x (tw + 1): column j <-> node i0 - 1 + j
    const int RW = tw + 1;
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      if (g.n0 + k > nt) break;
      if (i < nn) R[k * RW + t + 1] = resid(k, HL + t, i, c, fv[k]);
      if (t == 0) R[k * RW] = g.i0 >= 1 ? resid(k, HL - 1, g.i0 - 1, ch, fh[k]) : 0.0;
    }
    __syncthreads();
    if (t < tw / 2) {
      const int64_t I = g.i0 / 2 + t;
      if (I < nnc) {
#pragma unroll
        for (int k = 0; k < NT; ++k) {
          const int64_t n = g.n0 + k;
          if (n > nt) break;
          const double* rr = R + k * RW + 2 * t;  // nodes 2I-1, 2I, 2I+1
          Acc a;
          if (I >= 1) a.add(0.5 * rr[0]);
          a.add(1.0 * rr[1]);
          if (2 * I + 1 <= F.n_el) a.add(0.5 * rr[2]);
          fc[n * nnc + I] = a.result();
        }
      }
    }
  } else {
    if (i >= nn) return;
    double rv[NT];
#pragma unroll
    for (int k = 0; k < NT; ++k) rv[k] = (g.n0 + k <= nt) ? resid(k, HL + t, i, c, fv[k]) : 0.0;
#pragma unroll
    for (int s2 = 0; s2 < NT / 2; ++s2) {
      const int64_t n2 = g.n0 + 2 * s2;  // fine level 2N
      if (n2 > nt) break;
      Acc a;
      a.add(0.5 * rv[2 * s2]);
      if (n2 + 1 <= nt) a.add(0.5 * rv[2 * s2 + 1]);
      fc[(n2 / 2) * nnc + i] = a.result();
    }
  }
}

// Streaming stencil kernels.  Block (blockIdx.x, blockIdx.y) covers node tile
// [i0, i0 + TW) (TW = blockDim.x) for rows n in [nA, nB), a long chunk of time
// levels; each warp streams its own 32-node strip through the chunk with no
// block barrier (a barrier would wait on the prefetched loads).  A rolling
// register queue keeps the next kQ levels' loads in flight (x, f, and the
// strip-edge halo nodes loaded by lanes 0 and 31), so every vector element is
// read from HBM once per pass with ~2 kQ independent loads per thread
// outstanding.  Same-level neighbours come from warp shuffles.
//   J   (ADJ = false): step j stages level m = nA - 1 + j, computes row m.
//   J^T (ADJ = true) : step j stages level m = nA + j,     computes row m - 1.
constexpr int kQ = 8;  // prefetch depth (levels)

struct StreamGeom {
  int64_t i0, nA, nB, first, count;
};

template <bool ADJ>
__device__ __forceinline__ StreamGeom stream_geom(const LevelView& L, int64_t chunk) {
  StreamGeom g;
  g.i0 = (int64_t)blockIdx.y * blockDim.x;
  g.nA = (int64_t)blockIdx.x * chunk;
  g.nB = g.nA + chunk < L.n_t + 1 ? g.nA + chunk : L.n_t + 1;
  g.first = ADJ ? g.nA : g.nA - 1;
  g.count = g.nB - g.nA + 1;  // levels staged; rows computed at steps 1 .. count-1
  return g;
}

// One staged level as seen by a lane: x at i-1, i, i+1, and (X2, lane 0 of a
// strip only) x at i-2 plus f at i-1 for the extra residual of restriction.
struct Staged {
  double xm, x0, xp, x2, f, f1;
};

// Drives the per-level pipeline of a warp strip and calls
// body(m, cur, prev) for every staged level m after the first, where cur is
// level m and prev level m - 1.
template <bool X2, class Ld, class Body>
__device__ __forceinline__ void warp_stream(const LevelView& L, const Ld& ld,
                                            const double* __restrict__ f, const StreamGeom& g,
                                            Body&& body) {
  const int lane = threadIdx.x & 31;
  const int64_t nn = L.nn;
  const int64_t i = g.i0 + threadIdx.x;
  const bool own_ok = i < nn;
  // lane 0 loads i-1 (and i-2), lane 31 loads i+1
  const int64_t ih = lane == 0 ? i - 1 : i + 1;
  const bool has_h = (lane == 0 || lane == 31) && ih >= 0 && ih < nn;
  const bool has_h2 = X2 && lane == 0 && i - 2 >= 0 && i - 2 < nn;
  const bool has_f1 = X2 && lane == 0 && i - 1 >= 0 && i - 1 < nn;
  double qx[kQ], qh[kQ], qf[kQ], qx2[kQ], qf1[kQ];
  auto load = [&](int64_t m, int k) {
    const bool mok = m >= 0 && m <= L.n_t;
    qx[k] = (mok && own_ok) ? ld(m, i) : 0.0;
    qh[k] = (mok && has_h) ? ld(m, ih) : 0.0;
    qf[k] = (mok && own_ok) ? f[m * nn + i] : 0.0;
    if (X2) {
      qx2[k] = (mok && has_h2) ? ld(m, i - 2) : 0.0;
      qf1[k] = (mok && has_f1) ? f[m * nn + i - 1] : 0.0;
    }
  };
#pragma unroll
  for (int k = 0; k < kQ; ++k)
    if (k < g.count) load(g.first + k, k);
  Staged prev{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int64_t base = 0; base < g.count; base += kQ) {
#pragma unroll
    for (int k = 0; k < kQ; ++k) {
      const int64_t j = base + k;
      if (j >= g.count) break;
      Staged cur;
      cur.x0 = qx[k];
      const double h = qh[k];
      cur.f = qf[k];
      cur.x2 = X2 ? qx2[k] : 0.0;
      cur.f1 = X2 ? qf1[k] : 0.0;
      if (j + kQ < g.count) load(g.first + j + kQ, k);
      cur.xm = __shfl_up_sync(kFull, cur.x0, 1);
      cur.xp = __shfl_down_sync(kFull, cur.x0, 1);
      if (lane == 0) cur.xm = h;
      if (lane == 31) cur.xp = h;
      if (j >= 1) body(g.first + j, cur, prev);
      prev = cur;
    }
  }
}

// Damped-Jacobi sweep / residual / residual-norm pass over a level.
template <bool ADJ, int MODE, bool NORM, class Ld>
__global__ void __launch_bounds__(kMaxTW, 2) k_stream(LevelView L, Ld ld, const double* __restrict__ f,
                                                      double* __restrict__ y, double omega,
                                                      double* __restrict__ partials, int64_t chunk) {
  pdl_entry();
  const StreamGeom g = stream_geom<ADJ>(L, chunk);
  const int64_t nn = L.nn;
  const int64_t i = g.i0 + threadIdx.x;
  const bool valid = i < nn;
  Coefs c{};
  if (valid) c = load_coefs(L, i);
  double acc = 0.0;
  warp_stream<false>(L, ld, f, g, [&](int64_t m, const Staged& cu, const Staged& pv) {
    if (!valid) return;
    const int64_t n = ADJ ? m - 1 : m;  // row
    const Staged& rowl = ADJ ? pv : cu;  // level n
    const Staged& oth = ADJ ? cu : pv;   // coupled level
    const double row = row_sum<ADJ>(L, n, i, c, rowl.xm, rowl.x0, rowl.xp, oth.xm, oth.x0, oth.xp);
    const double r = rowl.f - row;
    if (NORM) acc = acc + r * r;
    if (MODE == kSweep) {
      const double id = (n == 0 || i == 0) ? L.inv_w : c.invd;
      y[n * nn + i] = rowl.x0 + omega * (r * id);
    } else if (MODE == kResidual) {
      y[n * nn + i] = r;
    }
  });
  if (NORM) {
    const double s = block_sum(acc);
    if (threadIdx.x == 0) partials[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
  }
}

// f_c = R (f - J x), R = s P^T (proj/src/transfer.cpp:95-104); the fine
// residual never reaches memory.  x step (DIR 0): lane l of a strip computes
// the residual at node i0 + l (lane 0 also at i0 - 1), lanes 0..15 then gather
// nodes 2I-1, 2I, 2I+1 of coarse node I = (i0 + 2l) / 2 by shuffles.  Causal t
// step (DIR 1): coarse level N = (fine 2N, fine 2N+1) at the same node; time
// chunks are even so pairs never straddle blocks.
template <bool ADJ, int DIR>
__global__ void __launch_bounds__(kMaxTW, 2) k_restrict_stream(LevelView F, LevelView C,
                                                               const double* __restrict__ f,
                                                               const double* __restrict__ x,
                                                               double* __restrict__ fc,
                                                               int64_t chunk) {
  pdl_entry();
  const StreamGeom g = stream_geom<ADJ>(F, chunk);
  const int lane = threadIdx.x & 31;
  const int64_t nn = F.nn, nnc = C.nn;
  const int64_t i = g.i0 + threadIdx.x;
  const int64_t istrip = i - lane;  // first node of this warp's strip (even)
  const bool valid = i < nn;
  const PlainLoad ld{x, nn};
  Coefs c{}, ch{};
  if (valid) c = load_coefs(F, i);
  if (DIR == 0 && lane == 0 && i >= 1 && i - 1 < nn) ch = load_coefs(F, i - 1);
  double r_even = 0.0;
  warp_stream<DIR == 0>(F, ld, f, g, [&](int64_t m, const Staged& cu, const Staged& pv) {
    const int64_t n = ADJ ? m - 1 : m;
    const Staged& rowl = ADJ ? pv : cu;
    const Staged& oth = ADJ ? cu : pv;
    double r = 0.0;
    if (valid)
      r = rowl.f - row_sum<ADJ>(F, n, i, c, rowl.xm, rowl.x0, rowl.xp, oth.xm, oth.x0, oth.xp);
    if (DIR == 0) {
      double r1 = 0.0;  // residual at node i - 1 (lane 0 only)
      if (lane == 0 && i >= 1 && i - 1 < nn)
        r1 = rowl.f1 - row_sum<ADJ>(F, n, i - 1, ch, rowl.x2, rowl.xm, rowl.x0, oth.x2, oth.xm,
                                    oth.x0);
      // lane l < 16: coarse node I = istrip/2 + l needs r at fine lanes 2l-1, 2l, 2l+1
      const int src = 2 * lane;
      const double ra = __shfl_sync(kFull, r, (src - 1) & 31);
      const double rb = __shfl_sync(kFull, r, src & 31);
      const double rc = __shfl_sync(kFull, r, (src + 1) & 31);
      if (lane < 16) {
        const int64_t I = istrip / 2 + lane;
        if (I < nnc && 2 * I <= F.n_el) {
          const double rm1 = lane == 0 ? r1 : ra;
          Acc a;
          if (I >= 1) a.add(0.5 * rm1);
          a.add(1.0 * rb);
          if (2 * I + 1 <= F.n_el) a.add(0.5 * rc);
          fc[n * nnc + I] = a.result();
        }
      }
    } else {
      if (!valid) return;
      if ((n & 1) == 0) {
        r_even = r;
        if (n == F.n_t) {  // last coarse level: truncated row (0.5 * r(2N) only)
          Acc a;
          a.add(0.5 * r);
          fc[(n >> 1) * nnc + i] = a.result();
        }
      } else {
        Acc a;
        a.add(0.5 * r_even);
        a.add(0.5 * r);
        fc[(n >> 1) * nnc + i] = a.result();
      }
    }
  });
}

__global__ void k_sweep_from_zero(LevelView L, const double* __restrict__ f, double* __restrict__ y,
                                  double omega, int64_t total) {
  pdl_entry();
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
  pdl_entry();
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
  pdl_entry();
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
  pdl_entry();
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

// ---------------------------------------------------------------------------
// Bulk-copy pipelined fused sweeps (k_bulk): the k_leanD computation (depth D,
// overlapping warps, canonical row order -- bit-identical to D separate
// sweeps), fed by cp.async.bulk copies of whole tile rows into a STAGES-deep
// shared-memory ring instead of per-thread global loads.  The CTAs are
// persistent (grid = resident CTAs) and walk the tiles node-tile fastest; warp
// 0 refills a stage as soon as every warp has moved the stage's values into
// registers, so the copies of the next STAGES - 1 tiles are in flight while a
// tile is computed.  One copy per staged row: x rows sbase .. sbase+S-1, f rows
// fbase .. fbase+F-1 of the nodes node0 .. node0+WN-1, the source rounded out
// to 16-byte boundaries (the smem row carries a 0/1-element shift).  Vectors
// are allocated with kVecPad doubles of tail padding so the rounding never
// leaves the allocation; out-of-grid nodes are never used (EDGE path).
// Full-range levels only.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int NT, int D, int W>
struct BulkGeom {
  static constexpr int S = NT + D;           // staged x rows
  static constexpr int F = NT + D - 1;       // f rows
  static constexpr int ROWS = S + F + kNumCoef;  // x rows, f rows, the 7 coefficient rows
  static constexpr int STORED = 32 - 2 * D;  // stored nodes per warp
  static constexpr int WN = W * STORED + 2 * D;
  static constexpr int RW = WN + 2;          // even: rows stay 16-byte aligned
  static constexpr int STAGE = ROWS * RW;    // doubles per stage
};

// Source range of staged row r of a tile: [gstart, gstart + bytes / 8), and the
// shift of node0 inside the smem row.
struct RowCopy {
  int64_t gstart;
  uint32_t bytes;
  int shift;
};
template <bool ADJ, int NT, int D, int W>
__device__ __forceinline__ RowCopy bulk_row(const LevelView& L, int r, int64_t n0, int64_t node0) {
  using G = BulkGeom<NT, D, W>;
  const int64_t sbase = ADJ ? n0 : n0 - D;
  const int64_t fbase = ADJ ? n0 : n0 - D + 1;
  RowCopy rc{0, 0u, 0};
  if (r >= G::ROWS) return rc;
  int64_t gs;
  if (r >= G::S + G::F) {  // coefficient array k = r - S - F: coef + k nn + node
    gs = (r - G::S - G::F) * L.nn + node0;
  } else {
    const int64_t n = r < G::S ? sbase + r : fbase + (r - G::S);
    if (n < 0 || n > L.n_t) return rc;
    gs = n * L.nn + node0;
  }
  const int64_t g0 = (gs < 0 ? 0 : gs) & ~int64_t{1};
  const int64_t g1 = (gs + G::WN + 1) & ~int64_t{1};
  rc.gstart = g0;
  rc.bytes = static_cast<uint32_t>((g1 - g0) * 8);
  rc.shift = static_cast<int>(gs - g0);
  return rc;
}

template <bool ADJ, int NT, int D, int W, bool EDGE>
__device__ __forceinline__ void bulk_body(const LevelView& L, const double* stage, double* __restrict__ y,
                                          double omega, int64_t n0, int64_t node0, int warp, int lane,
                                          uint64_t* empty_bar) {
  using G = BulkGeom<NT, D, W>;
  constexpr int S = G::S, F = G::F;
  const int64_t nn = L.nn, nt = L.n_t;
  const int q = warp * G::STORED + lane;  // smem position of this lane's node
  const int64_t i = node0 + q;
  const int64_t sbase = ADJ ? n0 : n0 - D;
  const int64_t fbase = ADJ ? n0 : n0 - D + 1;
  const bool in_grid = !EDGE || (i >= 0 && i < nn);
  double v[S], fv[F];
  // smem shift of a row: gs - (max(gs, 0) & ~1), gs = n nn + node0 (bulk_row)
  auto shift = [&](int64_t n) -> int {
    const int64_t gs = n * nn + node0;
    return gs < 0 ? static_cast<int>(gs) : static_cast<int>(gs & 1);
  };
  auto shift_c = [&](int k) -> int { return shift(k); };  // coefficient row k starts at k nn
#pragma unroll
  for (int j = 0; j < S; ++j) {
    const int64_t n = sbase + j;
    const bool ok = !EDGE || (in_grid && n >= 0 && n <= nt);
    v[j] = ok ? stage[j * G::RW + q + shift(n)] : 0.0;
  }
#pragma unroll
  for (int j = 0; j < F; ++j) {
    const int64_t n = fbase + j;
    const bool ok = !EDGE || (in_grid && n >= 0 && n <= nt);
    fv[j] = ok ? stage[(S + j) * G::RW + q + shift(n)] : 0.0;
  }
  Coefs c{};
  if (in_grid) {
    const double* cr = stage + (S + F) * G::RW + q;
    auto coef = [&](int k) { return cr[k * G::RW + shift_c(k)]; };
    c.cm = coef(kCm);
    c.c0 = coef(kC0);
    c.cp = coef(kCp);
    c.om = coef(kOm);
    c.o0 = coef(kO0);
    c.op = coef(kOp);
    c.invd = coef(kInvD);
  }
  // this warp's values are in registers: release the stage to the producer
  __syncwarp();
  if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty_bar)) : "memory");
#pragma unroll
  for (int st = 1; st <= D; ++st) {
    double pm = __shfl_up_sync(kFull, v[0], 1), pp = __shfl_down_sync(kFull, v[0], 1);
#pragma unroll
    for (int j = 0; j < S - st; ++j) {
      const double x1 = v[j + 1];
      const double qm = __shfl_up_sync(kFull, x1, 1), qp = __shfl_down_sync(kFull, x1, 1);
      const int64_t n = ADJ ? sbase + j : sbase + st + j;
      const double fval = ADJ ? fv[j] : fv[st - 1 + j];
      const double own = ADJ ? v[j] : x1;
      double out;
      if (!EDGE) {
        const double row = ADJ ? row_interior<true>(c, pm, v[j], pp, qm, x1, qp)
                               : row_interior<false>(c, qm, x1, qp, pm, v[j], pp);
        out = own + omega * ((fval - row) * c.invd);
      } else {
        out = 0.0;
        if (in_grid && n >= 0 && n <= nt) {
          const double row = ADJ ? row_sum<true>(L, n, i, c, pm, v[j], pp, qm, x1, qp)
                                 : row_sum<false>(L, n, i, c, qm, x1, qp, pm, v[j], pp);
          const double id = (n == 0 || i == 0) ? L.inv_w : c.invd;
          out = own + omega * ((fval - row) * id);
        }
      }
      v[j] = out;
      pm = qm;
      pp = qp;
    }
  }
  if (lane >= D && lane <= 31 - D && in_grid) {
    double* yp = y + (n0 * nn + i);
#pragma unroll
    for (int k = 0; k < NT; ++k)
      if (!EDGE || n0 + k <= nt) yp[k * nn] = v[k];
  }
}

// Tile walk of a persistent CTA: tiles blockIdx.x, +gridDim.x, ... (node tile
// fastest), advanced without 64-bit division.
struct TileWalk {
  int64_t tn, tt, step_tn, step_tt, nnt;
  __device__ __forceinline__ TileWalk(int64_t first, int64_t step, int64_t n_node_tiles)
      : tn(first % n_node_tiles), tt(first / n_node_tiles), step_tn(step % n_node_tiles),
        step_tt(step / n_node_tiles), nnt(n_node_tiles) {}
  __device__ __forceinline__ void next() {
    tn += step_tn;
    tt += step_tt;
    if (tn >= nnt) {
      tn -= nnt;
      ++tt;
    }
  }
};

// Warp-specialised: warp W is the producer (bulk copies into a STAGES-deep
// ring, full barriers with transaction counts), warps 0..W-1 consume (wait full,
// move the tile into registers, arrive on the stage's empty barrier, compute).
// No CTA-wide barrier inside the tile loop.
template <bool ADJ, int NT, int D, int W, int STAGES, int MINB>
__global__ void __launch_bounds__((W + 1) * 32, MINB) k_bulk(LevelView L, const double* __restrict__ f,
                                                            const double* __restrict__ x, double* __restrict__ y,
                                                            double omega, int64_t n_node_tiles, int64_t n_time_tiles) {
  using G = BulkGeom<NT, D, W>;
  extern __shared__ __align__(128) double bsm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(bsm + STAGES * G::STAGE);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < STAGES) {
    mbar_init(&full[threadIdx.x], 1);
    mbar_init(&empty[threadIdx.x], W);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  pdl_entry();
  const int64_t nt = L.n_t;
  TileWalk tw(blockIdx.x, gridDim.x, n_node_tiles);
  if (warp == W) {  // producer
    for (int64_t k = 0; tw.tt < n_time_tiles; ++k, tw.next()) {
      const int st = static_cast<int>(k % STAGES);
      if (k >= STAGES) mbar_wait_parity(&empty[st], static_cast<uint32_t>(((k / STAGES) - 1) & 1));
      const int64_t n0 = tw.tt * NT, node0 = tw.tn * (W * G::STORED) - D;
      const RowCopy rc = bulk_row<ADJ, NT, D, W>(L, lane, n0, node0);
      const uint32_t total = __reduce_add_sync(kFull, rc.bytes);
      if (lane == 0) mbar_arrive_expect_tx(&full[st], total);
      __syncwarp();
      if (rc.bytes) {
        const double* src = lane < G::S ? x : lane < G::S + G::F ? f : L.coef;
        bulk_g2s(bsm + st * G::STAGE + lane * G::RW, src + rc.gstart, rc.bytes, &full[st]);
      }
    }
    return;
  }
  for (int64_t k = 0; tw.tt < n_time_tiles; ++k, tw.next()) {
    const int st = static_cast<int>(k % STAGES);
    mbar_wait_parity(&full[st], static_cast<uint32_t>((k / STAGES) & 1));
    const int64_t n0 = tw.tt * NT, node0 = tw.tn * (W * G::STORED) - D;
    const double* stage = bsm + st * G::STAGE;
    const bool rows_in = ADJ ? (n0 >= 1 && n0 + NT + D - 1 <= nt) : (n0 >= D + 1 && n0 + NT - 1 <= nt);
    const int64_t first = node0 + warp * G::STORED + 1;  // lane 1's node
    const bool nodes_in = first >= 2 && first + 29 <= L.n_el - 1;
    if (rows_in && nodes_in) bulk_body<ADJ, NT, D, W, false>(L, stage, y, omega, n0, node0, warp, lane, &empty[st]);
    else bulk_body<ADJ, NT, D, W, true>(L, stage, y, omega, n0, node0, warp, lane, &empty[st]);
  }
}

// Parallel-in-time exact march for wide coarsest levels (n_el > 32).  The march
// x_n = T^-1 (f_n - S x_{n'}) (n' the coupled level) is affine in its start
// state, so the n_t steps are cut into C chunks of Lc steps:
//   PHASE 0 (C CTAs): each chunk marches from a zero start state (chunk 0's first
//     step is uncoupled, so chunk 0 is exact); CTA 0 also writes masked rows;
//   link (1 CTA): true chunk-end states s_c = y_end(c) + A^Lc s_{c-1};
//   PHASE 1 (C - 1 CTAs): chunk c >= 1 adds the homogeneous march from s_{c-1},
//     z_k = T^-1 (-S z_{k-1}), to its levels.
// Sequential depth 2 Lc + C instead of n_t.  Per step one tridiagonal solve by
// PCR over shared memory with the host-precomputed factors (as k_coarsest); the
// state stays in shared memory.  An exact solve like the reference's SparseLU,
// agreeing to rounding.
template <bool ADJ, int PHASE>
__global__ void __launch_bounds__(1024) k_coarsest_pint(CoarsestView cv, const double* __restrict__ f,
                                                        double* __restrict__ x,
                                                        const double* __restrict__ starts) {
  pdl_entry();
  extern __shared__ double smem[];
  const LevelView& L = cv.lv;
  const int m = cv.m;
  const int64_t nn = L.nn, nt = L.n_t;
  const int tid = threadIdx.x, bs = blockDim.x;
  // PHASE 2 (propagator build): CTA e marches the unit vector e through Lc
  // homogeneous steps and stores the result as column e of A^Lc (in `x`).
  const int c = PHASE == 0 ? blockIdx.x : blockIdx.x + 1;
  double* prev = smem;
  double* d0 = smem + m;
  double* d1 = smem + 2 * m;
  if (PHASE == 0 && c == 0) {
    for (int64_t i = tid; i < nn; i += bs) x[i] = f[i] / L.w;
    for (int64_t n = 1 + tid; n <= nt; n += bs) x[n * nn] = f[n * nn] / L.w;
  }
  for (int j = tid; j < m; j += bs)
    prev[j] = PHASE == 0 ? 0.0 : PHASE == 2 ? (j == (int)blockIdx.x ? 1.0 : 0.0) : starts[(int64_t)(c - 1) * m + j];
  const double* om = L.coef + kOm * nn;
  const double* o0 = L.coef + kO0 * nn;
  const double* op = L.coef + kOp * nn;
  const int64_t s0 = (int64_t)c * cv.pint_len + 1;
  __syncthreads();
  for (int64_t s = s0; s < s0 + cv.pint_len; ++s) {
    const int64_t n = ADJ ? nt + 1 - s : s;
    const bool coupled = PHASE == 2 || s >= 2;
    for (int j = tid; j < m; j += bs) {
      const int64_t i = j + 1;
      double acc = PHASE == 0 ? f[n * nn + i] : 0.0;
      if (coupled) {
        if (i >= 2) acc = acc - om[i] * prev[j - 1];
        acc = acc - o0[i] * prev[j];
        if (i <= m - 1) acc = acc - op[i] * prev[j + 1];
      }
      d0[j] = acc;
    }
    __syncthreads();
    double* a = d0;
    double* b = d1;
    for (int k = 0; k < cv.n_steps; ++k) {
      const int st = 1 << k;
      for (int j = tid; j < m; j += bs) {
        double v = a[j];
        if (j - st >= 0) v = v + cv.alpha[(int64_t)k * m + j] * a[j - st];
        if (j + st < m) v = v + cv.gamma[(int64_t)k * m + j] * a[j + st];
        b[j] = v;
      }
      __syncthreads();
      double* t = a;
      a = b;
      b = t;
    }
    for (int j = tid; j < m; j += bs) {
      const double v = a[j] / cv.bfin[j];
      prev[j] = v;
      if (PHASE != 2) {
        double* xp = x + n * nn + j + 1;
        *xp = PHASE == 0 ? v : *xp + v;
      }
    }
    __syncthreads();
  }
  if (PHASE == 2)
    for (int j = tid; j < m; j += bs) x[(int64_t)blockIdx.x * m + j] = prev[j];
}

// Chunk links of k_coarsest_pint by a Kogge-Stone scan.  The true end state of
// chunk c is s_c = sum_{j <= c} Q^(c-j) y_j (y_j: PHASE 0's end state of chunk j,
// Q = A^Lc).  Round r (stride d = 2^r) maps v_c <- v_c + Q^d v_{c-d} for c >= d,
// starting from v = y; after ceil(log2 C) rounds v_c = s_c.  One CTA per chunk,
// the matvec rows across threads (Q^d column-major, coalesced), the operand
// vector in shared memory.  Round 0 reads y from the chunk end levels of x.
template <bool ADJ>
__global__ void __launch_bounds__(1024) k_coarsest_pint_round(CoarsestView cv, const double* __restrict__ x,
                                                              const double* __restrict__ vin,
                                                              double* __restrict__ vout, int r) {
  pdl_entry();
  extern __shared__ double sv[];
  const int m = cv.m;
  const int64_t nn = cv.lv.nn, nt = cv.lv.n_t;
  const int c = blockIdx.x, tid = threadIdx.x, bs = blockDim.x;
  const int d = 1 << r;
  auto end_row = [&](int64_t cc) -> const double* {
    const int64_t s = (cc + 1) * cv.pint_len;
    return x + (ADJ ? nt + 1 - s : s) * nn + 1;
  };
  const double* own = r == 0 ? end_row(c) : vin + (int64_t)c * m;
  if (c < d) {
    for (int j = tid; j < m; j += bs) vout[(int64_t)c * m + j] = own[j];
    return;
  }
  const double* src = r == 0 ? end_row(c - d) : vin + (int64_t)(c - d) * m;
  for (int j = tid; j < m; j += bs) sv[j] = src[j];
  __syncthreads();
  const double* Q = cv.pint_pow + (int64_t)r * m * m;
  for (int j = tid; j < m; j += bs) {
    double acc = own[j];
    for (int k = 0; k < m; ++k) acc = fma(Q[(int64_t)k * m + j], sv[k], acc);
    vout[(int64_t)c * m + j] = acc;
  }
}

// C = A B for column-major m x m (the propagator squares; one-off per hierarchy).
__global__ void k_square(const double* __restrict__ A, double* __restrict__ C, int m) {
  __shared__ double ta[16][17], tb[16][17];
  const int i = blockIdx.y * 16 + threadIdx.y, j = blockIdx.x * 16 + threadIdx.x;
  double acc = 0.0;
  for (int k0 = 0; k0 < m; k0 += 16) {
    // A(i, k) at k * m + i; B = A
    ta[threadIdx.y][threadIdx.x] = (i < m && k0 + threadIdx.x < m) ? A[(int64_t)(k0 + threadIdx.x) * m + i] : 0.0;
    tb[threadIdx.y][threadIdx.x] = (k0 + threadIdx.y < m && j < m) ? A[(int64_t)j * m + k0 + threadIdx.y] : 0.0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) acc = fma(ta[threadIdx.y][k], tb[k][threadIdx.x], acc);
    __syncthreads();
  }
  if (i < m && j < m) C[(int64_t)j * m + i] = acc;
}

// Coarsest exact solve for n_el <= 32: one warp, lane j owns unmasked node
// j + 1.  Per time level: right-hand side with the coupled level's values
// (shuffles), then PCR by shuffles with the same precomputed factors and the
// same operation order as k_coarsest, so both give identical results; f is
// prefetched kPF levels ahead because the march itself is sequential.
constexpr int kPF = 8;

template <bool ADJ>
__global__ void __launch_bounds__(32) k_coarsest_warp(CoarsestView cv, const double* __restrict__ f,
                                                      double* __restrict__ x) {
  pdl_entry();
  const LevelView& L = cv.lv;
  const int m = cv.m;
  const int64_t nn = L.nn, nt = L.n_t;
  const int j = threadIdx.x;
  const int64_t i = j + 1;
  const bool active = j < m;
  for (int64_t k = j; k < nn; k += 32) x[k] = f[k] / L.w;
  for (int64_t n = 1 + j; n <= nt; n += 32) x[n * nn] = f[n * nn] / L.w;
  double al[5] = {0, 0, 0, 0, 0}, ga[5] = {0, 0, 0, 0, 0};
  double om = 0, o0 = 0, op = 0, bf = 1.0;
  if (active) {
#pragma unroll
    for (int k = 0; k < 5; ++k)
      if (k < cv.n_steps) {
        al[k] = cv.alpha[(int64_t)k * m + j];
        ga[k] = cv.gamma[(int64_t)k * m + j];
      }
    om = L.coef[kOm * nn + i];
    o0 = L.coef[kO0 * nn + i];
    op = L.coef[kOp * nn + i];
    bf = cv.bfin[j];
  }
  double q[kPF];
#pragma unroll
  for (int k = 0; k < kPF; ++k) {
    const int64_t s = 1 + k;
    const int64_t n = ADJ ? nt + 1 - s : s;
    q[k] = (active && s <= nt) ? f[n * nn + i] : 0.0;
  }
  double xprev = 0.0;
  for (int64_t base = 1; base <= nt; base += kPF) {
#pragma unroll
    for (int k = 0; k < kPF; ++k) {
      const int64_t s = base + k;
      if (s > nt) break;
      const int64_t n = ADJ ? nt + 1 - s : s;
      const bool coupled = ADJ ? (n + 1 <= nt) : (n - 1 >= 1);
      double acc = q[k];
      const int64_t s2 = s + kPF;
      if (s2 <= nt) {
        const int64_t n2 = ADJ ? nt + 1 - s2 : s2;
        q[k] = active ? f[n2 * nn + i] : 0.0;
      }
      const double xm = __shfl_up_sync(kFull, xprev, 1);
      const double xp = __shfl_down_sync(kFull, xprev, 1);
      if (coupled) {
        if (i >= 2) acc = acc - om * xm;
        acc = acc - o0 * xprev;
        if (i <= m - 1) acc = acc - op * xp;
      }
      double d = acc;
#pragma unroll
      for (int st = 0; st < 5; ++st) {
        if (st >= cv.n_steps) break;
        const int sh = 1 << st;
        const double dm = __shfl_up_sync(kFull, d, sh);
        const double dp = __shfl_down_sync(kFull, d, sh);
        double v = d;
        if (j - sh >= 0) v = v + al[st] * dm;
        if (j + sh < m) v = v + ga[st] * dp;
        d = v;
      }
      const double xv = active ? d / bf : 0.0;
      if (active) x[n * nn + i] = xv;
      xprev = xv;
    }
  }
}

// Adjoint sensitivities of the heat-compliance objective
// (objective_sensitivities, proj/src/optimisation.cpp:34-73): one thread per
// element, time levels accumulated in the reference's order, masked DOFs read
// as zero, so the result is the reference's bit for bit for the same u, lambda.
// The loads of kSensBatch levels are issued before their (sequential)
// accumulation, so the few element threads keep many loads in flight.
constexpr int kSensBatch = 16;
__global__ void k_sensitivities(int64_t n_el, int64_t n_t, double dt, const double* __restrict__ dk_dx,
                                const double* __restrict__ dc_dx6, const double* __restrict__ u,
                                const double* __restrict__ lam, double* __restrict__ sens) {
  pdl_entry();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_el) return;
  const int64_t nn = n_el + 1;
  const double kd = dk_dx[e], cd = dc_dx6[e];
  const bool left_masked = e == 0;  // node i = e is the Dirichlet node
  double acc = 0.0;
  double p0 = 0.0, p1 = 0.0;  // u at level n - 1 (level 0 is masked)
  for (int64_t n0 = 1; n0 <= n_t; n0 += kSensBatch) {
    double U0[kSensBatch], U1[kSensBatch], L0[kSensBatch], L1[kSensBatch];
#pragma unroll
    for (int k = 0; k < kSensBatch; ++k) {
      const int64_t n = n0 + k;
      const bool ok = n <= n_t;
      const int64_t r = (ok ? n : n_t) * nn + e;
      U0[k] = ok && !left_masked ? u[r] : 0.0;
      U1[k] = ok ? u[r + 1] : 0.0;
      L0[k] = ok && !left_masked ? lam[r] : 0.0;
      L1[k] = ok ? lam[r + 1] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kSensBatch; ++k) {
      if (n0 + k > n_t) break;
      const double u0 = U0[k], u1 = U1[k], l0 = L0[k], l1 = L1[k];
      acc = acc + (kd * (u0 - u1)) * (l0 - l1);
      const double v0 = (u0 - p0) / dt;
      const double v1 = (u1 - p1) / dt;
      acc = acc + cd * (l0 * (2.0 * v0 + v1) + l1 * (v0 + 2.0 * v1));
      p0 = u0;
      p1 = u1;
    }
  }
  sens[e] = -acc;
}

__global__ void k_dot(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                      double* __restrict__ partials);

// Exact coarsest solve for n_el <= 32 in two phases.  (1) Every warp of the
// block computes g_n = T^-1 f_n for its share of the time levels (T^-1 rows in
// registers, f broadcast by shuffles) into scratch.  (2) Warp 0 runs the
// causal recurrence x_n = g_n + A x_{n-1} (J; for J^T the anti-causal one
// with the next level), A = -T^-1 S, one 32 x 32 register mat-vec per step.
// Masked rows x = f / w as in k_coarsest.  Mathematically the block march of
// k_coarsest; agrees with it (and the oracle's Thomas march) to rounding.
template <bool ADJ>
__global__ void __launch_bounds__(256) k_coarsest_prop(CoarsestView cv, const double* __restrict__ f,
                                                       double* __restrict__ x,
                                                       double* __restrict__ gglobal, int use_smem) {
  pdl_entry();
  extern __shared__ double gsm[];
  double* g = use_smem ? gsm : gglobal;
  const LevelView& L = cv.lv;
  const int m = cv.m;
  const int64_t nn = L.nn, nt = L.n_t;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t k = threadIdx.x; k < nn; k += blockDim.x) x[k] = f[k] / L.w;
  for (int64_t n = 1 + threadIdx.x; n <= nt; n += blockDim.x) x[n * nn] = f[n * nn] / L.w;
  const bool active = lane < m;
  {
    double row[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) row[k] = cv.tinv[k * 32 + lane];
    for (int64_t n = 1 + warp; n <= nt; n += nw) {
      const double fl = active ? f[n * nn + lane + 1] : 0.0;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
      for (int k = 0; k < 32; k += 4) {
        a0 = a0 + row[k] * __shfl_sync(kFull, fl, k);
        a1 = a1 + row[k + 1] * __shfl_sync(kFull, fl, k + 1);
        a2 = a2 + row[k + 2] * __shfl_sync(kFull, fl, k + 2);
        a3 = a3 + row[k + 3] * __shfl_sync(kFull, fl, k + 3);
      }
      g[(n - 1) * 32 + lane] = (a0 + a1) + (a2 + a3);
    }
  }
  __syncthreads();
  if (warp != 0) return;
  double arow[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) arow[k] = cv.prop[k * 32 + lane];
  double xprev = 0.0;
  double gq = g[((ADJ ? nt : 1) - 1) * 32 + lane];
  for (int64_t s = 1; s <= nt; ++s) {
    const int64_t n = ADJ ? nt + 1 - s : s;
    const double gn = gq;
    if (s < nt) gq = g[((ADJ ? n - 1 : n + 1) - 1) * 32 + lane];
    double a0 = gn, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (s > 1) {  // the first level's coupled level is masked (J) / absent (J^T)
#pragma unroll
      for (int k = 0; k < 32; k += 4) {
        a0 = a0 + arow[k] * __shfl_sync(kFull, xprev, k);
        a1 = a1 + arow[k + 1] * __shfl_sync(kFull, xprev, k + 1);
        a2 = a2 + arow[k + 2] * __shfl_sync(kFull, xprev, k + 2);
        a3 = a3 + arow[k + 3] * __shfl_sync(kFull, xprev, k + 3);
      }
    }
    const double xv = (a0 + a1) + (a2 + a3);
    if (active) x[n * nn + lane + 1] = xv;
    xprev = active ? xv : 0.0;
  }
}

// Parallel-in-time exact coarsest solve (n_el <= 32).  The block march
// x_n = g_n + A x_{n-1} (g_n = T^-1 f_n, A = -T^-1 S; J^T: reversed in time)
// is linear, so the n_t steps are cut into C chunks of length Lc:
//   (1) all warps: g_n for every level (parallel);
//   (2) warp c: chunk c from a zero start -> its end state e_c;
//   (3) warp 0: chunk start states s_{c+1} = e_c + A^Lc s_c (C steps);
//   (4) warp c: chunk c again from s_c, writing x.
// Sequential depth 2 Lc + C instead of n_t.  Same solution up to rounding.

// Row `lane` of a 32 x 32 matrix (in registers) times v: four fused
// multiply-add accumulators over k mod 4, v broadcast through a per-warp
// shared slot (16 LDS.128).  The exact coarsest solve is not a bitwise-parity
// kernel (the reference factorises with a sparse LU), so FMA is used here.
__device__ __forceinline__ double matvec32s(const double (&row)[32], double v, double* vs) {
  __syncwarp();
  vs[threadIdx.x & 31] = v;
  __syncwarp();
  const double2* v2 = reinterpret_cast<const double2*>(vs);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
  for (int k = 0; k < 32; k += 4) {
    const double2 p = v2[k / 2], q = v2[k / 2 + 1];
    a0 = __fma_rn(row[k], p.x, a0);
    a1 = __fma_rn(row[k + 1], p.y, a1);
    a2 = __fma_rn(row[k + 2], q.x, a2);
    a3 = __fma_rn(row[k + 3], q.y, a3);
  }
  return (a0 + a1) + (a2 + a3);
}

template <bool ADJ>
__device__ __forceinline__ void dev_coarsest_chunked(const CoarsestView& cv, const double* __restrict__ f,
                                                     double* __restrict__ x, double* sm) {
  // sm: coarsest_chunked_smem(cv) bytes; every thread of the block calls this
  const LevelView& L = cv.lv;
  const int m = cv.m;
  const int64_t nn = L.nn, nt = L.n_t;
  const int C = cv.n_chunks, Lc = cv.chunk_len;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* g = sm;
  double* e = g + nt * 32;
  double* st = e + (int64_t)C * 32;
  double* vs = st + (int64_t)(C + 1) * 32 + warp * 32;  // this warp's vector slot
  for (int64_t k = threadIdx.x; k < nn; k += blockDim.x) x[k] = f[k] / L.w;
  for (int64_t n = 1 + threadIdx.x; n <= nt; n += blockDim.x) x[n * nn] = f[n * nn] / L.w;
  const bool active = lane < m;
  {
    double row[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) row[k] = cv.tinv[k * 32 + lane];
    for (int64_t n = 1 + warp; n <= nt; n += nw) {
      const double fl = active ? f[n * nn + lane + 1] : 0.0;
      g[(n - 1) * 32 + lane] = matvec32s(row, fl, vs);
    }
  }
  __syncthreads();
  double arow[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) arow[k] = cv.prop[k * 32 + lane];
  // step s = 1..nt in march order; level n(s) = s (J) or nt + 1 - s (J^T)
  auto level_of = [&](int64_t s) -> int64_t { return ADJ ? nt + 1 - s : s; };
  for (int c = warp; c < C; c += nw) {  // (2) zero-start chunk solves
    double xv = 0.0;
    for (int j = 0; j < Lc; ++j) {
      const int64_t s = (int64_t)c * Lc + j + 1;
      const double gn = g[(level_of(s) - 1) * 32 + lane];
      xv = (j == 0) ? gn : gn + matvec32s(arow, xv, vs);
    }
    e[c * 32 + lane] = xv;
  }
  __syncthreads();
  if (warp == 0) {  // (3) chunk start states
    double prow[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) prow[k] = cv.prop_chunk[k * 32 + lane];
    double sv = 0.0;
    st[lane] = 0.0;
    for (int c = 0; c < C; ++c) {
      sv = (c == 0) ? e[lane] : e[c * 32 + lane] + matvec32s(prow, sv, vs);
      st[(c + 1) * 32 + lane] = sv;
    }
  }
  __syncthreads();
  for (int c = warp; c < C; c += nw) {  // (4) final chunk solves from the true start
    double xv = st[c * 32 + lane];
    for (int j = 0; j < Lc; ++j) {
      const int64_t s = (int64_t)c * Lc + j + 1;
      const int64_t n = level_of(s);
      const double gn = g[(n - 1) * 32 + lane];
      xv = (s == 1) ? gn : gn + matvec32s(arow, xv, vs);
      if (active) x[n * nn + lane + 1] = xv;
    }
  }
}

template <bool ADJ>
__global__ void __launch_bounds__(512) k_coarsest_chunked(CoarsestView cv, const double* __restrict__ f,
                                                          double* __restrict__ x) {
  pdl_entry();
  extern __shared__ double sm[];
  dev_coarsest_chunked<ADJ>(cv, f, x, sm);
}

// ---------------------------------------------------------------------------
// Coarse tail in one thread-block cluster.  All CTAs of the cluster stride
// over the tiles of each pass (the same tile bodies as the stand-alone
// kernels, so results are bit-identical), a cluster barrier separates passes
// (it also invalidates L1, so each pass sees the previous one's stores), and
// CTA 0 runs the parallel-in-time coarsest solve.  One launch replaces
// ~(2 nu + 2) launches per tail level.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int tile_width(int64_t nn) {
  return nn >= kMaxTW ? kMaxTW : (int)((nn + 31) / 32 * 32);
}

// Barrier scopes for the tail: one thread-block cluster (<= 16 CTAs), or the
// whole grid of a cooperative launch (every SM; cg's grid barrier arrives with
// a release and polls with an acquire, so each pass sees the previous one's
// stores).
struct ClusterScope {
  __device__ static int64_t rank() { return cooperative_groups::this_cluster().block_rank(); }
  __device__ static int64_t size() { return cooperative_groups::this_cluster().num_blocks(); }
  __device__ static void sync() { cooperative_groups::this_cluster().sync(); }
};
struct GridScope {
  __device__ static int64_t rank() { return blockIdx.x; }
  __device__ static int64_t size() { return gridDim.x; }
  __device__ static void sync() { cooperative_groups::this_grid().sync(); }
};

template <bool ADJ, class Scope>
__global__ void __launch_bounds__(kMaxTW, 1) k_tail(TailParams p) {
  pdl_entry();
  extern __shared__ double sm[];
  struct {
    __device__ void sync() const { Scope::sync(); }
  } cluster;
  const int64_t rank = Scope::rank(), cs = Scope::size();
  const int nl = p.n_levels;
  int cur[kTailMaxLevels];
  auto sweep_pass = [&](int l, const double* xin, double* xout) {
    const LevelView& L = p.lv[l];
    const int tw = tile_width(L.nn);
    const int64_t node_tiles = (L.nn + (tw / 32) * 30 - 1) / ((tw / 32) * 30);
    const int64_t total = node_tiles * ((L.n_hi - L.n_lo + 7) / 8);
    const PlainLoad ld{xin, L.nn};
    for (int64_t t = rank; t < total; t += cs)
      dev_lean2<ADJ, kSweep, false, 8>(L, ld, p.f[l], xout, p.omega, t % node_tiles, t / node_tiles, tw);
    cluster.sync();
  };
  for (int l = 0; l + 1 < nl; ++l) {
    const LevelView& L = p.lv[l];
    const int tw = tile_width(L.nn);
    {
      const int64_t gx = (L.n_hi - L.n_lo + kFlatNT - 1) / kFlatNT, gy = (L.nn + tw - 1) / tw;
      for (int64_t t = rank; t < gx * gy; t += cs)
        dev_sweep_from_zero(L, p.f[l], p.xa[l], p.omega, t % gx, t / gx, tw);
      cluster.sync();
    }
    int c = 0;
    for (int k = 1; k < p.nu; ++k) {
      sweep_pass(l, c == 0 ? p.xa[l] : p.xb[l], c == 0 ? p.xb[l] : p.xa[l]);
      c ^= 1;
    }
    const LevelView& C = p.lv[l + 1];
    const double* x = c == 0 ? p.xa[l] : p.xb[l];
    {
      const int64_t warps = tw >> 5;
      const int64_t tiles = p.dir[l] == 0 ? ceil_div(ceil_div(C.nn, 14), warps) : ceil_div(L.nn, warps * 30);
      const int64_t total = tiles * ceil_div(L.n_hi - L.n_lo, 8);
      for (int64_t t = rank; t < total; t += cs) {
        if (p.dir[l] == 0) dev_restrict2<ADJ, 0, 8>(L, C, p.f[l], x, p.f[l + 1], t % tiles, t / tiles, tw);
        else dev_restrict2<ADJ, 1, 8>(L, C, p.f[l], x, p.f[l + 1], t % tiles, t / tiles, tw);
      }
    }
    cluster.sync();
    cur[l] = c;
  }
  if (rank == 0) dev_coarsest_chunked<ADJ>(p.cv, p.f[nl - 1], p.xa[nl - 1], sm);
  cluster.sync();
  int child = 0;
  for (int l = nl - 2; l >= 0; --l) {
    const LevelView& L = p.lv[l];
    const LevelView& C = p.lv[l + 1];
    const int tw = tile_width(L.nn);
    int c = cur[l];
    const double* xc = child == 0 ? p.xa[l + 1] : p.xb[l + 1];
    const int64_t node_tiles = (L.nn + (tw / 32) * 30 - 1) / ((tw / 32) * 30);
    const int64_t total = node_tiles * ((L.n_hi - L.n_lo + 7) / 8);
    double* xin = c == 0 ? p.xa[l] : p.xb[l];
    double* xout = c == 0 ? p.xb[l] : p.xa[l];
    if (p.dir[l] == 0) {
      const ProlongLoad<0> ld{xin, xc, L.nn, C.nn};
      for (int64_t t = rank; t < total; t += cs)
        dev_lean2<ADJ, kSweep, false, 8>(L, ld, p.f[l], xout, p.omega, t % node_tiles, t / node_tiles, tw);
    } else {
      const ProlongLoad<1> ld{xin, xc, L.nn, C.nn};
      for (int64_t t = rank; t < total; t += cs)
        dev_lean2<ADJ, kSweep, false, 8>(L, ld, p.f[l], xout, p.omega, t % node_tiles, t / node_tiles, tw);
    }
    cluster.sync();
    c ^= 1;
    for (int k = 1; k < p.nu; ++k) {
      sweep_pass(l, c == 0 ? p.xa[l] : p.xb[l], c == 0 ? p.xb[l] : p.xa[l]);
      c ^= 1;
    }
    child = c;
  }
}

__global__ void k_sumsq(const double* __restrict__ x, int64_t n, double* __restrict__ partials) {
  pdl_entry();
  double acc = 0.0;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[idx];
    acc = acc + v * v;
  }
  const double s = block_sum(acc);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void k_dot(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                      double* __restrict__ partials) {
  pdl_entry();
  double acc = 0.0;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x)
    acc = acc + x[idx] * y[idx];
  const double s = block_sum(acc);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void k_finalize_sum(const double* __restrict__ partials, int64_t n, double* out) {
  pdl_entry();
  double acc = 0.0;
  for (int64_t idx = threadIdx.x; idx < n; idx += blockDim.x) acc = acc + partials[idx];
  const double s = block_sum(acc);
  if (threadIdx.x == 0) *out = s;
}

// k_finalize_sum into scalars[1], then the cycle bookkeeping (one launch less
// per cycle of the device-side solve loop).
__global__ void k_finalize_check(const double* __restrict__ partials, int64_t n, double* scalars,
                                 SolveLoopCtl* ctl, double* hist, cudaGraphConditionalHandle handle) {
  pdl_entry();
  double acc = 0.0;
  for (int64_t idx = threadIdx.x; idx < n; idx += blockDim.x) acc = acc + partials[idx];
  const double s = block_sum(acc);
  if (threadIdx.x == 0) {
    scalars[1] = s;
    cycle_check_body(scalars[0], s, ctl, hist, handle);
  }
}

// Launchers return the cudaError_t of the launch (0 on success).
inline int check_launch() { return static_cast<int>(cudaGetLastError()); }

constexpr int kBlocksPerSM = 2;  // stream kernels: __launch_bounds__(kMaxTW, 2)
constexpr int kNumSMs = 148;

// Kernel design selection (benchmarking knob; 5 is the production default):
//   0: lean NT=8   1: lean NT=4   2: tile NT=4   3: warp streaming   4: tile NT=8
//   5: lean2 (overlapping warps, node-fastest order) NT=8   6: lean2 NT=16
constexpr int kDefaultVariant = 5;
int g_variant = kDefaultVariant;

inline int64_t rows(const LevelView& L) { return L.n_hi - L.n_lo; }
inline dim3 march_block(const LevelView& L) {
  int tw = L.nn >= kMaxTW ? kMaxTW : (int)((L.nn + 31) / 32 * 32);
  return dim3(tw);
}
inline int64_t stream_chunk(const LevelView& L, dim3 blk) {
  const int64_t tiles = (L.nn + blk.x - 1) / blk.x;
  int64_t chunks = (kNumSMs * kBlocksPerSM) / tiles;
  if (chunks < 1) chunks = 1;
  int64_t chunk = (L.n_t + 1 + chunks - 1) / chunks;
  if (chunk < 16) chunk = 16;
  chunk = (chunk + 1) & ~int64_t(1);
  return chunk;
}
inline int variant_nt(int v) { return (v == 1 || v == 2) ? 4 : v == 6 ? 16 : 8; }
// Overlapping-warp kernels: warps per block chosen so that the node tiles cover
// the level evenly (<= 8 warps per block).  E.g. 257 nodes -> 2 blocks of 5
// warps, not one full and one almost empty block of 8.
// At most 4 warps per block on levels of >= g_wpb4_dofs DOFs (STMG_WPB4_DOFS),
// 8 below: on large levels smaller blocks retire and refill SM slots sooner
// (cfg1 A/B 43.10 -> 42.69 ms with 4 everywhere; cfg2-scale sweep 4.51 -> 4.21 ms),
// on small levels the extra blocks cost more than they gain.
int64_t g_wpb4_dofs = 1000000;
inline int wpb_for(const LevelView& L) { return L.nn * (L.n_t + 1) >= g_wpb4_dofs ? 4 : 8; }
inline dim3 balanced_block(int64_t warps, int max_wpb) {
  if (warps < 1) warps = 1;
  const int64_t bx = (warps + max_wpb - 1) / max_wpb;
  return dim3((unsigned)(32 * ((warps + bx - 1) / bx)));
}
inline int lean_nt(const LevelView& L) { return L.tile_nt == 2 ? 2 : L.tile_nt == 4 ? 4 : 8; }
inline int64_t lean2_tiles(const LevelView& L, dim3 blk) {
  const int64_t per = (int64_t)(blk.x / 32) * 30;
  return (L.nn + per - 1) / per;
}
// Sub-range (slab) launches always use the production design.
inline int eff_variant(const LevelView& L) { return full_range(L) ? g_variant : kDefaultVariant; }
// time tiles on (y, z): tile = z * gridDim.y + y (gridDim.y <= 65535)
inline dim3 tgrid(int64_t x, int64_t t) {
  if (t < 1) t = 1;
  const int64_t y = t < 65535 ? t : 65535;
  return dim3((unsigned)x, (unsigned)y, (unsigned)((t + y - 1) / y));
}
inline dim3 pass_block(const LevelView& L, int v) {
  return (v == 5 || v == 6) ? balanced_block((L.nn + 29) / 30, wpb_for(L)) : march_block(L);
}
inline dim3 grid_for(const LevelView& L, dim3 blk, int v) {
  if (v == 5 || v == 6) {
    const int nt = v == 5 ? lean_nt(L) : 16;
    return tgrid(lean2_tiles(L, blk), (rows(L) + nt - 1) / nt);
  }
  const unsigned tiles = (unsigned)((L.nn + blk.x - 1) / blk.x);
  if (v == 3) {
    const int64_t chunk = stream_chunk(L, blk);
    return dim3((unsigned)((L.n_t + 1 + chunk - 1) / chunk), tiles);
  }
  const int nt = variant_nt(v);
  return dim3((unsigned)((L.n_t + 1 + nt - 1) / nt), tiles);
}
inline size_t tile_smem(dim3 blk, int nt, int halo) { return sizeof(double) * (nt + 1) * (blk.x + halo); }
inline unsigned flat_grid(int64_t total) { return (unsigned)((total + kFlatBlock - 1) / kFlatBlock); }

template <bool ADJ, int MODE, bool NORM, class Ld>
void launch_pass(const LevelView& L, const Ld& ld, const double* f, double* y, double omega,
                 double* partials, cudaStream_t s) {
  const int v = eff_variant(L);
  const dim3 blk = pass_block(L, v), grd = grid_for(L, blk, v);
  switch (v) {
    case 1:
      pdl_launch(k_lean<ADJ, MODE, NORM, 4, 3, Ld>, grd, blk, 0, s, L, ld, f, y, omega, partials);
      break;
    case 2:
      pdl_launch(k_tile<ADJ, MODE, NORM, 4, 4, Ld>, grd, blk, tile_smem(blk, 4, 2), s, L, ld, f, y, omega, partials);
      break;
    case 3:
      pdl_launch(k_stream<ADJ, MODE, NORM, Ld>, grd, blk, 0, s, L, ld, f, y, omega, partials, stream_chunk(L, blk));
      break;
    case 4:
      pdl_launch(k_tile<ADJ, MODE, NORM, 8, 2, Ld>, grd, blk, tile_smem(blk, 8, 2), s, L, ld, f, y, omega, partials);
      break;
    case 5:
      if (lean_nt(L) == 2 && L.nn * (L.n_t + 1) >= kMinB5Dofs)
        pdl_launch(k_lean2<ADJ, MODE, NORM, 2, 5, Ld>, grd, blk, 0, s, L, ld, f, y, omega, partials);
      else if (lean_nt(L) == 2)
        pdl_launch(k_lean2<ADJ, MODE, NORM, 2, 3, Ld>, grd, blk, 0, s, L, ld, f, y, omega, partials);
      else if (lean_nt(L) == 4)
        pdl_launch(k_lean2<ADJ, MODE, NORM, 4, 4, Ld>, grd, blk, 0, s, L, ld, f, y, omega, partials);
      else
        pdl_launch(k_lean2<ADJ, MODE, NORM, 8, 3, Ld>, grd, blk, 0, s, L, ld, f, y, omega, partials);
      break;
    case 6:
      pdl_launch(k_lean2<ADJ, MODE, NORM, 16, 2, Ld>, grd, blk, 0, s, L, ld, f, y, omega, partials);
      break;
    default:
      pdl_launch(k_lean<ADJ, MODE, NORM, 8, 2, Ld>, grd, blk, 0, s, L, ld, f, y, omega, partials);
  }
}

template <bool ADJ>
int sweep_impl(const LevelView& L, const double* f, const double* x, double* y, double omega,
               double* partials, cudaStream_t s) {
  const PlainLoad ld{x, L.nn};
  if (y != nullptr && partials != nullptr)
    launch_pass<ADJ, kSweep, true>(L, ld, f, y, omega, partials, s);
  else if (y != nullptr)
    launch_pass<ADJ, kSweep, false>(L, ld, f, y, omega, partials, s);
  else
    launch_pass<ADJ, kNormOnly, true>(L, ld, f, y, omega, partials, s);
  return check_launch();
}

template <bool ADJ, int DIR>
int sweep_prolong_impl(const LevelView& L, const LevelView& C, const double* f, const double* x,
                       const double* xc, double* y, double omega, cudaStream_t s) {
  const ProlongLoad<DIR> ld{x, xc, L.nn, C.nn};
  launch_pass<ADJ, kSweep, false>(L, ld, f, y, omega, nullptr, s);
  return check_launch();
}

template <bool ADJ, int DIR>
int restrict_tile_impl(const LevelView& F, const LevelView& C, const double* f, const double* x,
                       double* fc, cudaStream_t s, double* xc0, double omega) {
  const dim3 blk = march_block(F);
  const int v = eff_variant(F);
  if (xc0 != nullptr && !(v == 5 || v == 6)) {  // other designs: separate first coarse sweep
    const int e = restrict_tile_impl<ADJ, DIR>(F, C, f, x, fc, s, nullptr, 0.0);
    return e ? e : launch_sweep_from_zero(C, fc, xc0, omega, s);
  }
  if (v == 5 || v == 6) {
    // DIR 0: warp w owns coarse nodes 14 w .. 14 w + 13; DIR 1: fine nodes 30 w ..
    const int64_t warps = DIR == 0 ? ceil_div(C.nn, 14) : ceil_div(F.nn, 30);
    const dim3 rb = balanced_block(warps, wpb_for(F));
    const int64_t tiles = ceil_div(warps, rb.x / 32);
    if (lean_nt(F) == 2 && F.nn * (F.n_t + 1) >= kMinB5Dofs)
      pdl_launch(k_restrict2<ADJ, DIR, 2>, tgrid(tiles, (rows(F) + 1) / 2), rb, 0, s, F, C, f, x, fc, xc0, omega);
    else if (lean_nt(F) == 2)
      pdl_launch(k_restrict2<ADJ, DIR, 2, 3>, tgrid(tiles, (rows(F) + 1) / 2), rb, 0, s, F, C, f, x, fc, xc0, omega);
    else if (lean_nt(F) == 4)
      pdl_launch(k_restrict2<ADJ, DIR, 4>, tgrid(tiles, (rows(F) + 3) / 4), rb, 0, s, F, C, f, x, fc, xc0, omega);
    else
      pdl_launch(k_restrict2<ADJ, DIR, 8>, tgrid(tiles, (rows(F) + 7) / 8), rb, 0, s, F, C, f, x, fc, xc0, omega);
    return check_launch();
  }
  if (v == 0 || v == 1) {
    constexpr int NT = DIR == 0 ? 4 : 8;
    const dim3 grd((unsigned)((rows(F) + NT - 1) / NT), (unsigned)((F.nn + blk.x - 1) / blk.x));
    pdl_launch(k_lean_restrict<ADJ, DIR, NT>, grd, blk, 0, s, F, C, f, x, fc);
    return check_launch();
  }
  if (v == 3) {
    const dim3 grd = grid_for(F, blk, 3);
    pdl_launch(k_restrict_stream<ADJ, DIR>, grd, blk, 0, s, F, C, f, x, fc, stream_chunk(F, blk));
    return check_launch();
  }
  constexpr int NT = 8;
  const dim3 grd = grid_for(F, blk, 4);  // NT = 8 tiles
  size_t sm = tile_smem(blk, NT, DIR == 0 ? 3 : 2);
  if (DIR == 0) sm += sizeof(double) * NT * (blk.x + 1);
  pdl_launch(k_restrict_tile<ADJ, DIR, NT>, grd, blk, sm, s, F, C, f, x, fc);
  return check_launch();
}

}  // namespace

int64_t sweep_partials_needed(const LevelView& L) {
  // the largest grid any variant launches for this level
  const dim3 g1 = grid_for(L, march_block(L), 1), g5 = grid_for(L, pass_block(L, 5), 5);
  const int64_t a = (int64_t)g1.x * g1.y * g1.z, b = (int64_t)g5.x * g5.y * g5.z;
  return a > b ? a : b;
}

void set_kernel_variant(int v) { g_variant = (v >= 0 && v <= 6) ? v : kDefaultVariant; }
int kernel_variant() { return g_variant; }

int64_t sumsq_partials_needed(int64_t) { return kSumGrid; }

int launch_sweep(bool adjoint, const LevelView& L, const double* f, const double* x, double* y,
                 double omega, double* partials, int64_t* n_partials, cudaStream_t s) {
  if (n_partials) {
    const int v = eff_variant(L);
    const dim3 grd = grid_for(L, pass_block(L, v), v);
    *n_partials = (int64_t)grd.x * grd.y * grd.z;
  }
  return adjoint ? sweep_impl<true>(L, f, x, y, omega, partials, s)
                 : sweep_impl<false>(L, f, x, y, omega, partials, s);
}

// Streaming pair (k_march2) on levels built with L.march (STMG_MARCH_DOFS).
// Segments are sized so that the grid holds about g_march_waves x (148 SMs x
// resident warps per SM) warps; queue depth and residency: STMG_MARCH_Q / _MINB.
int g_march_q = 4;
double g_march_waves = 1.0;
int g_march_minb = 4;

template <bool ADJ, int Q>
void march2_launch(const LevelView& L, dim3 grd, dim3 blk, int64_t seg, const double* f, const double* x,
                   double* y, double omega, cudaStream_t s) {
  if (g_march_minb >= 4) pdl_launch(k_march2<ADJ, Q, 4>, grd, blk, 0, s, L, f, x, y, omega, seg);
  else pdl_launch(k_march2<ADJ, Q, 3>, grd, blk, 0, s, L, f, x, y, omega, seg);
}

int launch_sweep2_march(bool adjoint, const LevelView& L, const double* f, const double* x, double* y,
                        double omega, cudaStream_t s) {
  const int64_t warps = ceil_div(L.nn, 28);
  const dim3 blk = balanced_block(warps, wpb_for(L));
  const int64_t tiles = ceil_div(warps, blk.x / 32);
  const int64_t grid_warps = tiles * (blk.x / 32);
  const int64_t target = (int64_t)(g_march_waves * kNumSMs * 8 * (g_march_minb >= 4 ? 4 : 3));
  int64_t segs = target / grid_warps;
  if (segs < 1) segs = 1;
  int64_t seg = ceil_div(rows(L), segs);
  const int64_t q = g_march_q == 8 ? 8 : g_march_q == 2 ? 2 : 4;
  seg = ceil_div(seg, q) * q;  // whole queue groups
  const dim3 grd = tgrid(tiles, ceil_div(rows(L), seg));
  if (g_march_q == 8) {
    if (adjoint) march2_launch<true, 8>(L, grd, blk, seg, f, x, y, omega, s);
    else march2_launch<false, 8>(L, grd, blk, seg, f, x, y, omega, s);
  } else if (g_march_q == 2) {
    if (adjoint) march2_launch<true, 2>(L, grd, blk, seg, f, x, y, omega, s);
    else march2_launch<false, 2>(L, grd, blk, seg, f, x, y, omega, s);
  } else {
    if (adjoint) march2_launch<true, 4>(L, grd, blk, seg, f, x, y, omega, s);
    else march2_launch<false, 4>(L, grd, blk, seg, f, x, y, omega, s);
  }
  return check_launch();
}

// Power-of-two omega fast path of the fused pair (STMG_OMEGA_POW2=0 disables it
// for A/B measurements; read by kernels_init).
bool g_omega_pow2 = true;
inline bool omega_is_pow2(double w) {
  int e = 0;
  return w > 0.0 && std::isfinite(w) && std::frexp(w, &e) == 0.5;
}

int launch_sweep2(bool adjoint, const LevelView& L, const double* f, const double* x, double* y,
                  double omega, cudaStream_t s) {
  if (L.march) return launch_sweep2_march(adjoint, L, f, x, y, omega, s);
  const int64_t warps = ceil_div(L.nn, 28);
  const dim3 blk = balanced_block(warps, wpb_for(L));
  const int64_t tiles = ceil_div(warps, blk.x / 32);
  const bool w2 = g_omega_pow2 && omega_is_pow2(omega);
  auto go = [&](auto kern_w2, auto kern, dim3 grd) {
    if (w2) pdl_launch(kern_w2, grd, blk, 0, s, L, f, x, y, omega);
    else pdl_launch(kern, grd, blk, 0, s, L, f, x, y, omega);
  };
  if (lean_nt(L) == 2) {
    const dim3 grd = tgrid(tiles, (rows(L) + 1) / 2);
    if (L.nn * (L.n_t + 1) >= kMinB5Dofs) {
      if (adjoint) go(k_lean2x2<true, 2, minb_for_nt<2>(), true>, k_lean2x2<true, 2>, grd);
      else go(k_lean2x2<false, 2, minb_for_nt<2>(), true>, k_lean2x2<false, 2>, grd);
    } else {
      if (adjoint) go(k_lean2x2<true, 2, 3, true>, k_lean2x2<true, 2, 3>, grd);
      else go(k_lean2x2<false, 2, 3, true>, k_lean2x2<false, 2, 3>, grd);
    }
  } else if (lean_nt(L) == 4) {
    const dim3 grd = tgrid(tiles, (rows(L) + 3) / 4);
    if (adjoint) go(k_lean2x2<true, 4, minb_for_nt<4>(), true>, k_lean2x2<true, 4>, grd);
    else go(k_lean2x2<false, 4, minb_for_nt<4>(), true>, k_lean2x2<false, 4>, grd);
  } else {
    const dim3 grd = tgrid(tiles, (rows(L) + 7) / 8);
    if (adjoint) go(k_lean2x2<true, 8, minb_for_nt<8>(), true>, k_lean2x2<true, 8>, grd);
    else go(k_lean2x2<false, 8, minb_for_nt<8>(), true>, k_lean2x2<false, 8>, grd);
  }
  return check_launch();
}

// Fused pair (D = 2) through the bulk-copy pipeline (k_bulk); full-range levels.
constexpr int kBulkW = 8, kBulkStages = 2, kBulkNT = 8, kBulkMinB = 2;
template <bool ADJ>
int bulk_pair_impl(const LevelView& L, const double* f, const double* x, double* y, double omega,
                   cudaStream_t s) {
  using G = BulkGeom<kBulkNT, 2, kBulkW>;
  auto kern = k_bulk<ADJ, kBulkNT, 2, kBulkW, kBulkStages, kBulkMinB>;
  const size_t smem = sizeof(double) * (size_t)kBulkStages * G::STAGE + 16 * kBulkStages;
  static int ctas_per_sm[2] = {0, 0};
  int& cps = ctas_per_sm[ADJ ? 1 : 0];
  if (cps == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return static_cast<int>(e);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cps, kern, (kBulkW + 1) * 32, smem);
    if (e != cudaSuccess || cps < 1) return static_cast<int>(e != cudaSuccess ? e : cudaErrorInvalidConfiguration);
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n_node_tiles = ceil_div(L.nn, (int64_t)kBulkW * G::STORED);
  const int64_t n_time_tiles = ceil_div(L.n_t + 1, (int64_t)kBulkNT);
  const int64_t grid = std::min<int64_t>(n_node_tiles * n_time_tiles, (int64_t)sms * cps);
  pdl_launch(kern, (unsigned)grid, (kBulkW + 1) * 32, smem, s, L, f, x, y, omega, n_node_tiles, n_time_tiles);
  return check_launch();
}

int launch_sweep2_bulk(bool adjoint, const LevelView& L, const double* f, const double* x, double* y,
                       double omega, cudaStream_t s) {
  if (!full_range(L)) return static_cast<int>(cudaErrorInvalidValue);
  return adjoint ? bulk_pair_impl<true>(L, f, x, y, omega, s) : bulk_pair_impl<false>(L, f, x, y, omega, s);
}

int launch_sweep_deep(bool adjoint, const LevelView& L, int depth, const double* f, const double* x,
                      double* y, double omega, cudaStream_t s) {
  if (!full_range(L) || (depth != 3 && depth != 4)) return static_cast<int>(cudaErrorInvalidValue);
  const int64_t warps = ceil_div(L.nn, 32 - 2 * depth);
  const dim3 blk = balanced_block(warps, wpb_for(L));
  const int64_t tiles = ceil_div(warps, blk.x / 32);
  if (lean_nt(L) == 2) {  // the level's time-tile depth (2, else 4)
    const dim3 grd = tgrid(tiles, (rows(L) + 1) / 2);
    if (depth == 3) {
      if (adjoint) pdl_launch(k_leanD<true, 2, 3>, grd, blk, 0, s, L, f, x, y, omega);
      else pdl_launch(k_leanD<false, 2, 3>, grd, blk, 0, s, L, f, x, y, omega);
    } else {
      if (adjoint) pdl_launch(k_leanD<true, 2, 4>, grd, blk, 0, s, L, f, x, y, omega);
      else pdl_launch(k_leanD<false, 2, 4>, grd, blk, 0, s, L, f, x, y, omega);
    }
    return check_launch();
  }
  const dim3 grd = tgrid(tiles, (rows(L) + 3) / 4);
  if (depth == 3) {
    if (adjoint) pdl_launch(k_leanD<true, 4, 3>, grd, blk, 0, s, L, f, x, y, omega);
    else pdl_launch(k_leanD<false, 4, 3>, grd, blk, 0, s, L, f, x, y, omega);
  } else {
    if (adjoint) pdl_launch(k_leanD<true, 4, 4>, grd, blk, 0, s, L, f, x, y, omega);
    else pdl_launch(k_leanD<false, 4, 4>, grd, blk, 0, s, L, f, x, y, omega);
  }
  return check_launch();
}

int launch_sweep_from_zero(const LevelView& L, const double* f, double* y, double omega,
                           cudaStream_t s) {
  const dim3 blk = march_block(L);
  const dim3 grd((unsigned)((rows(L) + kFlatNT - 1) / kFlatNT), (unsigned)((L.nn + blk.x - 1) / blk.x));
  pdl_launch(k_sweep_from_zero2, grd, blk, 0, s, L, f, y, omega);
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
  const PlainLoad ld{x, L.nn};
  if (adjoint)
    launch_pass<true, kResidual, false>(L, ld, f, r, 0.0, nullptr, s);
  else
    launch_pass<false, kResidual, false>(L, ld, f, r, 0.0, nullptr, s);
  return check_launch();
}

int launch_restrict_residual(bool adjoint, const LevelView& F, const LevelView& C, int dir,
                             const double* f, const double* x, double* fc, cudaStream_t s, double* xc0,
                             double omega) {
  if (adjoint)
    return dir == 0 ? restrict_tile_impl<true, 0>(F, C, f, x, fc, s, xc0, omega)
                    : restrict_tile_impl<true, 1>(F, C, f, x, fc, s, xc0, omega);
  return dir == 0 ? restrict_tile_impl<false, 0>(F, C, f, x, fc, s, xc0, omega)
                  : restrict_tile_impl<false, 1>(F, C, f, x, fc, s, xc0, omega);
}

int launch_restrict(const LevelView& F, const LevelView& C, int dir, const double* r, double* fc,
                    cudaStream_t s) {
  const int64_t total = C.nn * (C.n_t + 1);
  const unsigned g = flat_grid(total);
  if (dir == 0) pdl_launch(k_restrict<false, 0, true>, g, kFlatBlock, 0, s, F, C, nullptr, r, fc, total);
  else pdl_launch(k_restrict<false, 1, true>, g, kFlatBlock, 0, s, F, C, nullptr, r, fc, total);
  return check_launch();
}

int launch_prolong_add(const LevelView& F, const LevelView& C, int dir, const double* xc, double* x,
                       cudaStream_t s) {
  const dim3 blk = march_block(F);
  const dim3 grd((unsigned)((rows(F) + kFlatNT - 1) / kFlatNT), (unsigned)((F.nn + blk.x - 1) / blk.x));
  if (dir == 0) pdl_launch(k_prolong_add2<0>, grd, blk, 0, s, F, C, xc, x);
  else pdl_launch(k_prolong_add2<1>, grd, blk, 0, s, F, C, xc, x);
  return check_launch();
}

int launch_coarsest_pint_prop(const CoarsestView& cv, double* P, int rounds, cudaStream_t s) {
  const size_t smem = sizeof(double) * 3 * (size_t)cv.m;
  const int threads = cv.m >= 1024 ? 1024 : (int)((cv.m + 31) / 32 * 32);
  pdl_launch(k_coarsest_pint<false, 2>, cv.m, threads, smem, s, cv, (const double*)nullptr, P,
             (const double*)nullptr);
  const int64_t mm = (int64_t)cv.m * cv.m;
  const dim3 blk(16, 16), grd((cv.m + 15) / 16, (cv.m + 15) / 16);
  for (int r = 1; r < rounds; ++r) k_square<<<grd, blk, 0, s>>>(P + (r - 1) * mm, P + r * mm, cv.m);
  return check_launch();
}

int launch_coarsest(bool adjoint, const CoarsestView& cv, const double* f, double* x,
                    double* scratch, cudaStream_t s) {
  if (cv.m > 32 && cv.pint_chunks > 1 && scratch != nullptr) {
    const size_t smem = sizeof(double) * 3 * (size_t)cv.m;
    int threads = cv.m >= 1024 ? 1024 : (int)((cv.m + 31) / 32 * 32);
    const int C = cv.pint_chunks;
    // scan rounds ping-pong between the two halves of scratch; the last round
    // writes the half that PHASE 1 reads
    double* half[2] = {scratch, scratch + (int64_t)C * cv.m};
    const int R = cv.pint_rounds;
    const size_t vsm = sizeof(double) * (size_t)cv.m;
    auto outbuf = [&](int r) { return half[(R - 1 - r) & 1]; };
    if (adjoint) {
      pdl_launch(k_coarsest_pint<true, 0>, C, threads, smem, s, cv, f, x, (const double*)nullptr);
      for (int r = 0; r < R; ++r)
        pdl_launch(k_coarsest_pint_round<true>, C, threads, vsm, s, cv, (const double*)x,
                   (const double*)(r == 0 ? nullptr : outbuf(r - 1)), outbuf(r), r);
      pdl_launch(k_coarsest_pint<true, 1>, C - 1, threads, smem, s, cv, f, x, (const double*)half[0]);
    } else {
      pdl_launch(k_coarsest_pint<false, 0>, C, threads, smem, s, cv, f, x, (const double*)nullptr);
      for (int r = 0; r < R; ++r)
        pdl_launch(k_coarsest_pint_round<false>, C, threads, vsm, s, cv, (const double*)x,
                   (const double*)(r == 0 ? nullptr : outbuf(r - 1)), outbuf(r), r);
      pdl_launch(k_coarsest_pint<false, 1>, C - 1, threads, smem, s, cv, f, x, (const double*)half[0]);
    }
    return check_launch();
  }
  if (cv.m <= 32 && cv.prop_chunk != nullptr && cv.n_chunks > 1) {
    const size_t bytes = coarsest_chunked_smem(cv);
    if (bytes <= 160 * 1024) {
      const int threads = 32 * (cv.n_chunks < 16 ? cv.n_chunks : 16);
      if (adjoint) pdl_launch(k_coarsest_chunked<true>, 1, threads, bytes, s, cv, f, x);
      else pdl_launch(k_coarsest_chunked<false>, 1, threads, bytes, s, cv, f, x);
      return check_launch();
    }
  }
  if (cv.m <= 32 && cv.tinv != nullptr && scratch != nullptr) {
    const size_t gbytes = sizeof(double) * 32 * (size_t)cv.lv.n_t;
    const int sm = gbytes <= 160 * 1024 ? 1 : 0;
    if (adjoint) pdl_launch(k_coarsest_prop<true>, 1, 256, sm ? gbytes : 0, s, cv, f, x, scratch, sm);
    else pdl_launch(k_coarsest_prop<false>, 1, 256, sm ? gbytes : 0, s, cv, f, x, scratch, sm);
    return check_launch();
  }
  if (cv.m <= 32) {
    if (adjoint) pdl_launch(k_coarsest_warp<true>, 1, 32, 0, s, cv, f, x);
    else pdl_launch(k_coarsest_warp<false>, 1, 32, 0, s, cv, f, x);
    return check_launch();
  }
  const size_t smem = sizeof(double) * 2 * (size_t)cv.m;
  const int use_smem = smem <= 160 * 1024 ? 1 : 0;
  int threads = cv.m >= 1024 ? 1024 : (int)((cv.m + 31) / 32 * 32);
  if (threads < 32) threads = 32;
  const size_t dyn = use_smem ? smem : 0;
  if (adjoint) pdl_launch(k_coarsest<true>, 1, threads, dyn, s, cv, f, x, scratch, use_smem);
  else pdl_launch(k_coarsest<false>, 1, threads, dyn, s, cv, f, x, scratch, use_smem);
  return check_launch();
}

int kernels_init() {
  static bool env_read = false;
  if (!env_read) {  // STMG_KERNEL_VARIANT lets the test suite exercise every design
    env_read = true;
    if (const char* v = std::getenv("STMG_KERNEL_VARIANT")) set_kernel_variant(std::atoi(v));
    if (const char* v = std::getenv("STMG_PDL")) g_pdl = std::atoi(v) != 0;
    if (const char* v = std::getenv("STMG_OMEGA_POW2")) g_omega_pow2 = std::atoi(v) != 0;
    if (const char* v = std::getenv("STMG_WPB4_DOFS")) g_wpb4_dofs = std::atoll(v);
    if (const char* v = std::getenv("STMG_MARCH_Q")) g_march_q = std::atoi(v);
    if (const char* v = std::getenv("STMG_MARCH_WAVES")) g_march_waves = std::atof(v);
    if (const char* v = std::getenv("STMG_MARCH_MINB")) g_march_minb = std::atoi(v);
  }
  // The coarsest march keeps its two PCR work vectors in shared memory up to 160 KB.
  cudaError_t e = cudaFuncSetAttribute(k_coarsest<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  if (e != cudaSuccess) return static_cast<int>(e);
  e = cudaFuncSetAttribute(k_coarsest<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           160 * 1024);
  if (e != cudaSuccess) return static_cast<int>(e);
  e = cudaFuncSetAttribute(k_coarsest_prop<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           160 * 1024);
  if (e != cudaSuccess) return static_cast<int>(e);
  e = cudaFuncSetAttribute(k_coarsest_prop<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           160 * 1024);
  if (e != cudaSuccess) return static_cast<int>(e);
  e = cudaFuncSetAttribute(k_coarsest_chunked<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           160 * 1024);
  if (e != cudaSuccess) return static_cast<int>(e);
  e = cudaFuncSetAttribute(k_coarsest_chunked<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           160 * 1024);
  if (e != cudaSuccess) return static_cast<int>(e);
  for (auto fn : {k_tail<true, ClusterScope>, k_tail<false, ClusterScope>}) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e != cudaSuccess) return static_cast<int>(e);
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  for (auto fn : {k_tail<true, GridScope>, k_tail<false, GridScope>}) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  for (auto fn : {k_coarsest_pint<true, 0>, k_coarsest_pint<true, 1>, k_coarsest_pint<false, 0>,
                  k_coarsest_pint<false, 1>, k_coarsest_pint<false, 2>}) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  return 0;
}

bool tail_supported(const CoarsestView& cv) {
  if (!(cv.m <= 32 && cv.prop_chunk != nullptr && cv.n_chunks > 1)) return false;
  const size_t bytes = coarsest_chunked_smem(cv);
  return bytes <= 160 * 1024;
}

int tail_grid_blocks(const TailParams& p) {
  const size_t smem = coarsest_chunked_smem(p.cv);
  int per_sm = 0, dev = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tail<false, GridScope>, kMaxTW, smem) != cudaSuccess)
    return 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return 0;
  return per_sm * sms;
}

int launch_tail(bool adjoint, const TailParams& p, int cluster, int* final_buf, cudaStream_t s) {
  if (p.nu < 1 || p.n_levels < 1 || p.n_levels > kTailMaxLevels || !tail_supported(p.cv)) return 1;
  const size_t smem = coarsest_chunked_smem(p.cv);
  int c = (p.nu - 1) & 1;  // result buffer of tail level 0: from-zero sweep -> 0, nu-1 flips, nu flips up
  if (p.n_levels > 1) c = (c + p.nu) & 1;
  else c = 0;
  if (final_buf) *final_buf = c;
  if (cluster <= 0) {  // whole-grid cooperative launch, every CTA co-resident
    const int blocks = tail_grid_blocks(p);
    if (blocks < 1) return 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(kMaxTW);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = adjoint ? cudaLaunchKernelEx(&cfg, k_tail<true, GridScope>, p)
                                  : cudaLaunchKernelEx(&cfg, k_tail<false, GridScope>, p);
    return static_cast<int>(e);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cluster);
  cfg.blockDim = dim3(kMaxTW);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl ? 2 : 1;
  const cudaError_t e = adjoint ? cudaLaunchKernelEx(&cfg, k_tail<true, ClusterScope>, p)
                                : cudaLaunchKernelEx(&cfg, k_tail<false, ClusterScope>, p);
  return static_cast<int>(e);
}

int launch_finalize_sum(const double* partials, int64_t n, double* out, cudaStream_t s) {
  pdl_launch(k_finalize_sum, 1, 1024, 0, s, partials, n, out);
  return check_launch();
}

int launch_finalize_check(const double* partials, int64_t n, double* scalars, SolveLoopCtl* ctl, double* hist,
                          cudaGraphConditionalHandle handle, cudaStream_t s) {
  pdl_launch(k_finalize_check, 1, 1024, 0, s, partials, n, scalars, ctl, hist, handle);
  return check_launch();
}

int launch_sensitivities(int64_t n_el, int64_t n_t, double dt, const double* dk_dx,
                         const double* dc_dx6, const double* u, const double* lam, double* sens,
                         cudaStream_t s) {
  // 32-thread blocks spread the n_el element threads over every SM
  pdl_launch(k_sensitivities, (unsigned)((n_el + 31) / 32), 32, 0, s, n_el, n_t, dt, dk_dx, dc_dx6, u, lam, sens);
  return check_launch();
}

int launch_dot(const double* x, const double* y, int64_t n, double* partials, int64_t* n_partials,
               cudaStream_t s) {
  pdl_launch(k_dot, kSumGrid, 256, 0, s, x, y, n, partials);
  if (n_partials) *n_partials = kSumGrid;
  return check_launch();
}

int launch_sumsq(const double* x, int64_t n, double* partials, int64_t* n_partials, cudaStream_t s) {
  pdl_launch(k_sumsq, kSumGrid, 256, 0, s, x, n, partials);
  if (n_partials) *n_partials = kSumGrid;
  return check_launch();
}

}  // namespace stmgb
