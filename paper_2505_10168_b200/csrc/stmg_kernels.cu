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

#include <cmath>
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
constexpr bool g_pdl = true;

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
// A row stride, optionally hidden from the optimiser's uniformity analysis.  Known
// uniform, k * stride is computed in 64-bit on the uniform datapath (UIMAD / USHF /
// ULOP3 per access, then IADD3 + IADD3.X: ~6 instructions per access); as a per-thread
// value it is one IMAD (shared by the row's accesses) and one IMAD.WIDE per access:
// 12-19 % fewer instructions in the sweep and restriction tiles.  Measured per kernel
// family (same box, 1.3e8 DOFs): x-step kernels and the t-step ZX restriction gain
// 2-6 %, the t-step stored restriction and prolong-sweeps and k_up lose 3-12 %, so those
// keep the uniform form.  Config-2 solve 65.5 -> 64.2 ms.
// Unsigned: k * stride wraps at 32 bits and is then scaled to bytes, which the compiler
// emulates with 64-bit products and masks (~3.7 integer instructions per access in k_up).
// Signed strides (-DSTMG_SIGNED_STRIDES: overflow undefined, free to widen) were measured
// per kernel on 1.3e8 DOFs: sweep +1.3 %, ZX prolong-sweep +4 %, ZX restriction +1 %, but
// pair -7 %, restriction -15 %, k_up -0.7 % -- the address code ptxas emits is erratic
// either way; unsigned stays (profiles/round2_march_experiment.md).
#ifdef STMG_SIGNED_STRIDES
using stride_t = int32_t;
#else
using stride_t = uint32_t;
#endif
template <bool OPAQUE>
__device__ __forceinline__ stride_t stride32(int64_t n) {
  stride_t v = (stride_t)n;
  if (OPAQUE) asm("mov.b32 %0, %0;" : "+r"(v));
  return v;
}
template <class Ld>
struct OpaqueStride {
  static constexpr bool value = true;
};

// Row strides of a level whose width is known at compile time (NNW = nodes per time level,
// 0 = run time): every row offset of a tile becomes an immediate of its load / store, which
// removes most of the integer address arithmetic (3.7 instructions per access in k_up,
// 31 % of its instructions).  Same box, 1.3e8 DOFs, run-time -> compile-time width: ZX
// restriction 0.359 -> 0.325 ms, ZX prolong-sweep 0.558 -> 0.508, k_up 0.903 -> 0.867; the
// stored restriction, the sweep and the pair do not gain (+-2 %) and keep the run-time form.
// Instantiated for the x-step forms of those three kernel families on the widths of
// kFixedWidths (n_el = 2048 .. 16384, the large levels of power-of-two grids); every other
// level takes NNW = 0.  x step: the coarse level has (NNW + 1) / 2 nodes.
template <int NNW, bool OPAQUE>
__device__ __forceinline__ stride_t fine_stride(int64_t nn) {
  if (NNW > 0) return (stride_t)NNW;
  return stride32<OPAQUE>(nn);
}
template <int NNW, bool OPAQUE>
__device__ __forceinline__ stride_t coarse_stride_x(int64_t nnc) {
  if (NNW > 0) return (stride_t)((NNW + 1) / 2);
  return stride32<OPAQUE>(nnc);
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
// EDGE: also short four-entry forms for node 1 / node n_el (see below); compiled into the
// tiles of small levels only (time tiles of <= 4 levels), where the edge warps' blocks set
// the pace; in the 8- and 16-level tiles the extra code costs registers (spills) and
// measured slower.
template <bool ADJ, bool EDGE = false>
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
  // Node 1 (no i - 1 entries) and node n_el (no i + 1 entries) on a row that has its coupled
  // level: four entries, one per canonical lane, (s0 + s1) + (s2 + s3) with s = 0 + v, folded
  // to a final + 0.0 as in row_interior.  These are the rows of the first and last warp of
  // every interior time tile: without this short form they took the generic accumulator below
  // (a data-dependent lane switch per entry) and made their block ~2x slower on narrow levels.
  if (EDGE && has_o && has_m != has_p) {
    if (!ADJ) {  // [SW, S, SE, W, D, E] without the missing side
      if (has_p) return ((c.o0 * y0 + c.op * yp) + (c.c0 * x0 + c.cp * xp)) + 0.0;
      return ((c.om * ym + c.o0 * y0) + (c.cm * xm + c.c0 * x0)) + 0.0;
    }
    // [W, D, E, NW, N, NE] without the missing side
    if (has_p) return ((c.c0 * x0 + c.cp * xp) + (c.o0 * y0 + c.op * yp)) + 0.0;
    return ((c.cm * xm + c.c0 * x0) + (c.om * ym + c.o0 * y0)) + 0.0;
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


// Edge warps of an interior time tile (every row has its coupled level and is unmasked): the
// warps holding node 0 / node 1 (first) and node n_el (last) run the interior tile body too,
// with the lane's node clamped into the grid for addresses (out-of-grid lanes stage finite
// duplicates that no stored lane couples to), and the three special rows re-evaluated in
// their own canonical forms (row_sum's: node 0 masked, node 1 without i - 1, node n_el
// without i + 1).  Without this the edge warps took the fully general tile body (64-bit
// indexing, per-row masks, the lane-switching accumulator), ~5x an interior warp: 2 of 10
// warps per row on a 257-node level, which made narrow levels ~2x slower per DOF than wide ones.
struct EdgeLane {
  int64_t ia;    // node used for addresses (clamped)
  int cls;       // 0 interior row, 1 node 0, 2 node 1, 3 node n_el
  bool in_grid;  // the lane's node exists
};
template <bool EDGE>
__device__ __forceinline__ EdgeLane edge_lane(const LevelView& L, int64_t i) {
  EdgeLane e{i, 0, true};
  if (EDGE) {
    e.ia = i < 0 ? 0 : (i > L.n_el ? L.n_el : i);
    e.in_grid = e.ia == i;
    e.cls = i == 0 ? 1 : (i == 1 ? 2 : (i == L.n_el ? 3 : 0));
  }
  return e;
}
// Needs n_el >= 2 (node 1 and node n_el distinct).
template <bool ADJ, bool EDGE>
__device__ __forceinline__ double row_tile(const LevelView& L, int cls, const Coefs& c, double xm, double x0,
                                           double xp, double ym, double y0, double yp) {
  double row = row_interior<ADJ>(c, xm, x0, xp, ym, y0, yp);
  if (EDGE && cls != 0) {
    if (cls == 1) {
      row = 0.0 + L.w * x0;
    } else if (!ADJ) {  // [SW, S, SE, W, D, E] without the missing side
      row = cls == 2 ? ((c.o0 * y0 + c.op * yp) + (c.c0 * x0 + c.cp * xp)) + 0.0
                     : ((c.om * ym + c.o0 * y0) + (c.cm * xm + c.c0 * x0)) + 0.0;
    } else {  // [W, D, E, NW, N, NE] without the missing side
      row = cls == 2 ? ((c.c0 * x0 + c.cp * xp) + (c.o0 * y0 + c.op * yp)) + 0.0
                     : ((c.cm * xm + c.c0 * x0) + (c.om * ym + c.o0 * y0)) + 0.0;
    }
  }
  return row;
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

// Staged-row loaders of the single-sweep chassis (dev_lean2).  operator()(n, i)
// is the per-lane form (boundary tiles, any lane subset).  Interior tiles use
// the three-phase form: lane() once per lane (64-bit row bases, hoisted out of
// the row loop), load(l, r, nn32) for staged row r (32-bit element offsets
// from those bases; every load of a tile is issued before the first use), and
// finish() to combine (invd: the lane's inverse diagonal -- interior rows and
// nodes are unmasked).
// The first sweep from a zero iterate, S(0) = 0 + omega (f * inv_diag) (the
// dev_sweep_from_zero / coarse_from_zero expression), recomputed from f where
// the iterate is read instead of being stored by the parent's restriction and
// read back: the coarse-level iterate after its first pre-smoothing sweep.
__device__ __forceinline__ double zero_sweep(double fv, double id, double omega) { return 0.0 + omega * (fv * id); }

struct PlainLoad {
  const double* __restrict__ x;
  int64_t nn;
  __device__ __forceinline__ double operator()(int64_t n, int64_t i) const { return x[n * nn + i]; }
  struct Lane {
    const double* __restrict__ xb;
  };
  struct Raw {
    double x;
  };
  // nbase: staged row 0; i: the lane's node
  __device__ __forceinline__ Lane lane(int64_t nbase, int64_t i, int64_t, int) const {
    return {opaque(x + (nbase * nn + i))};
  }
  template <int NNW = 0>
  __device__ __forceinline__ Raw load(const Lane& l, int r, stride_t nn32) const {
    return {__ldg(l.xb + (stride_t)r * nn32)};
  }
  __device__ __forceinline__ double finish(const Raw& w, const Lane&, int64_t, double) const { return w.x; }
};

struct ZeroLoad {
  const double* __restrict__ f;
  const double* __restrict__ invd;  // the level's inv_diag row (coef + kInvD * nn)
  double inv_w, omega;
  int64_t nn;
  __device__ __forceinline__ double id(int64_t n, int64_t i) const {
    return (n == 0 || i == 0) ? inv_w : __ldg(invd + i);
  }
  __device__ __forceinline__ double operator()(int64_t n, int64_t i) const {
    return zero_sweep(f[n * nn + i], id(n, i), omega);
  }
  struct Lane {
    const double* __restrict__ fb;
  };
  struct Raw {
    double f;
  };
  __device__ __forceinline__ Lane lane(int64_t nbase, int64_t i, int64_t, int) const {
    return {opaque(f + (nbase * nn + i))};
  }
  template <int NNW = 0>
  __device__ __forceinline__ Raw load(const Lane& l, int r, stride_t nn32) const {
    return {__ldg(l.fb + (stride_t)r * nn32)};
  }
  __device__ __forceinline__ double finish(const Raw& w, const Lane&, int64_t, double invd_i) const {
    return zero_sweep(w.f, invd_i, omega);
  }
};

// x + P xc at the staged rows (csr_spmv_add, proj/src/transfer.cpp:74-88), the
// fine iterate x given by Base (PlainLoad, or ZeroLoad for nu = 1 coarse
// levels).  x step (DIR 0): each lane reads its coarse values xc[i >> 1] and
// xc[(i + 1) >> 1] directly (one or two distinct values, L1-resident across the
// warp); causal t step (DIR 1): xc[n >> 1] at the same node.  The arithmetic is
// prolong_row's: even i 0 + 1.0 a, odd i (0.5 a + 0.5 b) + 0.
template <int DIR, class Base>
struct ProlongOn {
  Base base;
  const double* __restrict__ xc;
  int64_t nnc;
  __device__ __forceinline__ double operator()(int64_t n, int64_t i) const {
    return base(n, i) + prolong_row<DIR>(xc, nnc, n, i);
  }
  struct Lane {
    typename Base::Lane b;
    const double* __restrict__ cb;
    uint32_t odd;  // DIR 0: i & 1; DIR 1: nbase & 1
  };
  struct Raw {
    typename Base::Raw b;
    double a, c;
  };
  __device__ __forceinline__ Lane lane(int64_t nbase, int64_t i, int64_t wfirst, int ln) const {
    Lane l;
    l.b = base.lane(nbase, i, wfirst, ln);
    if (DIR == 0) {
      l.cb = opaque(xc + (nbase * nnc + (i >> 1)));
      l.odd = (uint32_t)(i & 1);
    } else {
      l.cb = opaque(xc + ((nbase >> 1) * nnc + i));
      l.odd = (uint32_t)(nbase & 1);
    }
    return l;
  }
  template <int NNW = 0>
  __device__ __forceinline__ Raw load(const Lane& l, int r, stride_t nn32) const {
    Raw w;
    w.b = base.template load<NNW>(l.b, r, nn32);
    const stride_t nnc32 = DIR == 0 ? coarse_stride_x<NNW, true>(nnc) : stride32<false>(nnc);
    if (DIR == 0) {
      const double* p = l.cb + (stride_t)r * nnc32;
      w.a = __ldg(p);
      w.c = __ldg(p + l.odd);
    } else {
      w.a = __ldg(l.cb + (stride_t)((l.odd + (uint32_t)r) >> 1) * nnc32);
      w.c = 0.0;
    }
    return w;
  }
  __device__ __forceinline__ double finish(const Raw& w, const Lane& l, int64_t i, double invd_i) const {
    const double x = base.finish(w.b, l.b, i, invd_i);
    if (DIR == 1) return x + (0.0 + 1.0 * w.a);  // prolong_row<1>
    const double pe = 0.0 + 1.0 * w.a;
    const double po = (0.5 * w.a + 0.5 * w.c) + 0.0;
    return x + (l.odd ? po : pe);
  }
};
template <class Base>
struct OpaqueStride<ProlongOn<1, Base>> {  // t-step prolong-sweeps: uniform strides measured faster
  static constexpr bool value = false;
};
template <int DIR>
using ProlongLoad = ProlongOn<DIR, PlainLoad>;
template <int DIR>
using ProlongZeroLoad = ProlongOn<DIR, ZeroLoad>;

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
template <bool ADJ, int MODE, bool NORM, int NT, class Ld, int NNW = 0>
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
  // interior time tile: the predicate-free body; EDGE (std::true_type) for the warps that hold
  // node 0 / 1 / n_el (see edge_lane)
  auto body = [&](auto edge_tag) -> double {
    constexpr bool EDGE = decltype(edge_tag)::value;
    // every lane's (clamped) node is inside the grid: lanes 0 / 31 load too (unused values).
    // 64-bit row bases once per lane, 32-bit element offsets per row.
    const EdgeLane e = edge_lane<EDGE>(L, i);
    const int64_t ia = e.ia;
    const bool computes = lane >= 1 && lane <= 30 && e.in_grid;
    const stride_t nn32 = fine_stride<NNW, OpaqueStride<Ld>::value>(nn);
    const double* __restrict__ fp = opaque(f + (n0 * nn + ia));
#pragma unroll
    for (int k = 0; k < NT; ++k) fv[k] = __ldg(fp + (stride_t)k * nn32);
    const typename Ld::Lane lc = ld.lane(nbase, ia, wfirst, lane);
    typename Ld::Raw raw[NT + 1];
#pragma unroll
    for (int r = 0; r <= NT; ++r) raw[r] = ld.template load<NNW>(lc, r, nn32);
    Coefs c = load_coefs(L, ia);
    if (EDGE && e.cls == 1) c.invd = L.inv_w;
#pragma unroll
    for (int r = 0; r <= NT; ++r) xr[r] = ld.finish(raw[r], lc, ia, c.invd);
    double* __restrict__ yp = opaque(y + (n0 * nn + ia));
    double pm = __shfl_up_sync(kFull, xr[0], 1);
    double pp = __shfl_down_sync(kFull, xr[0], 1);
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const double x1 = xr[k + 1];
      const double qm = __shfl_up_sync(kFull, x1, 1);
      const double qp = __shfl_down_sync(kFull, x1, 1);
      const double x0 = ADJ ? xr[k] : x1;
      const double row = ADJ ? row_tile<true, EDGE>(L, e.cls, c, pm, xr[k], pp, qm, x1, qp)
                             : row_tile<false, EDGE>(L, e.cls, c, qm, x1, qp, pm, xr[k], pp);
      const double r = fv[k] - row;
      if (NORM) acc = acc + (computes ? r * r : 0.0);  // a select: keeps the row out of the store's branch
      if (MODE != kNormOnly && computes) *(yp + (stride_t)k * nn32) = MODE == kSweep ? x0 + omega * (r * c.invd) : r;
      pm = qm;
      pp = qp;
    }
    return acc;
  };
  if (rows_in && nodes_in) return body(std::false_type{});
  if (rows_in && L.n_el >= 2) return body(std::true_type{});
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
      const double row = ADJ ? row_sum<true, (NT <= 4)>(L, n, i, c, pm, xr[k], pp, qm, x1, qp)
                             : row_sum<false, (NT <= 4)>(L, n, i, c, qm, x1, qp, pm, xr[k], pp);
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

template <bool ADJ, int MODE, bool NORM, int NT, int MINB, class Ld, int NNW = 0>
__global__ void __launch_bounds__(kMaxTW, MINB) k_lean2(LevelView L, Ld ld,
                                                        const double* __restrict__ f,
                                                        double* __restrict__ y, double omega,
                                                        double* __restrict__ partials) {
  pdl_entry();
  const int64_t tt = (int64_t)blockIdx.z * gridDim.y + blockIdx.y;  // time tile
  double acc = 0.0;
  if (tt < ceil_div(L.n_hi - L.n_lo, NT))
    acc = dev_lean2<ADJ, MODE, NORM, NT, Ld, NNW>(L, ld, f, y, omega, blockIdx.x, tt, blockDim.x);
  if (NORM) {  // one partial per warp (no block barrier), fixed order
    for (int o = 16; o > 0; o >>= 1) acc = acc + __shfl_xor_sync(kFull, acc, o);
    if ((threadIdx.x & 31) == 0)
      partials[(tt * gridDim.x + blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)] = acc;
  }
}

// Two damped-Jacobi sweeps fused into one pass over memory (temporal
// blocking), bit-identical to two separate sweeps.  Warps overlap by two
// nodes on each side: lanes 1..30 evaluate sweep 1, lanes 2..29 evaluate and
// store sweep 2 (28 nodes per warp).  Sweep 1 is also evaluated on the one
// staged row before the tile (J) / after it (J^T) that sweep 2 couples to.
// Staged: x on NT + 2 levels, f on NT + 1 levels.  Grid as k_lean2.
// ZX: x is the first sweep from a zero iterate, S(0) = 0 + omega (f * inv_diag),
// recomputed from f on the staged levels (x is not read; NT + 2 f levels).
template <bool ADJ, int NT, bool ZX = false>
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
  // interior time tile; EDGE for the warps that hold node 0 / 1 / n_el (see edge_lane)
  auto body = [&](auto edge_tag) {
    constexpr bool EDGE = decltype(edge_tag)::value;
    const EdgeLane e = edge_lane<EDGE>(L, i);
    // one 64-bit row base for x, f and y; 32-bit element offsets from it
    // (o[j] = node i on staged row sbase + j), so each access is one IMAD.WIDE
    const int64_t rowbase = sbase * nn;
    const double* __restrict__ xb = opaque(x + rowbase);
    const double* __restrict__ fb = opaque(f + rowbase);
    double* __restrict__ yb = opaque(y + rowbase);
    const stride_t nn32 = stride32<false>(nn);
    stride_t o[NT + 2];
    o[0] = (stride_t)e.ia;
#pragma unroll
    for (int r = 1; r < NT + 2; ++r) o[r] = o[r - 1] + nn32;
    if (ZX) {
      // staged f rows sbase + r; the sweep-1 rows are staged rows r (J^T) / r + 1 (J)
      double fs[NT + 2];
#pragma unroll
      for (int r = 0; r < NT + 2; ++r) fs[r] = __ldg(fb + o[r]);
#pragma unroll
      for (int r = 0; r < NT + 1; ++r) fv[r] = fs[ADJ ? r : r + 1];
      double idv = __ldg(L.coef + kInvD * nn + e.ia);
      if (EDGE && e.cls == 1) idv = L.inv_w;
#pragma unroll
      for (int r = 0; r < NT + 2; ++r) xs[r] = zero_sweep(fs[r], idv, omega);
    } else {
#pragma unroll
      for (int r = 0; r < NT + 2; ++r) xs[r] = __ldg(xb + o[r]);
#pragma unroll
      for (int r = 0; r < NT + 1; ++r) fv[r] = __ldg(fb + o[ADJ ? r : r + 1]);  // f rows s1base + r
    }
    Coefs c = load_coefs(L, e.ia);
    if (EDGE && e.cls == 1) c.invd = L.inv_w;
    auto upd = [&](double x0, double fval, double row) { return x0 + omega * ((fval - row) * c.invd); };
    double pm = __shfl_up_sync(kFull, xs[0], 1), pp = __shfl_down_sync(kFull, xs[0], 1);
#pragma unroll
    for (int r = 0; r <= NT; ++r) {
      const double x1 = xs[r + 1];
      const double qm = __shfl_up_sync(kFull, x1, 1), qp = __shfl_down_sync(kFull, x1, 1);
      if (ADJ) y1[r] = upd(xs[r], fv[r], row_tile<true, EDGE>(L, e.cls, c, pm, xs[r], pp, qm, x1, qp));
      else y1[r] = upd(x1, fv[r], row_tile<false, EDGE>(L, e.cls, c, qm, x1, qp, pm, xs[r], pp));
      pm = qm;
      pp = qp;
    }
    const bool lane2 = lane >= 2 && lane <= 29 && e.in_grid;
    double am = __shfl_up_sync(kFull, y1[0], 1), ap = __shfl_down_sync(kFull, y1[0], 1);
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const double z1 = y1[k + 1];
      const double bm = __shfl_up_sync(kFull, z1, 1), bp = __shfl_down_sync(kFull, z1, 1);
      // evaluated on every lane (no divergence around the shuffles); stored on
      // lanes 2..29; row n0 + k is staged row k (J^T) / k + 2 (J)
      const double v = ADJ ? upd(y1[k], fv[k], row_tile<true, EDGE>(L, e.cls, c, am, y1[k], ap, bm, z1, bp))
                           : upd(z1, fv[k + 1], row_tile<false, EDGE>(L, e.cls, c, bm, z1, bp, am, y1[k], ap));
      if (lane2) *(yb + o[ADJ ? k : k + 2]) = v;
      am = bm;
      ap = bp;
    }
  };
  if (rows_in && nodes_in) return body(std::false_type{});
  if (rows_in && L.n_el >= 2) return body(std::true_type{});
  const bool in_grid = i >= 0 && i < nn;
  const bool lane1 = lane >= 1 && lane <= 30 && in_grid;
  const bool lane2 = lane >= 2 && lane <= 29 && in_grid;
  const double idz = (ZX && in_grid) ? __ldg(L.coef + kInvD * nn + i) : 0.0;
#pragma unroll
  for (int r = 0; r < NT + 2; ++r) {
    const int64_t n = sbase + r;
    if (ZX)
      xs[r] = (n >= 0 && n <= nt && in_grid) ? zero_sweep(f[n * nn + i], (n == 0 || i == 0) ? L.inv_w : idz, omega)
                                             : 0.0;
    else
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
        const double row = row_sum<true, (NT <= 4)>(L, n, i, c, pm, xs[r], pp, qm, x1, qp);
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
        const double row = row_sum<false, (NT <= 4)>(L, n, i, c, qm, x1, qp, pm, xs[r], pp);
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
        row = row_sum<true, (NT <= 4)>(L, n, i, c, am, y1[k], ap, bm, z1, bp);
        x0 = y1[k];
        fval = fv[k];
      } else {  // row n = y1[k+1] level, coupled y1[k]
        row = row_sum<false, (NT <= 4)>(L, n, i, c, bm, z1, bp, am, y1[k], ap);
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

// Fine up-pass of a V(1,1) cycle in one pass over memory (level 0, nu = 1): the
// prolongation, the post-smoothing sweep, the residual norm that closes the cycle and
// the speculative first sweep of the next cycle,
//   v = x + P x_c               (proj/src/multigrid.cpp:202, staged, never stored)
//   u = v + omega ((f - A v) inv_diag)    the cycle's result          -> u_out
//   r = f - A u, sum r^2        (multigrid.cpp:246-249)               -> partial per warp
//   w = u + omega (r inv_diag)  the next cycle's pre-smoothing sweep  -> w_out
// i.e. the fused pair (dev_lean2x2) on the prolongated iterate with both sweeps stored
// and the second residual's squares summed: 36 B/DOF instead of 28 (prolong-sweep) + 24
// (norm pass).  u_out, w_out and x are three distinct buffers (every tile reads x rows
// that other tiles own).  Values are the separate kernels' bit for bit; the norm's
// summation order differs (deterministic).
template <bool ADJ, int NT, class Ld, int NNW = 0>
__device__ __forceinline__ double dev_up(const LevelView& L, const Ld& ld, const double* __restrict__ f,
                                         double* __restrict__ u_out, double* __restrict__ w_out, double omega,
                                         int64_t tile, int64_t ttile) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nn = L.nn, nt = L.n_t;
  const int64_t node1 = tile * ((int64_t)(blockDim.x >> 5) * 28) + warp * 28 - 1;  // node of lane 1
  if (node1 + 1 >= nn) return 0.0;  // no stored node in this warp (whole warp exits)
  const int64_t i = node1 + lane - 1;  // node of this lane
  const int64_t n0 = L.n_lo + ttile * NT;
  const int64_t sbase = ADJ ? n0 : n0 - 2;   // staged rows (NT + 2)
  const int64_t s1base = ADJ ? n0 : n0 - 1;  // sweep-1 rows (NT + 1)
  const bool rows_in = (ADJ ? (n0 >= 1 && n0 + NT <= nt - 1) : (n0 >= 3 && n0 + NT - 1 <= nt)) &&
                       n0 + NT - 1 < L.n_hi;
  const bool nodes_in = node1 >= 2 && node1 + 29 <= L.n_el - 1;
  double xs[NT + 2], fv[NT + 1], y1[NT + 1];
  double acc = 0.0;
  // interior time tile; EDGE for the warps that hold node 0 / 1 / n_el (see edge_lane)
  auto body = [&](auto edge_tag) -> double {
    constexpr bool EDGE = decltype(edge_tag)::value;
    const EdgeLane e = edge_lane<EDGE>(L, i);
    const int64_t ia = e.ia;
    const stride_t nn32 = fine_stride<NNW, false>(nn);
    const double* __restrict__ fb = opaque(f + (s1base * nn + ia));
#pragma unroll
    for (int r = 0; r < NT + 1; ++r) fv[r] = __ldg(fb + (stride_t)r * nn32);  // f rows s1base + r
    const typename Ld::Lane lc = ld.lane(sbase, ia, node1 - 1, lane);
    typename Ld::Raw raw[NT + 2];
#pragma unroll
    for (int r = 0; r < NT + 2; ++r) raw[r] = ld.template load<NNW>(lc, r, nn32);
    Coefs c = load_coefs(L, ia);
    if (EDGE && e.cls == 1) c.invd = L.inv_w;
#pragma unroll
    for (int r = 0; r < NT + 2; ++r) xs[r] = ld.finish(raw[r], lc, ia, c.invd);
    double* __restrict__ ub = opaque(u_out + (s1base * nn + ia));
    double* __restrict__ wb = opaque(w_out + (n0 * nn + ia));
    const bool lane2 = lane >= 2 && lane <= 29 && e.in_grid;
    double pm = __shfl_up_sync(kFull, xs[0], 1), pp = __shfl_down_sync(kFull, xs[0], 1);
#pragma unroll
    for (int r = 0; r <= NT; ++r) {
      const double x1 = xs[r + 1];
      const double qm = __shfl_up_sync(kFull, x1, 1), qp = __shfl_down_sync(kFull, x1, 1);
      if (ADJ) y1[r] = xs[r] + omega * ((fv[r] - row_tile<true, EDGE>(L, e.cls, c, pm, xs[r], pp, qm, x1, qp)) * c.invd);
      else y1[r] = x1 + omega * ((fv[r] - row_tile<false, EDGE>(L, e.cls, c, qm, x1, qp, pm, xs[r], pp)) * c.invd);
      const bool own_row = ADJ ? r < NT : r >= 1;  // rows n0 .. n0 + NT - 1 (compile-time per r)
      if (own_row && lane2) *(ub + (stride_t)r * nn32) = y1[r];
      pm = qm;
      pp = qp;
    }
    double am = __shfl_up_sync(kFull, y1[0], 1), ap = __shfl_down_sync(kFull, y1[0], 1);
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const double z1 = y1[k + 1];
      const double bm = __shfl_up_sync(kFull, z1, 1), bp = __shfl_down_sync(kFull, z1, 1);
      const double res = ADJ ? fv[k] - row_tile<true, EDGE>(L, e.cls, c, am, y1[k], ap, bm, z1, bp)
                             : fv[k + 1] - row_tile<false, EDGE>(L, e.cls, c, bm, z1, bp, am, y1[k], ap);
      const double x0 = ADJ ? y1[k] : z1;
      // the squared residual is summed by a select on every lane: the row evaluation then
      // cannot be sunk into the divergent branch around the store (BSSY / BRA / BSYNC and
      // a convergence check before the next shuffles, every row: 0.99 -> 0.93 ms)
      acc = acc + (lane2 ? res * res : 0.0);
      if (lane2) *(wb + (stride_t)k * nn32) = x0 + omega * (res * c.invd);
      am = bm;
      ap = bp;
    }
    return acc;
  };
  if (rows_in && nodes_in) return body(std::false_type{});
  if (rows_in && L.n_el >= 2) return body(std::true_type{});
  // ---- general path (boundary tiles): per-row-class evaluation
  const bool in_grid = i >= 0 && i < nn;
  const bool lane1 = lane >= 1 && lane <= 30 && in_grid;
  const bool lane2 = lane >= 2 && lane <= 29 && in_grid;
#pragma unroll
  for (int r = 0; r < NT + 2; ++r) {
    const int64_t n = sbase + r;
    xs[r] = (n >= 0 && n <= nt && in_grid) ? ld(n, i) : 0.0;
  }
#pragma unroll
  for (int r = 0; r < NT + 1; ++r) {
    const int64_t n = s1base + r;
    fv[r] = (n >= 0 && n <= nt && lane1) ? f[n * nn + i] : 0.0;
  }
  Coefs c{};
  if (lane1) c = load_coefs(L, i);
  double pm = __shfl_up_sync(kFull, xs[0], 1), pp = __shfl_down_sync(kFull, xs[0], 1);
#pragma unroll
  for (int r = 0; r <= NT; ++r) {
    const double x1 = xs[r + 1];
    const double qm = __shfl_up_sync(kFull, x1, 1), qp = __shfl_down_sync(kFull, x1, 1);
    const int64_t n = s1base + r;
    double v = 0.0;
    if (lane1 && n >= 0 && n <= nt) {
      const double row = ADJ ? row_sum<true, (NT <= 4)>(L, n, i, c, pm, xs[r], pp, qm, x1, qp)
                             : row_sum<false, (NT <= 4)>(L, n, i, c, qm, x1, qp, pm, xs[r], pp);
      const double id = (n == 0 || i == 0) ? L.inv_w : c.invd;
      v = (ADJ ? xs[r] : x1) + omega * ((fv[r] - row) * id);
      if (lane2 && n >= n0 && n < n0 + NT && n < L.n_hi) u_out[n * nn + i] = v;
    }
    y1[r] = v;
    pm = qm;
    pp = qp;
  }
  double am = __shfl_up_sync(kFull, y1[0], 1), ap = __shfl_down_sync(kFull, y1[0], 1);
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const double z1 = y1[k + 1];
    const double bm = __shfl_up_sync(kFull, z1, 1), bp = __shfl_down_sync(kFull, z1, 1);
    const int64_t n = n0 + k;
    if (lane2 && n < L.n_hi) {
      double row, x0, fval;
      if (ADJ) {
        row = row_sum<true, (NT <= 4)>(L, n, i, c, am, y1[k], ap, bm, z1, bp);
        x0 = y1[k];
        fval = fv[k];
      } else {
        row = row_sum<false, (NT <= 4)>(L, n, i, c, bm, z1, bp, am, y1[k], ap);
        x0 = z1;
        fval = fv[k + 1];
      }
      const double res = fval - row;
      const double id = (n == 0 || i == 0) ? L.inv_w : c.invd;
      acc = acc + res * res;
      w_out[n * nn + i] = x0 + omega * (res * id);
    }
    am = bm;
    ap = bp;
  }
  return acc;
}

// Resident 256-thread blocks per SM k_up is compiled for.  8-level tiles: 2 (up to 128
// registers, no spills) measured faster than 3 (80 registers, ~100 B of spills): probe
// 0.99 vs 1.05 ms on 1.3e8 DOFs, config-2 solve 69.4 vs 70.7 ms; register caps of 96 /
// 104 (__maxnreg__) are slower still (1.00 / 1.09 vs 0.94 ms).
template <int NT>
// (with compile-time widths the 80-register build spills only ~50 B, but still measures
// 0.881 vs 0.873 ms, config 2 60.6 vs 60.3 ms)
#ifndef STMG_UP_MINB8
#define STMG_UP_MINB8 2
#endif
constexpr int up_minb() { return NT <= 2 ? 4 : NT <= 4 ? 3 : STMG_UP_MINB8; }

// x_ind: optional device-resident pointer to the input iterate (overrides the
// loader's x): the solve loop alternates the speculative iterate between two
// buffers from cycle to cycle with the graph's kernel arguments fixed.
template <int DIR>
__device__ __forceinline__ void set_base_x(ProlongOn<DIR, PlainLoad>& ld, const double* x) { ld.base.x = x; }
template <int DIR>
__device__ __forceinline__ void set_base_x(ProlongOn<DIR, ZeroLoad>&, const double*) {}  // S(0) comes from f

template <bool ADJ, int NT, class Ld, int MINB = up_minb<NT>(), int NNW = 0>
__global__ void __launch_bounds__(kMaxTW, MINB) k_up(LevelView L, Ld ld, const double* __restrict__ f,
                                                     double* __restrict__ u_out, double* const* w_ind,
                                                     const double* const* x_ind, double omega,
                                                     double* __restrict__ partials) {
  pdl_entry();
  if (x_ind != nullptr) set_base_x(ld, *x_ind);
  double* w_out = *w_ind;
  const int64_t tt = (int64_t)blockIdx.z * gridDim.y + blockIdx.y;  // time tile
  double acc = 0.0;
  if (tt < ceil_div(L.n_hi - L.n_lo, NT)) acc = dev_up<ADJ, NT, Ld, NNW>(L, ld, f, u_out, w_out, omega, blockIdx.x, tt);
  for (int o = 16; o > 0; o >>= 1) acc = acc + __shfl_xor_sync(kFull, acc, o);
  if ((threadIdx.x & 31) == 0)
    partials[(tt * gridDim.x + blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)] = acc;
}

// Resident blocks per SM the kernels are compiled for: 5 (48 registers) pays on
// mid-sized levels, where the launch fills the GPU and latency is hidden by
// warps; on small levels the few blocks never fill the SMs and the spills of the
// tighter register budget cost latency, so 3 is used there (launch sites).
constexpr int64_t kMinB5Dofs = 200000;
// Resident blocks the 8-level norm-pass sweep (NORM) is compiled for
// (compile-time A/B switch, profiles/ab_build.py).
#ifndef STMG_NORM_MINB8
#define STMG_NORM_MINB8 3
#endif
template <int NT>
constexpr int minb_for_nt() { return NT <= 2 ? 5 : NT <= 4 ? 4 : 3; }

template <bool ADJ, int NT, int MINB = minb_for_nt<NT>(), bool ZX = false>
__global__ void __launch_bounds__(kMaxTW, MINB) k_lean2x2(LevelView L, const double* __restrict__ f,
                                                       const double* __restrict__ x,
                                                       double* __restrict__ y, double omega) {
  pdl_entry();
  const int64_t tt = (int64_t)blockIdx.z * gridDim.y + blockIdx.y;  // time tile
  if (tt < ceil_div(L.n_hi - L.n_lo, NT)) dev_lean2x2<ADJ, NT, ZX>(L, f, x, y, omega, blockIdx.x, tt);
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

// ZX: x is S(0) = 0 + omega (f * inv_diag), recomputed from f (x is not read).
// OPEN (with ZX): the opening pass of a solve from a zero iterate rides along: the
// owned entries of S(0) are stored to y_open and the thread's sum of f^2 over its owned
// entries is returned (||b||^2 = ||r0||^2), so one pass over f gives the first sweep,
// the norm and level 1's right-hand side.
template <bool ADJ, int DIR, int NT, bool ZX = false, bool OPEN = false, int NNW = 0>
__device__ __forceinline__ double dev_restrict2(const LevelView& F, const LevelView& C,
                                                const double* __restrict__ f, const double* __restrict__ x,
                                                double* __restrict__ fc, int64_t tile, int64_t ttile, int tw,
                                                double* __restrict__ /*xc0: unused*/ = nullptr, double omega = 0.0,
                                                double* __restrict__ y_open = nullptr) {
  static_assert(!OPEN || ZX, "the opening pass restricts the virtual zero iterate");
  if ((int)threadIdx.x >= tw) return 0.0;
  constexpr int kAdv = DIR == 0 ? 28 : 30;  // nodes per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nn = F.nn, nt = F.n_t, nnc = C.nn;
  const int64_t base = tile * ((tw >> 5) * kAdv) + warp * kAdv + (DIR == 0 ? -2 : 0);
  if (DIR == 0 ? (base / 2 + 1 >= nnc) : (base >= nn)) return 0.0;  // whole warp past the grid
  // fine nodes this warp owns (OPEN): x step 28 w .. 28 w + 27 = lanes 3..30; t step lanes 1..30
  const bool owns = DIR == 0 ? (lane >= 3 && lane <= 30) : (lane >= 1 && lane <= 30);
  double acc = 0.0;
  const int64_t i = base - 1 + lane;
  const int64_t n0 = F.n_lo + ttile * NT;
  const int64_t nbase = ADJ ? n0 : n0 - 1;
  const bool rows_in = (ADJ ? (n0 >= 1 && n0 + NT - 1 <= nt - 1) : (n0 >= 2 && n0 + NT - 1 <= nt)) &&
                       n0 + NT - 1 < F.n_hi;
  const bool nodes_in = base >= 2 && base + 29 <= F.n_el - 1;
  double xr[NT + 1], fv[NT];
  // interior time tile; EDGE for the warps that hold node 0 / 1 / n_el (see edge_lane).  The
  // x step's truncated coarse rows (I = 0 without 2I - 1, I = n_el / 2 without 2I + 1) are the
  // interior form with the absent residual an exact zero: ((.5 0 + r) + .5 rc) + 0 is
  // (0 + r) + (0 + .5 rc) up to the sign of a zero, which the final + 0 removes.
  auto body = [&](auto edge_tag) -> double {
    constexpr bool EDGE = decltype(edge_tag)::value;
    const EdgeLane e = edge_lane<EDGE>(F, i);
    const int64_t ia = e.ia;
    const bool own = owns && e.in_grid;
    // 64-bit row bases once per lane, 32-bit element offsets per row
    const stride_t nn32 = fine_stride<NNW, DIR == 0 || ZX>(nn);
    const stride_t nnc32 = DIR == 0 ? coarse_stride_x<NNW, true>(nnc) : stride32<ZX>(nnc);
    const double* __restrict__ fp = opaque(f + (n0 * nn + ia));
#pragma unroll
    for (int k = 0; k < NT; ++k) fv[k] = __ldg(fp + (stride_t)k * nn32);
    double fx = 0.0;  // ZX: the one staged level outside the f rows
    if (ZX) fx = ADJ ? __ldg(fp + (stride_t)NT * nn32) : __ldg(opaque(f + (nbase * nn + ia)));
    if (!ZX) {
      const double* __restrict__ xp = opaque(x + (nbase * nn + ia));
#pragma unroll
      for (int r = 0; r <= NT; ++r) xr[r] = __ldg(xp + (stride_t)r * nn32);
    }
    Coefs c = load_coefs(F, ia);
    if (EDGE && e.cls == 1) c.invd = F.inv_w;
    if (ZX) {
      // staged level nbase + r: f row r - 1 (J) / r (J^T)
#pragma unroll
      for (int r = 0; r <= NT; ++r) {
        const double fr = ADJ ? (r < NT ? fv[r] : fx) : (r == 0 ? fx : fv[r - 1]);
        xr[r] = zero_sweep(fr, c.invd, omega);
      }
    }
    if (OPEN) {
      double* __restrict__ yb = y_open != nullptr ? opaque(y_open + (n0 * nn + ia)) : nullptr;
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        acc = acc + (own ? fv[k] * fv[k] : 0.0);
        if (own && y_open != nullptr) *(yb + (stride_t)k * nn32) = xr[ADJ ? k : k + 1];  // S(0) on row n0 + k
      }
    }
    // Output lanes and their coarse node: x step, the lanes at even fine nodes
    // i = 2I (odd lanes 3..29); t step, every computing lane (I = i).
    const bool out = (DIR == 0 ? ((lane & 1) && lane >= 3 && lane <= 29) : (lane >= 1 && lane <= 30)) && e.in_grid;
    const int64_t I = DIR == 0 ? (ia >> 1) : ia;
    const int64_t crow = DIR == 0 ? n0 : (n0 >> 1);
    double* __restrict__ fcb = opaque(fc + (crow * nnc + I));
    double pm = __shfl_up_sync(kFull, xr[0], 1), pp = __shfl_down_sync(kFull, xr[0], 1);
    double r_even = 0.0;
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const double x1 = xr[k + 1];
      const double qm = __shfl_up_sync(kFull, x1, 1), qp = __shfl_down_sync(kFull, x1, 1);
      double r = fv[k] - (ADJ ? row_tile<true, EDGE>(F, e.cls, c, pm, xr[k], pp, qm, x1, qp)
                              : row_tile<false, EDGE>(F, e.cls, c, qm, x1, qp, pm, xr[k], pp));
      if (DIR == 0) {
        if (EDGE && !e.in_grid) r = 0.0;  // the absent neighbour of a truncated coarse row
        // fine nodes 2I - 1, 2I, 2I + 1 are lanes l - 1, l, l + 1 of output lane l;
        // canonical ((0 + .5 ra) + (0 + rb)) + ((0 + .5 rc) + 0), folded (see row_interior)
        const double ra = __shfl_up_sync(kFull, r, 1);
        const double rc = __shfl_down_sync(kFull, r, 1);
        const double v = ((0.5 * ra + 1.0 * r) + 0.5 * rc) + 0.0;
        if (out) *(fcb + (stride_t)k * nnc32) = v;
      } else {
        if ((k & 1) == 0) {
          r_even = r;
        } else {
          const double v = (0.5 * r_even + 0.5 * r) + 0.0;
          if (out) *(fcb + (stride_t)(k >> 1) * nnc32) = v;
        }
      }
      pm = qm;
      pp = qp;
    }
    return acc;
  };
  if (rows_in && nodes_in) return body(std::false_type{});
  if (rows_in && F.n_el >= 2 && (DIR == 1 || (F.n_el & 1) == 0)) return body(std::true_type{});
  const bool in_grid = i >= 0 && i < nn;
  const bool computes = lane >= 1 && lane <= 30 && in_grid;
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const int64_t n = n0 + k;
    fv[k] = (computes && n < F.n_hi) ? f[n * nn + i] : 0.0;
  }
  if (!ZX) {
#pragma unroll
    for (int r = 0; r <= NT; ++r) {
      const int64_t n = nbase + r;
      xr[r] = (n >= 0 && n <= nt && in_grid) ? x[n * nn + i] : 0.0;
    }
  }
  if (ZX) {
    const double idz = in_grid ? __ldg(F.coef + kInvD * nn + i) : 0.0;
#pragma unroll
    for (int r = 0; r <= NT; ++r) {
      const int64_t n = nbase + r;
      xr[r] = (n >= 0 && n <= nt && in_grid) ? zero_sweep(f[n * nn + i], (n == 0 || i == 0) ? F.inv_w : idz, omega)
                                             : 0.0;
    }
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
    if (OPEN && owns && in_grid) {
      acc = acc + fv[k] * fv[k];
      if (y_open != nullptr) y_open[n * nn + i] = xr[ADJ ? k : k + 1];  // S(0) on row n
    }
    double r = 0.0;
    if (computes)
      r = fv[k] - (ADJ ? row_sum<true, (NT <= 4)>(F, n, i, c, pm, xr[k], pp, qm, x1, qp)
                       : row_sum<false, (NT <= 4)>(F, n, i, c, qm, x1, qp, pm, xr[k], pp));
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
      }
    } else if (computes) {
      if ((k & 1) == 0) {
        r_even = r;
        if (n == nt) {  // last coarse level: truncated row, 0.5 * r(2N) only
          Acc a;
          a.add(0.5 * r);
          const double v = a.result();
          fc[(n >> 1) * nnc + i] = v;
        }
      } else {
        Acc a;
        a.add(0.5 * r_even);
        a.add(0.5 * r);
        const double v = a.result();
        fc[(n >> 1) * nnc + i] = v;
      }
    }
    pm = qm;
    pp = qp;
  }
  return acc;
}

// omega: the coarse first sweep's (xc0) and, with ZX, the fine iterate's S(0).
// x_ind: optional device-resident pointer to the iterate, read instead of x (the
// fine up-pass alternates the speculative iterate between two buffers).
template <bool ADJ, int DIR, int NT, int MINB = minb_for_nt<NT>(), bool ZX = false, int NNW = 0>
__global__ void __launch_bounds__(kMaxTW, MINB) k_restrict2(LevelView F, LevelView C, const double* __restrict__ f,
                                                         const double* x, double* __restrict__ fc,
                                                         double* __restrict__ xc0, double omega,
                                                         const double* const* x_ind) {
  pdl_entry();
  if (!ZX && x_ind != nullptr) x = *x_ind;
  const int64_t tt = (int64_t)blockIdx.z * gridDim.y + blockIdx.y;
  if (tt < ceil_div(F.n_hi - F.n_lo, NT))
    dev_restrict2<ADJ, DIR, NT, ZX, false, NNW>(F, C, f, x, fc, blockIdx.x, tt, blockDim.x, xc0, omega);
}

// The opening pass of a solve from a zero iterate fused with cycle 1's level-0
// restriction: y = S(0) = 0 + omega (f * inv_diag), f_c = R (f - A S(0)), and one partial
// per warp of sum f^2 (= ||b||^2 = ||r0||^2): 20 B/DOF instead of 16 (opening pass) + 20.
template <bool ADJ, int DIR, int NT, int MINB, int NNW = 0>
__global__ void __launch_bounds__(kMaxTW, MINB) k_restrict_open(LevelView F, LevelView C, const double* __restrict__ f,
                                                             double* __restrict__ fc, double* __restrict__ xc0,
                                                             double* __restrict__ y, double omega,
                                                             double* __restrict__ partials) {
  pdl_entry();
  const int64_t tt = (int64_t)blockIdx.z * gridDim.y + blockIdx.y;
  double acc = 0.0;
  if (tt < ceil_div(F.n_hi - F.n_lo, NT))
    acc = dev_restrict2<ADJ, DIR, NT, true, true, NNW>(F, C, f, nullptr, fc, blockIdx.x, tt, blockDim.x, xc0, omega, y);
  for (int o = 16; o > 0; o >>= 1) acc = acc + __shfl_xor_sync(kFull, acc, o);
  if ((threadIdx.x & 31) == 0)
    partials[(tt * gridDim.x + blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)] = acc;
}

// Fine down-pass of a V(1,1) cycle in one pass over memory (level 0, nu = 1):
//   stage 1: r1 = f - J x (its squares summed: the cycle's residual norm,
//            proj/src/multigrid.cpp:246-249), y = x + omega (r1 * inv_diag)
//            (the one pre-smoothing sweep, :190-193), y stored;
//   stage 2: r2 = f - J y restricted, f_c = R r2 (:197-199), and optionally the
//            coarse first sweep from zero x_c0 = S(0) (as dev_restrict2).
// Temporal blocking as dev_lean2x2: stage 1 is also evaluated on the staged row
// before the tile (J) / after it (J^T) that stage 2 couples to, and on one
// node more on each side than stage 2.  Lane l holds node base - 1 + l:
//   x step (DIR 0): stage 1 on lanes 1..30, stage 2 on lanes 2..29; coarse node
//     I = base/2 + j (j = 1..13) takes fine nodes 2I-1, 2I, 2I+1 = lanes 2j,
//     2j+1, 2j+2; warps advance 26 fine nodes (13 coarse), base = 26 w - 2, so
//     warp w owns coarse nodes 13 w .. 13 w + 12 and fine nodes 26 w .. 26 w + 25
//     (lanes 3..28: y stores and the norm);
//   causal t step (DIR 1): lanes 2..29 own nodes 28 w .. 28 w + 27; coarse level
//     N = fine levels 2N, 2N+1 at the same node (NT even, tiles start even).
// Every value is the separate kernels' bit for bit: the same row evaluations,
// lane orders and restriction sums; only the norm's summation order differs
// (block partials, deterministic).
template <bool ADJ, int DIR, int NT>
__device__ __forceinline__ double dev_down(const LevelView& F, const LevelView& C, const double* __restrict__ f,
                                           const double* __restrict__ x, double* __restrict__ y,
                                           double* __restrict__ fc, double* __restrict__ xc0, double omega,
                                           int64_t tile, int64_t ttile) {
  constexpr int kAdv = DIR == 0 ? 26 : 28;  // owned fine nodes per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nn = F.nn, nt = F.n_t, nnc = C.nn;
  const int64_t w = tile * (int64_t)(blockDim.x >> 5) + warp;
  const int64_t base = w * kAdv - 2;
  if (base + 2 >= nn) return 0.0;  // no owned node (whole warp exits)
  const int64_t i = base - 1 + lane;
  const int64_t n0 = F.n_lo + ttile * NT;
  const int64_t sbase = ADJ ? n0 : n0 - 2;   // staged x rows (NT + 2)
  const int64_t s1base = ADJ ? n0 : n0 - 1;  // stage-1 rows (NT + 1)
  const int own_lo = DIR == 0 ? 3 : 2, own_hi = DIR == 0 ? 28 : 29;
  const bool owns = lane >= own_lo && lane <= own_hi;
  const bool rows_in = (ADJ ? (n0 >= 1 && n0 + NT <= nt - 1) : (n0 >= 3 && n0 + NT - 1 <= nt)) &&
                       n0 + NT - 1 < F.n_hi;
  const bool nodes_in = base >= 2 && base + 29 <= F.n_el - 1;
  double xs[NT + 2], fv[NT + 1], y1[NT + 1];
  double acc = 0.0;
  if (rows_in && nodes_in) {
    const int64_t rowbase = sbase * nn;
    const double* __restrict__ xb = opaque(x + rowbase);
    const double* __restrict__ fb = opaque(f + rowbase);
    double* __restrict__ yb = opaque(y + rowbase);
    const stride_t nn32 = stride32<false>(nn);
    stride_t o[NT + 2];
    o[0] = (stride_t)i;
#pragma unroll
    for (int r = 1; r < NT + 2; ++r) o[r] = o[r - 1] + nn32;
#pragma unroll
    for (int r = 0; r < NT + 2; ++r) xs[r] = __ldg(xb + o[r]);
#pragma unroll
    for (int r = 0; r < NT + 1; ++r) fv[r] = __ldg(fb + o[ADJ ? r : r + 1]);  // f rows s1base + r
    const Coefs c = load_coefs(F, i);
    // output lanes and their coarse node: x step, even fine nodes i = 2I (odd lanes
    // 3..27); t step, the owned lanes (I = i)
    const bool out = DIR == 0 ? ((lane & 1) && lane >= 3 && lane <= 27) : owns;
    const int64_t I = DIR == 0 ? (i >> 1) : i;
    const int64_t crow = DIR == 0 ? n0 : (n0 >> 1);
    const stride_t nnc32 = stride32<false>(nnc);
    double* __restrict__ fcb = opaque(fc + (crow * nnc + I));
    double* __restrict__ xcb = xc0 != nullptr ? opaque(xc0 + (crow * nnc + I)) : nullptr;
    // coarse inverse diagonal at this lane's coarse node (x_c0)
    const double idc = (xc0 != nullptr && out) ? __ldg(C.coef + kInvD * nnc + I) : 0.0;
    // ---- stage 1: y1[r] = S(x) on row s1base + r; norm on the tile's own rows
    double pm = __shfl_up_sync(kFull, xs[0], 1), pp = __shfl_down_sync(kFull, xs[0], 1);
#pragma unroll
    for (int r = 0; r <= NT; ++r) {
      const double x1 = xs[r + 1];
      const double qm = __shfl_up_sync(kFull, x1, 1), qp = __shfl_down_sync(kFull, x1, 1);
      double res, x0;
      if (ADJ) {
        res = fv[r] - row_interior<true>(c, pm, xs[r], pp, qm, x1, qp);
        x0 = xs[r];
      } else {
        res = fv[r] - row_interior<false>(c, qm, x1, qp, pm, xs[r], pp);
        x0 = x1;
      }
      y1[r] = x0 + omega * (res * c.invd);
      const bool own_row = ADJ ? r < NT : r >= 1;  // row n0 .. n0 + NT - 1
      if (own_row && owns) {
        acc = acc + res * res;
        *(yb + o[ADJ ? r : r + 1]) = y1[r];
      }
      pm = qm;
      pp = qp;
    }
    // ---- stage 2: r2 = f - J y on rows n0 .. n0 + NT - 1, restricted
    double am = __shfl_up_sync(kFull, y1[0], 1), ap = __shfl_down_sync(kFull, y1[0], 1);
    double r_even = 0.0;
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const double z1 = y1[k + 1];
      const double bm = __shfl_up_sync(kFull, z1, 1), bp = __shfl_down_sync(kFull, z1, 1);
      const double r2 = ADJ ? fv[k] - row_interior<true>(c, am, y1[k], ap, bm, z1, bp)
                            : fv[k + 1] - row_interior<false>(c, bm, z1, bp, am, y1[k], ap);
      if (DIR == 0) {
        // output lanes (even fine node 2I: odd lanes 3..27) take lanes l - 1, l, l + 1
        const double ra = __shfl_up_sync(kFull, r2, 1);
        const double rc = __shfl_down_sync(kFull, r2, 1);
        if (out) {
          const double v = ((0.5 * ra + 1.0 * r2) + 0.5 * rc) + 0.0;
          *(fcb + (stride_t)k * nnc32) = v;
          if (xc0 != nullptr) *(xcb + (stride_t)k * nnc32) = 0.0 + omega * (v * idc);
        }
      } else {
        if ((k & 1) == 0) {
          r_even = r2;
        } else if (out) {
          const double v = (0.5 * r_even + 0.5 * r2) + 0.0;
          *(fcb + (stride_t)(k >> 1) * nnc32) = v;
          if (xc0 != nullptr) *(xcb + (stride_t)(k >> 1) * nnc32) = 0.0 + omega * (v * idc);
        }
      }
      am = bm;
      ap = bp;
    }
    return acc;
  }
  // ---- general path (boundary tiles): per-row-class evaluation
  const bool in_grid = i >= 0 && i < nn;
  const bool lane1 = lane >= 1 && lane <= 30 && in_grid;
  const bool own_g = owns && in_grid;
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
  if (lane1) c = load_coefs(F, i);
  double pm = __shfl_up_sync(kFull, xs[0], 1), pp = __shfl_down_sync(kFull, xs[0], 1);
#pragma unroll
  for (int r = 0; r <= NT; ++r) {
    const double x1 = xs[r + 1];
    const double qm = __shfl_up_sync(kFull, x1, 1), qp = __shfl_down_sync(kFull, x1, 1);
    const int64_t n = s1base + r;
    double v = 0.0;
    if (lane1 && n >= 0 && n <= nt) {
      double row, x0;
      if (ADJ) {
        row = row_sum<true, (NT <= 4)>(F, n, i, c, pm, xs[r], pp, qm, x1, qp);
        x0 = xs[r];
      } else {
        row = row_sum<false, (NT <= 4)>(F, n, i, c, qm, x1, qp, pm, xs[r], pp);
        x0 = x1;
      }
      const double res = fv[r] - row;
      const double id = (n == 0 || i == 0) ? F.inv_w : c.invd;
      v = x0 + omega * (res * id);
      if (own_g && n >= n0 && n < n0 + NT && n < F.n_hi) {
        acc = acc + res * res;
        y[n * nn + i] = v;
      }
    }
    y1[r] = v;
    pm = qm;
    pp = qp;
  }
  double am = __shfl_up_sync(kFull, y1[0], 1), ap = __shfl_down_sync(kFull, y1[0], 1);
  double r_even = 0.0;
  const bool lane2 = lane >= 2 && lane <= 29 && in_grid;
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const int64_t n = n0 + k;
    if (n >= F.n_hi) break;
    const double z1 = y1[k + 1];
    const double bm = __shfl_up_sync(kFull, z1, 1), bp = __shfl_down_sync(kFull, z1, 1);
    double r2 = 0.0;
    if (lane2)
      r2 = ADJ ? fv[k] - row_sum<true, (NT <= 4)>(F, n, i, c, am, y1[k], ap, bm, z1, bp)
               : fv[k + 1] - row_sum<false, (NT <= 4)>(F, n, i, c, bm, z1, bp, am, y1[k], ap);
    if (DIR == 0) {
      const int src = 2 * lane;
      const double ra = __shfl_sync(kFull, r2, src & 31);
      const double rb = __shfl_sync(kFull, r2, (src + 1) & 31);
      const double rc = __shfl_sync(kFull, r2, (src + 2) & 31);
      const int64_t I = base / 2 + lane;
      if (lane >= 1 && lane <= 13 && I >= 0 && I < nnc) {
        Acc a;
        if (I >= 1) a.add(0.5 * ra);
        a.add(1.0 * rb);
        if (2 * I + 1 <= F.n_el) a.add(0.5 * rc);
        const double v = a.result();
        fc[n * nnc + I] = v;
        if (xc0 != nullptr) xc0[n * nnc + I] = coarse_from_zero(C, n, I, v, omega);
      }
    } else if (own_g) {
      if ((k & 1) == 0) {
        r_even = r2;
        if (n == nt) {  // last coarse level: truncated row, 0.5 * r(2N) only
          Acc a;
          a.add(0.5 * r2);
          const double v = a.result();
          fc[(n >> 1) * nnc + i] = v;
          if (xc0 != nullptr) xc0[(n >> 1) * nnc + i] = coarse_from_zero(C, n >> 1, i, v, omega);
        }
      } else {
        Acc a;
        a.add(0.5 * r_even);
        a.add(0.5 * r2);
        const double v = a.result();
        fc[(n >> 1) * nnc + i] = v;
        if (xc0 != nullptr) xc0[(n >> 1) * nnc + i] = coarse_from_zero(C, n >> 1, i, v, omega);
      }
    }
    am = bm;
    ap = bp;
  }
  return acc;
}

// Resident 256-thread blocks per SM k_down is compiled for.  8-level tiles: 3
// (80 registers, ~100 B of spills) measured faster than 2 (126 registers, no
// spills): 0.92 vs 1.00 ms on 1.3e8 DOFs (profiles/round2_march_experiment.md).
template <int NT>
constexpr int down_minb() { return NT <= 2 ? 4 : 3; }

template <bool ADJ, int DIR, int NT, int MINB = down_minb<NT>()>
__global__ void __launch_bounds__(kMaxTW, MINB) k_down(LevelView F, LevelView C, const double* __restrict__ f,
                                                    const double* __restrict__ x, double* __restrict__ y,
                                                    double* __restrict__ fc, double* __restrict__ xc0, double omega,
                                                    double* __restrict__ partials) {
  pdl_entry();
  const int64_t tt = (int64_t)blockIdx.z * gridDim.y + blockIdx.y;  // time tile
  double acc = 0.0;
  if (tt < ceil_div(F.n_hi - F.n_lo, NT))
    acc = dev_down<ADJ, DIR, NT>(F, C, f, x, y, fc, xc0, omega, blockIdx.x, tt);
  const double s = block_sum(acc);
  if (threadIdx.x == 0) partials[tt * gridDim.x + blockIdx.x] = s;
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

// The opening pass of a solve from a zero iterate: y = S(0) = 0 + omega (f * inv_diag)
// (the first pre-smoothing sweep) and one partial of sum f^2 per block.  With u = 0 the
// initial residual is f itself (every row of J 0 is +0), so this one pass over f replaces
// the separate ||b||^2 pass and the residual-norm + sweep pass (16 instead of 8 + 24 B/DOF).
__global__ void k_sweep_from_zero_norm(LevelView L, const double* __restrict__ f, double* __restrict__ y,
                                       double omega, double* __restrict__ partials) {
  pdl_entry();
  double acc = 0.0;
  const int64_t i = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  if (i < L.nn) {
    const int64_t n0 = L.n_lo + (int64_t)blockIdx.x * kFlatNT;
    const double idv = __ldg(L.coef + kInvD * L.nn + i);
#pragma unroll
    for (int k = 0; k < kFlatNT; ++k) {
      const int64_t n = n0 + k;
      if (n >= L.n_hi) break;
      const double fv = f[n * L.nn + i];
      const double id = (n == 0 || i == 0) ? L.inv_w : idv;
      y[n * L.nn + i] = 0.0 + omega * (fv * id);
      acc = acc + fv * fv;
    }
  }
  const double s = block_sum(acc);
  if (threadIdx.x == 0) partials[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
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

// Adjoint sensitivities of the heat-compliance objective
// (objective_sensitivities, proj/src/optimisation.cpp:34-73), bit for bit: per
// element e the terms of time level n,
//   t_n = (dk_dx (u0 - u1)) (l0 - l1),   s_n = dc_dx6 (l0 (2 v0 + v1) + l1 (v0 + 2 v1)),
// v = (u_n - u_{n-1}) / dt, masked DOFs (n == 0, node 0) read as zero, are
// accumulated in the reference's order acc = ((acc + t_1) + s_1) + t_2 + ....
// The terms are independent, the sums are a chain.  A block owns kSensE = 16
// elements: warps 1..kSensWarps-1 compute the terms of a tile of kSensTile
// levels (a half warp per level, 16 consecutive elements = one 128-byte row
// segment of u and lambda at nodes e and e + 1) into one of two shared-memory
// buffers, while warp 0 adds the previous tile's terms in level order (double
// buffering: loads and the sequential chain overlap).  ceil(n_el / 16) blocks
// stream u and lambda once (config 4: 256 blocks over 1.07 GB).
constexpr int kSensE = 16, kSensWarps = 16, kSensLv = 3;
constexpr int kSensTile = (kSensWarps - 1) * 2 * kSensLv;  // levels per tile (90; 46 KB of buffers)
// POW2: dt is a power of two, so a / dt and a * (1 / dt) are the same correctly
// rounded number and the two divisions per level (~35 instructions each) become
// multiplications (config 4: dt = 2^-14).
template <bool POW2>
__global__ void __launch_bounds__(kSensWarps * 32, 2) k_sensitivities(
    int64_t n_el, int64_t n_t, double dt, const double* __restrict__ dk_dx, const double* __restrict__ dc_dx6,
    const double* __restrict__ u, const double* __restrict__ lam, double* __restrict__ sens) {
  pdl_entry();
  __shared__ double terms[2][2][kSensTile][kSensE];  // [buffer][t / s][level][element]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int el = lane & (kSensE - 1), half = lane >> 4;
  const int64_t e = (int64_t)blockIdx.x * kSensE + el;
  const bool active = e < n_el;
  const bool lm = e == 0;  // node i = e is the Dirichlet node
  const int64_t nn = n_el + 1;
  const double kd = active ? dk_dx[e] : 0.0, cd = active ? dc_dx6[e] : 0.0;
  const int64_t tiles = (n_t + kSensTile - 1) / kSensTile;
  const double inv_dt = 1.0 / dt;  // exact when POW2
  double acc = 0.0;
  for (int64_t t = 0; t <= tiles; ++t) {
    if (warp > 0 && t < tiles && active) {  // terms of tile t into buffer t & 1
      double(*T)[kSensTile][kSensE] = terms[t & 1];
#pragma unroll
      for (int k = 0; k < kSensLv; ++k) {
        const int j = ((warp - 1) * kSensLv + k) * 2 + half;  // level slot within the tile
        const int64_t n = 1 + t * kSensTile + j;
        if (n > n_t) continue;
        const int64_t r = n * nn + e;
        const double u0 = lm ? 0.0 : __ldg(u + r), u1 = __ldg(u + r + 1);
        const double l0 = lm ? 0.0 : __ldg(lam + r), l1 = __ldg(lam + r + 1);
        double p0 = 0.0, p1 = 0.0;  // level n - 1 (level 0 is masked)
        if (n >= 2) {
          p0 = lm ? 0.0 : __ldg(u + r - nn);
          p1 = __ldg(u + r - nn + 1);
        }
        const double v0 = POW2 ? (u0 - p0) * inv_dt : (u0 - p0) / dt;
        const double v1 = POW2 ? (u1 - p1) * inv_dt : (u1 - p1) / dt;
        T[0][j][el] = (kd * (u0 - u1)) * (l0 - l1);
        T[1][j][el] = cd * (l0 * (2.0 * v0 + v1) + l1 * (v0 + 2.0 * v1));
      }
    }
    if (warp == 0 && t > 0 && half == 0 && active) {  // tile t - 1, in level order
      double(*T)[kSensTile][kSensE] = terms[(t - 1) & 1];
      const int64_t first = 1 + (t - 1) * kSensTile;
      const int cnt = n_t - first + 1 < kSensTile ? (int)(n_t - first + 1) : kSensTile;
      for (int j = 0; j < cnt; ++j) {
        acc = acc + T[0][j][el];
        acc = acc + T[1][j][el];
      }
    }
    __syncthreads();
  }
  if (warp == 0 && half == 0 && active) sens[e] = -acc;
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

// Fixed-order sum of n block partials by one CTA: thread t adds entries t, t + B,
// t + 2B, ... into four interleaved accumulators (four independent load / add
// chains in flight), then ((a0 + a1) + (a2 + a3)) and the fixed block tree.
__device__ __forceinline__ double partials_sum(const double* __restrict__ partials, int64_t n) {
  const int64_t B = blockDim.x;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int64_t idx = threadIdx.x;
  for (; idx + 3 * B < n; idx += 4 * B) {
    a0 = a0 + partials[idx];
    a1 = a1 + partials[idx + B];
    a2 = a2 + partials[idx + 2 * B];
    a3 = a3 + partials[idx + 3 * B];
  }
  for (; idx < n; idx += B) a0 = a0 + partials[idx];
  return block_sum((a0 + a1) + (a2 + a3));
}

__global__ void k_finalize_sum(const double* __restrict__ partials, int64_t n, double* out) {
  pdl_entry();
  const double s = partials_sum(partials, n);
  if (threadIdx.x == 0) *out = s;
}

// First stage of a two-stage fixed-order sum of many partials: block b adds
// entries [b chunk, (b + 1) chunk) into out[b].
__global__ void k_partials_stage(const double* __restrict__ partials, int64_t n, int64_t chunk, double* out) {
  pdl_entry();
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t cnt = lo >= n ? 0 : (n - lo < chunk ? n - lo : chunk);
  const double s = partials_sum(partials + lo, cnt);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// k_finalize_sum into scalars[1], then the cycle bookkeeping (one launch less
// per cycle of the device-side solve loop).
__global__ void k_finalize_check(const double* __restrict__ partials, int64_t n, double* scalars,
                                 SolveLoopCtl* ctl, double* hist, cudaGraphConditionalHandle handle) {
  pdl_entry();
  const double s = partials_sum(partials, n);
  if (threadIdx.x == 0) {
    scalars[1] = s;
    cycle_check_body(scalars[0], s, ctl, hist, handle);
  }
}

// Launchers return the cudaError_t of the launch (0 on success).
inline int check_launch() { return static_cast<int>(cudaGetLastError()); }

inline int64_t rows(const LevelView& L) { return L.n_hi - L.n_lo; }
// one thread per node, up to kMaxTW nodes per block (elementwise kernels)
inline dim3 march_block(const LevelView& L) {
  int tw = L.nn >= kMaxTW ? kMaxTW : (int)((L.nn + 31) / 32 * 32);
  return dim3(tw);
}
// Overlapping-warp kernels: warps per block chosen so that the node tiles cover
// the level evenly (<= 8 warps per block).  E.g. 257 nodes -> 2 blocks of 5
// warps, not one full and one almost empty block of 8.
// At most 4 warps per block on levels of >= kWpb4Dofs DOFs, 8 below: on large
// levels smaller blocks retire and refill SM slots sooner (cfg1 A/B 43.10 ->
// 42.69 ms with 4 everywhere; cfg2-scale sweep 4.51 -> 4.21 ms), on small
// levels the extra blocks cost more than they gain.
constexpr int64_t kWpb4Dofs = 1000000;
inline int wpb_for(const LevelView& L) { return L.nn * (L.n_t + 1) >= kWpb4Dofs ? 4 : 8; }
inline dim3 balanced_block(int64_t warps, int max_wpb) {
  if (warps < 1) warps = 1;
  const int64_t bx = (warps + max_wpb - 1) / max_wpb;
  return dim3((unsigned)(32 * ((warps + bx - 1) / bx)));
}
inline int lean_nt(const LevelView& L) { return L.tile_nt == 2 ? 2 : L.tile_nt == 4 ? 4 : 8; }
// time tiles on (y, z): tile = z * gridDim.y + y (gridDim.y <= 65535)
inline dim3 tgrid(int64_t x, int64_t t) {
  if (t < 1) t = 1;
  const int64_t y = t < 65535 ? t : 65535;
  return dim3((unsigned)x, (unsigned)y, (unsigned)((t + y - 1) / y));
}
// single-sweep chassis: 30 computing lanes per warp
inline dim3 pass_block(const LevelView& L) { return balanced_block((L.nn + 29) / 30, wpb_for(L)); }
inline dim3 pass_grid(const LevelView& L, dim3 blk) {
  const int64_t per = (int64_t)(blk.x / 32) * 30;
  return tgrid((L.nn + per - 1) / per, (rows(L) + lean_nt(L) - 1) / lean_nt(L));
}
inline unsigned flat_grid(int64_t total) { return (unsigned)((total + kFlatBlock - 1) / kFlatBlock); }

// Compile-time level widths (fine_stride): fn(std::integral_constant<int, NNW>) with NNW the
// level's nodes per time level when an instantiation exists for it, else 0 (run-time width).
// MINW: the smallest width instantiated for the caller's kernel (the level-0-only kernels skip 2049).
template <int MINW = 2049, class Fn>
inline void dispatch_width(const LevelView& F, const LevelView& C, Fn&& fn) {
  const int64_t nn = (C.nn == (F.nn + 1) / 2 && F.nn >= MINW) ? F.nn : 0;  // an x step halves the elements
  switch (nn) {
    case 16385: fn(std::integral_constant<int, 16385>{}); break;
    case 8193: fn(std::integral_constant<int, 8193>{}); break;
    case 4097: fn(std::integral_constant<int, 4097>{}); break;
    case 2049: fn(std::integral_constant<int, MINW <= 2049 ? 2049 : 0>{}); break;
    default: fn(std::integral_constant<int, 0>{});
  }
}

// Resident blocks the 8-level single-sweep tiles are compiled for, by loader: 3 (80
// registers); the x-step virtual-zero prolong-sweep 4 (64 registers: 0.577 -> 0.556 ms on
// 1.3e8 DOFs; 2 blocks: 0.617).
template <class Ld>
struct Minb8 {
  static constexpr int value = 3;
};
template <>
struct Minb8<ProlongZeroLoad<0>> {
  static constexpr int value = 4;
};

template <bool ADJ, int MODE, bool NORM, class Ld>
void launch_pass(const LevelView& L, const Ld& ld, const double* f, double* y, double omega,
                 double* partials, cudaStream_t s) {
  const dim3 blk = pass_block(L), grd = pass_grid(L, blk);
  if (lean_nt(L) == 2 && L.nn * (L.n_t + 1) >= kMinB5Dofs)
    pdl_launch(k_lean2<ADJ, MODE, NORM, 2, 5, Ld>, grd, blk, 0, s, L, ld, f, y, omega, partials);
  else if (lean_nt(L) == 2)
    pdl_launch(k_lean2<ADJ, MODE, NORM, 2, 3, Ld>, grd, blk, 0, s, L, ld, f, y, omega, partials);
  else if (lean_nt(L) == 4)
    pdl_launch(k_lean2<ADJ, MODE, NORM, 4, 4, Ld>, grd, blk, 0, s, L, ld, f, y, omega, partials);
  else if constexpr (std::is_same<Ld, ProlongZeroLoad<0>>::value && MODE == kSweep && !NORM) {
    LevelView C = L;  // only its width matters here
    C.nn = ld.nnc;
    dispatch_width(L, C, [&](auto w) {
      pdl_launch(k_lean2<ADJ, MODE, NORM, 8, Minb8<Ld>::value, Ld, decltype(w)::value>, grd, blk, 0, s, L, ld, f, y,
                 omega, partials);
    });
  } else
    pdl_launch(k_lean2<ADJ, MODE, NORM, 8, NORM ? STMG_NORM_MINB8 : Minb8<Ld>::value, Ld>, grd, blk, 0, s, L, ld, f, y,
               omega, partials);
}

inline ZeroLoad zero_load(const LevelView& L, const double* f, double omega) {
  return ZeroLoad{f, L.coef + kInvD * L.nn, L.inv_w, omega, L.nn};
}

template <bool ADJ>
int sweep_impl(const LevelView& L, const double* f, const double* x, double* y, double omega,
               double* partials, cudaStream_t s) {
  if (x == nullptr) {  // x = S(0), recomputed from f
    if (y == nullptr || partials != nullptr) return static_cast<int>(cudaErrorInvalidValue);
    launch_pass<ADJ, kSweep, false>(L, zero_load(L, f, omega), f, y, omega, partials, s);
    return check_launch();
  }
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
  if (x == nullptr) {  // fine iterate S(0), recomputed from f
    const ProlongZeroLoad<DIR> ld{zero_load(L, f, omega), xc, C.nn};
    launch_pass<ADJ, kSweep, false>(L, ld, f, y, omega, nullptr, s);
  } else {
    const ProlongLoad<DIR> ld{PlainLoad{x, L.nn}, xc, C.nn};
    launch_pass<ADJ, kSweep, false>(L, ld, f, y, omega, nullptr, s);
  }
  return check_launch();
}

template <bool ADJ, int DIR, bool ZX>
void restrict_launch(const LevelView& F, const LevelView& C, const double* f, const double* x,
                     double* fc, cudaStream_t s, double* xc0, double omega, const double* const* x_ind) {
  // DIR 0: warp w owns coarse nodes 14 w .. 14 w + 13; DIR 1: fine nodes 30 w ..
  const int64_t warps = DIR == 0 ? ceil_div(C.nn, 14) : ceil_div(F.nn, 30);
  const dim3 rb = balanced_block(warps, wpb_for(F));
  const int64_t tiles = ceil_div(warps, rb.x / 32);
  // x step on a virtual zero iterate (12 B/DOF, instruction-bound): 16-level tiles halve
  // the per-tile prologue and the extra staged level (0.483 -> 0.420 ms on 1.3e8 DOFs,
  // config-2 solve 69.8 -> 69.1 ms); the t step and the stored-iterate form do not gain
  // x step on a stored iterate: 16-level tiles with 2 resident blocks (no spills) 0.463 ->
  // 0.442 ms on 1.3e8 DOFs (with 3 blocks / 80 registers: 0.530)
  if (!ZX && DIR == 0 && lean_nt(F) == 8) {
    pdl_launch(k_restrict2<ADJ, DIR, 16, 2, ZX>, tgrid(tiles, (rows(F) + 15) / 16), rb, 0, s, F, C, f, x, fc, xc0,
               omega, x_ind);
    return;
  }
  if (ZX && DIR == 0 && lean_nt(F) == 8) {
    dispatch_width(F, C, [&](auto w) {
      pdl_launch(k_restrict2<ADJ, DIR, 16, 3, ZX, (ZX && DIR == 0) ? decltype(w)::value : 0>,
                 tgrid(tiles, (rows(F) + 15) / 16), rb, 0, s, F, C, f, x, fc, xc0, omega, x_ind);
    });
    return;
  }
  if (lean_nt(F) == 2 && F.nn * (F.n_t + 1) >= kMinB5Dofs)
    pdl_launch(k_restrict2<ADJ, DIR, 2, minb_for_nt<2>(), ZX>, tgrid(tiles, (rows(F) + 1) / 2), rb, 0, s, F, C,
               f, x, fc, xc0, omega, x_ind);
  else if (lean_nt(F) == 2)
    pdl_launch(k_restrict2<ADJ, DIR, 2, 3, ZX>, tgrid(tiles, (rows(F) + 1) / 2), rb, 0, s, F, C, f, x, fc, xc0,
               omega, x_ind);
  else if (lean_nt(F) == 4)
    pdl_launch(k_restrict2<ADJ, DIR, 4, minb_for_nt<4>(), ZX>, tgrid(tiles, (rows(F) + 3) / 4), rb, 0, s, F, C,
               f, x, fc, xc0, omega, x_ind);
  else
    pdl_launch(k_restrict2<ADJ, DIR, 8, minb_for_nt<8>(), ZX>, tgrid(tiles, (rows(F) + 7) / 8), rb, 0, s, F, C,
               f, x, fc, xc0, omega, x_ind);
}

// grid of the opening restriction: the ZX restriction's, with 16-level tiles on large x-step levels
template <int DIR>
inline void restrict_open_geometry(const LevelView& F, const LevelView& C, dim3* blk, dim3* grd, int* nt) {
  const int64_t warps = DIR == 0 ? ceil_div(C.nn, 14) : ceil_div(F.nn, 30);
  *blk = balanced_block(warps, wpb_for(F));
  const int64_t tiles = ceil_div(warps, blk->x / 32);
  *nt = (DIR == 0 && lean_nt(F) == 8) ? 16 : lean_nt(F);
  *grd = tgrid(tiles, ceil_div(rows(F), *nt));
}
template <bool ADJ, int DIR>
void restrict_open_launch(const LevelView& F, const LevelView& C, const double* f, double* fc, double* xc0, double* y,
                          double omega, double* partials, cudaStream_t s) {
  dim3 blk, grd;
  int nt = 0;
  restrict_open_geometry<DIR>(F, C, &blk, &grd, &nt);
  if (nt == 16) {
    if (DIR == 0)
      dispatch_width<4097>(F, C, [&](auto w) {
        pdl_launch(k_restrict_open<ADJ, 0, 16, 3, DIR == 0 ? decltype(w)::value : 0>, grd, blk, 0, s, F, C, f, fc, xc0,
                   y, omega, partials);
      });
  } else if (nt == 8) {
    pdl_launch(k_restrict_open<ADJ, DIR, 8, 3>, grd, blk, 0, s, F, C, f, fc, xc0, y, omega, partials);
  } else if (nt == 4) {
    pdl_launch(k_restrict_open<ADJ, DIR, 4, 4>, grd, blk, 0, s, F, C, f, fc, xc0, y, omega, partials);
  } else {
    pdl_launch(k_restrict_open<ADJ, DIR, 2, 3>, grd, blk, 0, s, F, C, f, fc, xc0, y, omega, partials);
  }
}

template <bool ADJ, int DIR>
int restrict_impl(const LevelView& F, const LevelView& C, const double* f, const double* x,
                  double* fc, cudaStream_t s, double* xc0, double omega, const double* const* x_ind) {
  // the stored coarse first sweep is no longer written by the restriction tiles (dead code on
  // the default path: 8 % of the ZX tile's instructions); the child sweeps from zero itself
  if (xc0 != nullptr) return static_cast<int>(cudaErrorInvalidValue);
  if (x == nullptr) restrict_launch<ADJ, DIR, true>(F, C, f, x, fc, s, xc0, omega, nullptr);  // x = S(0) from f
  else restrict_launch<ADJ, DIR, false>(F, C, f, x, fc, s, xc0, omega, x_ind);
  return check_launch();
}

}  // namespace

int64_t sweep_partials_needed(const LevelView& L) {
  const dim3 b = pass_block(L), g = pass_grid(L, b);
  return (int64_t)g.x * g.y * g.z * (b.x / 32);  // one per warp
}

int64_t sumsq_partials_needed(int64_t) { return kSumGrid; }

int launch_sweep(bool adjoint, const LevelView& L, const double* f, const double* x, double* y,
                 double omega, double* partials, int64_t* n_partials, cudaStream_t s) {
  if (n_partials) *n_partials = sweep_partials_needed(L);
  return adjoint ? sweep_impl<true>(L, f, x, y, omega, partials, s)
                 : sweep_impl<false>(L, f, x, y, omega, partials, s);
}

namespace {
template <bool ADJ, bool ZX>
void sweep2_launch(const LevelView& L, const double* f, const double* x, double* y, double omega, cudaStream_t s) {
  const int64_t warps = ceil_div(L.nn, 28);
  const dim3 blk = balanced_block(warps, wpb_for(L));
  const int64_t tiles = ceil_div(warps, blk.x / 32);
  if (lean_nt(L) == 2) {
    const dim3 grd = tgrid(tiles, (rows(L) + 1) / 2);
    if (L.nn * (L.n_t + 1) >= kMinB5Dofs)
      pdl_launch(k_lean2x2<ADJ, 2, minb_for_nt<2>(), ZX>, grd, blk, 0, s, L, f, x, y, omega);
    else
      pdl_launch(k_lean2x2<ADJ, 2, 3, ZX>, grd, blk, 0, s, L, f, x, y, omega);
  } else if (lean_nt(L) == 4) {
    pdl_launch(k_lean2x2<ADJ, 4, minb_for_nt<4>(), ZX>, tgrid(tiles, (rows(L) + 3) / 4), blk, 0, s, L, f, x, y,
               omega);
  } else {
    pdl_launch(k_lean2x2<ADJ, 8, minb_for_nt<8>(), ZX>, tgrid(tiles, (rows(L) + 7) / 8), blk, 0, s, L, f, x, y,
               omega);
  }
}
}  // namespace

// x == nullptr: x is S(0), recomputed from f (the pair then applies sweeps 2 and 3 from zero)
int launch_sweep2(bool adjoint, const LevelView& L, const double* f, const double* x, double* y,
                  double omega, cudaStream_t s) {
  if (adjoint) {
    if (x == nullptr) sweep2_launch<true, true>(L, f, x, y, omega, s);
    else sweep2_launch<true, false>(L, f, x, y, omega, s);
  } else {
    if (x == nullptr) sweep2_launch<false, true>(L, f, x, y, omega, s);
    else sweep2_launch<false, false>(L, f, x, y, omega, s);
  }
  return check_launch();
}

namespace {
template <bool ADJ, int DIR>
void down_launch(const LevelView& F, const LevelView& C, const double* f, const double* x, double* y, double* fc,
                 double* xc0, double omega, double* partials, cudaStream_t s) {
  const int64_t warps = DIR == 0 ? ceil_div(C.nn, 13) : ceil_div(F.nn, 28);
  const dim3 blk = balanced_block(warps, wpb_for(F));
  const int64_t tiles = ceil_div(warps, blk.x / 32);
  const int nt = lean_nt(F);
  const dim3 grd = tgrid(tiles, (rows(F) + nt - 1) / nt);
  if (nt == 2)
    pdl_launch(k_down<ADJ, DIR, 2>, grd, blk, 0, s, F, C, f, x, y, fc, xc0, omega, partials);
  else if (nt == 4)
    pdl_launch(k_down<ADJ, DIR, 4>, grd, blk, 0, s, F, C, f, x, y, fc, xc0, omega, partials);
  else
    pdl_launch(k_down<ADJ, DIR, 8>, grd, blk, 0, s, F, C, f, x, y, fc, xc0, omega, partials);
}
}  // namespace

int64_t down_partials_needed(const LevelView& F, const LevelView& C, int dir) {
  const int64_t warps = dir == 0 ? ceil_div(C.nn, 13) : ceil_div(F.nn, 28);
  const dim3 blk = balanced_block(warps, wpb_for(F));
  const int64_t tiles = ceil_div(warps, blk.x / 32);
  const dim3 grd = tgrid(tiles, (rows(F) + lean_nt(F) - 1) / lean_nt(F));
  return (int64_t)grd.x * grd.y * grd.z;
}

int launch_down(bool adjoint, const LevelView& F, const LevelView& C, int dir, const double* f, const double* x,
                double* y, double* fc, double* xc0, double omega, double* partials, int64_t* n_partials,
                cudaStream_t s) {
  if (F.tile_nt % 2 != 0 || (F.n_lo & 1) != 0) return static_cast<int>(cudaErrorInvalidValue);
  if (n_partials) *n_partials = down_partials_needed(F, C, dir);
  if (adjoint) {
    if (dir == 0) down_launch<true, 0>(F, C, f, x, y, fc, xc0, omega, partials, s);
    else down_launch<true, 1>(F, C, f, x, y, fc, xc0, omega, partials, s);
  } else {
    if (dir == 0) down_launch<false, 0>(F, C, f, x, y, fc, xc0, omega, partials, s);
    else down_launch<false, 1>(F, C, f, x, y, fc, xc0, omega, partials, s);
  }
  return check_launch();
}

namespace {
// 4-warp blocks on large levels as for the other tiles (8-warp blocks: config-2 solve 71.1 vs 69.8 ms)
inline dim3 up_block(const LevelView& L) { return balanced_block(ceil_div(L.nn, 28), wpb_for(L)); }
inline dim3 up_grid(const LevelView& L, dim3 blk) {
  const int64_t tiles = ceil_div(ceil_div(L.nn, 28), blk.x / 32);
  return tgrid(tiles, ceil_div(rows(L), lean_nt(L)));
}
template <bool ADJ, int DIR>
void up_launch(const LevelView& L, const LevelView& C, const double* f, const double* x, const double* xc,
               double* u_out, double* const* w_ind, const double* const* x_ind, double omega, double* partials,
               cudaStream_t s) {
  const dim3 blk = up_block(L), grd = up_grid(L, blk);
  if (x == nullptr) {  // the iterate is S(0), recomputed from f (cycle 1 of a zero-guess solve)
    const ProlongZeroLoad<DIR> lz{zero_load(L, f, omega), xc, C.nn};
    if (lean_nt(L) == 2)
      pdl_launch(k_up<ADJ, 2, ProlongZeroLoad<DIR>>, grd, blk, 0, s, L, lz, f, u_out, w_ind, x_ind, omega, partials);
    else if (lean_nt(L) == 4)
      pdl_launch(k_up<ADJ, 4, ProlongZeroLoad<DIR>>, grd, blk, 0, s, L, lz, f, u_out, w_ind, x_ind, omega, partials);
    else
      dispatch_width<4097>(L, C, [&](auto w) {
        pdl_launch(k_up<ADJ, 8, ProlongZeroLoad<DIR>, up_minb<8>(), DIR == 0 ? decltype(w)::value : 0>, grd, blk, 0, s, L,
                   lz, f, u_out, w_ind, x_ind, omega, partials);
      });
    return;
  }
  const ProlongLoad<DIR> ld{PlainLoad{x, L.nn}, xc, C.nn};
  if (lean_nt(L) == 2)
    pdl_launch(k_up<ADJ, 2, ProlongLoad<DIR>>, grd, blk, 0, s, L, ld, f, u_out, w_ind, x_ind, omega, partials);
  else if (lean_nt(L) == 4)
    pdl_launch(k_up<ADJ, 4, ProlongLoad<DIR>>, grd, blk, 0, s, L, ld, f, u_out, w_ind, x_ind, omega, partials);
  else  // 8-level tiles: 6 / 10 levels measured slower (1.05 / 0.99 vs 0.94 ms on 1.3e8 DOFs)
    dispatch_width<4097>(L, C, [&](auto w) {
      pdl_launch(k_up<ADJ, 8, ProlongLoad<DIR>, up_minb<8>(), DIR == 0 ? decltype(w)::value : 0>, grd, blk, 0, s, L, ld,
                 f, u_out, w_ind, x_ind, omega, partials);
    });
}
}  // namespace

int64_t up_partials_needed(const LevelView& L) {
  const dim3 b = up_block(L), g = up_grid(L, b);
  return (int64_t)g.x * g.y * g.z * (b.x / 32);  // one per warp
}

// Fine up-pass (k_up): u_out = S(x + P xc), *w_ind = S(u_out), partials of ||f - A u_out||^2.
// x_ind (optional): device-resident pointer to the input iterate, read instead of x.
int launch_up(bool adjoint, const LevelView& L, const LevelView& C, int dir, const double* f, const double* x,
              const double* xc, double* u_out, double* const* w_ind, const double* const* x_ind, double omega,
              double* partials, int64_t* n_partials, cudaStream_t s) {
  if (n_partials) *n_partials = up_partials_needed(L);
  if (adjoint) {
    if (dir == 0) up_launch<true, 0>(L, C, f, x, xc, u_out, w_ind, x_ind, omega, partials, s);
    else up_launch<true, 1>(L, C, f, x, xc, u_out, w_ind, x_ind, omega, partials, s);
  } else {
    if (dir == 0) up_launch<false, 0>(L, C, f, x, xc, u_out, w_ind, x_ind, omega, partials, s);
    else up_launch<false, 1>(L, C, f, x, xc, u_out, w_ind, x_ind, omega, partials, s);
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

int64_t zero_norm_partials_needed(const LevelView& L) {
  const dim3 blk = march_block(L);
  return ((rows(L) + kFlatNT - 1) / kFlatNT) * ((L.nn + blk.x - 1) / blk.x);
}

int launch_sweep_from_zero_norm(const LevelView& L, const double* f, double* y, double omega, double* partials,
                                int64_t* n_partials, cudaStream_t s) {
  const dim3 blk = march_block(L);
  const dim3 grd((unsigned)((rows(L) + kFlatNT - 1) / kFlatNT), (unsigned)((L.nn + blk.x - 1) / blk.x));
  if (n_partials) *n_partials = (int64_t)grd.x * grd.y;
  pdl_launch(k_sweep_from_zero_norm, grd, blk, 0, s, L, f, y, omega, partials);
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
                             double omega, const double* const* x_ind) {
  if (adjoint)
    return dir == 0 ? restrict_impl<true, 0>(F, C, f, x, fc, s, xc0, omega, x_ind)
                    : restrict_impl<true, 1>(F, C, f, x, fc, s, xc0, omega, x_ind);
  return dir == 0 ? restrict_impl<false, 0>(F, C, f, x, fc, s, xc0, omega, x_ind)
                  : restrict_impl<false, 1>(F, C, f, x, fc, s, xc0, omega, x_ind);
}

int64_t restrict_open_partials_needed(const LevelView& F, const LevelView& C, int dir) {
  dim3 blk, grd;
  int nt = 0;
  if (dir == 0) restrict_open_geometry<0>(F, C, &blk, &grd, &nt);
  else restrict_open_geometry<1>(F, C, &blk, &grd, &nt);
  return (int64_t)grd.x * grd.y * grd.z * (blk.x / 32);
}

// Opening pass of a zero-guess solve fused with cycle 1's level-0 restriction
// (k_restrict_open): y = S(0), f_c = R (f - A S(0)) (and the stored coarse first sweep
// x_c0 when not null), one partial per warp of sum f^2.
int launch_restrict_open(bool adjoint, const LevelView& F, const LevelView& C, int dir, const double* f, double* fc,
                         double* xc0, double* y, double omega, double* partials, int64_t* n_partials,
                         cudaStream_t s) {
  if (dir == 1 && (F.tile_nt % 2 != 0 || (F.n_lo & 1) != 0)) return static_cast<int>(cudaErrorInvalidValue);
  if (xc0 != nullptr) return static_cast<int>(cudaErrorInvalidValue);  // see restrict_impl
  if (n_partials) *n_partials = restrict_open_partials_needed(F, C, dir);
  if (adjoint) {
    if (dir == 0) restrict_open_launch<true, 0>(F, C, f, fc, xc0, y, omega, partials, s);
    else restrict_open_launch<true, 1>(F, C, f, fc, xc0, y, omega, partials, s);
  } else {
    if (dir == 0) restrict_open_launch<false, 0>(F, C, f, fc, xc0, y, omega, partials, s);
    else restrict_open_launch<false, 1>(F, C, f, fc, xc0, y, omega, partials, s);
  }
  return check_launch();
}

namespace {
__global__ void k_swap_ptrs(double** p) {
  pdl_entry();
  if (threadIdx.x == 0) {
    double* t = p[0];
    p[0] = p[1];
    p[1] = t;
  }
}
}  // namespace

int launch_swap_ptrs(double** p, cudaStream_t s) {
  pdl_launch(k_swap_ptrs, 1, 32, 0, s, p);
  return check_launch();
}

// Small host <-> device transfers of a solve as kernels instead of copy-engine
// operations: values up travel as kernel arguments, values down are stored to page-locked
// host memory (device-addressable under unified addressing).  A copy-engine operation
// queues behind whatever large transfer another stream has in flight (the neighbouring
// entries of stmg_mg_solve_stream), a kernel does not.
namespace {
__global__ void k_poke(double* dst, PokeWords w, int count) {
  pdl_entry();
  if ((int)threadIdx.x < count) dst[threadIdx.x] = w.v[threadIdx.x];
}
__global__ void k_peek(double* host_dst, const double* src, int count) {
  pdl_entry();
  for (int k = threadIdx.x; k < count; k += blockDim.x) host_dst[k] = src[k];
  __threadfence_system();
}
}  // namespace

int launch_poke(double* dst, const PokeWords& w, int count, cudaStream_t s) {
  if (count < 0 || count > kPokeWords) return cudaErrorInvalidValue;
  pdl_launch(k_poke, 1, 32, 0, s, dst, w, count);
  return check_launch();
}

int launch_peek(double* host_dst, const double* src, int count, cudaStream_t s) {
  pdl_launch(k_peek, 1, 256, 0, s, host_dst, src, count);
  return check_launch();
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

// Exact coarsest solve, by the shape of the level:
//   m > 32 with chunks: parallel-in-time march (k_coarsest_pint + Kogge-Stone links);
//   m <= 32 with chunks whose tables fit in shared memory: k_coarsest_chunked (one CTA);
//   m <= 32 otherwise: k_coarsest_prop (T^-1 and A tables, g_n in scratch);
//   else the sequential block-PCR march k_coarsest.
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
  // shared-memory opt-ins of the coarsest marches (up to 160 KB of tables / work vectors)
  cudaError_t e = cudaSuccess;
  auto opt_in = [&](auto fn) {
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  };
  opt_in(k_coarsest<true>);
  opt_in(k_coarsest<false>);
  opt_in(k_coarsest_prop<true>);
  opt_in(k_coarsest_prop<false>);
  opt_in(k_coarsest_chunked<true>);
  opt_in(k_coarsest_chunked<false>);
  opt_in(k_coarsest_pint<true, 0>);
  opt_in(k_coarsest_pint<true, 1>);
  opt_in(k_coarsest_pint<false, 0>);
  opt_in(k_coarsest_pint<false, 1>);
  opt_in(k_coarsest_pint<false, 2>);
  return static_cast<int>(e);
}

namespace {
// More than this many partials are summed in two stages (kPartialsScratch blocks,
// then one), through the scratch doubles every partials buffer has past its end.
constexpr int64_t kOneStagePartials = int64_t{1} << 16;  // finalize_launches agrees
const double* stage_partials(const double* partials, int64_t* n, cudaStream_t s) {
  if (*n <= kOneStagePartials) return partials;
  const int64_t chunk = ceil_div(*n, kPartialsScratch);
  const unsigned blocks = (unsigned)ceil_div(*n, chunk);
  double* scratch = const_cast<double*>(partials) + *n;
  pdl_launch(k_partials_stage, blocks, 256, 0, s, partials, *n, chunk, scratch);
  *n = blocks;
  return scratch;
}
}  // namespace

int launch_finalize_sum(const double* partials, int64_t n, double* out, cudaStream_t s) {
  const double* p = stage_partials(partials, &n, s);
  pdl_launch(k_finalize_sum, 1, 1024, 0, s, p, n, out);
  return check_launch();
}

int launch_finalize_check(const double* partials, int64_t n, double* scalars, SolveLoopCtl* ctl, double* hist,
                          cudaGraphConditionalHandle handle, cudaStream_t s) {
  const double* p = stage_partials(partials, &n, s);
  pdl_launch(k_finalize_check, 1, 1024, 0, s, p, n, scalars, ctl, hist, handle);
  return check_launch();
}

int launch_sensitivities(int64_t n_el, int64_t n_t, double dt, const double* dk_dx,
                         const double* dc_dx6, const double* u, const double* lam, double* sens,
                         cudaStream_t s) {
  // one block of kSensWarps warps per kSensE elements; dt a power of two (frexp
  // mantissa 0.5, finite reciprocal): multiply by the exact 1 / dt instead of dividing
  int ex = 0;
  const bool pow2 = dt > 0.0 && std::frexp(dt, &ex) == 0.5 && std::isfinite(1.0 / dt);
  const unsigned grid = (unsigned)((n_el + kSensE - 1) / kSensE);
  if (pow2)
    pdl_launch(k_sensitivities<true>, grid, kSensWarps * 32, 0, s, n_el, n_t, dt, dk_dx, dc_dx6, u, lam, sens);
  else
    pdl_launch(k_sensitivities<false>, grid, kSensWarps * 32, 0, s, n_el, n_t, dt, dk_dx, dc_dx6, u, lam, sens);
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
