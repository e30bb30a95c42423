// Streaming-march chassis of the level kernels (included by stmg_kernels.cu inside
// namespace stmgb::{anonymous}; uses its row evaluators and loaders' arithmetic).
//
// The register-staged chassis (k_lean2 / k_restrict2) spends ~55 instructions per
// 30-node row: 64-bit addressing per load, four 32-bit shuffles plus moves per
// staged value, two idle halo lanes, a ~130-instruction tile prologue every 8 rows.
// On the low-byte kernels (restriction of the virtual zero iterate: 12 B/DOF) that
// instruction stream, not HBM, is the bound.  Here each warp owns a strip of 32 (or
// 30) consecutive nodes and MARCHES through a chunk of consecutive time levels:
//   * rows are staged by per-lane 8-byte cp.async copies into a warp-private ring
//     of kRing rows in shared memory (34 nodes per row: the strip and its two
//     halo nodes), so kRing - 1 rows per warp are in flight without holding
//     registers and without a block barrier (one __syncwarp per row);
//   * the three same-level values x[i-1], x[i], x[i+1] are three LDS with
//     immediate offsets (no shuffles, all 32 lanes compute); the coupled level's
//     three values stay in registers from the previous step of the march, so a
//     level is read from HBM once and from shared memory once;
//   * the time direction never re-stages a level inside a chunk (one extra row per
//     chunk of up to 256 rows instead of one per 8-row tile).
// Arithmetic is the register-staged kernels' bit for bit: the same row_interior /
// row_sum evaluations, the same zero_sweep / prolong_row / restriction sums.
//
// SRC: where the staged iterate comes from
//   kSrcPlain    stored x                                   (stage x and f)
//   kSrcZero     S(0) = 0 + omega (f * inv_diag) from f     (stage f with halo)
//   kSrcProlong  stored x + P xc                            (stage x, f, xc)
//   kSrcProlongZ S(0) + P xc                                (stage f with halo, xc)
// OUT: what a row produces
//   kOutSweep    y = x + omega ((f - A x) * inv_diag)       (+ r^2 partial: NORM)
//   kOutRestrict f_c = R (f - A x), x step (RDIR 0: warps advance 30 nodes, the
//                odd lanes hold the even fine nodes 2I) or causal t step (RDIR 1)
#pragma once

namespace march {

constexpr int kWarps = 4;   // warps (strips) per block
constexpr int kRing = 8;    // staged rows per warp
constexpr int kXW = 36;     // doubles per staged row (34 used; [0] and [33] are the halo nodes)

enum Src { kSrcPlain = 0, kSrcZero = 1, kSrcProlong = 2, kSrcProlongZ = 3 };
enum Out { kOutSweep = 0, kOutRestrict = 1 };

__device__ __forceinline__ void cp8(double* smem_dst, const double* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct Args {
  LevelView F;           // the level the rows are evaluated on
  LevelView C;           // coarse level (prolongation source / restriction target)
  const double* f;       // right-hand side of F
  const double* x;       // stored iterate (Plain / Prolong)
  const double* xc;      // coarse correction (Prolong sources)
  double* y;             // sweep output
  double* fc;            // restriction output
  double* xc0;           // optional: first coarse sweep from zero, stored with fc
  double* partials;      // NORM: one r^2 partial per warp
  double omega;
  int32_t chunk;         // rows per warp chunk (even)
};

template <int SRC>
__host__ __device__ constexpr bool src_zero() { return SRC == kSrcZero || SRC == kSrcProlongZ; }
template <int SRC>
__host__ __device__ constexpr bool src_prolong() { return SRC == kSrcProlong || SRC == kSrcProlongZ; }

template <int SRC>
struct Smem {
  double xs[kWarps][kRing][kXW];                                   // staged iterate rows (raw f rows for Zero sources)
  double fs[src_zero<SRC>() ? 1 : kWarps][src_zero<SRC>() ? 1 : kRing][32];  // f rows (Plain / Prolong)
  double cs[src_prolong<SRC>() ? kWarps : 1][src_prolong<SRC>() ? kRing : 1][kXW];  // coarse rows
};

// FAST: the warp's 34 staged nodes are interior nodes and every row of the chunk is an
// interior row (warp-uniform, decided by the kernel): no range checks, no boundary
// row classes, predicate-free copies.  !FAST: the general per-row-class evaluation.
template <bool ADJ, int SRC, int PDIR, int OUT, int RDIR, bool NORM, bool FAST>
__device__ __forceinline__ double body(const Args& a, Smem<SRC>& sm, int64_t i_first, int64_t ra, int64_t rb) {
  constexpr bool kZero = src_zero<SRC>(), kProl = src_prolong<SRC>();
  const LevelView& L = a.F;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nn = L.nn, nt = L.n_t, nnc = a.C.nn;
  double acc = 0.0;
  const int64_t i = i_first + lane;
  const bool in_grid = FAST || (i >= 0 && i < nn);
  // halo nodes handled by lanes 0 (left, e = 0) and 1 (right, e = 33)
  const int64_t ih = lane == 0 ? i_first - 1 : i_first + 32;
  const int eh = lane == 0 ? 0 : 33;
  const bool halo = lane < 2 && (FAST || (ih >= 0 && ih < nn));
  double(*xs)[kXW] = sm.xs[warp];
  if (!FAST) {  // slots of nodes outside the grid are never copied into: clear them once
    for (int k = lane; k < kRing * kXW; k += 32) (&xs[0][0])[k] = 0.0;
    __syncwarp();
  }
  const int64_t sb = ADJ ? ra : ra - 1;  // first staged level
  const int S = (int)(rb - ra) + 1;      // staged levels sb .. sb + S - 1
  const uint32_t nn32 = (uint32_t)nn, nnc32 = (uint32_t)nnc;
  // 64-bit per-lane bases at staged level sb (sb may be -1: never dereferenced then),
  // 32-bit element offsets s * nn from them
  const double* __restrict__ X = kZero ? a.f : a.x;
  const double* __restrict__ xg = opaque(X + (sb * nn + i));
  const double* __restrict__ xh = opaque(X + (sb * nn + ih));
  const double* __restrict__ fg = opaque(a.f + ((ADJ ? sb - 1 : sb) * nn + i));  // f of the row of step s at offset s nn
  // coarse rows: x step, coarse level = fine level, nodes i_first / 2 - 1 + j (j < 18);
  // t step, coarse level = fine level >> 1, the fine nodes
  const int64_t ic = PDIR == 0 ? (i_first >> 1) - 1 + lane : i;
  const bool c_in = kProl && (PDIR == 0 ? (lane < 18 && (FAST || (ic >= 0 && ic < nnc))) : in_grid);
  const double* __restrict__ cg = kProl ? opaque(a.xc + ((PDIR == 0 ? sb : 0) * nnc + ic)) : nullptr;
  const double* __restrict__ ch = kProl && PDIR == 1 ? opaque(a.xc + ih) : nullptr;
  double* __restrict__ yg = OUT == kOutSweep && a.y != nullptr ? opaque(a.y + ((ADJ ? sb - 1 : sb) * nn + i)) : nullptr;
  Coefs c{};
  if (in_grid) c = load_coefs(L, i);
  double idh = 0.0;  // inverse diagonal at the lane's halo node (Zero sources)
  if (kZero && halo) idh = __ldg(L.coef + kInvD * nn + ih);

  auto issue = [&](int s, int slot) {
    const int64_t m = sb + s;
    const uint32_t ro = (uint32_t)s * nn32;
    if (s < S) {
      if (!kZero && s >= 1 && in_grid) cp8(&sm.fs[warp][slot][lane], fg + ro);
      if (FAST || (m >= 0 && m <= nt)) {
        if (in_grid) cp8(&xs[slot][lane + 1], xg + ro);
        if (halo) cp8(&xs[slot][eh], xh + ro);
        if (kProl) {
          if (PDIR == 0) {
            if (c_in) cp8(&sm.cs[warp][slot][lane], cg + (uint32_t)s * nnc32);
          } else {
            const uint32_t co = (uint32_t)((sb + s) >> 1) * nnc32;
            if (c_in) cp8(&sm.cs[warp][slot][lane + 1], cg + co);
            if (halo) cp8(&sm.cs[warp][slot][eh], ch + co);
          }
        }
      }
    }
    cp_commit();
  };

  // Zero / Prolong sources: turn the raw staged row into the iterate row in place
  // (each slot entry is read and rewritten by the one lane that owns it)
  auto prepare_at = [&](int slot, int64_t m, int e, int64_t node, double id_node) {
    double v = xs[slot][e];
    if (kZero) v = zero_sweep(v, (!FAST && (m == 0 || node == 0)) ? L.inv_w : id_node, a.omega);
    if (kProl) {
      if (PDIR == 0) {
        // node = i_first - 1 + e (i_first even): xc[node >> 1] at cs[(e + 1) >> 1],
        // xc[(node + 1) >> 1] at cs[(e >> 1) + 1]
        const double ca = sm.cs[warp][slot][(e + 1) >> 1];
        if (node & 1) {
          const double cb = sm.cs[warp][slot][(e >> 1) + 1];
          v = v + ((0.5 * ca + 0.5 * cb) + 0.0);
        } else {
          v = v + (0.0 + 1.0 * ca);
        }
      } else {
        v = v + (0.0 + 1.0 * sm.cs[warp][slot][e]);
      }
    }
    xs[slot][e] = v;
  };

  // previous staged level's values (i - 1, i, i + 1), its raw f (Zero sources, J^T)
  double pm = 0.0, p0 = 0.0, pp = 0.0, f_prev = 0.0, r_even = 0.0;

  auto step = [&](int s, int slot) {
    const int64_t m = sb + s;
    const bool m_in = FAST || (m >= 0 && m <= nt);
    double f_raw = 0.0;
    if (kZero) f_raw = xs[slot][lane + 1];
    if ((kZero || kProl) && m_in) {
      if (in_grid) prepare_at(slot, m, lane + 1, i, c.invd);
      if (halo) prepare_at(slot, m, eh, ih, idh);
      __syncwarp();
    }
    const double qm = xs[slot][lane], q0 = xs[slot][lane + 1], qp = xs[slot][lane + 2];
    if (s >= 1) {
      const int64_t n = ADJ ? m - 1 : m;  // the row evaluated at this step
      const uint32_t ro = (uint32_t)s * nn32;
      const double fv = kZero ? (ADJ ? f_prev : f_raw) : sm.fs[warp][slot][lane];
      double r = 0.0, x0 = ADJ ? p0 : q0, id = c.invd;
      if (FAST) {
        r = fv - (ADJ ? row_interior<true>(c, pm, p0, pp, qm, q0, qp)
                      : row_interior<false>(c, qm, q0, qp, pm, p0, pp));
      } else if (in_grid) {
        r = fv - (ADJ ? row_sum<true>(L, n, i, c, pm, p0, pp, qm, q0, qp)
                      : row_sum<false>(L, n, i, c, qm, q0, qp, pm, p0, pp));
        if (n == 0 || i == 0) id = L.inv_w;
      }
      if (OUT == kOutSweep) {
        if (in_grid) {
          if (NORM) acc = acc + r * r;
          if (yg != nullptr) *(yg + ro) = x0 + a.omega * (r * id);
        }
      } else if (RDIR == 0) {
        // lanes at even fine nodes 2I (odd lanes) take r at lanes l - 1, l, l + 1
        const double ra_ = __shfl_up_sync(kFull, r, 1);
        const double rc_ = __shfl_down_sync(kFull, r, 1);
        const int64_t I = i >> 1;
        const bool out = (lane & 1) && lane <= 29 && in_grid;
        if (out) {
          double v;
          if (FAST) {
            v = ((0.5 * ra_ + 1.0 * r) + 0.5 * rc_) + 0.0;
          } else {
            Acc t;
            if (I >= 1) t.add(0.5 * ra_);
            t.add(1.0 * r);
            if (2 * I + 1 <= L.n_el) t.add(0.5 * rc_);
            v = t.result();
          }
          a.fc[n * nnc + I] = v;
          if (a.xc0 != nullptr) a.xc0[n * nnc + I] = coarse_from_zero(a.C, n, I, v, a.omega);
        }
      } else {
        // causal t step: coarse level N = fine levels 2N, 2N + 1 at the same node
        if ((n & 1) == 0) {
          r_even = r;
          if (!FAST && n == nt && in_grid) {  // last coarse level: truncated row, 0.5 r(2N) only
            Acc t;
            t.add(0.5 * r);
            const double v = t.result();
            a.fc[(n >> 1) * nnc + i] = v;
            if (a.xc0 != nullptr) a.xc0[(n >> 1) * nnc + i] = coarse_from_zero(a.C, n >> 1, i, v, a.omega);
          }
        } else if (in_grid) {
          double v;
          if (FAST) {
            v = (0.5 * r_even + 0.5 * r) + 0.0;
          } else {
            Acc t;
            t.add(0.5 * r_even);
            t.add(0.5 * r);
            v = t.result();
          }
          a.fc[(n >> 1) * nnc + i] = v;
          if (a.xc0 != nullptr) a.xc0[(n >> 1) * nnc + i] = coarse_from_zero(a.C, n >> 1, i, v, a.omega);
        }
      }
    }
    pm = qm;
    p0 = q0;
    pp = qp;
    f_prev = f_raw;
  };

#pragma unroll
  for (int s = 0; s < kRing - 1; ++s) issue(s, s);
  for (int s0 = 0; s0 < S; s0 += kRing) {
#pragma unroll
    for (int j = 0; j < kRing; ++j) {
      const int s = s0 + j;
      if (s >= S) break;
      cp_wait<kRing - 2>();
      __syncwarp();
      issue(s + kRing - 1, (j + kRing - 1) % kRing);
      step(s, j);
    }
  }
  return acc;
}

template <bool ADJ, int SRC, int PDIR, int OUT, int RDIR, bool NORM, int MINB>
__global__ void __launch_bounds__(kWarps * 32, MINB) k_march(const Args a) {
  pdl_entry();
  __shared__ Smem<SRC> sm;
  constexpr int kAdv = (OUT == kOutRestrict && RDIR == 0) ? 30 : 32;
  const LevelView& L = a.F;
  const int64_t strip = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int64_t i_first = strip * kAdv - (kAdv == 30 ? 1 : 0);  // node of lane 0
  const int64_t ra = L.n_lo + (int64_t)blockIdx.y * a.chunk;
  const int64_t rb = ra + a.chunk < L.n_hi ? ra + a.chunk : L.n_hi;
  double acc = 0.0;
  if (strip * kAdv < L.nn && ra < rb) {  // warp-uniform
    // staged nodes i_first - 1 .. i_first + 32 interior (and their coarse nodes inside);
    // every evaluated row interior with its coupled level: J rows >= 2, J^T rows <= n_t - 1
    const bool fast = i_first >= 3 && i_first + 33 <= L.n_el - 1 && ra >= 2 && (ADJ ? rb <= L.n_t : rb <= L.n_t + 1);
    if (fast) acc = body<ADJ, SRC, PDIR, OUT, RDIR, NORM, true>(a, sm, i_first, ra, rb);
    else acc = body<ADJ, SRC, PDIR, OUT, RDIR, NORM, false>(a, sm, i_first, ra, rb);
  }
  if (NORM) {  // one partial per warp, fixed order
    for (int o = 16; o > 0; o >>= 1) acc = acc + __shfl_xor_sync(kFull, acc, o);
    if ((threadIdx.x & 31) == 0)
      a.partials[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * kWarps + (threadIdx.x >> 5)] = acc;
  }
}

}  // namespace march
