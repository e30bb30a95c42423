// Host-side construction of the general coarse discretisations (SURVEY.md
// §8(f) item 4): per-DOF 9-point level operators, the Galerkin product R J P
// in the reference's exact arithmetic, transposition, and the dense block
// factors of the coarsest exact solve.  Included by stmg_hierarchy.cu only.
//
// A level's operator is held as a "Dia9": per row, the 9 slots of columns
// (n + dn, i + di), dn, di in {-1, 0, 1}, plus a bit mask of the slots the
// reference's CSR row stores (structural entries, zeros included: the
// reference never drops them, proj/src/sparse.cpp:121-162).  Slot order is
// ascending column order, so a canonical CSR reduction over present slots is
// the reference's reduction.
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <thread>
#include <vector>

namespace stmgb {

inline int slot9(int dn, int di) { return 3 * (dn + 1) + (di + 1); }

struct Dia9Host {
  int64_t n_el = 0, n_t = 0;
  std::vector<double> v;        // 9 * ndofs, slot-major
  std::vector<uint16_t> mask;   // ndofs
  std::vector<double> inv_diag; // ndofs

  int64_t nn() const { return n_el + 1; }
  int64_t ndofs() const { return (n_el + 1) * (n_t + 1); }
  void init(int64_t ne, int64_t nt) {
    n_el = ne;
    n_t = nt;
    v.assign(static_cast<size_t>(9 * ndofs()), 0.0);
    mask.assign(static_cast<size_t>(ndofs()), 0);
    inv_diag.clear();
  }
  double& at(int k, int64_t r) { return v[static_cast<size_t>(k * ndofs() + r)]; }
  double at(int k, int64_t r) const { return v[static_cast<size_t>(k * ndofs() + r)]; }
};

// Run f(lo, hi) over [0, n) on the host's cores (row-independent work only).
template <class F>
void parallel_rows(int64_t n, F&& f, int64_t serial_below = 65536) {
  unsigned nt = std::max(1u, std::thread::hardware_concurrency());
  if (n < serial_below) nt = 1;
  nt = std::min<unsigned>(nt, 64);
  if (nt == 1) {
    f(int64_t{0}, n);
    return;
  }
  std::vector<std::thread> th;
  const int64_t chunk = (n + nt - 1) / nt;
  for (unsigned t = 0; t < nt; ++t) {
    const int64_t lo = t * chunk, hi = std::min<int64_t>(n, lo + chunk);
    if (lo < hi) th.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& x : th) x.join();
}

// reciprocal_diagonal, proj/src/multigrid.cpp:73-82
inline void dia9_invert_diagonal(Dia9Host& A) {
  A.inv_diag.assign(static_cast<size_t>(A.ndofs()), 0.0);
  const int c = slot9(0, 0);
  for (int64_t r = 0; r < A.ndofs(); ++r) {
    const double d = (A.mask[r] >> c) & 1u ? A.at(c, r) : 0.0;
    if (d == 0.0) throw std::runtime_error("build_hierarchy: level operator has a zero diagonal entry");
    A.inv_diag[r] = 1.0 / d;
  }
}

// The assembled J (proj/src/assembly.cpp:85-132) from a level's per-node
// primal entries W, D, E (same level) and SW, S, SE (level n - 1): masked rows
// (n == 0 || i == 0) hold only w; unmasked rows drop masked columns.
inline Dia9Host dia9_assembled(int64_t n_el, int64_t n_t, const std::vector<double>& W,
                               const std::vector<double>& D, const std::vector<double>& E,
                               const std::vector<double>& SW, const std::vector<double>& S,
                               const std::vector<double>& SE, double w) {
  Dia9Host A;
  A.init(n_el, n_t);
  const int64_t nn = n_el + 1;
  parallel_rows(A.ndofs(), [&](int64_t lo, int64_t hi) {
    for (int64_t r = lo; r < hi; ++r) {
      const int64_t n = r / nn, i = r - n * nn;
      uint16_t m = 0;
      auto put = [&](int dn, int di, double val) {
        A.at(slot9(dn, di), r) = val;
        m |= static_cast<uint16_t>(1u << slot9(dn, di));
      };
      if (n == 0 || i == 0) {
        put(0, 0, w);
      } else {
        if (n >= 2 && i >= 2) put(-1, -1, SW[i]);
        if (n >= 2) put(-1, 0, S[i]);
        if (n >= 2 && i <= n_el - 1) put(-1, 1, SE[i]);
        if (i >= 2) put(0, -1, W[i]);
        put(0, 0, D[i]);
        if (i <= n_el - 1) put(0, 1, E[i]);
      }
      A.mask[r] = m;
    }
  });
  return A;
}

// SparseMatrix::transposed (proj/src/sparse.cpp:74-96) moves values only:
// T(n, i)[dn, di] = A(n + dn, i + di)[-dn, -di].
inline Dia9Host dia9_transposed(const Dia9Host& A) {
  Dia9Host T;
  T.init(A.n_el, A.n_t);
  const int64_t nn = A.nn();
  parallel_rows(A.ndofs(), [&](int64_t lo, int64_t hi) {
    for (int64_t r = lo; r < hi; ++r) {
      const int64_t n = r / nn, i = r - n * nn;
      uint16_t m = 0;
      for (int dn = -1; dn <= 1; ++dn)
        for (int di = -1; di <= 1; ++di) {
          const int64_t n2 = n + dn, i2 = i + di;
          if (n2 < 0 || n2 > A.n_t || i2 < 0 || i2 > A.n_el) continue;
          const int64_t r2 = n2 * nn + i2;
          const int ks = slot9(-dn, -di);
          if ((A.mask[r2] >> ks) & 1u) {
            T.at(slot9(dn, di), r) = A.at(ks, r2);
            m |= static_cast<uint16_t>(1u << slot9(dn, di));
          }
        }
      T.mask[r] = m;
    }
  });
  T.inv_diag = A.inv_diag;  // transposition keeps the diagonal (multigrid.cpp:154)
  return T;
}

// One sparse row entry.
struct Ent {
  int64_t col;
  double val;
};

// Row (N, I) of R = s P^T (proj/src/transfer.cpp:39-104): fine (2N + dn, 2I + dx)
// ascending, value (P value) * s.
inline void restriction_row(int dir, bool bilinear, int64_t f_nel, int64_t f_nt, int64_t c_nn, int64_t q,
                            std::vector<Ent>& out) {
  out.clear();
  const bool hx = dir != 1, ht = dir != 0;
  const double s = dir == 0 ? 1.0 : 0.5;
  const int64_t N = q / c_nn, I = q - N * c_nn, f_nn = f_nel + 1;
  int dns[3];
  double ws[3];
  int nte = 0;
  if (!ht) {
    dns[0] = 0, ws[0] = 1.0, nte = 1;
  } else if (!bilinear) {
    dns[0] = 0, ws[0] = 1.0, dns[1] = 1, ws[1] = 1.0, nte = 2;
  } else {
    dns[0] = -1, ws[0] = 0.5, dns[1] = 0, ws[1] = 1.0, dns[2] = 1, ws[2] = 0.5, nte = 3;
  }
  for (int te = 0; te < nte; ++te) {
    const int64_t nf = ht ? 2 * N + dns[te] : N;
    if (nf < 0 || nf > f_nt) continue;
    const double wt = ws[te];
    if (hx) {
      const int64_t i0 = 2 * I;
      if (i0 - 1 >= 0) out.push_back({nf * f_nn + i0 - 1, (0.5 * wt) * s});
      out.push_back({nf * f_nn + i0, wt * s});
      if (i0 + 1 <= f_nel) out.push_back({nf * f_nn + i0 + 1, (0.5 * wt) * s});
    } else {
      out.push_back({nf * f_nn + I, wt * s});
    }
  }
}

// Row (n, i) of P: coarse columns ascending.
inline void prolongation_row(int dir, bool bilinear, int64_t f_nn, int64_t c_nn, int64_t r,
                             std::vector<Ent>& out) {
  out.clear();
  const bool hx = dir != 1, ht = dir != 0;
  const int64_t n = r / f_nn, i = r - n * f_nn;
  int64_t Nc[2];
  double wt[2];
  int ntm;
  if (!ht) {
    Nc[0] = n, wt[0] = 1.0, ntm = 1;
  } else if (!bilinear || (n & 1) == 0) {
    Nc[0] = n >> 1, wt[0] = 1.0, ntm = 1;
  } else {
    Nc[0] = (n - 1) >> 1, wt[0] = 0.5, Nc[1] = (n + 1) >> 1, wt[1] = 0.5, ntm = 2;
  }
  for (int a = 0; a < ntm; ++a) {
    if (!hx) {
      out.push_back({Nc[a] * c_nn + i, wt[a]});
    } else if ((i & 1) == 0) {
      out.push_back({Nc[a] * c_nn + (i >> 1), wt[a]});
    } else {
      out.push_back({Nc[a] * c_nn + ((i - 1) >> 1), 0.5 * wt[a]});
      out.push_back({Nc[a] * c_nn + ((i + 1) >> 1), 0.5 * wt[a]});
    }
  }
}

// Gustavson row merge (proj/src/sparse.cpp:121-162): acc[j] starts at 0.0 on
// first touch and accumulates in (a-entry, b-entry) order; the row is emitted
// with ascending columns.  Rows here are short, so a linear marker list stands
// in for the dense marker array without changing any accumulation order.
struct RowAcc {
  std::vector<Ent> e;
  void clear() { e.clear(); }
  void add(int64_t col, double prod) {
    for (Ent& x : e)
      if (x.col == col) {
        x.val += prod;
        return;
      }
    e.push_back({col, 0.0});
    e.back().val += prod;
  }
  void sorted(std::vector<Ent>& out) {
    std::sort(e.begin(), e.end(), [](const Ent& a, const Ent& b) { return a.col < b.col; });
    out = e;
  }
};

// galerkin_operator (proj/src/rediscretisation.cpp:112-115): multiply(multiply(R, J), P),
// row by row (row q of R J, then row q of (R J) P, exactly as the two full products).
inline Dia9Host dia9_galerkin(const Dia9Host& J, int dir, bool bilinear, int64_t c_nel, int64_t c_nt) {
  Dia9Host C;
  C.init(c_nel, c_nt);
  const int64_t f_nn = J.nn(), c_nn = c_nel + 1;
  const int64_t f_nd = J.ndofs();
  std::atomic<int> fail{0};
  parallel_rows(C.ndofs(), [&](int64_t lo, int64_t hi) {
    std::vector<Ent> rrow, rj, prow, crow;
    RowAcc acc1, acc2;
    for (int64_t q = lo; q < hi; ++q) {
      restriction_row(dir, bilinear, J.n_el, J.n_t, c_nn, q, rrow);
      acc1.clear();
      for (const Ent& a : rrow) {
        const int64_t k = a.col;
        const unsigned m = J.mask[k];
        for (int s = 0; s < 9; ++s)
          if ((m >> s) & 1u) {
            const int64_t j = k + (s / 3 - 1) * f_nn + (s % 3 - 1);
            acc1.add(j, a.val * J.v[static_cast<size_t>(s * f_nd + k)]);
          }
      }
      acc1.sorted(rj);
      acc2.clear();
      for (const Ent& a : rj) {
        prolongation_row(dir, bilinear, f_nn, c_nn, a.col, prow);
        for (const Ent& p : prow) acc2.add(p.col, a.val * p.val);
      }
      acc2.sorted(crow);
      const int64_t N = q / c_nn, I = q - N * c_nn;
      uint16_t m = 0;
      for (const Ent& e : crow) {
        const int64_t Nc = e.col / c_nn, Ic = e.col - Nc * c_nn;
        const int64_t dn = Nc - N, di = Ic - I;
        if (dn < -1 || dn > 1 || di < -1 || di > 1) {
          fail.store(1);
          continue;
        }
        const int s = slot9(static_cast<int>(dn), static_cast<int>(di));
        C.at(s, q) = e.val;
        m |= static_cast<uint16_t>(1u << s);
      }
      C.mask[q] = m;
    }
  });
  if (fail.load()) throw std::runtime_error("build_hierarchy: Galerkin operator wider than a 3x3 stencil");
  return C;
}

// Dense block factors of a 9-point operator, block-tridiagonal in time with
// m = n_el + 1: M_0 = B_0, M_n = B_n - A_n H_{n-1}, G_n = M_n^-1, H_n = G_n C_n.
// Column-major blocks.  has_upper = 0 when every dn = +1 slot is absent.
struct BlockTables {
  int64_t m = 0, n_t = 0;
  std::vector<double> G, H;
  bool has_upper = false;
};

// In-place inverse of a column-major m x m matrix (LU with partial pivoting).
inline void dense_inverse(std::vector<double>& a, int64_t m) {
  std::vector<int64_t> piv(static_cast<size_t>(m));
  auto A = [&](int64_t i, int64_t j) -> double& { return a[static_cast<size_t>(j * m + i)]; };
  for (int64_t k = 0; k < m; ++k) {
    int64_t p = k;
    for (int64_t i = k + 1; i < m; ++i)
      if (std::fabs(A(i, k)) > std::fabs(A(p, k))) p = i;
    if (A(p, k) == 0.0) throw std::runtime_error("coarsest solver: singular block");
    piv[k] = p;
    if (p != k)
      for (int64_t j = 0; j < m; ++j) std::swap(A(k, j), A(p, j));
    const double inv = 1.0 / A(k, k);
    for (int64_t i = k + 1; i < m; ++i) A(i, k) *= inv;
    for (int64_t j = k + 1; j < m; ++j) {
      const double akj = A(k, j);
      if (akj == 0.0) continue;
      for (int64_t i = k + 1; i < m; ++i) A(i, j) -= A(i, k) * akj;
    }
  }
  // solve A X = I column by column
  std::vector<double> inv(static_cast<size_t>(m * m), 0.0);
  std::vector<double> col(static_cast<size_t>(m));
  for (int64_t c = 0; c < m; ++c) {
    std::fill(col.begin(), col.end(), 0.0);
    col[c] = 1.0;
    for (int64_t k = 0; k < m; ++k)
      if (piv[k] != k) std::swap(col[k], col[piv[k]]);
    for (int64_t k = 0; k < m; ++k)
      for (int64_t i = k + 1; i < m; ++i) col[i] -= A(i, k) * col[k];
    for (int64_t k = m - 1; k >= 0; --k) {
      col[k] /= A(k, k);
      for (int64_t i = 0; i < k; ++i) col[i] -= A(i, k) * col[k];
    }
    std::copy(col.begin(), col.end(), inv.begin() + c * m);
  }
  a.swap(inv);
}

inline BlockTables block_tables(const Dia9Host& A, int64_t max_bytes) {
  BlockTables T;
  const int64_t m = A.nn(), nt = A.n_t;
  T.m = m;
  T.n_t = nt;
  for (int64_t r = 0; r < A.ndofs() && !T.has_upper; ++r)
    for (int di = -1; di <= 1; ++di)
      if ((A.mask[r] >> slot9(1, di)) & 1u) T.has_upper = true;
  const int64_t blocks = (nt + 1) + (T.has_upper ? nt : 0);
  if (static_cast<double>(blocks) * m * m * 8.0 > static_cast<double>(max_bytes))
    throw std::runtime_error(
        "build_hierarchy: coarsest Galerkin level too large for the dense block solver; use more levels");
  T.G.assign(static_cast<size_t>((nt + 1) * m * m), 0.0);
  if (T.has_upper) T.H.assign(static_cast<size_t>(nt * m * m), 0.0);
  std::vector<double> M(static_cast<size_t>(m * m));
  auto entry = [&](int64_t n, int64_t i, int dn, int di) -> double {
    const int64_t r = n * m + i;
    return (A.mask[r] >> slot9(dn, di)) & 1u ? A.at(slot9(dn, di), r) : 0.0;
  };
  for (int64_t n = 0; n <= nt; ++n) {
    std::fill(M.begin(), M.end(), 0.0);
    for (int64_t i = 0; i < m; ++i)
      for (int di = -1; di <= 1; ++di)
        if (i + di >= 0 && i + di < m) M[static_cast<size_t>((i + di) * m + i)] = entry(n, i, 0, di);
    if (n > 0 && T.has_upper) {
      // M -= A_n H_{n-1}; A_n row i has columns i-1..i+1 (dn = -1)
      const double* Hp = T.H.data() + (n - 1) * m * m;
      for (int64_t j = 0; j < m; ++j)
        for (int64_t i = 0; i < m; ++i) {
          double s = 0.0;
          for (int di = -1; di <= 1; ++di)
            if (i + di >= 0 && i + di < m) s += entry(n, i, -1, di) * Hp[j * m + (i + di)];
          M[static_cast<size_t>(j * m + i)] -= s;
        }
    }
    dense_inverse(M, m);
    std::copy(M.begin(), M.end(), T.G.begin() + n * m * m);
    if (T.has_upper && n < nt) {
      // H_n = G_n C_n; C_n row i has columns i-1..i+1 of level n+1
      double* Hn = T.H.data() + n * m * m;
      for (int64_t j = 0; j < m; ++j) {
        // column j of C_n: rows i with i + di == j
        for (int64_t i = 0; i < m; ++i) {
          double s = 0.0;
          for (int di = -1; di <= 1; ++di) {
            const int64_t row = j - di;
            if (row < 0 || row >= m) continue;
            const double c = entry(n, row, 1, di);
            if (c != 0.0) s += M[static_cast<size_t>(row * m + i)] * c;
          }
          Hn[j * m + i] = s;
        }
      }
    }
  }
  return T;
}

}  // namespace stmgb
