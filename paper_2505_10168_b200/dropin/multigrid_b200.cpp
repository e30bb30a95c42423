// Drop-in replacement for the reference's proj/src/multigrid.cpp on the B200
// library: the reference's own solver API (proj/include/stmg/multigrid.hpp:33-108,
// namespace stmg, unchanged signatures) implemented over the C ABI of
// include/stmg_b200.h.  A maintainer compiles this file against the reference's
// headers in place of multigrid.cpp and links libstmg_b200.so; every caller of
// build_hierarchy / transposed_hierarchy / mg_solve -- optimise()
// (proj/src/optimisation.cpp:116-139), the experiments, the CLI -- then runs its
// V-cycles on the GPU with no source change.  INTEGRATION.md shows the build line;
// tests/test_gpu_dropin.py runs the reference's own optimise() and mg_solve
// through it (oracle/Makefile target `dropin`).
//
// What differs from multigrid.cpp, by design:
//  * No CSR operator, transfer matrix or sparse LU is formed on the host: the
//    per-level operators, transfers and the exact coarsest solver live on the
//    device (that host assembly is the cost the GPU path removes, SURVEY §8(a)
//    rows a8-a10).  Level::J, Level::inv_diag and LevelHierarchy::transfers stay
//    empty; Level::grid carries each level's geometry and materials, built with
//    the reference's own coarsen_grid / coarsen_materials.  Callers that inspect
//    the host operators (the reference's structural tests do) can set
//    STMG_B200_HOST_OPERATORS=1: build_hierarchy / transposed_hierarchy then also
//    fill those members with the reference's own assemble_system / build_transfer /
//    galerkin_operator (host cost and memory as in the reference; the solve does
//    not read them).
//  * LevelHierarchy::coarsest still owns the hierarchy's exact solver: its pimpl
//    (DirectSolver::Impl) owns the device hierarchy handle, so the handle follows
//    the LevelHierarchy through moves and dies with it.
//  * A stand-alone DirectSolver / direct_solve on a caller's CSR matrix (the
//    reference's tests and its gradient check use it as an exact host solver,
//    proj/src/multigrid.cpp:24-66) is a host banded LU with partial pivoting here,
//    so the drop-in needs no Eigen; it is not on the solve path.
//
// Errors keep the reference's classes: std::invalid_argument, std::runtime_error
// and std::out_of_range, mapped from the C ABI's codes.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <cstdlib>

#include "stmg/assembly.hpp"
#include "stmg/multigrid.hpp"
#include "stmg/rediscretisation.hpp"
#include "stmg/transfer.hpp"
#include "stmg_b200.h"

namespace stmg {

// Host LU of a banded matrix with partial pivoting (stand-alone DirectSolver
// only).  Row r keeps columns r - kl .. r + ku + kl (interchanges widen the upper
// band by kl).  Interchanges swap the active part of two rows (columns >= k); the
// multipliers of earlier steps stay where they were computed, and solve() replays
// interchange k before eliminating with column k's multipliers.
struct BandLU {
  std::int64_t n = 0, kl = 0, ku = 0, w = 0;
  std::vector<double> a;          // entry (r, c) at a[r * w + (c - r + kl)]
  std::vector<std::int64_t> piv;  // row interchanged with row k at step k
  double& at(std::int64_t r, std::int64_t c) { return a[static_cast<std::size_t>(r * w + (c - r + kl))]; }
  double at(std::int64_t r, std::int64_t c) const { return a[static_cast<std::size_t>(r * w + (c - r + kl))]; }

  bool factor(const SparseMatrix& m) {
    n = m.rows();
    for (std::int32_t r = 0; r < m.rows(); ++r)
      for (std::int32_t p = m.row_ptr()[r]; p < m.row_ptr()[r + 1]; ++p) {
        const std::int64_t c = m.col_idx()[p];
        kl = std::max<std::int64_t>(kl, r - c);
        ku = std::max<std::int64_t>(ku, c - r);
      }
    w = 2 * kl + ku + 1;
    a.assign(static_cast<std::size_t>(n * w), 0.0);
    piv.assign(static_cast<std::size_t>(n), 0);
    for (std::int32_t r = 0; r < m.rows(); ++r)
      for (std::int32_t p = m.row_ptr()[r]; p < m.row_ptr()[r + 1]; ++p) at(r, m.col_idx()[p]) += m.values()[p];
    for (std::int64_t k = 0; k < n; ++k) {
      const std::int64_t rmax = std::min(n - 1, k + kl), cmax = std::min(n - 1, k + ku + kl);
      std::int64_t best = k;
      double vbest = std::abs(at(k, k));
      for (std::int64_t r = k + 1; r <= rmax; ++r)
        if (std::abs(at(r, k)) > vbest) vbest = std::abs(at(r, k)), best = r;
      if (!(vbest > 0.0) || !std::isfinite(vbest)) return false;
      piv[static_cast<std::size_t>(k)] = best;
      if (best != k)
        for (std::int64_t c = k; c <= cmax; ++c) std::swap(at(k, c), at(best, c));
      const double d = at(k, k);
      for (std::int64_t r = k + 1; r <= rmax; ++r) {
        const double l = at(r, k) / d;
        at(r, k) = l;
        if (l != 0.0)
          for (std::int64_t c = k + 1; c <= cmax; ++c) at(r, c) -= l * at(k, c);
      }
    }
    return true;
  }
  void solve(std::span<const double> rhs, std::span<double> x) const {
    std::vector<double> y(rhs.begin(), rhs.end());
    for (std::int64_t k = 0; k < n; ++k) {
      std::swap(y[static_cast<std::size_t>(k)], y[static_cast<std::size_t>(piv[static_cast<std::size_t>(k)])]);
      const std::int64_t rmax = std::min(n - 1, k + kl);
      const double yk = y[static_cast<std::size_t>(k)];
      if (yk != 0.0)
        for (std::int64_t r = k + 1; r <= rmax; ++r) y[static_cast<std::size_t>(r)] -= at(r, k) * yk;
    }
    for (std::int64_t k = n - 1; k >= 0; --k) {
      const std::int64_t cmax = std::min(n - 1, k + ku + kl);
      double s = y[static_cast<std::size_t>(k)];
      for (std::int64_t c = k + 1; c <= cmax; ++c) s -= at(k, c) * x[static_cast<std::size_t>(c)];
      x[static_cast<std::size_t>(k)] = s / at(k, k);
    }
  }
};

struct DirectSolver::Impl {
  stmg_hierarchy* h = nullptr;  // a hierarchy's device handle (build_hierarchy), or
  BandLU lu;                    // a stand-alone host factorisation
  ~Impl() {
    if (h) stmg_hierarchy_destroy(h);
  }
};

namespace {

// The structs passed across the C ABI (stmg_solve_report) are this header's: a library
// built from another version must not be called.
void check_abi() {
  static const bool ok = stmg_abi_version() == STMG_ABI_VERSION;
  if (!ok)
    throw std::runtime_error("libstmg_b200.so has C ABI version " + std::to_string(stmg_abi_version()) +
                             ", multigrid_b200.cpp was compiled for " + std::to_string(STMG_ABI_VERSION));
}

void check(int rc) {
  if (rc == STMG_OK) return;
  const std::string what = stmg_last_error();
  switch (rc) {
    case STMG_EINVAL: throw std::invalid_argument(what);
    case STMG_ERANGE: throw std::out_of_range(what);
    default: throw std::runtime_error(what);
  }
}

// DirectSolver objects of hierarchies built here -> their device handles (the
// pimpl is private to the class; the registry is how mg_solve finds it).
std::mutex g_mu;
std::map<const DirectSolver*, stmg_hierarchy*> g_handles;
thread_local stmg_hierarchy* t_adopt = nullptr;  // handed to the next DirectSolver constructed

std::unique_ptr<DirectSolver> owning_solver(stmg_hierarchy* h) {
  t_adopt = h;
  try {
    auto ds = std::make_unique<DirectSolver>(SparseMatrix{});
    t_adopt = nullptr;
    return ds;
  } catch (...) {
    t_adopt = nullptr;
    stmg_hierarchy_destroy(h);
    throw;
  }
}

stmg_hierarchy* handle_of(const LevelHierarchy& h) {
  std::lock_guard<std::mutex> lk(g_mu);
  const auto it = g_handles.find(h.coarsest.get());
  if (it == g_handles.end() || it->second == nullptr)
    throw std::invalid_argument("mg_solve: hierarchy was not built by build_hierarchy");
  return it->second;
}

bool host_operators_wanted() {
  const char* e = std::getenv("STMG_B200_HOST_OPERATORS");
  return e != nullptr && e[0] != '\0' && e[0] != '0';
}

// 1 / diag(J) as Level::inv_diag holds it (proj/src/multigrid.cpp:72-82)
std::vector<double> inverse_diagonal(const SparseMatrix& J) {
  std::vector<double> d = J.diagonal();
  for (double& v : d) {
    if (v == 0.0) throw std::runtime_error("build_hierarchy: level operator has a zero diagonal entry");
    v = 1.0 / v;
  }
  return d;
}

// Host mirrors of the level operators and transfers (opt-in, see the header note).
void fill_host_operators(LevelHierarchy& h) {
  for (std::size_t l = 0; l < h.levels.size(); ++l) {
    Level& lv = h.levels[l];
    if (l > 0) {
      h.transfers.push_back(build_transfer(h.levels[l - 1].grid, lv.grid, h.path.dirs[l - 1], h.method.interp));
      const TransferPair& t = h.transfers.back();
      lv.J = h.method.reassembly == ReassemblyMethod::P ? galerkin_operator(t.R, h.levels[l - 1].J, t.P)
                                                        : assemble_system(lv.grid).J;
    } else {
      lv.J = assemble_system(lv.grid).J;
    }
    lv.inv_diag = inverse_diagonal(lv.J);
  }
}

int32_t dir_code(CoarseningDirection d) {
  switch (d) {
    case CoarseningDirection::SpaceX: return STMG_DIR_X;
    case CoarseningDirection::TimeT: return STMG_DIR_T;
    default: return STMG_DIR_XT;
  }
}

}  // namespace

DirectSolver::DirectSolver(const SparseMatrix& m) : impl_(new Impl) {
  if (t_adopt == nullptr) {  // stand-alone exact solver (proj/src/multigrid.cpp:24-41)
    if (m.rows() != m.cols()) throw std::invalid_argument("DirectSolver: matrix must be square");
    if (!impl_->lu.factor(m))
      throw std::runtime_error("DirectSolver: sparse LU factorisation failed (singular operator?)");
    return;
  }
  impl_->h = t_adopt;
  std::lock_guard<std::mutex> lk(g_mu);
  g_handles[this] = impl_->h;
}

DirectSolver::DirectSolver(DirectSolver&& o) noexcept : impl_(std::move(o.impl_)) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_handles.erase(&o);
  if (impl_ && impl_->h) g_handles[this] = impl_->h;
}

DirectSolver& DirectSolver::operator=(DirectSolver&& o) noexcept {
  if (this != &o) {
    std::lock_guard<std::mutex> lk(g_mu);
    impl_ = std::move(o.impl_);
    g_handles.erase(&o);
    if (impl_ && impl_->h) g_handles[this] = impl_->h;
    else g_handles.erase(this);
  }
  return *this;
}

DirectSolver::~DirectSolver() {
  std::lock_guard<std::mutex> lk(g_mu);
  g_handles.erase(this);
}

void DirectSolver::solve(std::span<const double> rhs, std::span<double> x) const {
  if (impl_->h != nullptr)
    throw std::logic_error("DirectSolver::solve: a hierarchy's coarsest solve runs on the device inside mg_solve");
  if (std::cmp_not_equal(rhs.size(), impl_->lu.n) || std::cmp_not_equal(x.size(), impl_->lu.n))
    throw std::invalid_argument("DirectSolver::solve: size mismatch");
  impl_->lu.solve(rhs, x);
}

// proj/src/multigrid.cpp:59-66
std::vector<double> direct_solve(const SparseMatrix& m, std::span<const double> rhs) {
  const DirectSolver ds(m);
  std::vector<double> x(rhs.size());
  ds.solve(rhs, x);
  return x;
}

// proj/src/multigrid.cpp:86-143
LevelHierarchy build_hierarchy(const SpaceTimeGrid& fine, const RediscretisationMethod& method,
                               const CoarseningPath& path, const DesignField* chi, const MaterialPair* mat) {
  if (!fine.has_materials()) throw std::invalid_argument("build_hierarchy: fine grid has no materials");
  check_abi();
  const bool track_chi = method.reassembly == ReassemblyMethod::D;
  if (track_chi && (chi == nullptr || mat == nullptr))
    throw std::invalid_argument("build_hierarchy: D reassembly needs the design field and materials");

  LevelHierarchy h;
  h.path = path;
  h.method = method;
  h.levels.reserve(path.dirs.size() + 1);
  {
    Level l0;
    l0.grid = fine;
    h.levels.push_back(std::move(l0));
  }
  // level geometry and materials (the reference's coarsen_grid / coarsen_materials)
  DesignField chi_level;
  if (track_chi) chi_level = *chi;
  for (const CoarseningDirection dir : path.dirs) {
    const SpaceTimeGrid& prev = h.levels.back().grid;
    SpaceTimeGrid cg = coarsen_grid(prev, dir);
    CoarsenedMaterials cm = coarsen_materials(prev, dir, method.reassembly, track_chi ? &chi_level : nullptr, mat);
    cg.k = std::move(cm.k);
    cg.c = std::move(cm.c);
    if (track_chi) chi_level = std::move(*cm.chi);
    Level lc;
    lc.grid = std::move(cg);
    h.levels.push_back(std::move(lc));
  }

  // the device hierarchy: operators, transfers and the exact coarsest solver
  const stmg_grid g{fine.L, fine.t_T, fine.n_el, fine.n_t};
  std::vector<int32_t> dirs;
  for (const CoarseningDirection d : path.dirs) dirs.push_back(dir_code(d));
  stmg_material_pair m{};
  if (mat) m = {mat->k_ins, mat->k_con, mat->c_ins, mat->c_con, mat->p_k, mat->p_c};
  const std::string name = method_name(method);
  stmg_hierarchy* dh = nullptr;
  check(stmg_hierarchy_create(&g, fine.k.data(), fine.c.data(), chi ? chi->chi.data() : nullptr,
                              mat ? &m : nullptr, name.c_str(), static_cast<int32_t>(dirs.size()),
                              dirs.empty() ? nullptr : dirs.data(), 0, &dh));
  h.coarsest = owning_solver(dh);
  if (host_operators_wanted()) fill_host_operators(h);
  return h;
}

// proj/src/multigrid.cpp:145-160
LevelHierarchy transposed_hierarchy(const LevelHierarchy& h) {
  stmg_hierarchy* t = nullptr;
  check(stmg_hierarchy_transposed(handle_of(h), &t));
  LevelHierarchy out;
  out.levels = h.levels;
  out.transfers = h.transfers;
  out.path = h.path;
  out.method = h.method;
  out.coarsest = owning_solver(t);
  for (Level& l : out.levels)  // host mirrors, when present: J^T, same diagonal
    if (l.J.rows() > 0) l.J = l.J.transposed();
  return out;
}

const char* status_name(SolveStatus s) {
  switch (s) {
    case SolveStatus::Converged: return "converged";
    case SolveStatus::MaxCycles: return "max-cycles";
    case SolveStatus::Diverged: return "diverged";
  }
  return "unknown";
}

// proj/src/multigrid.cpp:212-279
SolveReport mg_solve(const LevelHierarchy& h, std::span<const double> b, std::span<double> u,
                     const SolveOptions& opts) {
  const std::size_t n = h.levels.front().grid.n_dofs();
  if (b.size() != n || u.size() != n) throw std::invalid_argument("mg_solve: vector size mismatch");
  stmg_hierarchy* dh = handle_of(h);
  const stmg_solve_options o{opts.nu, opts.omega, opts.tol, opts.div_tol, opts.max_cycles};
  std::vector<double> hist(static_cast<std::size_t>(std::max(opts.max_cycles, 0)) + 1);
  stmg_solve_report rep{};
  check(stmg_mg_solve(dh, b.data(), u.data(), &o, &rep, hist.data(), static_cast<int32_t>(hist.size())));
  SolveReport out;
  out.status = static_cast<SolveStatus>(rep.status);
  out.cycles = rep.cycles;
  out.factor = rep.factor;
  out.history.assign(hist.begin(), hist.begin() + rep.n_history);
  out.absolute_norms = rep.absolute_norms != 0;
  out.seconds = rep.seconds;
  return out;
}

}  // namespace stmg
