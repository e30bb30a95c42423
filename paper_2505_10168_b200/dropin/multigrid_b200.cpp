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
//    the reference's own coarsen_grid / coarsen_materials.
//  * LevelHierarchy::coarsest still owns the hierarchy's exact solver: its pimpl
//    (DirectSolver::Impl) owns the device hierarchy handle, so the handle follows
//    the LevelHierarchy through moves and dies with it.
//  * A stand-alone DirectSolver / direct_solve on an arbitrary CSR matrix is not
//    part of the solve path and is not provided (std::logic_error).
//
// Errors keep the reference's classes: std::invalid_argument, std::runtime_error
// and std::out_of_range, mapped from the C ABI's codes.
#include <chrono>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "stmg/multigrid.hpp"
#include "stmg_b200.h"

namespace stmg {

struct DirectSolver::Impl {
  stmg_hierarchy* h = nullptr;
  ~Impl() {
    if (h) stmg_hierarchy_destroy(h);
  }
};

namespace {

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

int32_t dir_code(CoarseningDirection d) {
  switch (d) {
    case CoarseningDirection::SpaceX: return STMG_DIR_X;
    case CoarseningDirection::TimeT: return STMG_DIR_T;
    default: return STMG_DIR_XT;
  }
}

}  // namespace

DirectSolver::DirectSolver(const SparseMatrix&) : impl_(new Impl) {
  if (t_adopt == nullptr)
    throw std::logic_error(
        "DirectSolver: stand-alone sparse LU solves are not part of the B200 drop-in "
        "(the exact coarsest solve runs on the device inside mg_solve)");
  impl_->h = t_adopt;
  std::lock_guard<std::mutex> lk(g_mu);
  g_handles[this] = impl_->h;
}

DirectSolver::DirectSolver(DirectSolver&& o) noexcept : impl_(std::move(o.impl_)) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_handles.erase(&o);
  if (impl_) g_handles[this] = impl_->h;
}

DirectSolver& DirectSolver::operator=(DirectSolver&& o) noexcept {
  if (this != &o) {
    std::lock_guard<std::mutex> lk(g_mu);
    impl_ = std::move(o.impl_);
    g_handles.erase(&o);
    if (impl_) g_handles[this] = impl_->h;
    else g_handles.erase(this);
  }
  return *this;
}

DirectSolver::~DirectSolver() {
  std::lock_guard<std::mutex> lk(g_mu);
  g_handles.erase(this);
}

void DirectSolver::solve(std::span<const double> rhs, std::span<double> x) const {
  (void)rhs;
  (void)x;
  throw std::logic_error("DirectSolver::solve: the coarsest solve runs on the device inside mg_solve");
}

std::vector<double> direct_solve(const SparseMatrix& m, std::span<const double> rhs) {
  (void)rhs;
  DirectSolver ds(m);  // throws std::logic_error
  return {};
}

// proj/src/multigrid.cpp:86-143
LevelHierarchy build_hierarchy(const SpaceTimeGrid& fine, const RediscretisationMethod& method,
                               const CoarseningPath& path, const DesignField* chi, const MaterialPair* mat) {
  if (!fine.has_materials()) throw std::invalid_argument("build_hierarchy: fine grid has no materials");
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
