// stmg_b200.hpp — header-only C++ face of the C ABI in stmg_b200.h, shaped like
// the reference's solver API (namespace stmg, proj/include/stmg/*.hpp) so a
// caller can switch with minimal edits:
//
//   reference                                   here (namespace stmg_b200)
//   build_fine_grid       mesh.hpp:62           Grid{L, t_T, n_el, n_t}
//   plan_coarsening       strategy.hpp:104      plan_coarsening(...)
//   build_hierarchy       multigrid.hpp:70-74   Hierarchy::build(...)
//   transposed_hierarchy  multigrid.hpp:77      Hierarchy::transposed()
//   mg_solve              multigrid.hpp:107     mg_solve(h, b, u, opts)
//
// Errors are rethrown as the reference's exception classes:
// std::invalid_argument, std::runtime_error, std::out_of_range (and
// std::bad_alloc for allocation failures).  Link with libstmg_b200.so.
#pragma once

#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "stmg_b200.h"

namespace stmg_b200 {

inline void check(int rc) {
  if (rc == STMG_OK) return;
  const std::string msg = stmg_last_error();
  switch (rc) {
    case STMG_EINVAL: throw std::invalid_argument(msg);
    case STMG_ERANGE: throw std::out_of_range(msg);
    case STMG_ENOMEM: throw std::bad_alloc();
    default: throw std::runtime_error(msg);
  }
}

enum class SolveStatus { Converged = STMG_CONVERGED, MaxCycles = STMG_MAX_CYCLES, Diverged = STMG_DIVERGED };

struct SolveOptions {  // proj/include/stmg/multigrid.hpp:83-89
  int nu = 5;
  double omega = 0.5;
  double tol = 1e-9;
  double div_tol = 1e9;
  int max_cycles = 100;
};

struct SolveReport {  // proj/include/stmg/multigrid.hpp:91-102
  SolveStatus status = SolveStatus::MaxCycles;
  int cycles = 0;
  double factor = 1.0;
  std::vector<double> history;
  bool absolute_norms = false;
  double seconds = 0.0;
  double device_seconds = 0.0;
  double smoother_dof_updates = 0.0;
};

struct Grid {
  double L = 1.0, t_T = 1.0;
  long long n_el = 0, n_t = 0;
  stmg_grid c() const { return {L, t_T, n_el, n_t}; }
};

// plan_coarsening with the reference's PlanRequest fields; returns the
// direction list (0 = x, 1 = t).
inline std::vector<int> plan_coarsening(const Grid& g, std::span<const double> k,
                                        std::span<const double> c, int n_levels,
                                        int strategy = STMG_PLAN_CONTRAST,
                                        int reassembly = STMG_REASM_K, long long min_elements = 0,
                                        double lambda_crit = 0.25,
                                        const stmg_material_pair* mat = nullptr,
                                        const double* chi = nullptr,
                                        std::vector<double>* indicators = nullptr) {
  const stmg_grid gc = g.c();
  const stmg_plan_request req{n_levels, lambda_crit, strategy, reassembly, min_elements};
  std::vector<int32_t> dirs(static_cast<size_t>(n_levels > 1 ? n_levels - 1 : 1));
  std::vector<double> ind(dirs.size());
  check(stmg_plan_coarsening(&gc, k.empty() ? nullptr : k.data(), c.empty() ? nullptr : c.data(),
                             chi, mat, &req, dirs.data(), ind.data()));
  dirs.resize(static_cast<size_t>(n_levels - 1));
  ind.resize(dirs.size());
  if (indicators) *indicators = ind;
  return std::vector<int>(dirs.begin(), dirs.end());
}

class Hierarchy {
 public:
  static Hierarchy build(const Grid& g, std::span<const double> k, std::span<const double> c,
                         const std::string& method, const std::vector<int>& dirs, int device = 0,
                         const double* chi = nullptr, const stmg_material_pair* mat = nullptr) {
    const stmg_grid gc = g.c();
    std::vector<int32_t> d(dirs.begin(), dirs.end());
    stmg_hierarchy* h = nullptr;
    check(stmg_hierarchy_create(&gc, k.data(), c.data(), chi, mat, method.c_str(),
                                static_cast<int32_t>(d.size()), d.empty() ? nullptr : d.data(),
                                device, &h));
    return Hierarchy(h);
  }
  // proj/src/multigrid.cpp:145-160 (shares device workspaces with *this)
  Hierarchy transposed() const {
    stmg_hierarchy* t = nullptr;
    check(stmg_hierarchy_transposed(h_.get(), &t));
    return Hierarchy(t);
  }
  int n_levels() const {
    int32_t n = 0;
    check(stmg_hierarchy_n_levels(h_.get(), &n));
    return n;
  }
  stmg_hierarchy* get() const { return h_.get(); }

 private:
  struct Del {
    void operator()(stmg_hierarchy* p) const { stmg_hierarchy_destroy(p); }
  };
  explicit Hierarchy(stmg_hierarchy* h) : h_(h, Del{}) {}
  std::shared_ptr<stmg_hierarchy> h_;
};

namespace detail {
inline SolveReport to_report(const stmg_solve_report& r, const double* hist) {
  SolveReport out;
  out.status = static_cast<SolveStatus>(r.status);
  out.cycles = r.cycles;
  out.factor = r.factor;
  out.history.assign(hist, hist + r.n_history);
  out.absolute_norms = r.absolute_norms != 0;
  out.seconds = r.seconds;
  out.device_seconds = r.device_seconds;
  out.smoother_dof_updates = r.smoother_dof_updates;
  return out;
}
}  // namespace detail

// mg_solve: b and u are host or device pointers; u is in/out (warm start).  zero_guess: start
// from zero, u is output only (STMG_SOLVE_ZERO_GUESS; a host u is not uploaded).
inline SolveReport mg_solve(const Hierarchy& h, std::span<const double> b, std::span<double> u,
                            const SolveOptions& o = {}, bool zero_guess = false) {
  if (b.size() != u.size()) throw std::invalid_argument("mg_solve: vector size mismatch");
  const stmg_solve_options co{o.nu, o.omega, o.tol, o.div_tol, o.max_cycles};
  stmg_solve_report r{};
  std::vector<double> hist(static_cast<size_t>(o.max_cycles > 0 ? o.max_cycles : 0) + 1);
  check(stmg_mg_solve_ex(h.get(), b.data(), u.data(), &co, zero_guess ? STMG_SOLVE_ZERO_GUESS : 0, &r, hist.data(),
                         static_cast<int32_t>(hist.size())));
  return detail::to_report(r, hist.data());
}

// A stream of solves on one hierarchy with host vectors (stmg_mg_solve_stream): entry k is
// mg_solve(h, bs[k], us[k], o, zero_guess), in order, bit-identical; the upload of entry k + 1 and
// the download of entry k - 1 overlap solve k when the vectors are page-locked.
inline std::vector<SolveReport> mg_solve_stream(const Hierarchy& h, std::span<const std::span<const double>> bs,
                                                std::span<const std::span<double>> us, const SolveOptions& o = {},
                                                bool zero_guess = false) {
  if (bs.size() != us.size()) throw std::invalid_argument("mg_solve_stream: bs and us differ in length");
  const size_t k = bs.size(), cap = static_cast<size_t>(o.max_cycles > 0 ? o.max_cycles : 0) + 1;
  std::vector<const double*> bp(k);
  std::vector<double*> up(k), hp(k);
  std::vector<double> hist(k * cap);
  for (size_t i = 0; i < k; ++i) {
    if (bs[i].size() != us[i].size()) throw std::invalid_argument("mg_solve_stream: vector size mismatch");
    bp[i] = bs[i].data();
    up[i] = us[i].data();
    hp[i] = hist.data() + i * cap;
  }
  const stmg_solve_options co{o.nu, o.omega, o.tol, o.div_tol, o.max_cycles};
  std::vector<stmg_solve_report> rs(k);
  check(stmg_mg_solve_stream(h.get(), static_cast<int32_t>(k), bp.data(), up.data(), &co,
                             zero_guess ? STMG_SOLVE_ZERO_GUESS : 0, rs.data(), hp.data(), static_cast<int32_t>(cap)));
  std::vector<SolveReport> out;
  for (size_t i = 0; i < k; ++i) out.push_back(detail::to_report(rs[i], hp[i]));
  return out;
}

}  // namespace stmg_b200
