// TEST INFRASTRUCTURE — extern "C" harness over the UNMODIFIED reference
// (/root/reference/proj/src, compiled by oracle/Makefile into oracle/_ref/).
// It drives the reference's own public API (build_fine_grid, plan_coarsening,
// build_hierarchy, transposed_hierarchy, mg_solve, load_vector, assemble_system,
// SparseMatrix kernels) so tests can pin the C oracle and the GPU path to the
// reference's actual outputs.  Only tests/, smoke() and bench.py's reference /
// cpu_baseline legs load this library.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "stmg/assembly.hpp"
#include "stmg/kernels.hpp"
#include "stmg/materials.hpp"
#include "stmg/mesh.hpp"
#include "stmg/multigrid.hpp"
#include "stmg/optimisation.hpp"
#include "stmg/rediscretisation.hpp"
#include "stmg/strategy.hpp"

using namespace stmg;

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(1, e.what());
  } catch (const std::out_of_range& e) {
    return fail(3, e.what());
  } catch (const std::runtime_error& e) {
    return fail(2, e.what());
  } catch (const std::exception& e) {
    return fail(2, e.what());
  }
}

SpaceTimeGrid make_grid(double L, double tT, int n_el, int n_t, const double* k, const double* c) {
  SpaceTimeGrid g = build_fine_grid(L, tT, n_el, n_t);
  if (k && c) {
    g.k.assign(k, k + n_el);
    g.c.assign(c, c + n_el);
  }
  return g;
}

MaterialPair make_mat(const double* m) {
  MaterialPair p;
  p.k_ins = m[0];
  p.k_con = m[1];
  p.c_ins = m[2];
  p.c_con = m[3];
  p.p_k = m[4];
  p.p_c = m[5];
  return p;
}

CoarseningDirection to_dir(int d) {
  switch (d) {
    case 0: return CoarseningDirection::SpaceX;
    case 1: return CoarseningDirection::TimeT;
    case 2: return CoarseningDirection::FullST;
  }
  throw std::invalid_argument("ref harness: bad direction");
}

int from_dir(CoarseningDirection d) {
  return d == CoarseningDirection::SpaceX ? 0 : d == CoarseningDirection::TimeT ? 1 : 2;
}

PlanStrategy to_strategy(int s) {
  switch (s) {
    case 0: return PlanStrategy::Uniform;
    case 1: return PlanStrategy::Contrast;
    case 2: return PlanStrategy::Resolution;
    case 3: return PlanStrategy::DesignIndependent;
  }
  throw std::invalid_argument("ref harness: bad strategy");
}

ReassemblyMethod to_reasm(int r) {
  switch (r) {
    case 0: return ReassemblyMethod::K;
    case 1: return ReassemblyMethod::D;
    case 2: return ReassemblyMethod::R;
    case 3: return ReassemblyMethod::P;
  }
  throw std::invalid_argument("ref harness: bad reassembly");
}

double source_value(int kind, const double* p, double x, double t, double L, double tT) {
  switch (kind) {
    case 0: return p[0];
    case 1: return (L - x < p[1]) ? p[0] : 0.0;
    case 2: return (L - x < p[2]) ? 1.0 + p[0] * std::sin(2.0 * M_PI * p[1] * t) : 0.0;
    case 3: return heat_load_value(x, t, L, tT);
  }
  throw std::invalid_argument("ref harness: unknown source kind");
}

struct RefHier {
  LevelHierarchy h;
  std::unique_ptr<DesignField> chi;
  std::unique_ptr<MaterialPair> mat;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_plan(double L, double tT, int n_el, int n_t, const double* k, const double* c,
             const double* chi, const double* mat6, int n_levels, double lambda_crit, int strategy,
             int reassembly, int min_elements, int* dirs_out, double* ind_out) {
  return guarded([&] {
    SpaceTimeGrid g = make_grid(L, tT, n_el, n_t, k, c);
    DesignField d;
    MaterialPair m;
    PlanRequest req;
    req.n_levels = n_levels;
    req.lambda_crit = lambda_crit;
    req.strategy = to_strategy(strategy);
    req.reassembly = to_reasm(reassembly);
    req.min_elements = min_elements;
    if (chi) {
      d.chi.assign(chi, chi + n_el);
      req.chi = &d;
    }
    if (mat6) {
      m = make_mat(mat6);
      req.mat = &m;
    }
    const CoarseningPath p = plan_coarsening(g, req);
    for (std::size_t i = 0; i < p.dirs.size(); ++i) {
      dirs_out[i] = from_dir(p.dirs[i]);
      if (ind_out) ind_out[i] = p.indicator_at_decision[i];
    }
  });
}

int ref_hier_create(double L, double tT, int n_el, int n_t, const double* k, const double* c,
                    const double* chi, const double* mat6, const char* method, int n_dirs,
                    const int* dirs, int adjoint, void** out, double* build_seconds) {
  *out = nullptr;
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    auto rh = std::make_unique<RefHier>();
    SpaceTimeGrid g = make_grid(L, tT, n_el, n_t, k, c);
    if (chi) rh->chi = std::make_unique<DesignField>(DesignField{std::vector<double>(chi, chi + n_el)});
    if (mat6) rh->mat = std::make_unique<MaterialPair>(make_mat(mat6));
    CoarseningPath path;
    for (int i = 0; i < n_dirs; ++i) path.dirs.push_back(to_dir(dirs[i]));
    LevelHierarchy h = build_hierarchy(g, parse_method(method), path, rh->chi.get(), rh->mat.get());
    rh->h = adjoint ? transposed_hierarchy(h) : std::move(h);
    if (build_seconds)
      *build_seconds =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = rh.release();
  });
}

void ref_hier_free(void* h) { delete static_cast<RefHier*>(h); }

int ref_hier_n_levels(void* h) { return static_cast<RefHier*>(h)->h.n_levels(); }

long long ref_hier_level_dofs(void* h, int l) {
  return static_cast<long long>(static_cast<RefHier*>(h)->h.levels.at(l).grid.n_dofs());
}

long long ref_hier_level_nnz(void* h, int l) {
  return static_cast<long long>(static_cast<RefHier*>(h)->h.levels.at(l).J.nnz());
}

// Dump level l's CSR (row_ptr[n+1], col[nnz], val[nnz]) and inv_diag[n].
int ref_hier_level_csr(void* hp, int l, int* row_ptr, int* col, double* val, double* inv_diag) {
  return guarded([&] {
    const Level& lv = static_cast<RefHier*>(hp)->h.levels.at(l);
    const auto rp = lv.J.row_ptr();
    const auto ci = lv.J.col_idx();
    const auto v = lv.J.values();
    std::memcpy(row_ptr, rp.data(), rp.size() * sizeof(int));
    std::memcpy(col, ci.data(), ci.size() * sizeof(int));
    std::memcpy(val, v.data(), v.size() * sizeof(double));
    std::memcpy(inv_diag, lv.inv_diag.data(), lv.inv_diag.size() * sizeof(double));
  });
}

// r = f - J_l x (the reference's dispatched csr_residual).
int ref_residual(void* hp, int l, const double* f, const double* x, double* r) {
  return guarded([&] {
    const Level& lv = static_cast<RefHier*>(hp)->h.levels.at(l);
    const std::size_t n = lv.grid.n_dofs();
    lv.J.residual({f, n}, {x, n}, {r, n});
  });
}

// `sweeps` damped-Jacobi sweeps exactly as v_cycle does them (multigrid.cpp:193-196).
int ref_jacobi_sweeps(void* hp, int l, const double* f, double* x, int sweeps, double omega) {
  return guarded([&] {
    const Level& lv = static_cast<RefHier*>(hp)->h.levels.at(l);
    const std::size_t n = lv.grid.n_dofs();
    std::vector<double> r(n);
    for (int s = 0; s < sweeps; ++s) {
      lv.J.residual({f, n}, {x, n}, r);
      kernels::jacobi_update(omega, lv.inv_diag, r, {x, n});
    }
  });
}

int ref_restrict(void* hp, int l, const double* r_fine, double* f_coarse) {
  return guarded([&] {
    const LevelHierarchy& h = static_cast<RefHier*>(hp)->h;
    const std::size_t nf = h.levels.at(l).grid.n_dofs(), nc = h.levels.at(l + 1).grid.n_dofs();
    h.transfers.at(l).R.multiply({r_fine, nf}, {f_coarse, nc});
  });
}

int ref_prolong_add(void* hp, int l, const double* x_coarse, double* x_fine) {
  return guarded([&] {
    const LevelHierarchy& h = static_cast<RefHier*>(hp)->h;
    const std::size_t nf = h.levels.at(l).grid.n_dofs(), nc = h.levels.at(l + 1).grid.n_dofs();
    h.transfers.at(l).P.multiply_add({x_coarse, nc}, {x_fine, nf});
  });
}

int ref_coarsest_solve(void* hp, const double* f, double* x) {
  return guarded([&] {
    const LevelHierarchy& h = static_cast<RefHier*>(hp)->h;
    const std::size_t n = h.levels.back().grid.n_dofs();
    h.coarsest->solve({f, n}, {x, n});
  });
}

int ref_mg_solve(void* hp, const double* b, double* u, int nu, double omega, double tol,
                 double div_tol, int max_cycles, int* status, int* cycles, double* factor,
                 int* absolute_norms, double* history, int* n_history, double* seconds) {
  return guarded([&] {
    const LevelHierarchy& h = static_cast<RefHier*>(hp)->h;
    const std::size_t n = h.levels.front().grid.n_dofs();
    SolveOptions o;
    o.nu = nu;
    o.omega = omega;
    o.tol = tol;
    o.div_tol = div_tol;
    o.max_cycles = max_cycles;
    const SolveReport rep = mg_solve(h, {b, n}, {u, n}, o);
    *status = static_cast<int>(rep.status);
    *cycles = rep.cycles;
    *factor = rep.factor;
    *absolute_norms = rep.absolute_norms ? 1 : 0;
    for (std::size_t i = 0; i < rep.history.size(); ++i) history[i] = rep.history[i];
    *n_history = static_cast<int>(rep.history.size());
    if (seconds) *seconds = rep.seconds;
  });
}

int ref_load_vector(double L, double tT, int n_el, int n_t, int kind, const double* params,
                    int masked, double* b) {
  return guarded([&] {
    const SpaceTimeGrid g = build_fine_grid(L, tT, n_el, n_t);
    std::vector<double> v = kind == 3 ? load_vector(g)
                                      : load_vector(g, [&](double x, double t) {
                                          return source_value(kind, params, x, t, L, tT);
                                        });
    if (masked)
      for (std::size_t f = 0; f < v.size(); ++f)
        if (dof_is_masked(g, static_cast<std::int32_t>(f))) v[f] = 0.0;
    std::memcpy(b, v.data(), v.size() * sizeof(double));
  });
}

int ref_apply_design(const double* chi, int n, const double* mat6, double* k, double* c) {
  return guarded([&] {
    std::vector<double> kk, cc;
    apply_design(kk, cc, DesignField{std::vector<double>(chi, chi + n)}, make_mat(mat6));
    std::memcpy(k, kk.data(), sizeof(double) * static_cast<std::size_t>(n));
    std::memcpy(c, cc.data(), sizeof(double) * static_cast<std::size_t>(n));
  });
}

// optimise(), proj/src/optimisation.cpp:83-186.  rec: per iteration 12 doubles
// {theta, volume, constraint, change, primal_status, adjoint_status,
//  primal_cycles, adjoint_cycles, primal_factor, adjoint_factor, primal_s, adjoint_s}
int ref_optimise(double L, double tT, int n_el, int n_t, const double* mat6, const char* method,
                 int strategy, int n_levels, double lambda_crit, int min_elements, int warm_start,
                 double volume_limit, double theta_ref, double chi_init, int max_iterations,
                 double rel_change_tol, int stable_iterations, int nu, double omega, double tol,
                 double div_tol, int max_cycles, double* chi_out, double* rec, int* n_rec,
                 double* theta, int* converged, double* seconds) {
  return guarded([&] {
    const SpaceTimeGrid g = build_fine_grid(L, tT, n_el, n_t);
    OptimisationOptions o;
    o.method = parse_method(method);
    o.strategy = to_strategy(strategy);
    o.n_levels = n_levels;
    o.lambda_crit = lambda_crit;
    o.min_elements = min_elements;
    o.warm_start = warm_start != 0;
    o.volume_limit = volume_limit;
    o.theta_ref = theta_ref;
    o.chi_init = chi_init;
    o.max_iterations = max_iterations;
    o.rel_change_tol = rel_change_tol;
    o.stable_iterations = stable_iterations;
    o.solve.nu = nu;
    o.solve.omega = omega;
    o.solve.tol = tol;
    o.solve.div_tol = div_tol;
    o.solve.max_cycles = max_cycles;
    const OptimisationResult r = optimise(g, make_mat(mat6), o);
    std::memcpy(chi_out, r.chi.chi.data(), sizeof(double) * r.chi.chi.size());
    for (std::size_t i = 0; i < r.history.size(); ++i) {
      const IterationRecord& h = r.history[i];
      double* d = rec + 12 * i;
      d[0] = h.theta; d[1] = h.volume; d[2] = h.constraint; d[3] = h.change;
      d[4] = static_cast<double>(h.primal_status); d[5] = static_cast<double>(h.adjoint_status);
      d[6] = h.primal_cycles; d[7] = h.adjoint_cycles; d[8] = h.primal_factor;
      d[9] = h.adjoint_factor; d[10] = h.primal_seconds; d[11] = h.adjoint_seconds;
    }
    *n_rec = static_cast<int>(r.history.size());
    *theta = r.theta;
    *converged = r.converged ? 1 : 0;
    *seconds = r.seconds;
  });
}

// objective_sensitivities, proj/src/optimisation.cpp:34-73
int ref_objective_sensitivities(double L, double tT, int n_el, int n_t, const double* mat6, const double* chi,
                                const double* u, const double* lam, double* sens) {
  return guarded([&] {
    const SpaceTimeGrid g = build_fine_grid(L, tT, n_el, n_t);
    const std::size_t n = g.n_dofs();
    const std::vector<double> s = objective_sensitivities(
        g, make_mat(mat6), DesignField{std::vector<double>(chi, chi + n_el)}, {u, n}, {lam, n});
    std::memcpy(sens, s.data(), sizeof(double) * s.size());
  });
}

double ref_norm2(const double* x, long long n) {
  return kernels::norm2({x, static_cast<std::size_t>(n)});
}

int ref_set_backend(int b) {
  return kernels::set_backend(b == 0 ? kernels::Backend::Scalar : kernels::Backend::Avx2) ? 0 : 1;
}

}  // extern "C"
