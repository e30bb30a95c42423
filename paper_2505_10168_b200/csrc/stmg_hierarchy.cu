// Host side of stmg_b200: grids, materials, planner, level build, device
// hierarchy, V-cycle orchestration (CUDA graphs) and the C ABI of
// include/stmg_b200.h.  Semantics follow the reference module by module;
// each function cites the reference code it restates.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/stmg_b200.h"
#include "stmg_internal.h"
#include "stmg_galerkin.h"

namespace stmgb {
namespace {

thread_local std::string g_error;

// NVTX range for Nsight timelines (header-only NVTX 3: a no-op unless a tool
// is attached).  Graph replays show as one range per V-cycle.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NoMem : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      throw NoMem(std::string(what) + ": " + cudaGetErrorString(e));
    }
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
  }
}
void launch_check(int rc, const char* what) {
  if (rc != 0) cuda_check(static_cast<cudaError_t>(rc), what);
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return STMG_OK;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return STMG_EINVAL;
  } catch (const std::out_of_range& e) {
    g_error = e.what();
    return STMG_ERANGE;
  } catch (const NoMem& e) {
    g_error = e.what();
    return STMG_ENOMEM;
  } catch (const CudaError& e) {
    g_error = e.what();
    return STMG_ECUDA;
  } catch (const std::bad_alloc&) {
    g_error = "host allocation failed";
    return STMG_ENOMEM;
  } catch (const std::runtime_error& e) {
    g_error = e.what();
    return STMG_ERUNTIME;
  } catch (const std::exception& e) {
    g_error = e.what();
    return STMG_ERUNTIME;
  }
}

// ---------------------------------------------------------------------------
// Host model (proj/src/{mesh,materials,assembly,rediscretisation,strategy}.cpp)
// ---------------------------------------------------------------------------

struct HostGrid {
  double L = 0, t_T = 0, dx = 0, dt = 0;
  int64_t n_el = 0, n_t = 0;
};

// build_fine_grid, proj/src/mesh.cpp:16-29
HostGrid make_grid(double L, double t_T, int64_t n_el, int64_t n_t) {
  if (L <= 0.0 || t_T <= 0.0) throw std::invalid_argument("build_fine_grid: non-positive extent");
  if (n_el <= 0 || n_t <= 0) throw std::invalid_argument("build_fine_grid: non-positive count");
  HostGrid g;
  g.L = L;
  g.t_T = t_T;
  g.n_el = n_el;
  g.n_t = n_t;
  g.dx = L / static_cast<double>(n_el);
  g.dt = t_T / static_cast<double>(n_t);
  return g;
}

// coarsen_grid, proj/src/mesh.cpp:31-42
HostGrid coarsen(const HostGrid& g, int dir) {
  const bool hx = dir != STMG_DIR_T, ht = dir != STMG_DIR_X;
  if ((hx && g.n_el % 2 != 0)) throw std::invalid_argument("coarsen_grid: odd element count");
  if ((ht && g.n_t % 2 != 0)) throw std::invalid_argument("coarsen_grid: odd step count");
  if ((hx && g.n_el < 2) || (ht && g.n_t < 2))
    throw std::invalid_argument("coarsen_grid: grid too small to coarsen");
  return make_grid(g.L, g.t_T, hx ? g.n_el / 2 : g.n_el, ht ? g.n_t / 2 : g.n_t);
}

void check_material(const stmg_material_pair& m) {
  if (m.k_ins <= 0.0 || m.k_con <= 0.0 || m.c_ins <= 0.0 || m.c_con <= 0.0)
    throw std::invalid_argument("material properties must be positive");
  if (m.p_k <= 0.0 || m.p_c <= 0.0)
    throw std::invalid_argument("penalisation exponents must be positive");
}

// simp_eval / apply_design, proj/src/materials.cpp:27-32, 44-50
void simp(const double* chi, int64_t n, const stmg_material_pair& m, double* k, double* c) {
  check_material(m);
  for (int64_t e = 0; e < n; ++e) {
    if (!(chi[e] >= 0.0 && chi[e] <= 1.0)) throw std::invalid_argument("volume fraction outside [0, 1]");
    k[e] = m.k_ins + (m.k_con - m.k_ins) * std::pow(chi[e], m.p_k);
    c[e] = m.c_ins + (m.c_con - m.c_ins) * std::pow(chi[e], m.p_c);
  }
}

// coarsen_materials, proj/src/rediscretisation.cpp:53-110 (x step; t copies)
void coarsen_materials_x(const std::vector<double>& k, const std::vector<double>& c,
                         const std::vector<double>* chi, const stmg_material_pair* mat, int reasm,
                         std::vector<double>& kc, std::vector<double>& cc, std::vector<double>* chic) {
  const size_t nc = k.size() / 2;
  kc.resize(nc);
  cc.resize(nc);
  if (reasm == STMG_REASM_D) {
    if (!chi || !mat)
      throw std::invalid_argument("coarsen_materials: D method needs the design field and materials");
    chic->resize(nc);
    for (size_t e = 0; e < nc; ++e) (*chic)[e] = 0.5 * ((*chi)[2 * e] + (*chi)[2 * e + 1]);
    simp(chic->data(), static_cast<int64_t>(nc), *mat, kc.data(), cc.data());
    return;
  }
  for (size_t e = 0; e < nc; ++e) {
    const double a = k[2 * e], b = k[2 * e + 1];
    kc[e] = reasm == STMG_REASM_R ? 2.0 * a * b / (a + b) : 0.5 * (a + b);
    cc[e] = 0.5 * (c[2 * e] + c[2 * e + 1]);
  }
}

// design_independent_diffusivity, proj/src/strategy.cpp:85-106
double design_independent_d(const stmg_material_pair& m) {
  const double d0 = m.k_ins / m.c_ins, d1 = m.k_con / m.c_con;
  const double lo = std::min(d0, d1), hi = std::max(d0, d1);
  for (int i = 0; i < 1001; ++i) {
    const double chi = static_cast<double>(i) / (1001 - 1);
    double k, c;
    simp(&chi, 1, m, &k, &c);
    const double d = k / c;
    if (d < lo * (1.0 - 1e-9) || d > hi * (1.0 + 1e-9))
      throw std::invalid_argument(
          "design_independent_diffusivity: interpolated diffusivity has an interior extremum; "
          "the design-independent indicator is invalid for this material pair");
  }
  return std::sqrt(d0 * d1);
}

// anisotropy / effective_lambda, proj/src/strategy.cpp:9-28
double lambda_eff(const std::vector<double>& k, const std::vector<double>& c, double dx, double dt) {
  const double scale = dt / (dx * dx);
  double lo = 0, hi = 0;
  for (size_t e = 0; e < k.size(); ++e) {
    const double le = (k[e] / c[e]) * scale;
    if (e == 0 || le < lo) lo = le;
    if (e == 0 || le > hi) hi = le;
  }
  return std::sqrt(lo * hi);
}

// plan_coarsening, proj/src/strategy.cpp:127-234
void plan(const HostGrid& fine, const double* k, const double* c, const double* chi,
          const stmg_material_pair* mat, const stmg_plan_request& req, int32_t* dirs,
          double* ind) {
  if (req.n_levels < 1) throw std::invalid_argument("plan_coarsening: need at least one level");
  if (req.lambda_crit <= 0.0)
    throw std::invalid_argument("plan_coarsening: lambda_crit must be positive");
  double fixed_d = 0.0;
  if (req.strategy == STMG_PLAN_DESIGN_INDEPENDENT) {
    if (!mat)
      throw std::invalid_argument("plan_coarsening: design-independent planning needs the material pair");
    fixed_d = design_independent_d(*mat);
  } else if (!k || !c) {
    throw std::invalid_argument("plan_coarsening: grid has no materials");
  }
  if (req.strategy < 0 || req.strategy > 3) throw std::invalid_argument("plan_coarsening: bad strategy");
  const bool track_chi = req.reassembly == STMG_REASM_D && req.strategy != STMG_PLAN_DESIGN_INDEPENDENT;
  if (track_chi && (!chi || !mat))
    throw std::invalid_argument("plan_coarsening: D reassembly needs the design field and materials");
  HostGrid lev = fine;
  std::vector<double> lk, lc, lchi;
  if (req.strategy != STMG_PLAN_DESIGN_INDEPENDENT) {
    lk.assign(k, k + fine.n_el);
    lc.assign(c, c + fine.n_el);
    if (track_chi) lchi.assign(chi, chi + fine.n_el);
  }
  for (int l = 1; l < req.n_levels; ++l) {
    double lambda = 0.0;
    if (req.strategy == STMG_PLAN_UNIFORM) {
      for (size_t e = 1; e < lk.size(); ++e)
        if (lk[e] != lk[0] || lc[e] != lc[0])
          throw std::invalid_argument("plan_coarsening: uniform strategy on non-uniform materials");
      lambda = (lk[0] / lc[0]) * lev.dt / (lev.dx * lev.dx);
    } else if (req.strategy == STMG_PLAN_DESIGN_INDEPENDENT) {
      lambda = fixed_d * lev.dt / (lev.dx * lev.dx);
    } else {
      lambda = lambda_eff(lk, lc, lev.dx, lev.dt);
    }
    const bool guard = req.strategy == STMG_PLAN_RESOLUTION && lev.n_el / 2 < req.min_elements;
    const bool want_time = lambda < req.lambda_crit || guard;
    const bool x_ok = lev.n_el % 2 == 0 && lev.n_el >= 2;
    const bool t_ok = lev.n_t % 2 == 0 && lev.n_t >= 2;
    int dir;
    if (want_time) {
      if (t_ok) dir = STMG_DIR_T;
      else if (guard)
        throw std::runtime_error(
            "plan_coarsening: forced time-coarsening impossible and the element floor forbids "
            "space-coarsening");
      else if (x_ok) dir = STMG_DIR_X;
      else throw std::runtime_error("plan_coarsening: no legal coarsening step");
    } else {
      if (x_ok) dir = STMG_DIR_X;
      else if (t_ok) dir = STMG_DIR_T;
      else throw std::runtime_error("plan_coarsening: no legal coarsening step");
    }
    dirs[l - 1] = dir;
    if (ind) ind[l - 1] = lambda;
    HostGrid next = coarsen(lev, dir);
    if (req.strategy != STMG_PLAN_DESIGN_INDEPENDENT && dir == STMG_DIR_X) {
      std::vector<double> kc, cc, chic;
      coarsen_materials_x(lk, lc, track_chi ? &lchi : nullptr, mat, req.reassembly, kc, cc,
                          track_chi ? &chic : nullptr);
      lk.swap(kc);
      lc.swap(cc);
      if (track_chi) lchi.swap(chic);
    }
    lev = next;
  }
}

// One level's stencil in the reference's exact arithmetic:
// element terms proj/src/assembly.cpp:17-32, per-row triplets :99-121, masked
// weight :52-57, 1/diag proj/src/multigrid.cpp:73-82.  Duplicate (row, col)
// entries are pairs, so from_triplets' summation order does not matter.
struct HostLevel {
  HostGrid g;
  std::vector<double> k, c, chi;
  double w = 0, inv_w = 0;
  std::vector<double> W, D, E, SW, S, SE, invD;  // primal, per node i (0 unused)

  void build() {
    const int64_t ne = g.n_el, nn = ne + 1;
    for (int64_t e = 0; e < ne; ++e)
      if (!(k[e] > 0.0) || !(c[e] > 0.0) || !(g.dx > 0.0))
        throw std::invalid_argument("element_matrices: non-positive input");
    const double kmax = *std::max_element(k.begin(), k.end());
    const double cmax = *std::max_element(c.begin(), c.end());
    w = cmax * g.dx / g.dt + kmax / g.dx;
    inv_w = 1.0 / w;
    for (auto* v : {&W, &D, &E, &SW, &S, &SE, &invD}) v->assign(static_cast<size_t>(nn), 0.0);
    for (int64_t i = 1; i <= ne; ++i) {
      const double kdl = k[i - 1] / g.dx;
      const double cdl = c[i - 1] * g.dx / 6.0;
      const double c11 = (2.0 * cdl) / g.dt, c10 = cdl / g.dt;
      double d = c11 + kdl;
      double s = -c11;
      W[i] = c10 + (-kdl);
      SW[i] = -c10;
      if (i <= ne - 1) {
        const double kdr = k[i] / g.dx;
        const double cdr = c[i] * g.dx / 6.0;
        const double c00 = (2.0 * cdr) / g.dt, c01 = cdr / g.dt;
        d = d + (c00 + kdr);
        s = s + (-c00);
        E[i] = c01 + (-kdr);
        SE[i] = -c01;
      }
      D[i] = d;
      S[i] = s;
      if (d == 0.0)
        throw std::runtime_error("build_hierarchy: level operator has a zero diagonal entry");
      invD[i] = 1.0 / d;
    }
    invD[0] = inv_w;
  }

  // Coefficient table in a row orientation (see LevelView).  The transposed
  // operator's row (n, i) is J's column (n, i) (proj/src/sparse.cpp:74-96).
  std::vector<double> table(bool adjoint) const {
    const int64_t nn = g.n_el + 1, ne = g.n_el;
    std::vector<double> t(static_cast<size_t>(kNumCoef * nn), 0.0);
    auto at = [&](int k, int64_t i) -> double& { return t[static_cast<size_t>(k * nn + i)]; };
    for (int64_t i = 0; i < nn; ++i) {
      if (!adjoint) {
        at(kCm, i) = W[i];
        at(kCp, i) = E[i];
        at(kOm, i) = SW[i];
        at(kOp, i) = SE[i];
      } else {
        at(kCm, i) = i >= 2 ? E[i - 1] : 0.0;
        at(kCp, i) = i <= ne - 1 ? W[i + 1] : 0.0;
        at(kOm, i) = i >= 2 ? SE[i - 1] : 0.0;
        at(kOp, i) = i <= ne - 1 ? SW[i + 1] : 0.0;
      }
      at(kC0, i) = D[i];
      at(kO0, i) = S[i];
      at(kInvD, i) = invD[i];
    }
    return t;
  }
};

// parse_method, proj/src/rediscretisation.cpp:19-38 (two letters: interpolation C/B,
// reassembly K/D/R/P); *bilinear receives the interpolation.
int parse_method(const char* name, bool* bilinear = nullptr) {
  if (!name || std::strlen(name) != 2) throw std::invalid_argument("parse_method: expected two letters");
  if (name[0] != 'C' && name[0] != 'B')
    throw std::invalid_argument("parse_method: unknown interpolation letter");
  int re;
  switch (name[1]) {
    case 'K': re = STMG_REASM_K; break;
    case 'D': re = STMG_REASM_D; break;
    case 'R': re = STMG_REASM_R; break;
    case 'P': re = STMG_REASM_P; break;
    default: throw std::invalid_argument("parse_method: unknown reassembly letter");
  }
  if (bilinear) *bilinear = name[0] == 'B';
  return re;
}

// ---------------------------------------------------------------------------
// Device hierarchy
// ---------------------------------------------------------------------------

struct DeviceBuf {
  double* p = nullptr;
  int64_t n = 0;
  DeviceBuf() = default;
  explicit DeviceBuf(int64_t count) : n(count) {
    if (count > 0) cuda_check(cudaMalloc(&p, sizeof(double) * static_cast<size_t>(count)), "cudaMalloc");
  }
  DeviceBuf(const DeviceBuf&) = delete;
  DeviceBuf& operator=(const DeviceBuf&) = delete;
  ~DeviceBuf() {
    if (p) cudaFree(p);
  }
};

// Vector workspaces (f, x, y per level; level 0: b, u, u').  A hierarchy and
// its transpose share one Workspace (they are never solved concurrently),
// which halves the footprint for 1e9-DOF grids.
// Cycle cap of the device-side solve loop (longer solves use the host loop).
constexpr int kLoopHistory = 4096;

struct Workspace {
  std::vector<std::unique_ptr<DeviceBuf>> f, xa, xb;
  std::unique_ptr<DeviceBuf> partials, scalars, coarse_scratch;
  double* pinned = nullptr;  // 4 host doubles
  // device solve loop: SolveLoopCtl + history[kLoopHistory + 1], and a pinned mirror
  std::unique_ptr<DeviceBuf> loop;
  double* loop_host = nullptr;
  // device-resident buffer pointers the fine up-pass kernels read (the speculative
  // iterate alternates between two buffers from cycle to cycle): [0] in, [1] out
  std::unique_ptr<DeviceBuf> ptrs;
  std::unique_ptr<DeviceBuf> xz;  // third level-0 iterate buffer (fine up-pass), allocated on first use
  // stmg_mg_solve_stream: two (b, u) device slots, allocated on first use and kept (the cycle
  // graphs are cached per bound pointer pair); stmg_hierarchy_release_staging frees them
  std::unique_ptr<DeviceBuf> stage_b[2], stage_u[2];
  ~Workspace() {
    if (pinned) cudaFreeHost(pinned);
    if (loop_host) cudaFreeHost(loop_host);
  }
};
constexpr int64_t kLoopCtlDoubles = (sizeof(SolveLoopCtl) + 7) / 8;

struct GraphKey {
  int nu;
  double omega;
  int profiling;
  // level-0 vectors the graph reads and writes (the caller's b and u when they
  // are bound in place, else the workspace's)
  const void* b = nullptr;
  const void* x = nullptr;
  // cycle 1 of a zero-guess solve whose level-0 restriction ran with the opening pass
  int first = 0;
  bool operator<(const GraphKey& o) const {
    return std::tie(nu, omega, profiling, b, x, first) < std::tie(o.nu, o.omega, o.profiling, o.b, o.x, o.first);
  }
};
// Graphs kept per hierarchy; a solve with new bound pointers beyond this many
// drops the cache (callers normally reuse the same b / u buffers).
constexpr size_t kMaxGraphs = 16;

// V-cycle fusions (stmg_hierarchy_set_fusion; all on by default).  Every
// combination gives bit-identical iterates; they differ in HBM traffic only.
enum FusionFlags {
  kFuseVirtualZero = 1,  // coarse first sweep from zero recomputed from f where read
  kFuseFineDown = 2,     // level 0 (nu = 1): norm + sweep + residual restriction in one pass
  kFuseFineUp = 4,       // level 0 (nu = 1): prolongation + post-sweep + norm + next pre-sweep in one pass
  kFuseAll = 7,
  // measured (cfg2): the virtual zero iterate pays (89 -> 85 ms), the fine up-pass pays
  // (75.9 -> 72.4 ms; 69.4 with 128 registers), the fine down-pass does not (k_down:
  // 0.92 ms vs 0.51 + 0.59 ms for the separate kernels on a 1.3e8-DOF level, but no
  // gain in the power-capped solve)
  kFuseDefault = kFuseVirtualZero | kFuseFineUp
};

enum TimedKind {
  kTimedSweep = 0,
  kTimedRestrict = 1,
  kTimedProlongSweep = 2,
  kTimedSweep2 = 3,
  kTimedFromZero = 4,
  kTimedCoarsest = 5,
  kTimedKinds = 6
};

struct TimedKernel {
  int kind;
  int level;
  cudaEvent_t start, stop;
};

struct GraphEntry {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int64_t kernels = 0;
  int final_buf = 0;
  std::vector<TimedKernel> timed;  // event pairs recorded inside the graph (profiling)
  // The whole cycle loop as one graph: a conditional WHILE node whose body is
  // the V-cycle, the residual norm and the bookkeeping kernel (solve_loop).
  cudaGraph_t loop_graph = nullptr;
  cudaGraphExec_t loop_exec = nullptr;
  bool loop_tried = false;
  // fine up-pass: the graph ends before level 0's prolongation; level 1's result buffer
  const double* up_xc = nullptr;
};

void destroy_graph_entry(GraphEntry& e) {
  if (e.exec) cudaGraphExecDestroy(e.exec);
  if (e.graph) cudaGraphDestroy(e.graph);
  if (e.loop_exec) cudaGraphExecDestroy(e.loop_exec);
  if (e.loop_graph) cudaGraphDestroy(e.loop_graph);
  for (auto& t : e.timed) {
    cudaEventDestroy(t.start);
    cudaEventDestroy(t.stop);
  }
  e = GraphEntry{};
}

}  // namespace
}  // namespace stmgb

struct stmg_hierarchy {
  int device = 0;
  bool adjoint = false;
  int reassembly = STMG_REASM_K;
  std::vector<int32_t> dirs;
  std::vector<stmgb::HostLevel> host;
  std::vector<std::unique_ptr<stmgb::DeviceBuf>> coef;  // per level
  std::vector<stmgb::LevelView> views;
  stmgb::CoarsestView coarsest{};
  std::unique_ptr<stmgb::DeviceBuf> pcr_alpha, pcr_gamma, pcr_bfin, prop_tinv, prop_a, prop_chunk, pint_pow;
  std::shared_ptr<stmgb::Workspace> ws;
  cudaStream_t stream = nullptr;      // where work runs (own_stream or a caller's)
  cudaStream_t own_stream = nullptr;  // created with the hierarchy
  cudaStream_t cap_stream = nullptr;  // private stream for graph capture
  int profiling = 0;  // 0 off, 1 finest-level kernels, 2 every kernel
  int fusion = stmgb::kFuseDefault;  // stmgb::kFuse* flags (stmg_hierarchy_set_fusion)
  // per (level, kind): launches and device seconds accumulated while profiling
  std::vector<std::array<std::pair<int64_t, double>, stmgb::kTimedKinds>> prof;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, norm_ev0 = nullptr, norm_ev1 = nullptr;
  std::map<stmgb::GraphKey, stmgb::GraphEntry> graphs;
  int64_t device_bytes = 0;
  // Level-0 right-hand side and iterate bound in place for the current solve
  // (the caller's device b and u, no copies); null: the workspace's f / xa.
  const double* bind_b = nullptr;
  double* bind_x = nullptr;
  double* f_ptr(int l) const { return l == 0 && bind_b ? const_cast<double*>(bind_b) : ws->f[l]->p; }
  double* xa_ptr(int l) const { return l == 0 && bind_x ? bind_x : ws->xa[l]->p; }
  // General coarse discretisations.
  bool bilinear = false;                 // temporal interpolation of the t transfers
  std::vector<stmgb::Dia9Host> gal;      // P reassembly: primal 9-point operators (level 0 empty)
  std::vector<std::unique_ptr<stmgb::DeviceBuf>> gbuf;  // per level: Galerkin v | inv_diag | mask
  std::vector<stmgb::Dia9View> dviews;   // per level; v == nullptr: per-node (rediscretised) level
  std::vector<stmgb::XferView> xviews;   // per transfer
  stmgb::BlockMarchView block{};         // Galerkin coarsest level's exact solver
  std::unique_ptr<stmgb::DeviceBuf> block_g, block_h;
  bool galerkin(int l) const { return l < static_cast<int>(dviews.size()) && dviews[l].v != nullptr; }
  // transfers the per-node fused kernels do not cover: bilinear t, FullST
  bool gen_xfer(int l) const {
    return dirs[l] == STMG_DIR_XT || (bilinear && dirs[l] == STMG_DIR_T);
  }
  bool general() const {
    for (int l = 0; l < n_levels(); ++l)
      if (galerkin(l) || (l + 1 < n_levels() && gen_xfer(l))) return true;
    return false;
  }

  ~stmg_hierarchy() {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (auto& kv : graphs) stmgb::destroy_graph_entry(kv.second);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (norm_ev0) cudaEventDestroy(norm_ev0);
    if (norm_ev1) cudaEventDestroy(norm_ev1);
    if (own_stream) cudaStreamDestroy(own_stream);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    coef.clear();
    gbuf.clear();
    block_g.reset();
    block_h.reset();
    pcr_alpha.reset();
    pcr_gamma.reset();
    pcr_bfin.reset();
    prop_tinv.reset();
    prop_a.reset();
    prop_chunk.reset();
    pint_pow.reset();
    ws.reset();
    cudaSetDevice(prev);
  }
  int n_levels() const { return static_cast<int>(host.size()); }
  int64_t ndofs(int l) const { return (host[l].g.n_el + 1) * (host[l].g.n_t + 1); }
};

namespace stmgb {
namespace {

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// Parallel-in-time march tables for a wide coarsest level (n_el > 32, see
// k_coarsest_pint): chunk length Lc, a power of two dividing n_t near
// sqrt(1.5 n_t) (balancing 2 Lc PCR steps against n_t / Lc dense links), and
// the chunk propagator A^Lc, A = -T^-1 S (column-major m x m), built on the
// device by m parallel homogeneous marches with the march's own PCR step.
// Needs the PCR tables.
void build_pint(stmg_hierarchy* h) {
  const int m = h->coarsest.m;
  const int64_t nt = h->host.back().g.n_t;
  if (m <= 32 || m > 2048 || nt < 64) return;
  int64_t Lc = 1;
  while (Lc * Lc < (3 * nt) / 2) Lc *= 2;
  while (Lc > 1 && nt % Lc != 0) Lc /= 2;
  const int64_t C = nt / Lc;
  if (C < 2 || Lc < 4) return;
  int rounds = 0;
  while ((int64_t{1} << rounds) < C) ++rounds;
  // reused across refresh_levels (optimise() rebuilds it every design iteration)
  const int64_t need = static_cast<int64_t>(rounds) * m * m;
  if (!h->pint_pow || h->pint_pow->n != need) h->pint_pow = std::make_unique<DeviceBuf>(need);
  h->coarsest.pint_len = static_cast<int32_t>(Lc);
  launch_check(launch_coarsest_pint_prop(h->coarsest, h->pint_pow->p, rounds,
                                         h->own_stream ? h->own_stream : nullptr),
               "pint propagator");
  cuda_check(cudaStreamSynchronize(h->own_stream ? h->own_stream : nullptr), "sync");
  h->coarsest.pint_pow = h->pint_pow->p;
  h->coarsest.pint_rounds = rounds;
  h->coarsest.pint_chunks = static_cast<int32_t>(C);
  h->device_bytes += static_cast<int64_t>(rounds) * m * m * 8;
}

// Parallel-cyclic-reduction factors of the coarsest step matrix (rows 1..n_el:
// sub cm, diag c0, super cp), shared by every time level.
void build_pcr(stmg_hierarchy* h) {
  const HostLevel& hl = h->host.back();
  const int64_t nn = hl.g.n_el + 1;
  const int m = static_cast<int>(hl.g.n_el);
  const std::vector<double> t = hl.table(h->adjoint);
  std::vector<double> a(m), b(m), c(m);
  for (int j = 0; j < m; ++j) {
    const int64_t i = j + 1;
    a[j] = i >= 2 ? t[kCm * nn + i] : 0.0;
    b[j] = t[kC0 * nn + i];
    c[j] = i <= m - 1 ? t[kCp * nn + i] : 0.0;
  }
  int steps = 0;
  while ((1 << steps) < m) ++steps;
  std::vector<double> alpha(static_cast<size_t>(std::max(steps, 1)) * m, 0.0), gamma(alpha.size(), 0.0);
  for (int k = 0; k < steps; ++k) {
    const int s = 1 << k;
    std::vector<double> a2(m, 0.0), b2(m), c2(m, 0.0);
    for (int j = 0; j < m; ++j) {
      double al = 0.0, ga = 0.0;
      double bb = b[j];
      if (j - s >= 0) {
        al = -a[j] / b[j - s];
        a2[j] = al * a[j - s];
        bb += al * c[j - s];
      }
      if (j + s < m) {
        ga = -c[j] / b[j + s];
        c2[j] = ga * c[j + s];
        bb += ga * a[j + s];
      }
      b2[j] = bb;
      alpha[static_cast<size_t>(k) * m + j] = al;
      gamma[static_cast<size_t>(k) * m + j] = ga;
    }
    a.swap(a2);
    b.swap(b2);
    c.swap(c2);
  }
  h->pcr_alpha = std::make_unique<DeviceBuf>(static_cast<int64_t>(alpha.size()));
  h->pcr_gamma = std::make_unique<DeviceBuf>(static_cast<int64_t>(gamma.size()));
  h->pcr_bfin = std::make_unique<DeviceBuf>(std::max(m, 1));
  cuda_check(cudaMemcpy(h->pcr_alpha->p, alpha.data(), alpha.size() * 8, cudaMemcpyHostToDevice), "pcr");
  cuda_check(cudaMemcpy(h->pcr_gamma->p, gamma.data(), gamma.size() * 8, cudaMemcpyHostToDevice), "pcr");
  if (m > 0) cuda_check(cudaMemcpy(h->pcr_bfin->p, b.data(), b.size() * 8, cudaMemcpyHostToDevice), "pcr");
  // n_el <= 32: T^-1 (Thomas on unit vectors) and A = -T^-1 S, 32 x 32 padded
  h->coarsest.tinv = nullptr;
  h->coarsest.prop = nullptr;
  h->coarsest.prop_chunk = nullptr;
  h->coarsest.n_chunks = 0;
  h->coarsest.chunk_len = 0;
  h->coarsest.pint_chunks = 0;
  h->coarsest.pint_len = 0;
  h->coarsest.pint_rounds = 0;
  h->coarsest.pint_pow = nullptr;
  if (m >= 1 && m <= 32) {
    std::vector<double> Ti(32 * 32, 0.0), A(32 * 32, 0.0), S(32 * 32, 0.0);
    std::vector<double> sub(m), dia(m), sup(m), cpv(m), col(m);
    for (int j = 0; j < m; ++j) {
      const int64_t i = j + 1;
      sub[j] = i >= 2 ? t[kCm * nn + i] : 0.0;
      dia[j] = t[kC0 * nn + i];
      sup[j] = i <= m - 1 ? t[kCp * nn + i] : 0.0;
      if (i >= 2) S[j * 32 + (j - 1)] = t[kOm * nn + i];
      S[j * 32 + j] = t[kO0 * nn + i];
      if (i <= m - 1) S[j * 32 + (j + 1)] = t[kOp * nn + i];
    }
    for (int e = 0; e < m; ++e) {  // column e of T^-1
      std::vector<double> rhs(m, 0.0);
      rhs[e] = 1.0;
      double piv = dia[0];
      cpv[0] = sup[0] / piv;
      col[0] = rhs[0] / piv;
      for (int j = 1; j < m; ++j) {
        piv = dia[j] - sub[j] * cpv[j - 1];
        cpv[j] = sup[j] / piv;
        col[j] = (rhs[j] - sub[j] * col[j - 1]) / piv;
      }
      for (int j = m - 2; j >= 0; --j) col[j] -= cpv[j] * col[j + 1];
      for (int j = 0; j < m; ++j) Ti[j * 32 + e] = col[j];
    }
    for (int j = 0; j < m; ++j)
      for (int k = 0; k < m; ++k) {
        double acc = 0.0;
        for (int q = 0; q < m; ++q) acc += Ti[j * 32 + q] * S[q * 32 + k];
        A[j * 32 + k] = -acc;
      }
    // device copies are column-major (element (j, k) at k * 32 + j): lane j
    // loads its row with 32 coalesced loads
    auto colmajor = [](const std::vector<double>& M) {
      std::vector<double> T(32 * 32);
      for (int j = 0; j < 32; ++j)
        for (int k = 0; k < 32; ++k) T[k * 32 + j] = M[j * 32 + k];
      return T;
    };
    const std::vector<double> TiT = colmajor(Ti), AT = colmajor(A);
    h->prop_tinv = std::make_unique<DeviceBuf>(32 * 32);
    h->prop_a = std::make_unique<DeviceBuf>(32 * 32);
    cuda_check(cudaMemcpy(h->prop_tinv->p, TiT.data(), TiT.size() * 8, cudaMemcpyHostToDevice), "tinv");
    cuda_check(cudaMemcpy(h->prop_a->p, AT.data(), AT.size() * 8, cudaMemcpyHostToDevice), "prop");
    h->coarsest.tinv = h->prop_tinv->p;
    h->coarsest.prop = h->prop_a->p;
    h->device_bytes += 2 * 32 * 32 * 8;
    // chunked march: C = largest power of two <= 16 dividing n_t with chunks >= 4 steps
    const int64_t nt = hl.g.n_t;
    int C = 16;
    while (C > 1 && (nt % C != 0 || nt / C < 4)) C /= 2;
    if (C > 1) {
      const int64_t Lc = nt / C;
      std::vector<double> P(A), T2(32 * 32);  // P = A^Lc by binary powering
      std::vector<double> R(32 * 32, 0.0);
      for (int j = 0; j < 32; ++j) R[j * 32 + j] = 1.0;
      auto mul = [](const std::vector<double>& X, const std::vector<double>& Y, std::vector<double>& Z) {
        for (int j = 0; j < 32; ++j)
          for (int k = 0; k < 32; ++k) {
            double acc = 0.0;
            for (int q = 0; q < 32; ++q) acc += X[j * 32 + q] * Y[q * 32 + k];
            Z[j * 32 + k] = acc;
          }
      };
      for (int64_t e = Lc; e > 0; e >>= 1) {
        if (e & 1) {
          mul(R, P, T2);
          R = T2;
        }
        mul(P, P, T2);
        P = T2;
      }
      h->prop_chunk = std::make_unique<DeviceBuf>(32 * 32);
      const std::vector<double> RT = colmajor(R);
      cuda_check(cudaMemcpy(h->prop_chunk->p, RT.data(), RT.size() * 8, cudaMemcpyHostToDevice), "prop^L");
      h->coarsest.prop_chunk = h->prop_chunk->p;
      h->coarsest.n_chunks = C;
      h->coarsest.chunk_len = static_cast<int32_t>(Lc);
      h->device_bytes += 32 * 32 * 8;
    }
  }
  h->coarsest.lv = h->views.back();
  h->coarsest.m = m;
  h->coarsest.n_steps = steps;
  h->coarsest.alpha = h->pcr_alpha->p;
  h->coarsest.gamma = h->pcr_gamma->p;
  h->coarsest.bfin = h->pcr_bfin->p;
  h->device_bytes += static_cast<int64_t>((alpha.size() * 2 + b.size()) * 8);
  build_pint(h);
}

// Level-API calls complete before returning, except while the caller is
// capturing the stream into a CUDA graph (then the launch is only recorded).
void sync_unless_capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cuda_check(cudaStreamIsCapturing(s, &st), "cudaStreamIsCapturing");
  if (st == cudaStreamCaptureStatusNone) cuda_check(cudaStreamSynchronize(s), "sync");
}

// Levels with at most this many DOFs use 4-level time tiles in the stencil
// kernels (shorter serial chains where a launch is latency-bound).  Fixed when
// a hierarchy is built; a handle's tile thresholds can be changed with
// stmg_hierarchy_set_tiling (A/B measurements, tests of every tile depth).
constexpr int64_t kSmallNtDofs = 5000000;  // measured: cfg1 solve 66.2 -> 57.7 ms (2.5M); 49.82 -> 49.68 ms (5M, A/B)
// Levels with at most kTinyNtDofs DOFs use 2-level tiles.
constexpr int64_t kTinyNtDofs = 600000;  // measured: cfg1 solve 53.3 -> 50.8 ms (1.1M); 41.34 -> 41.09 ms (600K, A/B)
int64_t tile_nt_for(int64_t dofs, int64_t small = kSmallNtDofs, int64_t tiny = kTinyNtDofs) {
  return dofs <= tiny ? 2 : dofs <= small ? 4 : 8;
}

// Device tables of the general coarse discretisations: Galerkin levels' 9-point
// operators (transposed for an adjoint hierarchy, proj/src/multigrid.cpp:145-160),
// transfer descriptors, and the dense block factors of a Galerkin coarsest level.
constexpr int64_t kBlockTableBytes = int64_t{4} << 30;
void upload_general(stmg_hierarchy* h) {
  const int nl = h->n_levels();
  h->dviews.assign(static_cast<size_t>(nl), Dia9View{});
  h->gbuf.clear();
  h->gbuf.resize(static_cast<size_t>(nl));
  h->xviews.clear();
  h->block_g.reset();
  h->block_h.reset();
  h->block = BlockMarchView{};
  for (int l = 0; l < nl; ++l) {
    Dia9View& v = h->dviews[l];
    v.n_el = h->host[l].g.n_el;
    v.n_t = h->host[l].g.n_t;
    v.nn = v.n_el + 1;
    if (l + 1 < nl) {
      const HostGrid& fg = h->host[l].g;
      const HostGrid& cg = h->host[l + 1].g;
      h->xviews.push_back(XferView{fg.n_el + 1, fg.n_t, cg.n_el + 1, cg.n_t, h->dirs[l], h->bilinear ? 1 : 0});
    }
    if (l >= static_cast<int>(h->gal.size()) || h->gal[l].mask.empty()) continue;
    Dia9Host tr;
    const Dia9Host* A = &h->gal[l];
    if (h->adjoint) {
      tr = dia9_transposed(*A);
      A = &tr;
    }
    const int64_t nd = A->ndofs();
    const int64_t words = 10 * nd + (2 * nd + 7) / 8;
    auto buf = std::make_unique<DeviceBuf>(words);
    cuda_check(cudaMemcpy(buf->p, A->v.data(), 9 * nd * 8, cudaMemcpyHostToDevice), "galerkin upload");
    cuda_check(cudaMemcpy(buf->p + 9 * nd, A->inv_diag.data(), nd * 8, cudaMemcpyHostToDevice), "galerkin upload");
    cuda_check(cudaMemcpy(buf->p + 10 * nd, A->mask.data(), nd * 2, cudaMemcpyHostToDevice), "galerkin upload");
    v.v = buf->p;
    v.inv_diag = buf->p + 9 * nd;
    v.mask = reinterpret_cast<const uint16_t*>(buf->p + 10 * nd);
    h->device_bytes += words * 8;
    if (l == nl - 1) {
      const BlockTables bt = block_tables(*A, kBlockTableBytes);
      h->block_g = std::make_unique<DeviceBuf>(static_cast<int64_t>(bt.G.size()));
      cuda_check(cudaMemcpy(h->block_g->p, bt.G.data(), bt.G.size() * 8, cudaMemcpyHostToDevice), "block upload");
      if (bt.has_upper) {
        h->block_h = std::make_unique<DeviceBuf>(static_cast<int64_t>(bt.H.size()));
        cuda_check(cudaMemcpy(h->block_h->p, bt.H.data(), bt.H.size() * 8, cudaMemcpyHostToDevice), "block upload");
      }
      h->device_bytes += static_cast<int64_t>(bt.G.size() + bt.H.size()) * 8;
      h->block = BlockMarchView{bt.m, bt.n_t, h->block_g->p, bt.has_upper ? h->block_h->p : nullptr,
                                bt.has_upper ? 1 : 0, v};
    }
    h->gbuf[l] = std::move(buf);
  }
}

void upload_levels(stmg_hierarchy* h) {
  h->coef.clear();
  h->views.clear();
  for (const HostLevel& hl : h->host) {
    const std::vector<double> t = hl.table(h->adjoint);
    auto buf = std::make_unique<DeviceBuf>(static_cast<int64_t>(t.size()) + kVecPad);
    cuda_check(cudaMemcpy(buf->p, t.data(), t.size() * 8, cudaMemcpyHostToDevice), "coef upload");
    LevelView v;
    v.n_el = hl.g.n_el;
    v.n_t = hl.g.n_t;
    v.nn = hl.g.n_el + 1;
    v.w = hl.w;
    v.inv_w = hl.inv_w;
    v.coef = buf->p;
    v.n_lo = 0;
    v.n_hi = hl.g.n_t + 1;
    v.tile_nt = tile_nt_for(v.nn * (v.n_t + 1));
    h->views.push_back(v);
    h->device_bytes += static_cast<int64_t>((t.size() + kVecPad) * 8);
    h->coef.push_back(std::move(buf));
  }
  build_pcr(h);
  upload_general(h);
}

std::shared_ptr<Workspace> make_workspace(const stmg_hierarchy* h, int64_t* bytes) {
  auto ws = std::make_shared<Workspace>();
  const int nl = h->n_levels();
  int64_t max_partials = sumsq_partials_needed(0);
  for (int l = 0; l < nl; ++l) {
    const int64_t nd = h->ndofs(l);
    ws->f.push_back(std::make_unique<DeviceBuf>(nd + kVecPad));
    ws->xa.push_back(std::make_unique<DeviceBuf>(nd + kVecPad));
    // the coarsest level never ping-pongs unless it is also level 0
    ws->xb.push_back(std::make_unique<DeviceBuf>(l < nl - 1 || nl == 1 ? nd + kVecPad : 0));
    *bytes += 8 * (3 * (nd + kVecPad));
    LevelView finest_tiles = h->views[l];  // the most partials any tiling can need
    finest_tiles.tile_nt = 2;
    max_partials = std::max(max_partials, sweep_partials_needed(finest_tiles));
    if (l == 0 && nl > 1)
      max_partials = std::max(max_partials, down_partials_needed(finest_tiles, h->views[1], h->dirs[0]));
    if (l + 1 < nl) max_partials = std::max(max_partials, up_partials_needed(finest_tiles));
    if (l == 0) max_partials = std::max(max_partials, zero_norm_partials_needed(h->views[0]));
    if (l == 0 && nl > 1 && !h->galerkin(0) && !h->gen_xfer(0))
      max_partials = std::max(max_partials, restrict_open_partials_needed(finest_tiles, h->views[1], h->dirs[0]));
  }
  ws->partials = std::make_unique<DeviceBuf>(max_partials + kPartialsScratch);
  ws->scalars = std::make_unique<DeviceBuf>(8);
  const int m = h->coarsest.m;
  const int64_t scratch = std::max<int64_t>(
      {2 * static_cast<int64_t>(m), 32 * h->host.back().g.n_t, coarsest_scratch(h->coarsest), 2});
  ws->coarse_scratch = std::make_unique<DeviceBuf>(scratch);
  *bytes += 8 * (max_partials + 8 + scratch);
  cuda_check(cudaMallocHost(&ws->pinned, 8 * sizeof(double)), "cudaMallocHost");
  ws->ptrs = std::make_unique<DeviceBuf>(8);
  ws->loop = std::make_unique<DeviceBuf>(kLoopCtlDoubles + kLoopHistory + 1);
  cuda_check(cudaMallocHost(&ws->loop_host, sizeof(double) * (kLoopCtlDoubles + kLoopHistory + 1)),
             "cudaMallocHost");
  *bytes += 8 * (kLoopCtlDoubles + kLoopHistory + 1);
  return ws;
}

void finish_create(stmg_hierarchy* h, bool share_ws_from_other, const stmg_hierarchy* other) {
  DeviceGuard dg(h->device);
  launch_check(kernels_init(), "kernels_init");
  upload_levels(h);
  if (share_ws_from_other) {
    // same tiling as the hierarchy whose workspace (norm partials) is shared
    for (size_t l = 0; l < h->views.size() && l < other->views.size(); ++l)
      h->views[l].tile_nt = other->views[l].tile_nt;
    h->ws = other->ws;
  } else {
    int64_t bytes = 0;
    h->ws = make_workspace(h, &bytes);
    h->device_bytes += bytes;
  }
  // A blocking stream: ordered with the legacy default stream, so device inputs
  // produced by a caller on the default stream (e.g. PyTorch) are complete
  // before the solve reads them, and results are visible to it afterwards.
  cuda_check(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamDefault), "cudaStreamCreate");
  cuda_check(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking), "cudaStreamCreate");
  h->stream = h->own_stream;
  cuda_check(cudaEventCreate(&h->ev0), "cudaEventCreate");
  cuda_check(cudaEventCreate(&h->ev1), "cudaEventCreate");
  cuda_check(cudaEventCreate(&h->norm_ev0), "cudaEventCreate");
  cuda_check(cudaEventCreate(&h->norm_ev1), "cudaEventCreate");
}

// ---------------------------------------------------------------------------
// V-cycle emission (proj/src/multigrid.cpp:184-208), recorded into a graph
// ---------------------------------------------------------------------------

// nu = 1 cycles whose level-0 residual restriction runs inside the norm pass
// that closes the previous cycle (k_down: norm + sweep + restriction).
// nu = 1 cycles whose level-0 prolongation, post-sweep, closing residual norm and the
// next cycle's speculative pre-sweep run as one pass (k_up); takes precedence over
// the fine down-pass (both would own the norm pass).
bool fine_up(const stmg_hierarchy* h, int nu) {
  return (h->fusion & kFuseFineUp) && nu == 1 && h->n_levels() >= 2 && !h->galerkin(0) && !h->gen_xfer(0);
}
bool fine_down(const stmg_hierarchy* h, int nu) {
  return (h->fusion & kFuseFineDown) && !fine_up(h, nu) && nu == 1 && h->n_levels() >= 2 && !h->galerkin(0) &&
         !h->gen_xfer(0);
}
// device-resident pointer table of the fine up-pass: [0] the speculative iterate the
// cycle reads (restriction, up-pass), [1] where the up-pass writes the next one
inline double** up_ptrs(const stmg_hierarchy* h) { return reinterpret_cast<double**>(h->ws->ptrs->p); }

// How level l + 1 gets its first sweep from zero: recomputed from f where it
// is read (virt), written by level l's restriction (store), or neither (the
// coarsest level, Galerkin levels, nu = 0).
struct ZeroMode {
  bool virt = false, store = false;
};
ZeroMode child_zero_mode(const stmg_hierarchy* h, int l, int nu) {
  ZeroMode m;
  const bool fused = !h->galerkin(l) && !h->gen_xfer(l);
  const bool plain = fused && nu >= 1 && l + 1 < h->n_levels() - 1 && !h->galerkin(l + 1);
  m.virt = plain && (h->fusion & kFuseVirtualZero) && !h->gen_xfer(l + 1);
  // without the virtual zero iterate the child sweeps from zero itself (launch_sweep_from_zero);
  // the restriction tiles no longer write the child's first sweep (the fine down-pass k_down can)
  m.store = plain && !m.virt && l == 0 && fine_down(h, nu);
  return m;
}

struct Emitter {
  stmg_hierarchy* h;
  int nu;
  double omega;
  cudaStream_t s;
  int64_t kernels = 0;
  std::vector<TimedKernel>* timed = nullptr;  // non-null: profiling
  int prof_mode = 0;
  // level 0's restriction was done by the norm pass closing the previous cycle
  // (fine_down); the V-cycle then starts at level 1
  bool down_done = false;
  // fine up-pass: level 0 reads its iterate through the pointer table and the cycle
  // graph ends after level 1 (the up-pass kernel follows it); up_xc: level 1's result
  bool up_fused = false;
  const double* up_xc = nullptr;

  template <class F>
  void timed_launch(int l, int kind, F&& launch) {
    if (timed && (prof_mode >= 2 || l == 0)) {
      TimedKernel t{kind, l, nullptr, nullptr};
      cuda_check(cudaEventCreate(&t.start), "cudaEventCreate");
      cuda_check(cudaEventCreate(&t.stop), "cudaEventCreate");
      cuda_check(cudaEventRecordWithFlags(t.start, s, cudaEventRecordExternal), "event record");
      launch();
      cuda_check(cudaEventRecordWithFlags(t.stop, s, cudaEventRecordExternal), "event record");
      timed->push_back(t);
    } else {
      launch();
    }
  }

  double* buf(int l, int which) {
    return which == 0 ? h->xa_ptr(l) : h->ws->xb[l]->p;
  }

  // kernel launches (= buffer flips) smooth(l, ., ., count) issues
  int smooth_launches(int l, int count) const {
    if (h->galerkin(l)) return count;
    return count / 2 + count % 2;
  }

  // `count` damped-Jacobi sweeps from buffer `cur`: fused pairs (one pass over
  // memory per two sweeps), then a single sweep if count is odd.  virt: the
  // iterate is the first sweep from zero, S(0), not stored; the first launch
  // recomputes it from f (and clears virt).
  void smooth(int l, const double* f, int& cur, int count, bool* virt = nullptr) {
    auto xin = [&]() -> const double* {
      if (virt && *virt) {
        *virt = false;
        return nullptr;
      }
      return buf(l, cur);
    };
    if (h->galerkin(l)) {  // 9-point level: one launch per sweep
      for (; count > 0; --count) {
        timed_launch(l, kTimedSweep, [&] {
          launch_check(launch_g_sweep(h->dviews[l], f, buf(l, cur), buf(l, 1 - cur), omega, s), "g_sweep");
        });
        ++kernels;
        cur = 1 - cur;
      }
      return;
    }
    const LevelView& L = h->views[l];
    for (; count >= 2; count -= 2) {
      timed_launch(l, kTimedSweep2, [&] {
        launch_check(launch_sweep2(h->adjoint, L, f, xin(), buf(l, 1 - cur), omega, s), "sweep2");
      });
      ++kernels;
      cur = 1 - cur;
    }
    if (count == 1) {
      timed_launch(l, kTimedSweep, [&] {
        launch_check(launch_sweep(h->adjoint, L, f, xin(), buf(l, 1 - cur), omega, nullptr, nullptr, s),
                     "sweep");
      });
      ++kernels;
      cur = 1 - cur;
    }
  }

  // Returns the buffer index (0 = xa, 1 = xb) holding the level's result.
  // start: buffer holding the current iterate; pre_done: sweeps already done;
  // from_zero: the iterate is identically zero (coarse levels).
  // zero_done: the first sweep from zero was already written into buffer 0 by
  // the parent's restriction (launch_restrict_residual with xc0).
  // zero_virtual: the first sweep from zero, S(0) = 0 + omega (f * inv_diag), is
  // never stored: the kernels that read this level's iterate next recompute it
  // from f (the first pre-smoothing launch; for nu = 1 the restriction and the
  // fused prolong-sweep), so the parent writes no iterate and this level
  // reads none (bit-identical to storing it).
  int level(int l, int start, int pre_done, bool from_zero, bool zero_done = false, bool zero_virtual = false) {
    const int nl = h->n_levels();
    const LevelView& L = h->views[l];
    double* f = h->f_ptr(l);
    if (l == nl - 1) {
      timed_launch(l, kTimedCoarsest, [&] {
        if (h->galerkin(l))
          launch_check(launch_block_march(h->block, f, buf(l, 0), s), "block march");
        else
          launch_check(launch_coarsest(h->adjoint, h->coarsest, f, buf(l, 0), h->ws->coarse_scratch->p, s),
                       "coarsest");
      });
      kernels += h->galerkin(l) ? 1 : coarsest_launches(h->coarsest);
      return 0;
    }
    int cur = start;
    int pre = nu - pre_done;
    bool virt = false;
    if (from_zero) {
      cur = 0;
      if (nu >= 1 && zero_virtual) {
        virt = true;
        pre = nu - 1;
      } else if (nu >= 1 && zero_done) {
        pre = nu - 1;
      } else if (nu >= 1) {
        timed_launch(l, kTimedFromZero, [&] {
          if (h->galerkin(l))
            launch_check(launch_g_from_zero(h->dviews[l], f, buf(l, 0), omega, s), "g_sweep0");
          else
            launch_check(launch_sweep_from_zero(L, f, buf(l, 0), omega, s), "sweep0");
        });
        ++kernels;
        pre = nu - 1;
      } else {
        cuda_check(cudaMemsetAsync(buf(l, 0), 0, sizeof(double) * h->ndofs(l), s), "memset");
        pre = 0;
      }
    }
    smooth(l, f, cur, pre, &virt);
    const LevelView& C = h->views[l + 1];
    // per-node level and causal x / t transfer: the fused kernels
    const bool fused = !h->galerkin(l) && !h->gen_xfer(l);
    // the child's first pre-smoothing sweep (from zero): recomputed where it is
    // read (per-node child with fused transfers of its own), else written by
    // this restriction; the coarsest level starts from its exact solve
    const ZeroMode zm = child_zero_mode(h, l, nu);
    const bool virt_zero = zm.virt, fuse_zero = zm.store;
    if (l == 0 && down_done) {
      if (!fused || pre != 0 || virt) throw std::logic_error("fine down-pass on a level that smooths first");
    } else if (fused) {
      timed_launch(l, kTimedRestrict, [&] {
        launch_check(launch_restrict_residual(h->adjoint, L, C, h->dirs[l], f, virt ? nullptr : buf(l, cur),
                                              h->ws->f[l + 1]->p, s, fuse_zero ? buf(l + 1, 0) : nullptr,
                                              omega, l == 0 && up_fused ? up_ptrs(h) : nullptr),
                     "restrict");
      });
      ++kernels;
    } else {
      // r = f - J x into the idle ping-pong buffer, then f_{l+1} = R r
      timed_launch(l, kTimedRestrict, [&] {
        if (h->galerkin(l))
          launch_check(launch_g_residual(h->dviews[l], f, buf(l, cur), buf(l, 1 - cur), s), "g_residual");
        else
          launch_check(launch_residual(h->adjoint, L, f, buf(l, cur), buf(l, 1 - cur), s), "residual");
        launch_check(launch_xfer_restrict(h->xviews[l], buf(l, 1 - cur), h->ws->f[l + 1]->p, s), "restrict");
      });
      kernels += 2;
    }
    const int child = level(l + 1, 0, 0, true, fuse_zero, virt_zero);
    const double* xc = buf(l + 1, child);
    if (l == 0 && up_fused) {  // the up-pass kernel (emit_up) prolongs, smooths and closes the cycle
      if (!fused || virt || nu != 1) throw std::logic_error("fine up-pass on an unsupported level 0");
      up_xc = xc;
      return 0;
    }
    int post = nu;
    if (virt && !fused) throw std::logic_error("virtual zero iterate on a level without fused transfers");
    if (!fused) {
      // level 0 must end in buffer 0 (the solve reads it): prolong out of place
      // when the post-smoothing launches would otherwise leave it in buffer 1
      const bool flip = l == 0 && (cur + smooth_launches(l, post)) % 2 != 0;
      launch_check(launch_xfer_prolong_add(h->xviews[l], xc, buf(l, cur), buf(l, flip ? 1 - cur : cur), s),
                   "prolong");
      ++kernels;
      if (flip) cur = 1 - cur;
    } else if (nu >= 1) {
      timed_launch(l, kTimedProlongSweep, [&] {
        launch_check(launch_sweep_prolong(h->adjoint, L, C, h->dirs[l], f, virt ? nullptr : buf(l, cur), xc,
                                          buf(l, 1 - cur), omega, s),
                     "sweep_prolong");
      });
      ++kernels;
      cur = 1 - cur;
      post = nu - 1;
    } else {
      launch_check(launch_prolong_add(L, C, h->dirs[l], xc, buf(l, cur), s), "prolong");
      ++kernels;
    }
    smooth(l, f, cur, post);
    return cur;
  }
};

bool speculative(const stmg_hierarchy* h, int nu) { return h->n_levels() > 1 && nu >= 1; }

// The level-0 pass that closes a cycle (and opens the solve): block partials
// of ||f - J x||^2 and, when the next cycle is speculated, its first
// pre-smoothing sweep into y; under fine_down also level 1's right-hand side
// (and stored zero iterate), i.e. the next cycle's level-0 restriction.
void launch_norm_pass(stmg_hierarchy* h, int nu, const double* f, const double* x, double* y, double omega,
                      cudaStream_t s, int64_t* np) {
  Workspace& ws = *h->ws;
  if (y != nullptr && fine_down(h, nu)) {
    const ZeroMode zm = child_zero_mode(h, 0, nu);
    launch_check(launch_down(h->adjoint, h->views[0], h->views[1], h->dirs[0], f, x, y, ws.f[1]->p,
                             zm.store ? ws.xa[1]->p : nullptr, omega, ws.partials->p, np, s),
                 "norm + sweep + restrict");
    return;
  }
  launch_check(launch_sweep(h->adjoint, h->views[0], f, x, y, omega, ws.partials->p, np, s), "norm sweep");
}

// Fine up-pass (k_up) closing a cycle: u = S(*P[0] + P x_c) into the primary buffer,
// the next speculative iterate into *P[1], partials of ||f - J u||^2.
// virtual_zero: the iterate read is S(0), recomputed from f (cycle 1 of a zero-guess solve:
// the opening pass then does not store it).
void launch_up_pass(stmg_hierarchy* h, const double* xc, double omega, cudaStream_t s, int64_t* np,
                    bool virtual_zero = false) {
  Workspace& ws = *h->ws;
  double** P = up_ptrs(h);
  launch_check(launch_up(h->adjoint, h->views[0], h->views[1], h->dirs[0], h->f_ptr(0),
                         virtual_zero ? nullptr : ws.xb[0]->p, xc, h->xa_ptr(0), P + 1, virtual_zero ? nullptr : P,
                         omega, ws.partials->p, np, s),
               "prolong + sweep + norm + sweep");
}

// first: the graph of cycle 1 after the opening restriction (launch_restrict_open): level 0's
// restriction is already done, the cycle starts at level 1.
GraphEntry& get_graph(stmg_hierarchy* h, int nu, double omega, bool first = false) {
  const GraphKey key{nu, omega, h->profiling, h->f_ptr(0), h->xa_ptr(0), first ? 1 : 0};  // profiling: int mode
  auto it = h->graphs.find(key);
  if (it != h->graphs.end()) return it->second;
  if (h->graphs.size() >= kMaxGraphs) {
    for (auto& kv : h->graphs) destroy_graph_entry(kv.second);
    h->graphs.clear();
  }
  Nvtx range("stmg::capture_v_cycle");
  GraphEntry e;
  Emitter em{h, nu, omega, h->cap_stream};
  em.down_done = first || fine_down(h, nu);
  em.up_fused = fine_up(h, nu);
  if (h->profiling) {
    em.timed = &e.timed;
    em.prof_mode = h->profiling;
  }
  cuda_check(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal), "capture");
  const bool spec = speculative(h, nu);
  e.final_buf = em.level(0, spec ? 1 : 0, spec ? 1 : 0, false);
  cuda_check(cudaStreamEndCapture(h->cap_stream, &e.graph), "end capture");
  cuda_check(cudaGraphInstantiate(&e.exec, e.graph, 0), "graph instantiate");
  e.kernels = em.kernels;
  e.up_xc = em.up_xc;
  return h->graphs.emplace(key, e).first->second;
}

// The solve loop of mg_solve (proj/src/multigrid.cpp:260-273) as one graph: a
// WHILE conditional node whose body is [V-cycle, speculative norm sweep,
// finalize, k_cycle_check].  The host launches it once per solve instead of
// one V-cycle graph plus a norm read-back per cycle.  Returns nullptr (and the
// host loop is used) when the graph cannot be built.
cudaGraphExec_t get_loop(stmg_hierarchy* h, int nu, double omega) {
  GraphEntry& e = get_graph(h, nu, omega);
  if (e.loop_tried) return e.loop_exec;
  e.loop_tried = true;
  Nvtx range("stmg::capture_solve_loop");
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ex = nullptr;
  auto fail = [&] {
    cudaGetLastError();
    if (ex) cudaGraphExecDestroy(ex);
    if (g) cudaGraphDestroy(g);
    return static_cast<cudaGraphExec_t>(nullptr);
  };
  if (cudaGraphCreate(&g, 0) != cudaSuccess) return fail();
  cudaGraphConditionalHandle handle;
  if (cudaGraphConditionalHandleCreate(&handle, g, 1, cudaGraphCondAssignDefault) != cudaSuccess) return fail();
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  if (cudaGraphAddNode(&node, g, nullptr, 0, &cp) != cudaSuccess) return fail();
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaStream_t cs = h->cap_stream;
  if (cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return fail();
  bool ok = true;
  try {
    Emitter em{h, nu, omega, cs};
    em.down_done = fine_down(h, nu);
    em.up_fused = fine_up(h, nu);
    const bool spec = h->n_levels() > 1 && nu >= 1;
    const int fin = em.level(0, spec ? 1 : 0, spec ? 1 : 0, false);
    if (fin != 0) throw std::logic_error("level-0 iterate left the primary buffer");
    Workspace& ws = *h->ws;
    int64_t np = 0;
    if (em.up_fused) launch_up_pass(h, em.up_xc, omega, cs, &np);
    else launch_norm_pass(h, nu, h->f_ptr(0), h->xa_ptr(0), spec ? ws.xb[0]->p : nullptr, omega, cs, &np);
    auto* ctl = reinterpret_cast<SolveLoopCtl*>(ws.loop->p);
    launch_check(launch_finalize_check(ws.partials->p, np, ws.scalars->p, ctl, ws.loop->p + kLoopCtlDoubles,
                                       handle, cs),
                 "finalize + cycle check");
    if (em.up_fused) launch_check(launch_swap_ptrs(up_ptrs(h), cs), "swap");
  } catch (...) {
    ok = false;
  }
  cudaGraph_t captured = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(cs, &captured);
  if (!ok || ec != cudaSuccess) return fail();
  if (cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) return fail();
  e.loop_graph = g;
  e.loop_exec = ex;
  return ex;
}

bool is_device_ptr(const void* p, int* device = nullptr) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (device) *device = a.device;
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Binds the caller's level-0 vectors for the duration of one solve.
struct Bind {
  stmg_hierarchy* h;
  Bind(stmg_hierarchy* hh, const double* b, double* x) : h(hh) {
    h->bind_b = b;
    h->bind_x = x;
  }
  ~Bind() {
    h->bind_b = nullptr;
    h->bind_x = nullptr;
  }
};

// sum of squares of the level-0 residual (and optionally a speculative sweep
// into xb) -> scalars[slot]
int64_t emit_norm(stmg_hierarchy* h, int nu, const double* f, const double* x, double* y, double omega,
                  int slot) {
  int64_t np = 0;
  launch_norm_pass(h, nu, f, x, y, omega, h->stream, &np);
  launch_check(launch_finalize_sum(h->ws->partials->p, np, h->ws->scalars->p + slot, h->stream),
               "finalize");
  return 1 + finalize_launches(np);
}

double fetch_scalars(stmg_hierarchy* h, int count, double* out) {
  launch_check(launch_peek(h->ws->pinned, h->ws->scalars->p, count, h->stream), "scalar read-back");
  cuda_check(cudaStreamSynchronize(h->stream), "stream sync");
  for (int i = 0; i < count; ++i) out[i] = h->ws->pinned[i];
  return out[0];
}

// mg_solve, proj/src/multigrid.cpp:212-279
// flags & STMG_SOLVE_ZERO_GUESS: the initial iterate is zero and u is output only
// (not read, not uploaded): the device iterate is cleared instead.
void solve(stmg_hierarchy* h, const double* b, double* u, const stmg_solve_options& o,
           stmg_solve_report* rep, double* history, int32_t cap, int32_t flags = 0) {
  if (!b || !u) throw std::invalid_argument("mg_solve: vector size mismatch");
  if (flags & ~STMG_SOLVE_ZERO_GUESS) throw std::invalid_argument("mg_solve: unknown flags");
  const bool zero_guess = (flags & STMG_SOLVE_ZERO_GUESS) != 0;
  if (o.nu < 0 || o.omega <= 0.0 || o.tol <= 0.0 || o.div_tol <= o.tol || o.max_cycles < 0)
    throw std::invalid_argument("mg_solve: invalid options");
  if (!history || cap < o.max_cycles + 1)
    throw std::invalid_argument("mg_solve: history buffer smaller than max_cycles + 1");
  Nvtx range(h->adjoint ? "stmg::mg_solve(adjoint)" : "stmg::mg_solve");
  DeviceGuard dg(h->device);
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t n = h->ndofs(0);
  const size_t bytes = sizeof(double) * static_cast<size_t>(n);
  Workspace& ws = *h->ws;
  int b_device = -1, u_device = -1;
  const bool b_dev = is_device_ptr(b, &b_device), u_dev = is_device_ptr(u, &u_device);
  // Device-resident b and u on the hierarchy's device are used in place: the V-cycle
  // reads b and updates u directly (u is in/out, as in the reference), no copies.
  // Host vectors (or other devices') are staged through the workspace.
  const bool in_place = b_dev && u_dev && b_device == h->device && u_device == h->device &&
                        static_cast<const void*>(b) != static_cast<const void*>(u);
  Bind bind(h, in_place ? b : nullptr, in_place ? u : nullptr);
  const double* B = h->f_ptr(0);
  double* X = h->xa_ptr(0);
  double* Y = ws.xb[0]->p;
  cuda_check(cudaEventRecord(h->ev0, h->stream), "event");
  if (!in_place) {
    cuda_check(cudaMemcpyAsync(ws.f[0]->p, b, bytes, b_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                               h->stream),
               "b copy");
    if (!zero_guess)
      cuda_check(cudaMemcpyAsync(X, u, bytes, u_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream),
                 "u copy");
  }
  int64_t launches = 0;
  int64_t np = 0;
  const bool spec = speculative(h, o.nu);
  // Zero initial guess with a speculated first sweep: the initial residual is b itself
  // (J 0 = +0 row by row), so ||r0||^2 = ||b||^2 and the first pre-smoothing sweep is
  // S(0) = 0 + omega (b * inv_diag): ONE pass over b gives the sweep and the norm
  // (history[0] is exactly 1, as in the reference).  The first cycle overwrites the
  // primary iterate, so it is cleared only when no cycle runs.
  // nu = 1 with fused level-0 transfers: cycle 1's level-0 restriction reads exactly S(0),
  // so it runs inside the opening pass too (launch_restrict_open: 20 B/DOF for the sweep,
  // the norm and level 1's right-hand side), and cycle 1 uses the graph that starts at level 1.
  const bool open_r = zero_guess && spec && o.max_cycles > 0 && o.nu == 1 && h->n_levels() >= 2 &&
                      !h->galerkin(0) && !h->gen_xfer(0) && !child_zero_mode(h, 0, o.nu).store;
  const bool zero_open = zero_guess && spec && o.max_cycles > 0 && (open_r || !fine_down(h, o.nu));
  if (zero_guess && !zero_open) cuda_check(cudaMemsetAsync(X, 0, bytes, h->stream), "u clear");
  GraphEntry* g = nullptr;
  GraphEntry* g1 = nullptr;  // cycle 1 after the opening restriction
  if (o.max_cycles > 0) g = &get_graph(h, o.nu, o.omega);
  if (open_r) g1 = &get_graph(h, o.nu, o.omega, true);
  if (open_r) {
    // with the fine up-pass, cycle 1 recomputes S(0) from b as well: it is not stored at all
    launch_check(launch_restrict_open(h->adjoint, h->views[0], h->views[1], h->dirs[0], B, ws.f[1]->p, nullptr,
                                      fine_up(h, o.nu) ? nullptr : Y, o.omega,
                                      ws.partials->p, &np, h->stream),
                 "sweep from zero + norm + restriction");
    launch_check(launch_finalize_sum(ws.partials->p, np, ws.scalars->p + 0, h->stream), "finalize");
    launch_check(launch_finalize_sum(ws.partials->p, np, ws.scalars->p + 1, h->stream), "finalize");
    launches += 1 + 2 * finalize_launches(np);
  } else if (zero_open) {
    launch_check(launch_sweep_from_zero_norm(h->views[0], B, Y, o.omega, ws.partials->p, &np, h->stream),
                 "sweep from zero + norm");
    launch_check(launch_finalize_sum(ws.partials->p, np, ws.scalars->p + 0, h->stream), "finalize");
    launch_check(launch_finalize_sum(ws.partials->p, np, ws.scalars->p + 1, h->stream), "finalize");
    launches += 1 + 2 * finalize_launches(np);
  } else {
    launch_check(launch_sumsq(B, n, ws.partials->p, &np, h->stream), "sumsq");
    launch_check(launch_finalize_sum(ws.partials->p, np, ws.scalars->p + 0, h->stream), "finalize");
    launches += 1 + finalize_launches(np);
    launches += emit_norm(h, o.nu, B, X, spec && o.max_cycles > 0 ? Y : nullptr, o.omega, 1);
  }
  double sc[2];
  fetch_scalars(h, 2, sc);
  const double norm_b = std::sqrt(sc[0]);
  rep->absolute_norms = norm_b == 0.0 ? 1 : 0;
  const double denom = rep->absolute_norms ? 1.0 : norm_b;
  const double r0 = std::sqrt(sc[1]) / denom;
  int nh = 0;
  history[nh++] = r0;
  rep->cycles = 0;
  rep->factor = 1.0;
  rep->smoother_dof_updates = 0.0;
  rep->fine_sweeps = rep->fine_restricts = rep->fine_prolong_sweeps = rep->fine_sweep_pairs = 0;
  rep->fine_sweep_seconds = rep->fine_restrict_seconds = rep->fine_prolong_sweep_seconds = 0.0;
  rep->fine_sweep_pair_seconds = 0.0;
  rep->fine_norm_passes = 0;
  rep->fine_norm_pass_seconds = 0.0;
  rep->fine_ups = 0;
  rep->fine_up_seconds = 0.0;
  double per_cycle_updates = 0.0;
  for (int l = 0; l + 1 < h->n_levels(); ++l) per_cycle_updates += 2.0 * o.nu * static_cast<double>(h->ndofs(l));
  const bool up = fine_up(h, o.nu) && o.max_cycles > 0;
  if (up && r0 >= o.tol) {
    // third level-0 buffer and the pointer table {speculative iterate in, out} = {Y, Z}
    if (!ws.xz) {
      ws.xz = std::make_unique<DeviceBuf>(n + kVecPad);
      h->device_bytes += 8 * (n + kVecPad);
    }
    double* tab[2] = {Y, ws.xz->p};
    PokeWords w{};
    static_assert(sizeof(tab) == 2 * sizeof(double), "pointer table travels as two words");
    std::memcpy(w.v, tab, sizeof(tab));
    launch_check(launch_poke(ws.ptrs->p, w, 2, h->stream), "ptrs");
  }
  cudaGraphExec_t loop = nullptr;
  if (r0 >= o.tol && o.max_cycles > (open_r ? 1 : 0) && o.max_cycles <= kLoopHistory && !h->profiling)
    loop = get_loop(h, o.nu, o.omega);
  // One cycle launched from the host: the V-cycle graph gg, the pass that closes the
  // cycle, a read-back of the norm and the reference's bookkeeping.  Returns true when
  // the solve stops after it.
  auto host_cycle = [&](GraphEntry* gg, int cycle) -> bool {
    Nvtx cyc("stmg::v_cycle");
    cuda_check(cudaGraphLaunch(gg->exec, h->stream), "graph launch");
    launches += gg->kernels;
    if (gg->final_buf != 0) throw std::logic_error("level-0 iterate left the primary buffer");
    const bool more = cycle < o.max_cycles;
    if (h->profiling) cuda_check(cudaEventRecord(h->norm_ev0, h->stream), "event");
    if (up) {
      int64_t npu = 0;
      launch_up_pass(h, gg->up_xc, o.omega, h->stream, &npu, open_r && cycle == 1);
      launch_check(launch_finalize_sum(ws.partials->p, npu, ws.scalars->p + 1, h->stream), "finalize");
      launches += 1 + finalize_launches(npu);
    } else {
      launches += emit_norm(h, o.nu, B, X, spec && more ? Y : nullptr, o.omega, 1);
    }
    if (h->profiling) cuda_check(cudaEventRecord(h->norm_ev1, h->stream), "event");
    if (up) {
      launch_check(launch_swap_ptrs(up_ptrs(h), h->stream), "swap");
      launches += 1;
    }
    fetch_scalars(h, 2, sc);
    if (h->profiling) {  // the pass closing the cycle (incl. its finalize launch)
      float ms = 0.f;
      cuda_check(cudaEventElapsedTime(&ms, h->norm_ev0, h->norm_ev1), "event elapsed");
      if (up) {
        rep->fine_ups += 1;
        rep->fine_up_seconds += ms * 1e-3;
      } else {
        rep->fine_norm_passes += 1;
        rep->fine_norm_pass_seconds += ms * 1e-3;
      }
    }
    for (const TimedKernel& t : gg->timed) {
      float ms = 0.f;
      cuda_check(cudaEventElapsedTime(&ms, t.start, t.stop), "event elapsed");
      if (h->prof.size() < h->host.size()) h->prof.resize(h->host.size());
      h->prof[t.level][t.kind].first += 1;
      h->prof[t.level][t.kind].second += ms * 1e-3;
      if (t.level != 0) continue;
      if (t.kind == kTimedSweep) {
        rep->fine_sweeps += 1;
        rep->fine_sweep_seconds += ms * 1e-3;
      } else if (t.kind == kTimedSweep2) {
        rep->fine_sweep_pairs += 1;
        rep->fine_sweep_pair_seconds += ms * 1e-3;
      } else if (t.kind == kTimedRestrict) {
        rep->fine_restricts += 1;
        rep->fine_restrict_seconds += ms * 1e-3;
      } else if (t.kind == kTimedProlongSweep) {
        rep->fine_prolong_sweeps += 1;
        rep->fine_prolong_sweep_seconds += ms * 1e-3;
      }
    }
    const double rn = std::sqrt(sc[1]) / denom;
    history[nh++] = rn;
    rep->cycles = cycle;
    rep->smoother_dof_updates += per_cycle_updates;
    if (rn < o.tol) {
      rep->status = STMG_CONVERGED;
      return true;
    }
    if (!std::isfinite(rn) || rn > o.div_tol) {
      rep->status = STMG_DIVERGED;
      return true;
    }
    return false;
  };
  if (r0 < o.tol) {
    rep->status = STMG_CONVERGED;
  } else {
    rep->status = STMG_MAX_CYCLES;
    int done = 0;  // cycles run so far
    bool stop = false;
    if (open_r) {  // cycle 1: its level-0 restriction ran with the opening pass
      stop = host_cycle(g1, 1);
      done = 1;
    }
    if (!stop && done < o.max_cycles && loop) {
      // the remaining cycle loop on the device: one launch, one read-back
      auto* ctl = reinterpret_cast<SolveLoopCtl*>(ws.loop_host);
      *ctl = SolveLoopCtl{o.tol, o.div_tol, o.max_cycles, done, STMG_MAX_CYCLES, 0};
      PokeWords w{};
      static_assert(sizeof(SolveLoopCtl) <= sizeof(w.v) && sizeof(SolveLoopCtl) % sizeof(double) == 0, "ctl words");
      std::memcpy(w.v, ctl, sizeof(SolveLoopCtl));
      launch_check(launch_poke(ws.loop->p, w, static_cast<int>(kLoopCtlDoubles), h->stream), "loop ctl");
      cuda_check(cudaGraphLaunch(loop, h->stream), "loop graph launch");
      launch_check(launch_peek(ws.loop_host, ws.loop->p, static_cast<int>(kLoopCtlDoubles + o.max_cycles + 1),
                               h->stream),
                   "loop read-back");
      cuda_check(cudaStreamSynchronize(h->stream), "stream sync");
      const double* dh = ws.loop_host + kLoopCtlDoubles;
      for (int c = done + 1; c <= ctl->cycles; ++c) history[nh++] = dh[c];
      const int ran = ctl->cycles - done;
      rep->cycles = ctl->cycles;
      rep->status = ctl->status;
      rep->smoother_dof_updates += per_cycle_updates * ran;
      // per cycle: the V-cycle graph, the pass closing the cycle and its fixed-order sum
      const int64_t norm_np = up ? up_partials_needed(h->views[0])
                                 : fine_down(h, o.nu) ? down_partials_needed(h->views[0], h->views[1], h->dirs[0])
                                                      : sweep_partials_needed(h->views[0]);
      launches += static_cast<int64_t>(ran) * (g->kernels + 1 + finalize_launches(norm_np) + (up ? 1 : 0));
    } else if (!stop) {
      for (int cycle = done + 1; cycle <= o.max_cycles; ++cycle)
        if (host_cycle(g, cycle)) break;
    }
  }
  if (rep->cycles > 0) rep->factor = std::pow(history[nh - 1] / r0, 1.0 / rep->cycles);
  if (zero_open && rep->cycles == 0) cuda_check(cudaMemsetAsync(X, 0, bytes, h->stream), "u clear");
  cuda_check(cudaEventRecord(h->ev1, h->stream), "event");
  if (!in_place)
    cuda_check(cudaMemcpyAsync(u, X, bytes, u_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->stream),
               "u copy back");
  cuda_check(cudaStreamSynchronize(h->stream), "stream sync");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, h->ev0, h->ev1);
  rep->device_seconds = ms * 1e-3;
  rep->n_history = nh;
  rep->kernel_launches = launches;
  rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

stmg_hierarchy* checked(stmg_hierarchy* h) {
  if (!h) throw std::invalid_argument("null hierarchy handle");
  return h;
}
void check_level(const stmg_hierarchy* h, int l) {
  if (l < 0 || l >= h->n_levels()) throw std::out_of_range("level index outside hierarchy");
}

// source kinds shared with paper_2505_10168_b200/configs.py
double source_value(int kind, const double* p, double x, double t, double L, double t_T) {
  switch (kind) {
    case 0: return p[0];
    case 1: return (L - x < p[1]) ? p[0] : 0.0;
    case 2: return (L - x < p[2]) ? 1.0 + p[0] * std::sin(2.0 * M_PI * p[1] * t) : 0.0;
    case 3: {  // heat_load_value, proj/src/assembly.cpp:59-63
      const double xs = x / L - 0.5, ts = t / t_T - 0.5;
      return (1.0 + std::cos(200.0 * (xs * xs + ts * ts))) * 1.0e6;
    }
  }
  throw std::invalid_argument("load_vector: unknown source kind");
}

// load_vector, proj/src/assembly.cpp:65-83; time levels are independent, so
// they are filled by several host threads with identical per-entry arithmetic.
template <class Q>
void load_vector_impl(const HostGrid& g, Q&& q, bool masked, double* b) {
  const int64_t nn = g.n_el + 1;
  const int64_t levels = g.n_t + 1;
  auto work = [&](int64_t lo, int64_t hi) {
    for (int64_t n = lo; n < hi; ++n) {
      double* row = b + n * nn;
      std::fill(row, row + nn, 0.0);
      if (n == 0) continue;
      const double t = static_cast<double>(n) * g.dt;
      for (int64_t e = 0; e < g.n_el; ++e) {
        const double qe = q((static_cast<double>(e) + 0.5) * g.dx, t) * g.dx / 2.0;
        row[e] += qe;
        row[e + 1] += qe;
      }
      if (masked) row[0] = 0.0;
    }
    if (masked && lo == 0)
      for (int64_t i = 0; i < nn; ++i) b[i] = 0.0;
  };
  const int64_t total = levels * nn;
  unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (total < (1 << 20)) nth = 1;
  std::vector<std::thread> th;
  const int64_t chunk = (levels + nth - 1) / nth;
  for (unsigned k = 0; k < nth; ++k) {
    const int64_t lo = k * chunk, hi = std::min(levels, lo + chunk);
    if (lo >= hi) break;
    th.emplace_back(work, lo, hi);
  }
  for (auto& t : th) t.join();
}

// build_hierarchy's host half (proj/src/multigrid.cpp:86-143): level grids,
// coarse materials and per-node coefficients, no device work.
// With P reassembly, *gal receives every level's operator as a 9-point stencil
// (level 0 assembled, coarser levels R J P, primal orientation); *bilinear_out
// the temporal interpolation.
std::vector<HostLevel> make_host_levels(const stmg_grid* g, const double* k, const double* c,
                                        const double* chi, const stmg_material_pair* mat,
                                        const char* method, int32_t n_dirs, const int32_t* dirs,
                                        int* reasm_out, bool* bilinear_out = nullptr,
                                        std::vector<Dia9Host>* gal = nullptr) {
  if (!g) throw std::invalid_argument("build_hierarchy: null grid");
  const HostGrid fine = make_grid(g->L, g->t_T, g->n_el, g->n_t);
  if (!k || !c) throw std::invalid_argument("build_hierarchy: fine grid has no materials");
  bool bilinear = false;
  const int reasm = parse_method(method, &bilinear);
  if (reasm == STMG_REASM_D && (!chi || !mat))
    throw std::invalid_argument("build_hierarchy: D reassembly needs the design field and materials");
  if (n_dirs < 0 || (n_dirs > 0 && !dirs)) throw std::invalid_argument("build_hierarchy: bad path");
  std::vector<HostLevel> host;
  HostLevel l0;
  l0.g = fine;
  l0.k.assign(k, k + fine.n_el);
  l0.c.assign(c, c + fine.n_el);
  if (chi) l0.chi.assign(chi, chi + fine.n_el);
  l0.build();
  host.push_back(std::move(l0));
  for (int32_t s = 0; s < n_dirs; ++s) {
    const int dir = dirs[s];
    if (dir != STMG_DIR_X && dir != STMG_DIR_T && dir != STMG_DIR_XT)
      throw std::invalid_argument("build_hierarchy: bad direction");
    const HostLevel& p = host.back();
    HostLevel lc;
    lc.g = coarsen(p.g, dir);
    if (dir == STMG_DIR_T) {
      lc.k = p.k;
      lc.c = p.c;
      lc.chi = p.chi;
    } else {
      coarsen_materials_x(p.k, p.c, p.chi.empty() ? nullptr : &p.chi, mat, reasm, lc.k, lc.c, &lc.chi);
      if (reasm != STMG_REASM_D) lc.chi.clear();
    }
    lc.build();
    // build_transfer -> build_prolongation's check (proj/src/transfer.cpp:44-47)
    if (dir == STMG_DIR_XT && bilinear)
      throw std::invalid_argument("build_prolongation: combined coarsening is causal-only");
    host.push_back(std::move(lc));
  }
  if (reasm_out) *reasm_out = reasm;
  if (bilinear_out) *bilinear_out = bilinear;
  if (gal) {
    gal->clear();
    if (reasm == STMG_REASM_P) {
      // lc.J = galerkin_operator(t.R, prev.J, t.P) (proj/src/multigrid.cpp:131-134)
      const HostLevel& h0 = host[0];
      gal->push_back(dia9_assembled(h0.g.n_el, h0.g.n_t, h0.W, h0.D, h0.E, h0.SW, h0.S, h0.SE, h0.w));
      for (int32_t s = 0; s < n_dirs; ++s) {
        const HostGrid& cg = host[s + 1].g;
        Dia9Host A = dia9_galerkin(gal->back(), dirs[s], bilinear, cg.n_el, cg.n_t);
        dia9_invert_diagonal(A);
        gal->push_back(std::move(A));
      }
      if (n_dirs > 0) (*gal)[0] = Dia9Host();  // level 0 stays the assembled (fast-path) operator
    }
  }
  return host;
}

// Replace the host levels of an existing hierarchy whose level shapes are
// unchanged (same grid and path, new materials) and refresh the device
// coefficient and PCR tables in place; graphs are re-captured on next use
// because w / 1/w are captured by value.
void refresh_levels(stmg_hierarchy* h, std::vector<HostLevel> host) {
  if (host.size() != h->host.size()) throw std::logic_error("refresh_levels: level count changed");
  DeviceGuard dg(h->device);
  sync_unless_capturing(h->stream);
  h->host = std::move(host);
  for (size_t l = 0; l < h->host.size(); ++l) {
    const HostLevel& hl = h->host[l];
    const std::vector<double> t = hl.table(h->adjoint);
    if (static_cast<int64_t>(t.size()) + kVecPad != h->coef[l]->n)
      throw std::logic_error("refresh_levels: shape changed");
    cuda_check(cudaMemcpy(h->coef[l]->p, t.data(), t.size() * 8, cudaMemcpyHostToDevice), "coef upload");
    h->views[l].w = hl.w;
    h->views[l].inv_w = hl.inv_w;
  }
  auto a = std::move(h->pcr_alpha);
  auto g = std::move(h->pcr_gamma);
  auto b = std::move(h->pcr_bfin);
  build_pcr(h);  // fresh factor tables (old ones freed after the sync above)
  for (auto& kv : h->graphs) destroy_graph_entry(kv.second);
  h->graphs.clear();
}

// MmaUpdater / mma_subsolve, restated from proj/src/mma.cpp:19-157 with the
// same loop order (sequential sums), so the design update is the reference's.
struct Mma {
  double x_min, x_max, move, asym_init, shrink, grow;
  size_t n;
  int iter = 0;
  std::vector<double> x_prev, x_prev2, low_, upp_;

  std::vector<double> subsolve(const std::vector<double>& x, const std::vector<double>& df,
                               const std::vector<double>& dg, double g, const std::vector<double>& lower,
                               const std::vector<double>& upper, const std::vector<double>& alpha,
                               const std::vector<double>& beta) const {
    std::vector<double> p0(n), q0(n), p1(n), q1(n), y(n);
    double r1 = g;
    for (size_t j = 0; j < n; ++j) {
      if (!(lower[j] < x[j] && x[j] < upper[j]))
        throw std::invalid_argument("mma_subsolve: x outside the asymptotes");
      const double du = upper[j] - x[j];
      const double dl = x[j] - lower[j];
      p0[j] = du * du * std::max(df[j], 0.0);
      q0[j] = dl * dl * std::max(-df[j], 0.0);
      p1[j] = du * du * std::max(dg[j], 0.0);
      q1[j] = dl * dl * std::max(-dg[j], 0.0);
      r1 -= p1[j] / du + q1[j] / dl;
    }
    auto x_of_eta = [&](double eta) {
      for (size_t j = 0; j < n; ++j) {
        const double p = p0[j] + eta * p1[j];
        const double q = q0[j] + eta * q1[j];
        double v;
        if (p == 0.0 && q == 0.0) {
          v = x[j];
        } else {
          const double sp = std::sqrt(p);
          const double sq = std::sqrt(q);
          v = (sp * lower[j] + sq * upper[j]) / (sp + sq);
        }
        y[j] = std::clamp(v, alpha[j], beta[j]);
      }
    };
    auto g_hat = [&] {
      double sacc = r1;
      for (size_t j = 0; j < n; ++j) sacc += p1[j] / (upper[j] - y[j]) + q1[j] / (y[j] - lower[j]);
      return sacc;
    };
    x_of_eta(0.0);
    if (g_hat() <= 0.0) return y;
    double eta_lo = 0.0, eta_hi = 1.0;
    x_of_eta(eta_hi);
    int guard = 0;
    while (g_hat() > 0.0) {
      eta_lo = eta_hi;
      eta_hi *= 2.0;
      x_of_eta(eta_hi);
      if (++guard > 100)
        throw std::runtime_error("mma_subsolve: constraint unreachable within the move limits");
    }
    for (int it = 0; it < 100; ++it) {
      const double mid = 0.5 * (eta_lo + eta_hi);
      x_of_eta(mid);
      if (g_hat() > 0.0) eta_lo = mid;
      else eta_hi = mid;
    }
    x_of_eta(eta_hi);
    return y;
  }

  std::vector<double> update(const std::vector<double>& x, const std::vector<double>& df,
                             const std::vector<double>& dg, double g) {
    const double range = x_max - x_min;
    ++iter;
    std::vector<double> low(n), upp(n);
    if (iter <= 2) {
      for (size_t j = 0; j < n; ++j) {
        low[j] = x[j] - asym_init * range;
        upp[j] = x[j] + asym_init * range;
      }
    } else {
      for (size_t j = 0; j < n; ++j) {
        const double osc = (x[j] - x_prev[j]) * (x_prev[j] - x_prev2[j]);
        const double gamma = osc < 0.0 ? shrink : osc > 0.0 ? grow : 1.0;
        low[j] = x[j] - gamma * (x_prev[j] - low_[j]);
        upp[j] = x[j] + gamma * (upp_[j] - x_prev[j]);
        low[j] = std::clamp(low[j], x[j] - 10.0 * range, x[j] - 0.01 * range);
        upp[j] = std::clamp(upp[j], x[j] + 0.01 * range, x[j] + 10.0 * range);
      }
    }
    std::vector<double> alpha(n), beta(n);
    for (size_t j = 0; j < n; ++j) {
      alpha[j] = std::max({x_min, low[j] + 0.1 * (x[j] - low[j]), x[j] - move * range});
      beta[j] = std::min({x_max, upp[j] - 0.1 * (upp[j] - x[j]), x[j] + move * range});
    }
    std::vector<double> x_new = subsolve(x, df, dg, g, low, upp, alpha, beta);
    x_prev2 = iter >= 2 ? x_prev : x;
    x_prev = x;
    low_ = std::move(low);
    upp_ = std::move(upp);
    return x_new;
  }
};

// optimise, proj/src/optimisation.cpp:83-186 (host loop; solves, objective and
// sensitivities on the GPU)
// Per-element scales of objective_sensitivities (proj/src/optimisation.cpp:54-56):
// dk_dx = k'(chi) / dx, dc_dx6 = c'(chi) dx / 6, with simp_derivatives'
// expressions (proj/src/materials.cpp).
void sensitivity_scales(const double* chi, int64_t ne, const stmg_material_pair& m, double dx, double* dk,
                        double* dc) {
  for (int64_t e = 0; e < ne; ++e) {
    if (!(chi[e] >= 0.0 && chi[e] <= 1.0)) throw std::invalid_argument("volume fraction outside [0, 1]");
    const double dkv = m.p_k * (m.k_con - m.k_ins) * std::pow(chi[e], m.p_k - 1.0);
    const double dcv = m.p_c * (m.c_con - m.c_ins) * std::pow(chi[e], m.p_c - 1.0);
    dk[e] = dkv / dx;
    dc[e] = dcv * dx / 6;
  }
}

void optimise(const stmg_grid* geom, const stmg_optimise_options& o, int device, double* chi_out,
              stmg_iteration_record* recs, int32_t* n_records, double* theta_out, int32_t* converged,
              double* seconds, double* design_history) {
  if (o.volume_limit <= 0.0 || o.volume_limit > 1.0)
    throw std::invalid_argument("optimise: volume limit must be in (0, 1]");
  if (o.max_iterations < 1 || o.stable_iterations < 1 || o.rel_change_tol <= 0.0 || o.theta_ref <= 0.0)
    throw std::invalid_argument("optimise: invalid options");
  if (!(o.mma_x_min < o.mma_x_max)) throw std::invalid_argument("MmaUpdater: empty box");
  if (o.mma_move_limit <= 0.0 || o.mma_asym_init <= 0.0 || o.mma_asym_shrink <= 0.0 ||
      o.mma_asym_shrink >= 1.0 || o.mma_asym_grow <= 1.0)
    throw std::invalid_argument("MmaUpdater: invalid options");
  const auto t0 = std::chrono::steady_clock::now();
  double ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  auto tick = std::chrono::steady_clock::now();
  auto lap = [&](int k) {
    const auto now = std::chrono::steady_clock::now();
    ph[k] += std::chrono::duration<double>(now - tick).count();
    tick = now;
  };
  const HostGrid g = make_grid(geom->L, geom->t_T, geom->n_el, geom->n_t);
  const int64_t ne = g.n_el, nn = ne + 1, ndof = nn * (g.n_t + 1);
  std::vector<double> chi(static_cast<size_t>(ne), o.chi_init), k(ne), c(ne);
  const double scale = g.dt / o.theta_ref;
  const std::vector<double> dg(static_cast<size_t>(ne), g.dx / (o.volume_limit * g.L));
  Mma mma{o.mma_x_min, o.mma_x_max, o.mma_move_limit, o.mma_asym_init, o.mma_asym_shrink,
          o.mma_asym_grow, static_cast<size_t>(ne)};
  DeviceGuard dgd(device);
  DeviceBuf d_b(ndof), d_c(ndof), d_u(ndof), d_lam(ndof), d_dk(ne), d_dc(ne), d_sens(ne), d_part(1184 * 2),
      d_s(2);
  // b = load_vector(g) with masking (optimisation.cpp:102; assembly.cpp:59-83, 128-130) and
  // the adjoint right-hand side c = b dt / theta_ref (adjoint_rhs, optimisation.cpp:26-32),
  // both generated on the device
  launch_check(launch_load_vector(3, nullptr, 0, g.L, g.t_T, g.n_el, g.n_t, 1, d_b.p, nullptr), "load_vector");
  launch_check(launch_scale(d_b.p, scale, d_c.p, ndof, nullptr), "scale");
  cuda_check(cudaMemset(d_u.p, 0, ndof * 8), "memset");
  cuda_check(cudaMemset(d_lam.p, 0, ndof * 8), "memset");
  std::unique_ptr<stmg_hierarchy> h, ht;
  std::vector<int32_t> cur_dirs;
  const stmg_grid gc{g.L, g.t_T, g.n_el, g.n_t};
  const stmg_plan_request preq{o.n_levels, o.lambda_crit, o.strategy, parse_method(o.method), o.min_elements};
  std::vector<double> hist(static_cast<size_t>(std::max(o.solve.max_cycles, 0)) + 1);
  double theta_prev = std::numeric_limits<double>::quiet_NaN();
  int stable = 0;
  *converged = 0;
  *n_records = 0;
  lap(0);
  for (int it = 1; it <= o.max_iterations; ++it) {
    Nvtx range("stmg::optimise_iteration");
    simp(chi.data(), ne, o.mat, k.data(), c.data());
    std::vector<int32_t> dirs(static_cast<size_t>(std::max(o.n_levels - 1, 0)));
    plan(g, k.data(), c.data(), chi.data(), &o.mat, preq, dirs.data(), nullptr);
    bool bilinear = false;
    std::vector<Dia9Host> gal;
    std::vector<HostLevel> host =
        make_host_levels(&gc, k.data(), c.data(), chi.data(), &o.mat, o.method,
                         static_cast<int32_t>(dirs.size()), dirs.data(), nullptr, &bilinear, &gal);
    // per-node levels with an unchanged path: refresh the coefficient tables in
    // place; Galerkin levels are rebuilt (their operators are per DOF)
    if (h && dirs == cur_dirs && gal.empty()) {
      refresh_levels(h.get(), host);
      refresh_levels(ht.get(), std::move(host));
    } else {
      ht.reset();
      h.reset();
      auto nh = std::make_unique<stmg_hierarchy>();
      nh->device = device;
      nh->dirs = dirs;
      nh->host = std::move(host);
      nh->bilinear = bilinear;
      nh->gal = std::move(gal);
      nh->reassembly = parse_method(o.method);
      finish_create(nh.get(), false, nullptr);
      stmg_hierarchy* tp = nullptr;
      const int rc = stmg_hierarchy_transposed(nh.get(), &tp);
      if (rc != STMG_OK) throw std::runtime_error(g_error);
      h = std::move(nh);
      ht.reset(tp);
      cur_dirs = dirs;
    }
    lap(1);
    if (!o.warm_start) cuda_check(cudaMemset(d_u.p, 0, ndof * 8), "memset");
    stmg_solve_report pr{}, ar{};
    solve(h.get(), d_b.p, d_u.p, o.solve, &pr, hist.data(), static_cast<int32_t>(hist.size()));
    lap(2);
    // objective_value = dot(b, u) dt / theta_ref (optimisation.cpp:21-24)
    int64_t np = 0;
    launch_check(launch_dot(d_b.p, d_u.p, ndof, d_part.p, &np, h->stream), "dot");
    launch_check(launch_finalize_sum(d_part.p, np, d_s.p, h->stream), "finalize");
    double dotbu = 0.0;
    cuda_check(cudaMemcpyAsync(&dotbu, d_s.p, 8, cudaMemcpyDeviceToHost, h->stream), "d2h");
    sync_unless_capturing(h->stream);
    const double theta = dotbu * g.dt / o.theta_ref;
    if (!o.warm_start) cuda_check(cudaMemset(d_lam.p, 0, ndof * 8), "memset");
    lap(3);
    solve(ht.get(), d_c.p, d_lam.p, o.solve, &ar, hist.data(), static_cast<int32_t>(hist.size()));
    lap(4);
    double vsum = 0.0;
    for (double v : chi) vsum += v;
    const double vol = vsum * g.dx / g.L;
    const double g_val = vol / o.volume_limit - 1.0;
    const double change = it == 1 ? std::numeric_limits<double>::infinity()
                                  : std::abs(theta - theta_prev) / std::abs(theta);
    stmg_iteration_record& r = recs[it - 1];
    r.iteration = it;
    r.theta = theta;
    r.volume = vol;
    r.constraint = g_val;
    r.change = change;
    r.primal_status = pr.status;
    r.adjoint_status = ar.status;
    r.primal_cycles = pr.cycles;
    r.adjoint_cycles = ar.cycles;
    r.primal_factor = pr.factor;
    r.adjoint_factor = ar.factor;
    r.primal_seconds = pr.seconds;
    r.adjoint_seconds = ar.seconds;
    {  // path_to_string (proj/src/strategy.cpp:118-125)
      std::string ps;
      for (size_t i = 0; i < dirs.size(); ++i) {
        if (i) ps += ',';
        ps += dirs[i] == STMG_DIR_X ? "x" : dirs[i] == STMG_DIR_T ? "t" : "xt";
      }
      const size_t m = std::min(ps.size(), sizeof(r.path) - 1);
      std::memcpy(r.path, ps.data(), m);
      r.path[m] = '\0';
    }
    if (design_history)  // the design this iteration evaluated
      std::memcpy(design_history + static_cast<size_t>(it - 1) * ne, chi.data(), sizeof(double) * ne);
    *n_records = it;
    *theta_out = theta;
    theta_prev = theta;
    stable = change < o.rel_change_tol ? stable + 1 : 0;
    if (stable >= o.stable_iterations) {
      *converged = 1;
      break;
    }
    if (it == o.max_iterations) break;
    // objective_sensitivities (optimisation.cpp:34-73) on the GPU
    std::vector<double> dk(ne), dc(ne), sens(ne);
    sensitivity_scales(chi.data(), ne, o.mat, g.dx, dk.data(), dc.data());
    cuda_check(cudaMemcpyAsync(d_dk.p, dk.data(), ne * 8, cudaMemcpyHostToDevice, h->stream), "h2d");
    cuda_check(cudaMemcpyAsync(d_dc.p, dc.data(), ne * 8, cudaMemcpyHostToDevice, h->stream), "h2d");
    launch_check(launch_sensitivities(ne, g.n_t, g.dt, d_dk.p, d_dc.p, d_u.p, d_lam.p, d_sens.p, h->stream),
                 "sensitivities");
    cuda_check(cudaMemcpyAsync(sens.data(), d_sens.p, ne * 8, cudaMemcpyDeviceToHost, h->stream), "d2h");
    sync_unless_capturing(h->stream);
    chi = mma.update(chi, sens, dg, g_val);
    lap(5);
  }
  std::memcpy(chi_out, chi.data(), sizeof(double) * static_cast<size_t>(ne));
  *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace
}  // namespace stmgb

#include "stmg_dist.cuh"

using namespace stmgb;

extern "C" {

const char* stmg_last_error(void) { return g_error.c_str(); }
int stmg_abi_version(void) { return STMG_ABI_VERSION; }

int stmg_apply_design(const double* chi, int64_t n, const stmg_material_pair* mat, double* k,
                      double* c) {
  return guarded([&] {
    if (!chi || !mat || !k || !c || n < 0) throw std::invalid_argument("apply_design: null argument");
    simp(chi, n, *mat, k, c);
  });
}

int stmg_load_vector(const stmg_grid* g, int32_t kind, const double* params, int32_t masked,
                     double* b) {
  return guarded([&] {
    if (!g || !b) throw std::invalid_argument("load_vector: null argument");
    const HostGrid hg = make_grid(g->L, g->t_T, g->n_el, g->n_t);
    double p[4] = {0, 0, 0, 0};
    const int np = kind == 0 ? 1 : kind == 1 ? 2 : kind == 2 ? 3 : 0;
    if (kind < 0 || kind > 3) throw std::invalid_argument("load_vector: unknown source kind");
    if (np > 0 && !params) throw std::invalid_argument("load_vector: missing source parameters");
    for (int i = 0; i < np; ++i) p[i] = params[i];
    load_vector_impl(hg, [&](double x, double t) { return source_value(kind, p, x, t, hg.L, hg.t_T); },
                     masked != 0, b);
  });
}

int stmg_load_vector_device(const stmg_grid* g, int32_t kind, const double* params, int32_t masked,
                            double* b, void* cuda_stream) {
  return guarded([&] {
    if (!g || !b) throw std::invalid_argument("load_vector: null argument");
    const HostGrid hg = make_grid(g->L, g->t_T, g->n_el, g->n_t);
    const int np = kind == 0 ? 1 : kind == 1 ? 2 : kind == 2 ? 3 : 0;
    if (kind < 0 || kind > 3) throw std::invalid_argument("load_vector: unknown source kind");
    if (np > 0 && !params) throw std::invalid_argument("load_vector: missing source parameters");
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, b) != cudaSuccess || a.type != cudaMemoryTypeDevice) {
      cudaGetLastError();
      throw std::invalid_argument("load_vector_device: b is not device memory");
    }
    DeviceGuard dg(a.device);
    launch_check(launch_load_vector(kind, params, np, hg.L, hg.t_T, hg.n_el, hg.n_t, masked != 0, b,
                                    static_cast<cudaStream_t>(cuda_stream)),
                 "load_vector");
    sync_unless_capturing(static_cast<cudaStream_t>(cuda_stream));
  });
}

int stmg_load_vector_cb(const stmg_grid* g, stmg_source_fn q, void* ctx, int32_t masked, double* b) {
  return guarded([&] {
    if (!g || !b || !q) throw std::invalid_argument("load_vector: null argument");
    const HostGrid hg = make_grid(g->L, g->t_T, g->n_el, g->n_t);
    const int64_t nn = hg.n_el + 1;
    // callbacks may not be thread-safe: sequential, same per-entry arithmetic
    std::fill(b, b + (hg.n_t + 1) * nn, 0.0);
    for (int64_t n = 1; n <= hg.n_t; ++n) {
      const double t = static_cast<double>(n) * hg.dt;
      for (int64_t e = 0; e < hg.n_el; ++e) {
        const double qe = q((static_cast<double>(e) + 0.5) * hg.dx, t, ctx) * hg.dx / 2.0;
        b[n * nn + e] += qe;
        b[n * nn + e + 1] += qe;
      }
    }
    if (masked) {
      for (int64_t i = 0; i < nn; ++i) b[i] = 0.0;
      for (int64_t n = 1; n <= hg.n_t; ++n) b[n * nn] = 0.0;
    }
  });
}

int stmg_plan_coarsening(const stmg_grid* g, const double* k, const double* c, const double* chi,
                         const stmg_material_pair* mat, const stmg_plan_request* req,
                         int32_t* dirs_out, double* indicator_out) {
  return guarded([&] {
    if (!g || !req || (!dirs_out && req->n_levels > 1))
      throw std::invalid_argument("plan_coarsening: null argument");
    const HostGrid hg = make_grid(g->L, g->t_T, g->n_el, g->n_t);
    plan(hg, k, c, chi, mat, *req, dirs_out, indicator_out);
  });
}

int stmg_hierarchy_create(const stmg_grid* g, const double* k, const double* c, const double* chi,
                          const stmg_material_pair* mat, const char* method, int32_t n_dirs,
                          const int32_t* dirs, int32_t device, stmg_hierarchy** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("build_hierarchy: null output handle");
    *out = nullptr;
    if (!g) throw std::invalid_argument("build_hierarchy: null grid");
    Nvtx range("stmg::build_hierarchy");
    auto h = std::make_unique<stmg_hierarchy>();
    // argument errors (the reference's invalid_argument) are raised before any device work
    h->host = make_host_levels(g, k, c, chi, mat, method, n_dirs, dirs, &h->reassembly, &h->bilinear, &h->gal);
    int n_dev = 0;
    cuda_check(cudaGetDeviceCount(&n_dev), "cudaGetDeviceCount");
    if (device < 0 || device >= n_dev) throw std::invalid_argument("build_hierarchy: bad device ordinal");
    h->device = device;
    h->dirs.assign(dirs, dirs + n_dirs);
    finish_create(h.get(), false, nullptr);
    *out = h.release();
  });
}

int stmg_hierarchy_transposed(const stmg_hierarchy* src, stmg_hierarchy** out) {
  return guarded([&] {
    if (!src || !out) throw std::invalid_argument("transposed_hierarchy: null argument");
    Nvtx range("stmg::transposed_hierarchy");
    auto h = std::make_unique<stmg_hierarchy>();
    h->device = src->device;
    h->adjoint = !src->adjoint;
    h->reassembly = src->reassembly;
    h->dirs = src->dirs;
    h->host = src->host;
    h->bilinear = src->bilinear;
    h->gal = src->gal;
    finish_create(h.get(), true, src);
    *out = h.release();
  });
}

void stmg_hierarchy_destroy(stmg_hierarchy* h) { delete h; }

int stmg_hierarchy_n_levels(const stmg_hierarchy* h, int32_t* n) {
  return guarded([&] {
    if (!h || !n) throw std::invalid_argument("null argument");
    *n = h->n_levels();
  });
}

int stmg_hierarchy_level_info(const stmg_hierarchy* h, int32_t l, int64_t* n_el, int64_t* n_t,
                              double* w) {
  return guarded([&] {
    if (!h) throw std::invalid_argument("null hierarchy handle");
    check_level(h, l);
    if (n_el) *n_el = h->host[l].g.n_el;
    if (n_t) *n_t = h->host[l].g.n_t;
    if (w) *w = h->host[l].w;
  });
}

int stmg_hierarchy_level_coeffs(const stmg_hierarchy* h, int32_t l, double* cm, double* c0,
                                double* cp, double* om, double* o0, double* op, double* invd) {
  return guarded([&] {
    if (!h) throw std::invalid_argument("null hierarchy handle");
    check_level(h, l);
    if (h->galerkin(l))
      throw std::invalid_argument("level_coeffs: Galerkin level (per-DOF operator); use stmg_hierarchy_level_stencil9");
    const std::vector<double> t = h->host[l].table(h->adjoint);
    const size_t nn = static_cast<size_t>(h->host[l].g.n_el + 1);
    double* outs[7] = {cm, c0, cp, om, o0, op, invd};
    for (int k = 0; k < 7; ++k)
      if (outs[k]) std::memcpy(outs[k], t.data() + k * nn, nn * sizeof(double));
  });
}

int stmg_hierarchy_level_stencil9(const stmg_hierarchy* h, int32_t l, double* v9, uint16_t* mask,
                                  double* invd) {
  return guarded([&] {
    if (!h) throw std::invalid_argument("null hierarchy handle");
    check_level(h, l);
    Dia9Host A;
    if (l < static_cast<int>(h->gal.size()) && !h->gal[l].mask.empty()) {
      A = h->gal[l];
    } else {
      const HostLevel& hl = h->host[l];
      A = dia9_assembled(hl.g.n_el, hl.g.n_t, hl.W, hl.D, hl.E, hl.SW, hl.S, hl.SE, hl.w);
      dia9_invert_diagonal(A);
    }
    if (h->adjoint) A = dia9_transposed(A);
    const size_t nd = static_cast<size_t>(A.ndofs());
    if (v9) std::memcpy(v9, A.v.data(), 9 * nd * sizeof(double));
    if (mask) std::memcpy(mask, A.mask.data(), nd * sizeof(uint16_t));
    if (invd) std::memcpy(invd, A.inv_diag.data(), nd * sizeof(double));
  });
}

int stmg_level_stencil9_host(const stmg_grid* g, const double* k, const double* c, const double* chi,
                             const stmg_material_pair* mat, const char* method, int32_t n_dirs,
                             const int32_t* dirs, int32_t level, int32_t adjoint, double* v9,
                             uint16_t* mask, double* invd) {
  return guarded([&] {
    int reasm = 0;
    bool bilinear = false;
    std::vector<Dia9Host> gal;
    const std::vector<HostLevel> host =
        make_host_levels(g, k, c, chi, mat, method, n_dirs, dirs, &reasm, &bilinear, &gal);
    if (level < 0 || level >= static_cast<int32_t>(host.size())) throw std::out_of_range("level out of range");
    Dia9Host A;
    if (level < static_cast<int32_t>(gal.size()) && !gal[level].mask.empty()) {
      A = std::move(gal[level]);
    } else {
      const HostLevel& hl = host[level];
      A = dia9_assembled(hl.g.n_el, hl.g.n_t, hl.W, hl.D, hl.E, hl.SW, hl.S, hl.SE, hl.w);
      dia9_invert_diagonal(A);
    }
    if (adjoint) A = dia9_transposed(A);
    const size_t nd = static_cast<size_t>(A.ndofs());
    if (v9) std::memcpy(v9, A.v.data(), 9 * nd * sizeof(double));
    if (mask) std::memcpy(mask, A.mask.data(), nd * sizeof(uint16_t));
    if (invd) std::memcpy(invd, A.inv_diag.data(), nd * sizeof(double));
  });
}

int stmg_hierarchy_set_stream(stmg_hierarchy* h, void* cuda_stream) {
  return guarded([&] {
    checked(h);
    DeviceGuard dg(h->device);
    sync_unless_capturing(h->stream);
    h->stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : h->own_stream;
  });
}

int stmg_hierarchy_set_profiling(stmg_hierarchy* h, int32_t on) {
  return guarded([&] {
    checked(h);
    h->profiling = on < 0 ? 0 : (on > 2 ? 2 : on);
  });
}

int stmg_hierarchy_set_fusion(stmg_hierarchy* h, int32_t flags) {
  return guarded([&] {
    checked(h);
    if (flags < 0 || flags > kFuseAll) throw std::invalid_argument("set_fusion: unknown flags");
    DeviceGuard dg(h->device);
    cuda_check(cudaStreamSynchronize(h->stream), "sync");
    h->fusion = flags;
    for (auto& kv : h->graphs) destroy_graph_entry(kv.second);
    h->graphs.clear();
  });
}

int stmg_hierarchy_set_tiling(stmg_hierarchy* h, int64_t small_dofs, int64_t tiny_dofs) {
  return guarded([&] {
    checked(h);
    DeviceGuard dg(h->device);
    cuda_check(cudaStreamSynchronize(h->stream), "sync");
    const int64_t small = small_dofs > 0 ? small_dofs : kSmallNtDofs;
    const int64_t tiny = tiny_dofs > 0 ? tiny_dofs : kTinyNtDofs;
    for (auto& v : h->views) v.tile_nt = tile_nt_for(v.nn * (v.n_t + 1), small, tiny);
    h->coarsest.lv = h->views.back();
    for (auto& kv : h->graphs) destroy_graph_entry(kv.second);
    h->graphs.clear();
  });
}

int stmg_hierarchy_profile(const stmg_hierarchy* h, int32_t level, int32_t kind, int64_t* launches,
                           double* seconds) {
  return guarded([&] {
    if (!h || !launches || !seconds) throw std::invalid_argument("null argument");
    check_level(h, level);
    if (kind < 0 || kind >= kTimedKinds) throw std::out_of_range("profile kind");
    *launches = 0;
    *seconds = 0.0;
    if (static_cast<size_t>(level) < h->prof.size()) {
      *launches = h->prof[level][kind].first;
      *seconds = h->prof[level][kind].second;
    }
  });
}

int stmg_hierarchy_device_bytes(const stmg_hierarchy* h, int64_t* bytes) {
  return guarded([&] {
    if (!h || !bytes) throw std::invalid_argument("null argument");
    *bytes = h->device_bytes;
  });
}

int stmg_mg_solve(stmg_hierarchy* h, const double* b, double* u, const stmg_solve_options* opts,
                  stmg_solve_report* report, double* history, int32_t cap) {
  return guarded([&] {
    checked(h);
    if (!opts || !report) throw std::invalid_argument("mg_solve: null argument");
    solve(h, b, u, *opts, report, history, cap);
  });
}

int stmg_mg_solve_ex(stmg_hierarchy* h, const double* b, double* u, const stmg_solve_options* opts, int32_t flags,
                     stmg_solve_report* report, double* history, int32_t cap) {
  return guarded([&] {
    checked(h);
    if (!opts || !report) throw std::invalid_argument("mg_solve: null argument");
    solve(h, b, u, *opts, report, history, cap, flags);
  });
}

int stmg_mg_solve_batch(int32_t count, stmg_hierarchy* const* hs, const double* const* bs, double* const* us,
                        const stmg_solve_options* opts, stmg_solve_report* reports, double* const* histories,
                        int32_t history_cap) {
  return guarded([&] {
    if (count < 0 || !opts) throw std::invalid_argument("mg_solve_batch: bad arguments");
    if (count == 0) return;
    if (!hs || !bs || !us || !reports || !histories) throw std::invalid_argument("mg_solve_batch: null argument");
    for (int32_t i = 0; i < count; ++i) {
      checked(hs[i]);
      for (int32_t j = 0; j < i; ++j)
        if (hs[i] == hs[j] || hs[i]->ws == hs[j]->ws)
          throw std::invalid_argument(
              "mg_solve_batch: two entries share a workspace (a repeat, or a hierarchy and its transpose)");
    }
    // one host worker per concurrent solve; each hierarchy runs on its own
    // stream (and device), so the solves overlap on the GPU(s)
    std::vector<int> rc(static_cast<size_t>(count), STMG_OK);
    std::vector<std::string> msg(static_cast<size_t>(count));
    std::atomic<int32_t> next{0};
    auto worker = [&] {
      for (int32_t i = next++; i < count; i = next++) {
        rc[i] = stmg_mg_solve(hs[i], bs[i], us[i], opts, &reports[i], histories[i], history_cap);
        if (rc[i] != STMG_OK) msg[i] = g_error;
      }
    };
    const int32_t n_workers = std::min<int32_t>(count, 64);
    std::vector<std::thread> th;
    for (int32_t w = 1; w < n_workers; ++w) th.emplace_back(worker);
    worker();
    for (auto& t : th) t.join();
    for (int32_t i = 0; i < count; ++i) {
      if (rc[i] == STMG_OK) continue;
      const std::string m = "mg_solve_batch[" + std::to_string(i) + "]: " + msg[i];
      switch (rc[i]) {
        case STMG_EINVAL: throw std::invalid_argument(m);
        case STMG_ERANGE: throw std::out_of_range(m);
        case STMG_ECUDA: throw CudaError(m);
        case STMG_ENOMEM: throw NoMem(m);
        default: throw std::runtime_error(m);
      }
    }
  });
}

namespace {
struct StreamRaii {
  cudaStream_t s = nullptr;
  StreamRaii() { cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate"); }
  ~StreamRaii() {
    if (s) cudaStreamDestroy(s);
  }
};
struct EventRaii {
  cudaEvent_t e = nullptr;
  EventRaii() { cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate"); }
  ~EventRaii() {
    if (e) cudaEventDestroy(e);
  }
};
}  // namespace

// The copy engines serve their queues one operation at a time, so any copy-engine operation
// of the solve itself would wait behind a whole 8.6 GB vector of a neighbouring entry, and
// the solve with it (measured with the solve's pointer table / loop control / read-back as
// cudaMemcpyAsync: 0.27 s per entry, the solve started only after the next upload).  The
// solve's small transfers are kernels now (launch_poke / launch_peek: 0.22 s per entry, the
// PCIe duplex bound); the vectors still go in pieces so that other small copies on the
// device (a caller's, another hierarchy's) are not held up either.  No bandwidth loss down to
// 8 MiB pieces (profiles/pcie_duplex.cu), but very small pieces fill the stream's launch queue.
size_t stream_chunk_bytes() {  // STMG_STREAM_CHUNK_MIB (0: whole vectors); default 64
  static const size_t v = [] {
    const char* e = std::getenv("STMG_STREAM_CHUNK_MIB");
    const long mib = e ? std::atol(e) : 64;
    return mib > 0 ? static_cast<size_t>(mib) << 20 : ~size_t(0);
  }();
  return v;
}
void copy_chunked(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s, const char* what) {
  const size_t chunk = stream_chunk_bytes();
  for (size_t o = 0; o < bytes; o += std::min(chunk, bytes - o))
    cuda_check(cudaMemcpyAsync(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                               std::min(chunk, bytes - o), kind, s),
               what);
}

// A sequence of solves on one hierarchy with host vectors, software-pipelined over two
// device (b, u) slots: while solve k runs on the hierarchy's stream, b_{k+1} (and u_{k+1}
// for a warm start) uploads on a second stream and u_{k-1} downloads on a third, so a
// stream of solves costs max(upload, solve, download) per entry instead of their sum.
// Each solve binds its slot in place, i.e. it is exactly stmg_mg_solve_ex on device
// vectors: the same kernels in the same order, bit-identical results.
int stmg_mg_solve_stream(stmg_hierarchy* h, int32_t count, const double* const* bs, double* const* us,
                         const stmg_solve_options* opts, int32_t flags, stmg_solve_report* reports,
                         double* const* histories, int32_t history_cap) {
  return guarded([&] {
    checked(h);
    if (count < 0 || !opts) throw std::invalid_argument("mg_solve_stream: bad arguments");
    if (count == 0) return;
    if (!bs || !us || !reports || !histories) throw std::invalid_argument("mg_solve_stream: null argument");
    if (flags & ~STMG_SOLVE_ZERO_GUESS) throw std::invalid_argument("mg_solve_stream: unknown flags");
    bool staged = count > 1;
    for (int32_t k = 0; k < count; ++k) {
      if (!bs[k] || !us[k] || !histories[k]) throw std::invalid_argument("mg_solve_stream: null entry");
      int dev = -1;
      if (is_device_ptr(bs[k], &dev) || is_device_ptr(us[k], &dev)) staged = false;  // nothing to overlap
    }
    if (!staged) {
      for (int32_t k = 0; k < count; ++k) solve(h, bs[k], us[k], *opts, &reports[k], histories[k], history_cap, flags);
      return;
    }
    Nvtx range("stmg::mg_solve_stream");
    DeviceGuard dg(h->device);
    Workspace& ws = *h->ws;
    const int64_t n = h->ndofs(0);
    const size_t bytes = sizeof(double) * static_cast<size_t>(n);
    const bool zero_guess = (flags & STMG_SOLVE_ZERO_GUESS) != 0;
    for (int s = 0; s < 2; ++s) {
      if (!ws.stage_b[s]) ws.stage_b[s] = std::make_unique<DeviceBuf>(n);
      if (!ws.stage_u[s]) ws.stage_u[s] = std::make_unique<DeviceBuf>(n);
    }
    StreamRaii up, down;
    EventRaii ev_up[2], ev_down[2];
    // upload entry k into slot k & 1: the slot's b was last read by solve k - 2 (finished:
    // solves are host-synchronous); its u may still be downloading (ev_down)
    auto upload = [&](int32_t k) {
      const int s = k & 1;
      if (!zero_guess) {
        if (k >= 2) cuda_check(cudaStreamWaitEvent(up.s, ev_down[s].e, 0), "wait");
        copy_chunked(ws.stage_u[s]->p, us[k], bytes, cudaMemcpyHostToDevice, up.s, "u upload");
      }
      copy_chunked(ws.stage_b[s]->p, bs[k], bytes, cudaMemcpyHostToDevice, up.s, "b upload");
      cuda_check(cudaEventRecord(ev_up[s].e, up.s), "event");
    };
    try {
      upload(0);
      for (int32_t k = 0; k < count; ++k) {
        const int s = k & 1;
        if (k + 1 < count) upload(k + 1);
        cuda_check(cudaStreamWaitEvent(h->stream, ev_up[s].e, 0), "wait");
        if (k >= 2) cuda_check(cudaStreamWaitEvent(h->stream, ev_down[s].e, 0), "wait");  // u_{k-2} has left the slot
        solve(h, ws.stage_b[s]->p, ws.stage_u[s]->p, *opts, &reports[k], histories[k], history_cap, flags);
        // the solve returned after its stream drained: the slot's u is final
        copy_chunked(us[k], ws.stage_u[s]->p, bytes, cudaMemcpyDeviceToHost, down.s, "u download");
        cuda_check(cudaEventRecord(ev_down[s].e, down.s), "event");
      }
      cuda_check(cudaStreamSynchronize(down.s), "stream sync");
    } catch (...) {
      cudaStreamSynchronize(up.s);  // no copy may outlive the caller's buffers
      cudaStreamSynchronize(down.s);
      throw;
    }
  });
}

int stmg_hierarchy_release_staging(stmg_hierarchy* h) {
  return guarded([&] {
    checked(h);
    DeviceGuard dg(h->device);
    cuda_check(cudaStreamSynchronize(h->stream), "stream sync");
    for (int s = 0; s < 2; ++s) {
      h->ws->stage_b[s].reset();
      h->ws->stage_u[s].reset();
    }
    for (auto& kv : h->graphs) destroy_graph_entry(kv.second);  // cycle graphs bound to the freed slots
    h->graphs.clear();
  });
}

int stmg_level_sweeps(stmg_hierarchy* h, int32_t l, const double* f, double* x, int32_t sweeps,
                      double omega) {
  return guarded([&] {
    checked(h);
    check_level(h, l);
    DeviceGuard dg(h->device);
    double* tmp = h->ws->xb[l]->p;
    std::unique_ptr<DeviceBuf> own;
    if (!tmp) {
      own = std::make_unique<DeviceBuf>(h->ndofs(l));
      tmp = own->p;
    }
    double* a = x;
    double* b = tmp;
    int left = sweeps;
    for (; h->galerkin(l) && left >= 1; --left) {
      launch_check(launch_g_sweep(h->dviews[l], f, a, b, omega, h->stream), "g_sweep");
      std::swap(a, b);
    }
    for (; left >= 2; left -= 2) {
      launch_check(launch_sweep2(h->adjoint, h->views[l], f, a, b, omega, h->stream), "sweep2");
      std::swap(a, b);
    }
    if (left == 1) {
      launch_check(launch_sweep(h->adjoint, h->views[l], f, a, b, omega, nullptr, nullptr, h->stream), "sweep");
      std::swap(a, b);
    }
    if (a != x)
      cuda_check(cudaMemcpyAsync(x, a, sizeof(double) * h->ndofs(l), cudaMemcpyDeviceToDevice, h->stream), "copy");
    sync_unless_capturing(h->stream);
  });
}

int stmg_level_sweep_kernels(stmg_hierarchy* h, int32_t l, const double* f, double* x, double* y,
                             int32_t launches, int32_t fused_pairs, double omega) {
  return guarded([&] {
    checked(h);
    check_level(h, l);
    if (!f || !x || !y || x == y || launches < 0) throw std::invalid_argument("sweep_kernels: bad arguments");
    DeviceGuard dg(h->device);
    double* a = x;
    double* b = y;
    for (int k = 0; k < launches; ++k) {
      if (h->galerkin(l))
        launch_check(launch_g_sweep(h->dviews[l], f, a, b, omega, h->stream), "g_sweep");
      else if (fused_pairs)
        launch_check(launch_sweep2(h->adjoint, h->views[l], f, a, b, omega, h->stream), "sweep2");
      else
        launch_check(launch_sweep(h->adjoint, h->views[l], f, a, b, omega, nullptr, nullptr, h->stream), "sweep");
      std::swap(a, b);
    }
  });
}

int stmg_level_residual(stmg_hierarchy* h, int32_t l, const double* f, const double* x, double* r) {
  return guarded([&] {
    checked(h);
    check_level(h, l);
    DeviceGuard dg(h->device);
    if (h->galerkin(l)) launch_check(launch_g_residual(h->dviews[l], f, x, r, h->stream), "g_residual");
    else launch_check(launch_residual(h->adjoint, h->views[l], f, x, r, h->stream), "residual");
    sync_unless_capturing(h->stream);
  });
}

int stmg_level_restrict_residual(stmg_hierarchy* h, int32_t l, const double* f, const double* x,
                                 double* fc) {
  return guarded([&] {
    checked(h);
    check_level(h, l);
    if (l + 1 >= h->n_levels()) throw std::out_of_range("no coarser level");
    DeviceGuard dg(h->device);
    if (h->galerkin(l) || h->gen_xfer(l)) {
      DeviceBuf r(h->ndofs(l));
      if (h->galerkin(l)) launch_check(launch_g_residual(h->dviews[l], f, x, r.p, h->stream), "g_residual");
      else launch_check(launch_residual(h->adjoint, h->views[l], f, x, r.p, h->stream), "residual");
      launch_check(launch_xfer_restrict(h->xviews[l], r.p, fc, h->stream), "restrict");
      cuda_check(cudaStreamSynchronize(h->stream), "sync");  // r is freed on return
    } else {
      launch_check(launch_restrict_residual(h->adjoint, h->views[l], h->views[l + 1], h->dirs[l], f, x,
                                            fc, h->stream),
                   "restrict");
    }
    sync_unless_capturing(h->stream);
  });
}

// Fused V-cycle kernel forms on device vectors (parity tests of the fusions).
int stmg_level_fused(stmg_hierarchy* h, int32_t l, int32_t kind, const double* f, const double* x,
                     const double* xc, double* y, double* fc, double omega, double* norm2) {
  return guarded([&] {
    checked(h);
    check_level(h, l);
    if (h->galerkin(l)) throw std::invalid_argument("level_fused: per-node levels only");
    if (!f) throw std::invalid_argument("level_fused: null f");
    const bool coarse_op = kind == STMG_FUSED_ZERO_RESTRICT || kind == STMG_FUSED_ZERO_PROLONG_SWEEP ||
                           kind == STMG_FUSED_FINE_DOWN || kind == STMG_FUSED_PROLONG_SWEEP ||
                           kind == STMG_FUSED_FINE_UP;
    if (coarse_op && (l + 1 >= h->n_levels() || h->gen_xfer(l)))
      throw std::out_of_range("level_fused: no fused transfer to a coarser level");
    DeviceGuard dg(h->device);
    const LevelView& L = h->views[l];
    switch (kind) {
      case STMG_FUSED_ZERO_SWEEP:
        if (!y) throw std::invalid_argument("level_fused: null y");
        launch_check(launch_sweep(h->adjoint, L, f, nullptr, y, omega, nullptr, nullptr, h->stream), "sweep");
        break;
      case STMG_FUSED_ZERO_PAIR:
        if (!y) throw std::invalid_argument("level_fused: null y");
        launch_check(launch_sweep2(h->adjoint, L, f, nullptr, y, omega, h->stream), "sweep2");
        break;
      case STMG_FUSED_ZERO_RESTRICT:
        if (!fc) throw std::invalid_argument("level_fused: null f_coarse");
        launch_check(launch_restrict_residual(h->adjoint, L, h->views[l + 1], h->dirs[l], f, nullptr, fc, h->stream,
                                              nullptr, omega),
                     "restrict");
        break;
      case STMG_FUSED_ZERO_PROLONG_SWEEP:
        if (!y || !xc) throw std::invalid_argument("level_fused: null y / x_coarse");
        launch_check(launch_sweep_prolong(h->adjoint, L, h->views[l + 1], h->dirs[l], f, nullptr, xc, y, omega,
                                          h->stream),
                     "sweep_prolong");
        break;
      case STMG_FUSED_FINE_DOWN: {
        if (!x || !y || !fc) throw std::invalid_argument("level_fused: null x / y / f_coarse");
        int64_t np = 0;
        launch_check(launch_down(h->adjoint, L, h->views[l + 1], h->dirs[l], f, x, y, fc, nullptr, omega,
                                 h->ws->partials->p, &np, h->stream),
                     "down");
        launch_check(launch_finalize_sum(h->ws->partials->p, np, h->ws->scalars->p + 2, h->stream), "finalize");
        double sc[3];
        fetch_scalars(h, 3, sc);
        if (norm2) *norm2 = sc[2];
        break;
      }
      case STMG_FUSED_PROLONG_SWEEP:
        if (!x || !y || !xc) throw std::invalid_argument("level_fused: null x / y / x_coarse");
        launch_check(launch_sweep_prolong(h->adjoint, L, h->views[l + 1], h->dirs[l], f, x, xc, y, omega, h->stream),
                     "sweep_prolong");
        break;
      case STMG_FUSED_FINE_UP: {
        if (!x || !y || !xc || !fc || x == y || x == fc || y == fc)
          throw std::invalid_argument("level_fused: fine up-pass needs distinct x, y and w (f_coarse)");
        double* const wptr = fc;
        cuda_check(cudaMemcpyAsync(h->ws->ptrs->p, &wptr, sizeof(wptr), cudaMemcpyHostToDevice, h->stream), "ptr");
        cuda_check(cudaStreamSynchronize(h->stream), "sync");  // wptr is a stack variable
        int64_t np = 0;
        launch_check(launch_up(h->adjoint, L, h->views[l + 1], h->dirs[l], f, x, xc, y,
                               reinterpret_cast<double* const*>(h->ws->ptrs->p), nullptr, omega, h->ws->partials->p,
                               &np, h->stream),
                     "up");
        launch_check(launch_finalize_sum(h->ws->partials->p, np, h->ws->scalars->p + 2, h->stream), "finalize");
        double sc[3];
        fetch_scalars(h, 3, sc);
        if (norm2) *norm2 = sc[2];
        break;
      }
      case STMG_FUSED_NORM_SWEEP: {
        if (!x || !y) throw std::invalid_argument("level_fused: null x / y");
        int64_t np = 0;
        launch_check(launch_sweep(h->adjoint, L, f, x, y, omega, h->ws->partials->p, &np, h->stream), "norm sweep");
        launch_check(launch_finalize_sum(h->ws->partials->p, np, h->ws->scalars->p + 2, h->stream), "finalize");
        double sc[3];
        fetch_scalars(h, 3, sc);
        if (norm2) *norm2 = sc[2];
        break;
      }
      default:
        throw std::invalid_argument("level_fused: unknown kind");
    }
    sync_unless_capturing(h->stream);
  });
}

int stmg_level_restrict(stmg_hierarchy* h, int32_t l, const double* r, double* fc) {
  return guarded([&] {
    checked(h);
    check_level(h, l);
    if (l + 1 >= h->n_levels()) throw std::out_of_range("no coarser level");
    DeviceGuard dg(h->device);
    if (h->gen_xfer(l)) launch_check(launch_xfer_restrict(h->xviews[l], r, fc, h->stream), "restrict");
    else launch_check(launch_restrict(h->views[l], h->views[l + 1], h->dirs[l], r, fc, h->stream), "restrict");
    sync_unless_capturing(h->stream);
  });
}

int stmg_level_prolong_add(stmg_hierarchy* h, int32_t l, const double* xc, double* x) {
  return guarded([&] {
    checked(h);
    check_level(h, l);
    if (l + 1 >= h->n_levels()) throw std::out_of_range("no coarser level");
    DeviceGuard dg(h->device);
    if (h->gen_xfer(l)) launch_check(launch_xfer_prolong_add(h->xviews[l], xc, x, x, h->stream), "prolong");
    else launch_check(launch_prolong_add(h->views[l], h->views[l + 1], h->dirs[l], xc, x, h->stream), "prolong");
    sync_unless_capturing(h->stream);
  });
}

int stmg_coarsest_solve(stmg_hierarchy* h, const double* f, double* x) {
  return guarded([&] {
    checked(h);
    DeviceGuard dg(h->device);
    if (h->galerkin(h->n_levels() - 1))
      launch_check(launch_block_march(h->block, f, x, h->stream), "block march");
    else
      launch_check(launch_coarsest(h->adjoint, h->coarsest, f, x, h->ws->coarse_scratch->p, h->stream),
                   "coarsest");
    sync_unless_capturing(h->stream);
  });
}

int stmg_residual_norm(stmg_hierarchy* h, const double* f, const double* x, double* norm) {
  return guarded([&] {
    checked(h);
    if (!norm) throw std::invalid_argument("null argument");
    DeviceGuard dg(h->device);
    emit_norm(h, 0, f, x, nullptr, 0.5, 1);
    double sc[2];
    fetch_scalars(h, 2, sc);
    *norm = std::sqrt(sc[1]);
  });
}

int stmg_norm2(stmg_hierarchy* h, const double* x, int64_t n, double* norm) {
  return guarded([&] {
    checked(h);
    if (!norm || n < 0) throw std::invalid_argument("bad argument");
    DeviceGuard dg(h->device);
    int64_t np = 0;
    launch_check(launch_sumsq(x, n, h->ws->partials->p, &np, h->stream), "sumsq");
    launch_check(launch_finalize_sum(h->ws->partials->p, np, h->ws->scalars->p, h->stream), "finalize");
    double sc[1];
    fetch_scalars(h, 1, sc);
    *norm = std::sqrt(sc[0]);
  });
}

int stmg_optimise(const stmg_grid* geom, const stmg_optimise_options* opts, int32_t device,
                  double* chi_out, stmg_iteration_record* records, int32_t* n_records, double* theta,
                  int32_t* converged, double* seconds, double* design_history) {
  return guarded([&] {
    if (!geom || !opts || !chi_out || !records || !n_records || !theta || !converged || !seconds)
      throw std::invalid_argument("optimise: null argument");
    optimise(geom, *opts, device, chi_out, records, n_records, theta, converged, seconds, design_history);
  });
}

// objective_sensitivities, proj/src/optimisation.cpp:34-73 (u, lambda host or device)
int stmg_objective_sensitivities(const stmg_grid* geom, const stmg_material_pair* mat, const double* chi,
                                 const double* u, const double* lam, double* sens, int32_t device) {
  return guarded([&] {
    if (!geom || !mat || !chi || !u || !lam || !sens) throw std::invalid_argument("objective_sensitivities: null argument");
    const HostGrid g = make_grid(geom->L, geom->t_T, geom->n_el, geom->n_t);
    const int64_t ne = g.n_el, ndof = (ne + 1) * (g.n_t + 1);
    std::vector<double> dk(ne), dc(ne);
    sensitivity_scales(chi, ne, *mat, g.dx, dk.data(), dc.data());
    DeviceGuard dgd(device);
    DeviceBuf d_dk(ne), d_dc(ne), d_sens(ne);
    std::unique_ptr<DeviceBuf> du, dl;
    const double* pu = u;
    const double* pl = lam;
    if (!is_device_ptr(u)) {
      du = std::make_unique<DeviceBuf>(ndof);
      cuda_check(cudaMemcpy(du->p, u, ndof * 8, cudaMemcpyHostToDevice), "h2d");
      pu = du->p;
    }
    if (!is_device_ptr(lam)) {
      dl = std::make_unique<DeviceBuf>(ndof);
      cuda_check(cudaMemcpy(dl->p, lam, ndof * 8, cudaMemcpyHostToDevice), "h2d");
      pl = dl->p;
    }
    cuda_check(cudaMemcpy(d_dk.p, dk.data(), ne * 8, cudaMemcpyHostToDevice), "h2d");
    cuda_check(cudaMemcpy(d_dc.p, dc.data(), ne * 8, cudaMemcpyHostToDevice), "h2d");
    launch_check(kernels_init(), "kernels_init");
    launch_check(launch_sensitivities(ne, g.n_t, g.dt, d_dk.p, d_dc.p, pu, pl, d_sens.p, nullptr), "sensitivities");
    cuda_check(cudaMemcpy(sens, d_sens.p, ne * 8, cudaMemcpyDeviceToHost), "d2h");
  });
}

// ---- time-slab multi-GPU --------------------------------------------------------
int stmg_dist_partition(int32_t n_levels, const int64_t* n_t, const int32_t* dirs, int32_t world,
                        int64_t min_slab, int32_t* n_distributed, int64_t* bounds) {
  return guarded([&] {
    if (n_levels < 1 || !n_t || (!dirs && n_levels > 1) || !n_distributed)
      throw std::invalid_argument("dist_partition: bad arguments");
    std::vector<int64_t> nts(n_t, n_t + n_levels);
    std::vector<int32_t> d(dirs, dirs + (n_levels - 1));
    const SlabPlan p = plan_slabs(nts, d, world, min_slab);
    *n_distributed = p.Lg;
    if (bounds)
      for (int l = 0; l < p.Lg; ++l)
        for (int g = 0; g <= world; ++g) bounds[static_cast<size_t>(l) * (world + 1) + g] = p.bounds[l][g];
  });
}

int stmg_dist_nccl_unique_id(void* id_out, int32_t cap) {
  return guarded([&] {
    if (!id_out || cap < static_cast<int32_t>(sizeof(ncclUniqueId)))
      throw std::invalid_argument("dist: unique-id buffer too small");
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int stmg_dist_create(const stmg_grid* g, const double* k, const double* c, const double* chi,
                     const stmg_material_pair* mat, const char* method, int32_t n_dirs,
                     const int32_t* dirs, int32_t adjoint, int32_t world, int32_t rank,
                     const void* nccl_id, int32_t device, int64_t min_slab, stmg_dist** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("dist_create: null output handle");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("dist_create: bad rank/world");
    if (!g) throw std::invalid_argument("dist_create: null grid");
    auto d = std::make_unique<stmg_dist>();
    bool bilinear = false;
    int reasm = 0;
    d->host = make_host_levels(g, k, c, chi, mat, method, n_dirs, dirs, &reasm, &bilinear);
    bool xt = false;
    for (int32_t s = 0; s < n_dirs; ++s) xt = xt || dirs[s] == STMG_DIR_XT;
    if (bilinear || reasm == STMG_REASM_P || xt)
      throw std::invalid_argument(
          "dist_create: time-slab hierarchies take causal x / t transfers with K, D or R reassembly");
    if (d->host.size() < 2) throw std::invalid_argument("dist_create: need at least two levels");
    int n_dev = 0;
    cuda_check(cudaGetDeviceCount(&n_dev), "cudaGetDeviceCount");
    if (device < 0 || device >= n_dev) throw std::invalid_argument("dist_create: bad device ordinal");
    d->device = device;
    d->adjoint = adjoint != 0;
    d->dirs.assign(dirs, dirs + n_dirs);
    dist_build(d.get(), world, rank, nccl_id, min_slab);
    *out = d.release();
  });
}

int stmg_dist_info(const stmg_dist* d, int32_t* n_distributed, int64_t* row_lo, int64_t* row_hi,
                   int32_t* n_local, int64_t* device_bytes) {
  return guarded([&] {
    if (!d) throw std::invalid_argument("null handle");
    if (n_distributed) *n_distributed = d->plan.Lg;
    if (row_lo) *row_lo = d->ranks.front().views[0].n_lo;
    if (row_hi) *row_hi = d->ranks.back().views[0].n_hi;
    if (n_local) *n_local = static_cast<int32_t>(d->ranks.size());
    if (device_bytes) *device_bytes = d->device_bytes;
  });
}

int stmg_dist_mg_solve(stmg_dist* d, const double* b, double* u, const stmg_solve_options* opts,
                       stmg_solve_report* report, double* history, int32_t cap) {
  return guarded([&] {
    if (!d || !opts || !report) throw std::invalid_argument("mg_solve: null argument");
    dist_solve(d, b, u, *opts, report, history, cap);
  });
}

int stmg_dist_mg_solve_local(stmg_dist* d, const double* b_local, double* u_local, const stmg_solve_options* opts,
                             stmg_solve_report* report, double* history, int32_t cap) {
  return guarded([&] {
    if (!d || !opts || !report) throw std::invalid_argument("mg_solve: null argument");
    dist_solve(d, b_local, u_local, *opts, report, history, cap, true);
  });
}

int stmg_dist_transport(const stmg_dist* d, char* name_out, int32_t cap) {
  return guarded([&] {
    if (!d || !name_out || cap < 1) throw std::invalid_argument("null handle or buffer");
    std::snprintf(name_out, static_cast<size_t>(cap), "%s", d->comm->name());
  });
}

int stmg_dist_split_passes(const stmg_dist* d, int64_t* count) {
  return guarded([&] {
    if (!d || !count) throw std::invalid_argument("null handle or argument");
    *count = d->split_passes;
  });
}

int stmg_dist_loop_on_device(const stmg_dist* d, int32_t* yes) {
  return guarded([&] {
    if (!d || !yes) throw std::invalid_argument("null handle or argument");
    *yes = d->last_on_device ? 1 : 0;
  });
}

void stmg_dist_destroy(stmg_dist* d) { delete d; }

int stmg_synchronize(stmg_hierarchy* h) {
  return guarded([&] {
    checked(h);
    DeviceGuard dg(h->device);
    sync_unless_capturing(h->stream);
  });
}

}  // extern "C"
