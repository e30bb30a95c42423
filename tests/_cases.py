"""Problem cases shared by the CPU (oracle vs reference) and GPU parity tests.

Each case is a small seeded instance of one BASELINE config family (or of a
reference unit-test situation) that the CPU checkers finish in seconds.
Planning uses the C oracle's restatement of plan_coarsening; the test suite
separately pins that planner to the reference's.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_2505_10168_b200 import configs as C


@dataclass
class Case:
    name: str
    L: float
    tT: float
    n_el: int
    n_t: int
    k: np.ndarray
    c: np.ndarray
    chi: np.ndarray | None
    mat: tuple | None
    method: str
    strategy: int
    n_levels: int
    min_elements: int = 0
    adjoint: bool = False
    nu: int = 1
    tol: float = 1e-10
    max_cycles: int = 100
    source_kind: int = 0
    source_params: tuple = (1.0,)
    rhs: str = "load"
    dirs: np.ndarray | None = None
    extra: dict = field(default_factory=dict)

    @property
    def reassembly(self) -> int:
        return {"K": 0, "D": 1, "R": 2, "P": 3}[self.method[1]]

    @property
    def n_dofs(self) -> int:
        return (self.n_el + 1) * (self.n_t + 1)

    def plan(self, port):
        if self.dirs is None:
            self.dirs, _ = port.plan(self.L, self.tT, self.n_el, self.n_t, self.k, self.c, self.n_levels,
                                     strategy=self.strategy, reassembly=self.reassembly,
                                     min_elements=self.min_elements, chi=self.chi, mat=self.mat)
        return self.dirs

    def rhs_vector(self, port):
        if self.rhs == "adjoint_uniform":
            return C.adjoint_uniform_rhs(self.n_el, self.n_t, self.L, self.tT)
        return port.load_vector(self.L, self.tT, self.n_el, self.n_t, self.source_kind,
                                self.source_params)


def _from_cfg(name, cfg, **kw) -> Case:
    c = Case(name, cfg.L, cfg.t_T, cfg.n_el, cfg.n_t, cfg.k, cfg.c, cfg.chi, cfg.mat, cfg.method,
             cfg.strategy, cfg.n_levels, cfg.min_elements, cfg.adjoint, cfg.nu, cfg.tol,
             cfg.max_cycles, cfg.source_kind, cfg.source_params, cfg.rhs)
    for k_, v in kw.items():
        setattr(c, k_, v)
    return c


def _uniform(name, n_el, n_t, nl, strategy=C.PLAN_UNIFORM, method="CK", **kw) -> Case:
    return Case(name, 1.0, 1.0, n_el, n_t, np.ones(n_el), np.ones(n_el), None, None, method,
                strategy, nl, source_kind=3, source_params=(), **kw)


def case(name: str) -> Case:
    if name == "cfg0":  # BASELINE config 0 exactly: reference-default two-grid, V(1,1)
        return _from_cfg(name, C.cfg0(), n_levels=2)
    if name == "cfg0_deep":
        return _from_cfg(name, C.cfg0(), n_levels=10, nu=2)
    if name == "cfg1_mini":
        return _from_cfg(name, C.cfg1(n_el=128, n_t=256), n_levels=8, nu=5)
    if name == "cfg2_mini":
        return _from_cfg(name, C.cfg2(n_el=256, n_t=512, min_elements=16), n_levels=9, nu=5)
    if name == "cfg3_mini":
        return _from_cfg(name, C.cfg3(n_el=256, n_t=512, min_elements=16), n_levels=9, nu=5)
    if name == "cfg1_mini_adj":
        return _from_cfg(name, C.cfg1(n_el=128, n_t=256), n_levels=8, nu=5, adjoint=True)
    if name == "cfgD":  # design-averaging reassembly
        cfg = C.cfg1(n_el=128, n_t=256)
        cc = _from_cfg(name, cfg, n_levels=6, nu=5)
        cc.method = "CD"
        return cc
    if name == "cfgK_contrast":
        return _from_cfg(name, C.cfg1(n_el=128, n_t=256), n_levels=6, nu=5, method="CK")
    if name == "time_first":  # proj/tests/test_multigrid.cpp:77-94 situation
        return _uniform(name, 4, 256, 4, nu=5)
    if name == "space_first":  # proj/tests/test_multigrid.cpp:55-75 situation
        return _uniform(name, 32, 32, 4, nu=5)
    if name == "single_level":  # proj/tests/test_multigrid.cpp:96-107
        return _uniform(name, 8, 8, 1, nu=5)
    if name == "tiny":  # one element, the hand-computed march (test_assembly.cpp:133-144)
        return Case(name, 1.0, 3.0, 1, 3, np.ones(1), np.ones(1), None, None, "CK", C.PLAN_UNIFORM,
                    1, source_kind=0, source_params=(1.0,), nu=1)
    if name == "wide_short":  # n_el > 256 exercises multi-tile node blocks; n_t not a tile multiple
        cc = _from_cfg(name, C.cfg2(n_el=1024, n_t=30, min_elements=0), n_levels=4, nu=2)
        cc.strategy = C.PLAN_CONTRAST
        return cc
    if name == "cfg4_mini":
        return _from_cfg(name, C.cfg4(n_el=256, n_t=1024), n_levels=8, nu=5)
    if name in ("wide_coarsest", "wide_coarsest_adj"):  # 64 x 1024 coarsest: the parallel-in-time march
        cc = _from_cfg(name, C.cfg4(n_el=256, n_t=1024), n_levels=3, nu=5,
                       adjoint=name.endswith("_adj"))
        cc.dirs = np.asarray([0, 0], np.int32)
        return cc
    if name.startswith("fixedw_"):  # fixedw_<n_el>[_adj]: see FIXEDW_CASES
        parts = name.split("_")
        ne, adjoint = int(parts[1]), parts[-1] == "adj"
        dirs = [0, 0, 1] if ne <= 4096 else [0, 0]
        cc = _from_cfg(name, C.cfg1(n_el=ne, n_t=48 if ne <= 4096 else 24), n_levels=len(dirs) + 1,
                       nu=1, adjoint=adjoint, method="CR")
        cc.dirs = np.asarray(dirs, np.int32)
        cc.max_cycles = 6
        return cc
    if name.startswith("edge_"):  # edge_<x|t>_<n_el>[_adj]: see EDGE_CASES
        parts = name.split("_")
        ne, adjoint = int(parts[2]), parts[-1] == "adj"
        cc = _from_cfg(name, C.cfg2(n_el=ne, n_t=48, min_elements=0), n_levels=2, nu=2, adjoint=adjoint,
                       method="CK")
        cc.dirs = np.asarray([0 if parts[1] == "x" else 1], np.int32)
        cc.max_cycles = 20
        return cc
    if name in GENERAL:
        kind, ne, nt, method, dirs, adjoint, nu = GENERAL[name]
        if kind == "cfg1":
            cc = _from_cfg(name, C.cfg1(n_el=ne, n_t=nt), n_levels=len(dirs) + 1, nu=nu, method=method,
                           adjoint=adjoint)
        else:
            cc = _uniform(name, ne, nt, len(dirs) + 1, method=method, nu=nu, adjoint=adjoint)
        cc.dirs = np.asarray(dirs, np.int32)
        cc.max_cycles = 40
        return cc
    raise KeyError(name)


# General coarse discretisations: Galerkin (P) coarse
# operators, bilinear temporal transfers (B*), combined space-time steps (2 =
# FullST).  Explicit paths (the planners never emit FullST).  Outcomes under the
# reference: converged (gen_bk, gen_br_deep, gen_cp_x4), diverged (gen_bp_div),
# the rest reach max_cycles = 40.
GENERAL = {
    # name: (inputs, n_el, n_t, method, dirs, adjoint, nu)
    "gen_cp": ("cfg1", 32, 64, "CP", [0, 1, 0], False, 2),
    "gen_bp_div": ("cfg1", 32, 64, "BP", [1, 0, 1], False, 2),
    "gen_cp_xt_adj": ("cfg1", 32, 64, "CP", [2, 0], True, 2),
    "gen_bk": ("cfg1", 32, 64, "BK", [1, 1, 0], False, 2),
    "gen_br_adj": ("cfg1", 32, 64, "BR", [0, 1, 1], True, 2),
    "gen_ck_xt": ("cfg1", 32, 64, "CK", [2, 2], False, 1),
    "gen_bd": ("cfg1", 32, 64, "BD", [0, 1], False, 2),
    "gen_br_deep": ("uniform", 32, 64, "BR", [0, 0, 1, 0, 1], False, 3),
    "gen_cp_x4": ("uniform", 128, 128, "CP", [0, 0, 0, 0], False, 1),
    "gen_bp_uni": ("uniform", 32, 64, "BP", [1, 0, 1], False, 2),
    # bilinear transfers above a rediscretised 64 x 64 coarsest level: the parallel-in-time march
    "gen_br_wide": ("cfg1", 64, 256, "BR", [1, 1], False, 2),
    "gen_bd_adj": ("cfg1", 32, 64, "BD", [0, 1, 1], True, 2),
    "gen_cp_deep_adj": ("uniform", 64, 128, "CP", [0, 1, 0, 1], True, 1),
}
GENERAL_CASES = list(GENERAL)


# Widths that put node n_el on every lane class of a row's last warp (warps advance 28 or
# 30 nodes, 26 in the fused down-pass) and make the first warp also the last: the edge-warp
# tile bodies (csrc/stmg_kernels.cu edge_lane / row_tile).  48 time steps give interior
# 8-level time tiles; x steps need an even n_el, odd widths take the causal t step.
EDGE_CASES = ([f"edge_x_{ne}" + ("_adj" if k % 2 else "") for k, ne in
               enumerate([2, 4, 6, 26, 28, 30, 32, 54, 56, 58, 60, 62, 84, 86, 88, 90])] +
              [f"edge_t_{ne}" + ("" if k % 2 else "_adj") for k, ne in
               enumerate([2, 3, 5, 27, 29, 30, 31, 33, 55, 57, 59, 61, 85, 87, 89, 91])])

# Level widths with compile-time instantiations of the x-step kernels (csrc/stmg_kernels.cu
# dispatch_width: 16385, 8193, 4097, 2049 nodes): short grids of those widths, run with the
# large-level tiling (tiles = 8) by the kernel tests.
FIXEDW_CASES = ["fixedw_4096", "fixedw_4096_adj", "fixedw_16384", "fixedw_16384_adj"]

SMALL_CASES = ["cfg0", "cfg0_deep", "cfg1_mini", "cfg1_mini_adj", "cfg2_mini", "cfg3_mini", "cfgD",
               "cfgK_contrast", "time_first", "space_first", "single_level", "tiny", "wide_short",
               "cfg4_mini", "wide_coarsest", "wide_coarsest_adj"]
