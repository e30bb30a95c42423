"""BASELINE.json configs as concrete, seeded synthetic inputs.

All inputs are produced in the reference's orientation: the Dirichlet node is
x = 0 (``dof_is_masked``: ``n == 0 || i == 0``, proj/src/assembly.cpp:85-88)
and x = L is insulated.  BASELINE.json states the configs the other way round
(insulated at x = 0, T = 0 at x = 1), so designs and sources are mirrored,
x' = L - x, element e' = N_el - 1 - e.

Randomness: ``std::mt19937_64(seed)``; Bernoulli(1/2) bit = ``rng() >> 63``;
Uniform[0,1) = ``(rng() >> 11) * 2**-53``.  No
``std::*_distribution`` is involved, so the streams are portable.

Source kinds (the ``kind`` argument of load_vector / stmg_load_vector):
  0  q = p0                                      (uniform)
  1  q = p0 * [L - x < p1]                       (mirrored box)
  2  q = (1 + p0 sin(2 pi p1 t)) * [L - x < p2]  (mirrored, time-modulated box)
  3  q = heat_load_value(x, t, L, t_T)           (the reference's Eq.-19 load,
                                                  proj/src/assembly.cpp:59-63)
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# Numbering shared with include/stmg_b200.h
DIR_X, DIR_T, DIR_XT = 0, 1, 2
REASM_K, REASM_D, REASM_R, REASM_P = 0, 1, 2, 3
PLAN_UNIFORM, PLAN_CONTRAST, PLAN_RESOLUTION, PLAN_DESIGN_INDEPENDENT = 0, 1, 2, 3

_M64 = (1 << 64) - 1


class MT19937_64:
    """Bit-exact std::mt19937_64."""

    N, M = 312, 156
    A = 0xB5026F5AA96619E9
    UPPER, LOWER = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int = 5489):
        mt = [0] * self.N
        mt[0] = seed & _M64
        for i in range(1, self.N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self.mt = mt
        self.idx = self.N

    def _twist(self):
        mt, N, M = self.mt, self.N, self.M
        for i in range(N):
            x = (mt[i] & self.UPPER) | (mt[(i + 1) % N] & self.LOWER)
            xa = x >> 1
            if x & 1:
                xa ^= self.A
            mt[i] = mt[(i + M) % N] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= self.N:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000 & _M64
        y ^= (y << 37) & 0xFFF7EEE000000000 & _M64
        y ^= y >> 43
        return y & _M64


def bernoulli_half(rng: MT19937_64) -> float:
    return float(rng() >> 63)


def uniform01(rng: MT19937_64) -> float:
    return float(rng() >> 11) * 2.0 ** -53


def simp(chi: np.ndarray, mat) -> tuple[np.ndarray, np.ndarray]:
    """apply_design (proj/src/materials.cpp:27-32, 44-50), elementwise with libm pow."""
    import math

    k_ins, k_con, c_ins, c_con, p_k, p_c = mat
    chi = np.asarray(chi, np.float64)
    if np.any(~((chi >= 0.0) & (chi <= 1.0))):
        raise ValueError("volume fraction outside [0, 1]")
    k = np.array([k_ins + (k_con - k_ins) * math.pow(v, p_k) for v in chi.tolist()])
    c = np.array([c_ins + (c_con - c_ins) * math.pow(v, p_c) for v in chi.tolist()])
    return k, c


@dataclass
class Config:
    name: str
    L: float
    t_T: float
    n_el: int
    n_t: int
    chi: np.ndarray | None
    mat: tuple | None
    k: np.ndarray
    c: np.ndarray
    source_kind: int
    source_params: tuple
    method: str  # two-letter reference name ("CR", "CK")
    strategy: int
    n_levels: int
    min_elements: int = 0
    lambda_crit: float = 0.25
    nu: int = 1
    omega: float = 0.5
    tol: float = 1e-10
    div_tol: float = 1e9
    max_cycles: int = 100
    adjoint: bool = False
    rhs: str = "load"  # "load" or "adjoint_uniform" (c = dx*dt at unmasked DOFs)
    notes: dict = field(default_factory=dict)

    @property
    def n_dofs(self) -> int:
        return (self.n_el + 1) * (self.n_t + 1)

    @property
    def reassembly(self) -> int:
        return {"K": REASM_K, "D": REASM_D, "R": REASM_R, "P": REASM_P}[self.method[1]]


def _mirror(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a[::-1])


def cfg0(n_el=128, n_t=128) -> Config:
    k = np.ones(n_el)
    c = np.ones(n_el)
    # "default coarsening": the reference's PlanRequest default, two levels (strategy.hpp:77)
    return Config("cfg0", 1.0, 1.0, n_el, n_t, None, None, k, c, 0, (1.0,), "CK", PLAN_CONTRAST,
                  n_levels=2, nu=1)


def cfg1(n_el=1024, n_t=4096, seed=1, n_levels=10, nu=5) -> Config:
    rng = MT19937_64(seed)
    n_blocks = n_el // 16
    bits = [bernoulli_half(rng) for _ in range(n_blocks)]
    chi = np.repeat(np.array(bits), 16)[:n_el]
    chi = _mirror(chi)
    mat = (1e-3, 1.0, 1.0, 1.0, 3.0, 2.0)
    k, c = simp(chi, mat)
    return Config("cfg1", 1.0, 1.0, n_el, n_t, chi, mat, k, c, 1, (1.0, 0.1), "CR", PLAN_CONTRAST,
                  n_levels=n_levels, nu=nu)


def cfg1_weak(world: int = 1, **kw) -> Config:
    """Weak-scaled config 1 for the time-slab runs: the horizon grows with the GPU
    count (t_T = world, n_t = 4096 world) so dt, the anisotropy and the planned
    coarsening path stay those of config 1; each GPU owns one 1024 x 4096 slab."""
    c = cfg1(n_t=4096 * world, **kw)
    c.t_T = float(world)
    c.name = f"cfg1-weak{world}"
    return c


def cfg2(n_el=16384, n_t=65536, seed=2, n_levels=18, nu=1, min_elements=256) -> Config:
    rng = MT19937_64(seed)
    u = np.array([uniform01(rng) for _ in range(n_el)])
    chi = _mirror((u >= 0.5).astype(np.float64))
    mat = (1e-4, 1.0, 1.0, 1.0, 3.0, 2.0)
    k, c = simp(chi, mat)
    return Config("cfg2", 1.0, 1.0, n_el, n_t, chi, mat, k, c, 2, (0.5, 8.0, 0.05), "CR",
                  PLAN_RESOLUTION, n_levels=n_levels, nu=nu, min_elements=min_elements)


def cfg3(n_el=16384, n_t=65536, seed=2, n_levels=18, nu=1, min_elements=256) -> Config:
    c2 = cfg2(n_el, n_t, seed, n_levels, nu, min_elements)
    c2.name = "cfg3"
    c2.adjoint = True
    c2.rhs = "adjoint_uniform"
    return c2


def cfg4(n_el=4096, n_t=16384) -> Config:
    chi = np.full(n_el, 0.5)
    mat = (1e-3, 1.0, 1.0, 1.0, 3.0, 2.0)
    k, c = simp(chi, mat)
    # OptimisationOptions defaults (proj/include/stmg/optimisation.hpp:59-75): CR, 6 levels,
    # nu = 20; strategy DesignIndependent as the paper's optimisation study
    return Config("cfg4", 1.0, 1.0, n_el, n_t, chi, mat, k, c, 3, (), "CR",
                  PLAN_DESIGN_INDEPENDENT, n_levels=6, nu=20, tol=1e-8)


def adjoint_uniform_rhs(n_el: int, n_t: int, L: float = 1.0, t_T: float = 1.0) -> np.ndarray:
    """dJ/dT for J = sum over unmasked DOFs of T * dx * dt (cfg3); 0 at masked DOFs."""
    dx, dt = L / n_el, t_T / n_t
    b = np.full((n_t + 1, n_el + 1), dx * dt)
    b[0, :] = 0.0
    b[:, 0] = 0.0
    return b.reshape(-1)


CONFIGS = {"cfg0": cfg0, "cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4}
