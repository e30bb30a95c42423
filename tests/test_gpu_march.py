"""GPU parity of the streaming-march chassis (csrc/stmg_march.cuh,
stmg_hierarchy_set_march): warp-private cp.async rings instead of register-staged
tiles for the single sweep, the norm pass, the fused prolong-sweep and the residual
restriction, with stored and virtual-zero iterates.

Every kernel form is forced onto the chassis on EVERY level of the small cases
(set_march(1): levels of a few nodes, ragged strips, one-row chunks) and checked
bit for bit against the oracle's composition of the reference's separate steps
(proj/src/multigrid.cpp:184-208; kernels proj/src/kernels/kernels.cpp:62-73);
whole solves on the chassis are bit-identical to solves on the register-staged
kernels.
"""
import numpy as np
import pytest

from tests._cases import SMALL_CASES, case
from tests.test_gpu_parity import bits, check_solve, gpu_hier, port_hier, special_values

pytestmark = pytest.mark.gpu

KERNEL_CASES = ["cfg0", "tiny", "cfg0_deep", "cfg1_mini", "cfg1_mini_adj", "cfg2_mini", "cfg3_mini", "cfgD",
                "time_first", "space_first", "wide_short", "cfg4_mini", "wide_coarsest_adj"]
SOLVE_CASES = [c for c in SMALL_CASES if c not in ("single_level",)]


@pytest.fixture(scope="module")
def torch():
    import torch as _t

    assert _t.cuda.is_available(), "GPU tests need CUDA (no CPU fallback exists)"
    return _t


@pytest.fixture(scope="module")
def S(torch):
    from paper_2505_10168_b200 import stmg

    return stmg


def extreme_values(rng, n):
    """special_values plus subnormals, values near DBL_MIN and huge values (whose
    squares overflow; products with the coefficients stay finite, so no NaN payloads)."""
    v = special_values(rng, n)
    idx = rng.choice(n, size=max(1, n // 24), replace=False)
    v[idx[0::3]] = 5e-324 * rng.integers(1, 1000, size=idx[0::3].size)
    v[idx[1::3]] = 1e150 * rng.standard_normal(idx[1::3].size)
    v[idx[2::3]] = 2.3e-308 * rng.standard_normal(idx[2::3].size)
    return v


@pytest.mark.parametrize("omega", [0.5, 0.6])
@pytest.mark.parametrize("name", KERNEL_CASES)
def test_march_kernels_bitwise(torch, S, port, name, omega):
    cs = case(name)
    h = gpu_hier(S, cs, port)
    h.set_march(1)
    hp = port_hier(port, cs)
    H = S.LevelHierarchy
    rng = np.random.default_rng(23)
    dev = torch.device("cuda:0")
    T = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
    for l in range(h.n_levels() - 1):
        n, nc = hp.ndofs(l), hp.ndofs(l + 1)
        gen = extreme_values if l % 2 else special_values
        x, f, xc = gen(rng, n), gen(rng, n), gen(rng, nc)
        xt, ft, xct = T(x), T(f), T(xc)
        nan = lambda k: torch.full((k,), np.nan, dtype=torch.float64, device=dev)  # noqa: E731
        # single sweep (stored iterate)
        y = nan(n)
        h.sweep_kernels(l, ft, xt, y, 1, False, omega)
        torch.cuda.synchronize()
        y_want = hp.sweeps(l, f, x, 1, omega)
        assert np.array_equal(bits(y), bits(y_want)), (l, "sweep")
        # norm pass: ||f - A x||^2 and the sweep
        y = nan(n)
        nrm2 = h.fused_kernel(l, H.FUSED_NORM_SWEEP, ft, x=xt, y=y, omega=omega)
        assert np.array_equal(bits(y), bits(y_want)), (l, "norm sweep")
        r = hp.residual(l, f, x)
        with np.errstate(over="ignore", invalid="ignore"):
            want2 = float(np.dot(r, r))
        if np.isfinite(want2):
            assert abs(nrm2 - want2) <= 1e-12 * want2, (l, "norm")
        # residual restriction (stored iterate)
        fc = nan(nc)
        h.restrict_residual(l, ft, xt, fc)
        assert np.array_equal(bits(fc), bits(hp.restrict(l, r))), (l, "restrict")
        # stored iterate + P xc, then the sweep
        y = nan(n)
        h.fused_kernel(l, H.FUSED_PROLONG_SWEEP, ft, x=xt, xc=xct, y=y, omega=omega)
        assert np.array_equal(bits(y), bits(hp.sweeps(l, f, hp.prolong_add(l, xc, x), 1, omega))), (l, "prolong")
        # virtual zero iterate S(0)
        x1 = hp.sweeps(l, f, np.zeros(n), 1, omega)
        y = nan(n)
        h.fused_kernel(l, H.FUSED_ZERO_SWEEP, ft, y=y, omega=omega)
        assert np.array_equal(bits(y), bits(hp.sweeps(l, f, x1, 1, omega))), (l, "zero sweep")
        fc = nan(nc)
        h.fused_kernel(l, H.FUSED_ZERO_RESTRICT, ft, fc=fc, omega=omega)
        assert np.array_equal(bits(fc), bits(hp.restrict(l, hp.residual(l, f, x1)))), (l, "zero restrict")
        y = nan(n)
        h.fused_kernel(l, H.FUSED_ZERO_PROLONG_SWEEP, ft, xc=xct, y=y, omega=omega)
        assert np.array_equal(bits(y), bits(hp.sweeps(l, f, hp.prolong_add(l, xc, x1), 1, omega))), (l, "zero prolong")


@pytest.mark.parametrize("nu", [1, 2, 3])
@pytest.mark.parametrize("name", SOLVE_CASES)
def test_march_solves_bitwise(torch, S, port, name, nu):
    """Solves with every level on the chassis: the register-staged solve's cycles,
    status and iterate bit for bit (histories to the norm's summation order), and
    parity with the oracle."""
    cs = case(name)
    b = cs.rhs_vector(port)
    opts = S.SolveOptions(nu=nu, tol=cs.tol, max_cycles=min(cs.max_cycles, 40))
    h = gpu_hier(S, cs, port)
    H = S.LevelHierarchy
    out = {}
    for march, flags in ((0, H.FUSE_DEFAULT), (1, H.FUSE_DEFAULT), (1, 0)):
        h.set_march(1 if march else 10 ** 18)
        h.set_fusion(flags)
        u = np.zeros_like(b)
        out[(march, flags)] = (S.mg_solve(h, b, u, opts), u)
    r0, u0 = out[(0, H.FUSE_DEFAULT)]
    for key in ((1, H.FUSE_DEFAULT), (1, 0)):
        r1, u1 = out[key]
        assert r1.cycles == r0.cycles and r1.status == r0.status, key
        np.testing.assert_allclose(r1.history, r0.history, rtol=1e-13, atol=0)
        assert np.array_equal(bits(u1), bits(u0)), key
    hp = port_hier(port, cs)
    u_p, rep_p = hp.solve(b, nu=nu, tol=cs.tol, max_cycles=min(cs.max_cycles, 40))
    check_solve(out[(1, H.FUSE_DEFAULT)][0], out[(1, H.FUSE_DEFAULT)][1], rep_p, u_p)
