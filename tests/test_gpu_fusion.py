"""GPU parity of the V-cycle fusions (stmg_hierarchy_set_fusion, stmg_level_fused).

* Virtual zero iterates: a coarse level's first sweep from zero, S(0), is
  recomputed from f by the kernels that read it (first pre-smoothing launch;
  for nu = 1 the residual restriction and the fused prolong-sweep).
* Fine down-pass (nu = 1): level 0's residual norm, pre-smoothing sweep and
  residual restriction in one pass.

Each fused kernel form is checked bit for bit against the oracle's composition
of the reference's separate steps (proj/src/multigrid.cpp:184-208; kernels
proj/src/kernels/kernels.cpp:62-73), and whole solves with every fusion on are
bit-identical to solves with every fusion off.
"""
import numpy as np
import pytest

from tests._cases import EDGE_CASES, FIXEDW_CASES, SMALL_CASES, case
from tests.test_gpu_parity import bits, check_solve, gpu_hier, port_hier, special_values

pytestmark = pytest.mark.gpu

KERNEL_CASES = ["cfg0_deep", "cfg1_mini", "cfg1_mini_adj", "cfg2_mini", "cfg3_mini", "cfgD", "time_first",
                "space_first", "wide_short", "cfg4_mini", "wide_coarsest_adj"]
SOLVE_CASES = [c for c in SMALL_CASES if c not in ("single_level",)] + ["gen_br_deep", "gen_ck_xt", "gen_bd_adj"]


@pytest.fixture(scope="module")
def torch():
    import torch as _t

    assert _t.cuda.is_available(), "GPU tests need CUDA (no CPU fallback exists)"
    return _t


@pytest.fixture(scope="module")
def S(torch):
    from paper_2505_10168_b200 import stmg

    return stmg


@pytest.mark.parametrize("tiles", [0, 8])
@pytest.mark.parametrize("omega", [0.5, 0.6])
@pytest.mark.parametrize("name", KERNEL_CASES + EDGE_CASES + FIXEDW_CASES)
def test_virtual_zero_kernels_bitwise(torch, S, port, name, omega, tiles):
    """tiles = 8 forces the large-level tiling (8-level tiles; 16-level tiles for the
    x-step restriction of a virtual zero iterate) onto every level."""
    cs = case(name)
    h = gpu_hier(S, cs, port)
    if tiles:
        h.set_tiling(small_dofs=1, tiny_dofs=1)
    hp = port_hier(port, cs)
    rng = np.random.default_rng(5)
    dev = torch.device("cuda:0")
    for l in range(h.n_levels() - 1):
        n = hp.ndofs(l)
        f = special_values(rng, n)
        ft = torch.from_numpy(f).to(dev)
        y = torch.empty_like(ft)
        x1 = hp.sweeps(l, f, np.zeros(n), 1, omega)  # S(0)
        h.fused_kernel(l, S.LevelHierarchy.FUSED_ZERO_SWEEP, ft, y=y, omega=omega)
        assert np.array_equal(bits(y), bits(hp.sweeps(l, f, x1, 1, omega))), (l, "sweep")
        h.fused_kernel(l, S.LevelHierarchy.FUSED_ZERO_PAIR, ft, y=y, omega=omega)
        assert np.array_equal(bits(y), bits(hp.sweeps(l, f, x1, 2, omega))), (l, "pair")
        fc = torch.empty(hp.ndofs(l + 1), dtype=torch.float64, device=dev)
        h.fused_kernel(l, S.LevelHierarchy.FUSED_ZERO_RESTRICT, ft, fc=fc, omega=omega)
        assert np.array_equal(bits(fc), bits(hp.restrict(l, hp.residual(l, f, x1)))), (l, "restrict")
        xc = special_values(rng, hp.ndofs(l + 1))
        h.fused_kernel(l, S.LevelHierarchy.FUSED_ZERO_PROLONG_SWEEP, ft, xc=torch.from_numpy(xc).to(dev), y=y,
                       omega=omega)
        want = hp.sweeps(l, f, hp.prolong_add(l, xc, x1), 1, omega)
        assert np.array_equal(bits(y), bits(want)), (l, "prolong_sweep")
        x = special_values(rng, n)
        h.fused_kernel(l, S.LevelHierarchy.FUSED_PROLONG_SWEEP, ft, x=torch.from_numpy(x).to(dev),
                       xc=torch.from_numpy(xc).to(dev), y=y, omega=omega)
        want = hp.sweeps(l, f, hp.prolong_add(l, xc, x), 1, omega)
        assert np.array_equal(bits(y), bits(want)), (l, "stored prolong_sweep")


@pytest.mark.parametrize("nu", [1, 2, 3])
@pytest.mark.parametrize("name", SOLVE_CASES)
def test_fused_solves_bitwise(torch, S, port, name, nu):
    """Every fusion combination (all on, off, each alone) gives the same cycles,
    history (to the norm's summation order) and iterate bit for bit; and parity
    with the oracle's solve."""
    cs = case(name)
    b = cs.rhs_vector(port)
    opts = S.SolveOptions(nu=nu, tol=cs.tol, max_cycles=min(cs.max_cycles, 40))
    h = gpu_hier(S, cs, port)
    out = {}
    H = S.LevelHierarchy
    combos = (H.FUSE_ALL, 0, H.FUSE_VIRTUAL_ZERO, H.FUSE_FINE_DOWN, H.FUSE_FINE_UP,
              H.FUSE_FINE_UP | H.FUSE_VIRTUAL_ZERO, H.FUSE_FINE_DOWN | H.FUSE_VIRTUAL_ZERO)
    for flags in combos:
        h.set_fusion(flags)
        u = np.zeros_like(b)
        out[flags] = (S.mg_solve(h, b, u, opts), u)
        if flags == H.FUSE_FINE_UP | H.FUSE_VIRTUAL_ZERO:  # repeated and warm-started solves, device vectors
            ut = torch.from_numpy(u).cuda()
            bt = torch.from_numpy(b).cuda()
            r_w = S.mg_solve(h, bt, ut, opts)
            u_w = u.copy()
            r_w2 = S.mg_solve(h, b, u_w, opts)
            assert r_w.history == r_w2.history and np.array_equal(bits(ut), bits(u_w))
    r0, u0 = out[H.FUSE_ALL]
    for flags in combos[1:]:
        r1, u1 = out[flags]
        assert r1.cycles == r0.cycles and r1.status == r0.status, flags
        # the iterates are bitwise; the fine down-pass sums the norm over other blocks
        np.testing.assert_allclose(r1.history, r0.history, rtol=1e-13, atol=0)
        assert np.array_equal(bits(u1), bits(u0)), flags
    if name.startswith("gen_"):
        return  # the general discretisations are pinned to the reference itself (test_gpu_general.py)
    hp = port_hier(port, cs)
    u_p, rep_p = hp.solve(b, nu=nu, tol=cs.tol, max_cycles=min(cs.max_cycles, 40))
    check_solve(r0, u0, rep_p, u_p)


@pytest.mark.parametrize("tiles", [8, 4, 2])
@pytest.mark.parametrize("name", KERNEL_CASES + ["cfg0", "tiny"])
def test_fine_down_kernel_bitwise(torch, S, port, name, tiles):
    """k_down: ||f - J x||^2, y = S(x) and f_c = R (f - J y) in one pass, against
    the oracle's separate residual, sweep and restriction; every level with a
    per-node transfer, every time-tile depth."""
    cs = case(name)
    h = gpu_hier(S, cs, port)
    if h.n_levels() < 2:
        pytest.skip("single-level hierarchy")
    h.set_tiling(small_dofs=10 ** 15 if tiles <= 4 else 1, tiny_dofs=10 ** 15 if tiles == 2 else 1)
    hp = port_hier(port, cs)
    rng = np.random.default_rng(41)
    dev = torch.device("cuda:0")
    for l in range(h.n_levels() - 1):
        n = hp.ndofs(l)
        x, f = special_values(rng, n), special_values(rng, n)
        xt, ft = torch.from_numpy(x).to(dev), torch.from_numpy(f).to(dev)
        y = torch.full_like(xt, np.nan)
        fc = torch.full((hp.ndofs(l + 1),), np.nan, dtype=torch.float64, device=dev)
        nrm2 = h.fused_kernel(l, S.LevelHierarchy.FUSED_FINE_DOWN, ft, x=xt, y=y, fc=fc)
        y_want = hp.sweeps(l, f, x, 1)
        assert np.array_equal(bits(y), bits(y_want)), (l, "sweep")
        assert np.array_equal(bits(fc), bits(hp.restrict(l, hp.residual(l, f, y_want)))), (l, "restrict")
        r = hp.residual(l, f, x)
        assert abs(nrm2 - float(np.dot(r, r))) <= 1e-13 * float(np.dot(r, r)), (l, "norm")


@pytest.mark.parametrize("tiles", [8, 4, 2])
@pytest.mark.parametrize("name", KERNEL_CASES + ["cfg0", "tiny"] + EDGE_CASES + FIXEDW_CASES)
def test_fine_up_kernel_bitwise(torch, S, port, name, tiles):
    """k_up: u = S(x + P x_c), w = S(u) and ||f - J u||^2 in one pass, against the
    oracle's separate prolongation, sweeps and residual; every level with a per-node
    transfer, every time-tile depth."""
    cs = case(name)
    h = gpu_hier(S, cs, port)
    if h.n_levels() < 2:
        pytest.skip("single-level hierarchy")
    h.set_tiling(small_dofs=10 ** 15 if tiles <= 4 else 1, tiny_dofs=10 ** 15 if tiles == 2 else 1)
    hp = port_hier(port, cs)
    rng = np.random.default_rng(43)
    dev = torch.device("cuda:0")
    for l in range(h.n_levels() - 1):
        n, nc = hp.ndofs(l), hp.ndofs(l + 1)
        x, f, xc = special_values(rng, n), special_values(rng, n), special_values(rng, nc)
        xt, ft, xct = torch.from_numpy(x).to(dev), torch.from_numpy(f).to(dev), torch.from_numpy(xc).to(dev)
        u = torch.full_like(xt, np.nan)
        w = torch.full_like(xt, np.nan)
        nrm2 = h.fused_kernel(l, S.LevelHierarchy.FUSED_FINE_UP, ft, x=xt, xc=xct, y=u, fc=w)
        u_want = hp.sweeps(l, f, hp.prolong_add(l, xc, x), 1)
        assert np.array_equal(bits(u), bits(u_want)), (l, "post-sweep")
        assert np.array_equal(bits(w), bits(hp.sweeps(l, f, u_want, 1))), (l, "speculative sweep")
        r = hp.residual(l, f, u_want)
        assert abs(nrm2 - float(np.dot(r, r))) <= 1e-13 * float(np.dot(r, r)), (l, "norm")


def test_shared_workspace_alternating_forward_and_adjoint_solves(torch, S, port):
    """A hierarchy and its transpose share the workspace (the third level-0 buffer and the
    pointer table of the fine up-pass included): alternating nu = 1 solves on both, flagged
    and in/out, give what fresh hierarchies give, bit for bit."""
    cs = case("cfg1_mini")
    b = cs.rhs_vector(port)
    b2 = b[::-1].copy()
    opts = S.SolveOptions(nu=1, tol=cs.tol, max_cycles=12)

    def fresh(adj, rhs):
        h = gpu_hier(S, cs, port)
        if adj:
            h = S.transposed_hierarchy(h)
        u = np.zeros_like(rhs)
        return S.mg_solve(h, rhs, u, opts), u

    want = {(adj, k): fresh(adj, rhs) for adj in (False, True) for k, rhs in enumerate((b, b2))}
    h = gpu_hier(S, cs, port)
    ht = S.transposed_hierarchy(h)
    for rnd in range(2):
        for adj, hh in ((False, h), (True, ht)):
            for k, rhs in enumerate((b, b2)):
                u = np.full_like(rhs, np.nan) if rnd else np.zeros_like(rhs)
                r = S.mg_solve(hh, rhs, u, opts, zero_guess=bool(rnd))
                rw, uw = want[(adj, k)]
                assert r.cycles == rw.cycles and r.status == rw.status and r.history[1:] == rw.history[1:]
                assert np.array_equal(bits(u), bits(uw)), (rnd, adj, k)


@pytest.mark.parametrize("zero_guess", [False, True])
@pytest.mark.parametrize("name", FIXEDW_CASES)
def test_fixed_width_kernels_in_the_solve(torch, S, port, name, zero_guess):
    """Levels of 16385 / 8193 / 4097 / 2049 nodes under the large-level tiling run the x-step
    kernels instantiated for their width (dispatch_width); the same solve under the small-level
    tiling runs the run-time-width kernels.  Same iterate bit for bit, same history to the
    norm's summation order; the oracle's solve agrees to the rounding of the (very wide)
    coarsest level's exact solve."""
    cs = case(name)
    b = cs.rhs_vector(port)
    opts = S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    out = []
    for big in (True, False):
        h = gpu_hier(S, cs, port)
        if big:
            h.set_tiling(small_dofs=1, tiny_dofs=1)
        u = np.zeros_like(b)
        out.append((S.mg_solve(h, b, u, opts, zero_guess=zero_guess), u))
    (r0, u0), (r1, u1) = out
    assert r0.cycles == r1.cycles and r0.status == r1.status
    np.testing.assert_allclose(r0.history, r1.history, rtol=1e-13, atol=0)
    assert np.array_equal(bits(u0), bits(u1))
    if cs.n_el > 4096:
        return  # a 4097-node coarsest level: the two exact coarsest solvers differ by cond x eps ~ 1e-4 there
    hp = port_hier(port, cs)
    u_p, rep_p = hp.solve(b, nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    assert r0.cycles == rep_p.cycles and int(r0.status) == rep_p.status
    np.testing.assert_allclose(r0.history, rep_p.history, rtol=1e-7, atol=0)
    assert np.max(np.abs(u0 - u_p)) <= 1e-7 * np.max(np.abs(u_p))
