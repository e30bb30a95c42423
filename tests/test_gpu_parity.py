"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Bar (BASELINE north_star): bit-identical level kernels; whole solves with the
same V-cycle count and status, per-cycle residual history within
1e-10 relative (+1e-13 absolute floor in units of ||b||, the fp64 cancellation
floor of evaluating b - J u), and fields within 1e-10 relative max-norm.
"""
import numpy as np
import pytest

from tests._cases import EDGE_CASES, FIXEDW_CASES, SMALL_CASES, case

pytestmark = pytest.mark.gpu

HIST_REL, HIST_ABS, FIELD_REL = 1e-10, 1e-13, 1e-10  # see tests/_tol.py


@pytest.fixture(scope="module")
def torch():
    import torch as _t

    assert _t.cuda.is_available(), "GPU tests need CUDA (no CPU fallback exists)"
    return _t


@pytest.fixture(scope="module")
def S(torch):
    from paper_2505_10168_b200 import stmg

    return stmg


def bits(a):
    if hasattr(a, "cpu"):
        a = a.cpu().numpy()
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def gpu_hier(S, cs, port):
    dirs = cs.plan(port)
    g = S.build_fine_grid(cs.L, cs.tT, cs.n_el, cs.n_t)
    g.k, g.c = cs.k, cs.c
    path = S.CoarseningPath([S.CoarseningDirection(int(d)) for d in dirs])
    h = S.build_hierarchy(g, cs.method, path, chi=cs.chi, mat=cs.mat)
    if cs.adjoint:
        h = S.transposed_hierarchy(h)
    return h


def port_hier(port, cs):
    return port.hierarchy(cs.L, cs.tT, cs.n_el, cs.n_t, cs.k, cs.c, cs.plan(port),
                          reassembly=cs.reassembly, adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat)


def special_values(rng, n):
    """Gaussian values salted with exact +0, -0 and powers of two."""
    v = rng.standard_normal(n)
    idx = rng.choice(n, size=max(1, n // 16), replace=False)
    v[idx[0::3]] = 0.0
    v[idx[1::3]] = -0.0
    v[idx[2::3]] = 2.0 ** rng.integers(-20, 20, size=idx[2::3].size)
    return v


@pytest.mark.parametrize("tiles", [0, 8])
@pytest.mark.parametrize("name", SMALL_CASES + EDGE_CASES + FIXEDW_CASES)
def test_level_kernels_bitwise(torch, S, port, name, tiles):
    """tiles = 8 forces the large-level tiling (8-level tiles, 16-level tiles for the
    x-step restrictions) onto every level of the small cases."""
    cs = case(name)
    h = gpu_hier(S, cs, port)
    if tiles:
        h.set_tiling(small_dofs=1, tiny_dofs=1)
    hp = port_hier(port, cs)
    assert h.n_levels() == hp.n_levels
    rng = np.random.default_rng(11)
    dev = torch.device("cuda:0")
    for l in range(h.n_levels()):
        n = hp.ndofs(l)
        x = special_values(rng, n)
        f = special_values(rng, n)
        xt = torch.from_numpy(x).to(dev)
        ft = torch.from_numpy(f).to(dev)
        r = torch.empty_like(xt)
        h.residual(l, ft, xt, r)
        assert np.array_equal(bits(r), bits(hp.residual(l, f, x))), f"residual level {l}"
        xs = xt.clone()
        h.sweeps(l, ft, xs, 3)
        assert np.array_equal(bits(xs), bits(hp.sweeps(l, f, x, 3))), f"sweeps level {l}"
        if l + 1 < h.n_levels():
            nc = hp.ndofs(l + 1)
            fc = torch.empty(nc, dtype=torch.float64, device=dev)
            h.restrict_residual(l, ft, xt, fc)
            want = hp.restrict(l, hp.residual(l, f, x))
            assert np.array_equal(bits(fc), bits(want)), f"restrict_residual level {l}"
            h.restrict(l, r, fc)
            assert np.array_equal(bits(fc), bits(want)), f"restrict level {l}"
            xc = special_values(rng, nc)
            xp = xt.clone()
            h.prolong_add(l, torch.from_numpy(xc).to(dev), xp)
            assert np.array_equal(bits(xp), bits(hp.prolong_add(l, xc, x))), f"prolong level {l}"
    if name.startswith("fixedw_"):
        return  # their coarsest levels are thousands of nodes wide: two exact solvers differ by cond x eps there
    # exact coarsest solve (PCR march vs Thomas march): rounding-level agreement
    nL = hp.ndofs(hp.n_levels - 1)
    f = rng.standard_normal(nL)
    x = torch.zeros(nL, dtype=torch.float64, device=dev)
    h.coarsest_solve(torch.from_numpy(f).to(dev), x)
    want = hp.coarsest(f)
    assert np.max(np.abs(x.cpu().numpy() - want)) <= 1e-12 * np.max(np.abs(want))


def check_solve(rep_g, u_g, rep_p, u_p, floor=HIST_ABS):
    from tests._tol import histories_match

    assert rep_g.cycles == rep_p.cycles
    assert int(rep_g.status) == rep_p.status
    assert histories_match(rep_g.history, rep_p.history, floor), floor
    scale = max(np.max(np.abs(u_p)), 1e-300)
    assert np.max(np.abs(u_g - u_p)) <= FIELD_REL * scale
    assert rep_g.absolute_norms == rep_p.absolute_norms


@pytest.mark.parametrize("name", SMALL_CASES)
def test_solve_parity(torch, S, port, name):
    cs = case(name)
    h = gpu_hier(S, cs, port)
    hp = port_hier(port, cs)
    b = cs.rhs_vector(port)
    u_p, rep_p = hp.solve(b, nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    u = np.zeros_like(b)
    rep = S.mg_solve(h, b, u, S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles))
    check_solve(rep, u, rep_p, u_p)
    # device-resident vectors give bit-identical results to host vectors
    bt = torch.from_numpy(b).cuda()
    ut = torch.zeros_like(bt)
    rep2 = S.mg_solve(h, bt, ut, S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles))
    assert np.array_equal(bits(ut), bits(u))
    assert rep2.history == rep.history


def test_solve_is_deterministic(torch, S, port):
    cs = case("cfg1_mini")
    h = gpu_hier(S, cs, port)
    b = cs.rhs_vector(port)
    outs = []
    for _ in range(2):
        u = np.zeros_like(b)
        rep = S.mg_solve(h, b, u, S.SolveOptions(nu=cs.nu, tol=cs.tol))
        outs.append((u, rep.history))
    assert np.array_equal(bits(outs[0][0]), bits(outs[1][0]))
    assert outs[0][1] == outs[1][1]


@pytest.mark.parametrize("nu", [0, 1, 2])
@pytest.mark.parametrize("name", ["cfg0", "cfg1_mini", "cfg1_mini_adj", "cfg2_mini", "cfg3_mini", "time_first",
                                  "cfgD", "tiny", "single_level"])
def test_zero_guess_flag_equals_a_zeroed_u(torch, S, port, name, nu):
    """stmg_mg_solve_ex with STMG_SOLVE_ZERO_GUESS: u is output only (garbage in, never
    read); host and device vectors give the in/out solve from a zero vector bit for bit.
    The flagged solve opens with one pass over b (first sweep + ||b||^2 = ||r0||^2), so its
    history[0] is exactly 1 as in the reference (the in/out path sums ||r0||^2 and ||b||^2 in
    two different fixed orders: 1 to rounding)."""
    cs = case(name)
    h = gpu_hier(S, cs, port)
    b = cs.rhs_vector(port)
    # nu = 0: the case's own smoothing count; 1: the opening pass also runs cycle 1's level-0
    # restriction (launch_restrict_open); 2: the plain one-pass opening
    opts = S.SolveOptions(nu=nu or cs.nu, tol=cs.tol, max_cycles=min(cs.max_cycles, 30))
    u0 = np.zeros_like(b)
    rep0 = S.mg_solve(h, b, u0, opts)
    u1 = np.full_like(b, np.nan)
    rep1 = S.mg_solve(h, b, u1, opts, zero_guess=True)
    assert np.array_equal(bits(u1), bits(u0)) and rep1.cycles == rep0.cycles and rep1.status == rep0.status
    assert abs(rep0.history[0] - 1.0) <= 1e-15 and abs(rep1.history[0] - 1.0) <= 1e-15
    if h.n_levels() > 1:
        assert rep1.history[0] == 1.0  # one pass gives ||b||^2 and ||r0||^2: exactly 1
    assert rep1.history[1:] == rep0.history[1:]
    for flags in (0, 1, 2, 3, 4, 6, 7):  # every other fusion set, max_cycles 1 and 2
        h.set_fusion(flags)
        for mc in (1, 2):
            o2 = S.SolveOptions(nu=opts.nu, tol=opts.tol, max_cycles=mc)
            ua, ub = np.zeros_like(b), np.full_like(b, np.nan)
            ra = S.mg_solve(h, b, ua, o2)
            rb = S.mg_solve(h, b, ub, o2, zero_guess=True)
            assert np.array_equal(bits(ua), bits(ub)) and ra.cycles == rb.cycles and ra.status == rb.status
            assert ra.history[1:] == rb.history[1:]
    h.set_fusion(S.LevelHierarchy.FUSE_DEFAULT)
    bt = torch.from_numpy(b).cuda()
    ut = torch.full_like(bt, float("nan"))
    rep2 = S.mg_solve(h, bt, ut, opts, zero_guess=True)
    assert np.array_equal(bits(ut), bits(u0)) and rep2.history == rep1.history
    # b = 0: converged before any cycle, u is cleared
    uz = np.full_like(b, np.nan)
    rz = S.mg_solve(h, np.zeros_like(b), uz, opts, zero_guess=True)
    assert rz.cycles == 0 and rz.absolute_norms and not uz.any()
    with pytest.raises(ValueError):
        from paper_2505_10168_b200.stmg import _lib, _check, _ptr  # unknown flag bits are rejected
        import ctypes as C

        hist = np.zeros(opts.max_cycles + 1)
        from paper_2505_10168_b200.stmg import _SolveOpts, _SolveRep

        co = _SolveOpts(int(opts.nu), float(opts.omega), float(opts.tol), float(opts.div_tol), int(opts.max_cycles))
        rep = _SolveRep()
        _check(_lib.stmg_mg_solve_ex(h.handle, _ptr(b), _ptr(u1), C.byref(co), 6, C.byref(rep), hist.ctypes.data,
                                     hist.size))


def test_tiny_hand_values(torch, S, port):
    """proj/tests/test_assembly.cpp:133-144: T = 0.375, 0.46875, 0.4921875."""
    cs = case("tiny")
    h = gpu_hier(S, cs, port)
    b = cs.rhs_vector(port)
    u = np.zeros_like(b)
    rep = S.mg_solve(h, b, u, S.SolveOptions(nu=1, tol=1e-12))
    assert rep.cycles == 1
    np.testing.assert_allclose(u[[3, 5, 7]], [0.375, 0.46875, 0.4921875], rtol=1e-14)
    assert u[0] == 0.0 and u[2] == 0.0


def test_bookkeeping_edge_cases(torch, S, port):
    """proj/tests/test_multigrid.cpp:109-162."""
    cs = case("space_first")
    h = gpu_hier(S, cs, port)
    b = cs.rhs_vector(port)
    u = np.zeros_like(b)
    rep = S.mg_solve(h, b, u, S.SolveOptions(nu=5, tol=1e-9))
    assert rep.history[0] == 1.0
    assert rep.status == S.SolveStatus.Converged and rep.history[-1] < 1e-9
    assert len(rep.history) == rep.cycles + 1
    assert rep.factor == pytest.approx((rep.history[-1] / rep.history[0]) ** (1.0 / rep.cycles))
    assert not rep.absolute_norms
    # warm start from a (much) tighter solution does no work
    u2 = np.zeros_like(b)
    S.mg_solve(h, b, u2, S.SolveOptions(nu=5, tol=1e-14, max_cycles=200))
    rep = S.mg_solve(h, b, u2, S.SolveOptions(nu=5, tol=1e-9))
    assert rep.status == S.SolveStatus.Converged and rep.cycles == 0 and rep.factor == 1.0
    assert len(rep.history) == 1
    # zero right-hand side: absolute norms, converged at once
    z = np.zeros_like(b)
    uz = np.zeros_like(b)
    rep = S.mg_solve(h, z, uz, S.SolveOptions())
    assert rep.absolute_norms and rep.cycles == 0 and rep.status == S.SolveStatus.Converged
    # invalid options / sizes raise ValueError (std::invalid_argument)
    for bad in (S.SolveOptions(nu=-1), S.SolveOptions(tol=0.0), S.SolveOptions(div_tol=1e-12)):
        with pytest.raises(ValueError):
            S.mg_solve(h, b, np.zeros_like(b), bad)
    with pytest.raises(ValueError):
        S.mg_solve(h, b, np.zeros(3), S.SolveOptions())


def test_one_cycle_is_linear(torch, S, port):
    """proj/tests/test_multigrid.cpp:164-194 / acceptance_main.cpp:513-550."""
    cs = case("cfg1_mini")
    h = gpu_hier(S, cs, port)
    b1 = cs.rhs_vector(port)
    b2 = np.sin(0.37 * np.arange(b1.size)) * 5.0
    one = S.SolveOptions(nu=5, tol=1e-300, max_cycles=1)
    us = []
    for bb in (b1, b2, b1 + b2):
        u = np.zeros_like(b1)
        S.mg_solve(h, bb, u, one)
        us.append(u)
    lin = us[0] + us[1]
    assert np.sqrt(np.sum((us[2] - lin) ** 2) / np.sum(lin ** 2)) < 1e-12


def test_nu_zero_and_max_cycles(torch, S, port):
    cs = case("cfg1_mini")
    h = gpu_hier(S, cs, port)
    hp = port_hier(port, cs)
    b = cs.rhs_vector(port)
    for nu, mc in ((0, 3), (1, 2), (2, 0)):
        u_p, rp = hp.solve(b, nu=nu, tol=1e-10, max_cycles=mc)
        u = np.zeros_like(b)
        rep = S.mg_solve(h, b, u, S.SolveOptions(nu=nu, tol=1e-10, max_cycles=mc))
        check_solve(rep, u, rp, u_p)


def test_adjoint_shares_workspace_with_primal(torch, S, port):
    cs = case("cfg2_mini")
    h = gpu_hier(S, cs, port)
    ht = S.transposed_hierarchy(h)
    b = cs.rhs_vector(port)
    c = np.ascontiguousarray(b * 0.01)
    cs_adj = case("cfg2_mini")
    cs_adj.adjoint = True
    hp_adj = port_hier(port, cs_adj)
    hp = port_hier(port, cs)
    for _ in range(2):  # interleave primal and adjoint solves on the shared workspace
        u = np.zeros_like(b)
        rep = S.mg_solve(h, b, u, S.SolveOptions(nu=2, tol=1e-10, max_cycles=20))
        check_solve(rep, u, *reversed(hp.solve(b, nu=2, tol=1e-10, max_cycles=20)))
        lam = np.zeros_like(b)
        rep = S.mg_solve(ht, c, lam, S.SolveOptions(nu=2, tol=1e-10, max_cycles=20))
        check_solve(rep, lam, *reversed(hp_adj.solve(c, nu=2, tol=1e-10, max_cycles=20)))


@pytest.mark.parametrize("name", ["cfg1_mini", "cfg1_mini_adj", "wide_short", "cfg0_deep"] + EDGE_CASES[::3])
def test_sweep_kernel_forms_bitwise(torch, S, port, name):
    """Single-sweep and fused two-sweep kernels, launched back to back."""
    cs = case(name)
    h = gpu_hier(S, cs, port)
    hp = port_hier(port, cs)
    rng = np.random.default_rng(3)
    for l in range(h.n_levels()):
        n = hp.ndofs(l)
        x, f = special_values(rng, n), special_values(rng, n)
        want = hp.sweeps(l, f, x, 4)
        for pairs, launches in ((False, 4), (True, 2)):
            xt, ft = torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda()
            yt = torch.empty_like(xt)
            h.sweep_kernels(l, ft, xt, yt, launches, pairs)
            torch.cuda.synchronize()
            assert np.array_equal(bits(xt), bits(want)), (l, pairs)


@pytest.mark.parametrize("tiles", [4, 2])
@pytest.mark.parametrize("name", ["cfg1_mini", "cfg1_mini_adj", "time_first", "wide_short", "cfg0_deep"] + EDGE_CASES)
def test_short_time_tiles_bitwise(torch, S, port, name, tiles):
    """4-level and 2-level time tiles (stmg_hierarchy_set_tiling), used on small
    latency-bound levels, on every level: kernels bit-identical to the oracle,
    solve parity."""
    cs = case(name)
    h = gpu_hier(S, cs, port)
    h.set_tiling(small_dofs=10 ** 15, tiny_dofs=10 ** 15 if tiles == 2 else 1)
    hp = port_hier(port, cs)
    rng = np.random.default_rng(17)
    dev = torch.device("cuda:0")
    for l in range(h.n_levels() - 1):
        n = hp.ndofs(l)
        x, f = special_values(rng, n), special_values(rng, n)
        xt, ft = torch.from_numpy(x).to(dev), torch.from_numpy(f).to(dev)
        for pairs, launches in ((False, 4), (True, 2)):
            xs, ys = xt.clone(), torch.empty_like(xt)
            h.sweep_kernels(l, ft, xs, ys, launches, pairs)
            torch.cuda.synchronize()
            assert np.array_equal(bits(xs), bits(hp.sweeps(l, f, x, 4))), (l, pairs)
        fc = torch.empty(hp.ndofs(l + 1), dtype=torch.float64, device=dev)
        h.restrict_residual(l, ft, xt, fc)
        assert np.array_equal(bits(fc), bits(hp.restrict(l, hp.residual(l, f, x)))), l
    b = cs.rhs_vector(port)
    u_p, rep_p = hp.solve(b, nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    u = np.zeros_like(b)
    rep = S.mg_solve(h, b, u, S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles))
    check_solve(rep, u, rep_p, u_p)


def extreme_values(rng, n):
    """special_values salted with subnormals, values whose scaled products are
    subnormal or overflow (|x| near DBL_MAX), and tiny normals."""
    v = special_values(rng, n)
    idx = rng.choice(n, size=max(4, n // 8), replace=False)
    v[idx[0::4]] = 5e-324 * rng.integers(1, 1 << 20, size=v[idx[0::4]].size)
    v[idx[1::4]] = 1.7e308 * rng.choice([-1.0, 1.0], size=v[idx[1::4]].size)
    v[idx[2::4]] = 2.2250738585072014e-308 * rng.standard_normal(v[idx[2::4]].size)
    v[idx[3::4]] = 1e300 * rng.standard_normal(v[idx[3::4]].size)
    return v


@pytest.mark.parametrize("omega", [0.5, 0.25, 1.0, 0.6, 2.0 / 3.0])
@pytest.mark.parametrize("name", ["cfg1_mini", "cfg1_mini_adj"])
@pytest.mark.parametrize("values", ["special", "extreme"])
def test_pair_kernel_omega_forms_bitwise(torch, S, port, name, omega, values):
    """Fused pairs compute omega * (r * invd) for every omega (the reference's
    form, proj/src/kernels/kernels.cpp:70-73), bitwise against the oracle's
    sweeps, including subnormal, overflowing and non-finite intermediates."""
    cs = case(name)
    h = gpu_hier(S, cs, port)
    hp = port_hier(port, cs)
    rng = np.random.default_rng(11)
    gen = special_values if values == "special" else extreme_values
    for l in range(h.n_levels() - 1):
        n = hp.ndofs(l)
        x, f = gen(rng, n), gen(rng, n)
        want = hp.sweeps(l, f, x, 4, omega)
        xt, ft = torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda()
        yt = torch.empty_like(xt)
        h.sweep_kernels(l, ft, xt, yt, 2, True, omega)
        torch.cuda.synchronize()
        got = xt.cpu().numpy()
        # NaN payloads differ between x86 and the GPU; every other value is bitwise
        same = (bits(got) == bits(want)) | (np.isnan(got) & np.isnan(want))
        assert same.all(), (l, omega, int((~same).sum()))
