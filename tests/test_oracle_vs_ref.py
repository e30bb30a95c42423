"""Pin the C oracle restatement to the UNMODIFIED reference (oracle/_ref).

Bitwise: planner paths and indicators, load vectors, every level kernel
(damped-Jacobi sweeps, residuals, restriction, prolongation) on primal and
transposed hierarchies.  Whole solves: identical cycle counts and status,
histories and fields within 1e-12 (the coarsest exact solver is Thomas in the
oracle and a sparse LU in the reference, proj/src/multigrid.cpp:20-57).
"""
import numpy as np
import pytest

from tests._cases import SMALL_CASES, case


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def test_reference_unit_suites_pass():
    """The reference's own doctest suites, unmodified, against the shims."""
    import os
    import subprocess

    from oracle import pyoracle

    exe = os.path.join(pyoracle.HERE, "_ref", "ref_unit_tests")
    if not os.path.exists(exe):
        pytest.skip("reference unit-test binary not built here")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    assert "0 failed" in r.stderr


@pytest.mark.parametrize("name", [c for c in SMALL_CASES if c not in ("single_level", "tiny")])
def test_plan_matches_reference(port, ref, name):
    cs = case(name)
    a = port.plan(cs.L, cs.tT, cs.n_el, cs.n_t, cs.k, cs.c, cs.n_levels, strategy=cs.strategy,
                  reassembly=cs.reassembly, min_elements=cs.min_elements, chi=cs.chi, mat=cs.mat)
    b = ref.plan(cs.L, cs.tT, cs.n_el, cs.n_t, cs.k, cs.c, cs.n_levels, strategy=cs.strategy,
                 reassembly=cs.reassembly, min_elements=cs.min_elements, chi=cs.chi, mat=cs.mat)
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(bits(a[1]), bits(b[1]))


@pytest.mark.parametrize("kind,params", [(0, (1.0,)), (1, (1.0, 0.1)), (2, (0.5, 8.0, 0.05)), (3, ())])
def test_load_vector_bitwise(port, ref, kind, params):
    for (ne, nt) in ((16, 8), (128, 64), (1000, 37)):
        a = port.load_vector(1.0, 1.0, ne, nt, kind, params)
        b = ref.load_vector(1.0, 1.0, ne, nt, kind, params)
        assert np.array_equal(bits(a), bits(b))


@pytest.mark.parametrize("name", SMALL_CASES)
def test_level_kernels_bitwise(port, ref, name):
    cs = case(name)
    dirs = cs.plan(port)
    hp = port.hierarchy(cs.L, cs.tT, cs.n_el, cs.n_t, cs.k, cs.c, dirs, reassembly=cs.reassembly,
                        adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat)
    hr = ref.hierarchy(cs.L, cs.tT, cs.n_el, cs.n_t, cs.k, cs.c, dirs, method=cs.method,
                       adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat)
    assert hp.n_levels == hr.n_levels
    rng = np.random.default_rng(7)
    for l in range(hp.n_levels):
        n = hp.ndofs(l)
        assert n == hr.ndofs(l)
        x = rng.standard_normal(n)
        f = rng.standard_normal(n)
        assert np.array_equal(bits(hp.residual(l, f, x)), bits(hr.residual(l, f, x)))
        assert np.array_equal(bits(hp.sweeps(l, f, x, 2)), bits(hr.sweeps(l, f, x, 2)))
        if l + 1 < hp.n_levels:
            r = hp.residual(l, f, x)
            assert np.array_equal(bits(hp.restrict(l, r)), bits(hr.restrict(l, r)))
            xc = rng.standard_normal(hp.ndofs(l + 1))
            assert np.array_equal(bits(hp.prolong_add(l, xc, x)), bits(hr.prolong_add(l, xc, x)))
    f = rng.standard_normal(hp.ndofs(hp.n_levels - 1))
    a, b = hp.coarsest(f), hr.coarsest(f)
    assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))


@pytest.mark.parametrize("name", SMALL_CASES)
def test_solve_matches_reference(port, ref, name):
    cs = case(name)
    dirs = cs.plan(port)
    b = cs.rhs_vector(port)
    hp = port.hierarchy(cs.L, cs.tT, cs.n_el, cs.n_t, cs.k, cs.c, dirs, reassembly=cs.reassembly,
                        adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat)
    hr = ref.hierarchy(cs.L, cs.tT, cs.n_el, cs.n_t, cs.k, cs.c, dirs, method=cs.method,
                       adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat)
    up, rp = hp.solve(b, nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    ur, rr = hr.solve(b, nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    assert rp.cycles == rr.cycles and rp.status == rr.status
    # |dh| <= 1e-12 h + 1e-13: the absolute floor (in units of ||b||) is the fp64
    # cancellation floor of evaluating b - J u once u is ~1e-10 accurate.
    assert np.all(np.abs(rp.history - rr.history) <= 1e-12 * np.abs(rr.history) + 1e-13)
    assert np.max(np.abs(up - ur)) <= 1e-12 * max(np.max(np.abs(ur)), 1e-300)


def test_masked_design_oracle_matches_reference_apply_design(port, ref):
    chi = np.linspace(0.0, 1.0, 101)
    mat = (1e-3, 1.0, 1.0, 2.0, 3.0, 2.0)
    kp, cp = port.apply_design(chi, mat)
    kr, cr = ref.apply_design(chi, mat)
    assert np.array_equal(bits(kp), bits(kr)) and np.array_equal(bits(cp), bits(cr))


def test_reference_errors_mirrored(port, ref):
    from oracle.pyoracle import OracleError

    k = np.ones(8)
    # lambda_crit must be positive (strategy.cpp:131-132)
    for o in (port, ref):
        with pytest.raises(OracleError):
            o.plan(1.0, 1.0, 8, 8, k, k, 3, lambda_crit=0.0)
    # resolution guard forbids a forced time step past the last level (strategy.cpp:196-200)
    for o in (port, ref):
        with pytest.raises(OracleError):
            o.plan(1.0, 1.0, 8, 8, k, k, 5, strategy=2, min_elements=8)
