"""The drop-in proven on the reference's side: the reference's own callers --
optimise() (proj/src/optimisation.cpp:83-186) and the harness's mg_solve /
build_hierarchy / transposed_hierarchy calls -- compiled unmodified and linked
against paper_2505_10168_b200/dropin/multigrid_b200.cpp (the reference's
multigrid.hpp API on libstmg_b200.so) instead of proj/src/multigrid.cpp
(oracle/Makefile target `dropin`).  Their outputs must match the committed
outputs of the unmodified reference (tests/golden).
"""
import os

import numpy as np
import pytest

from tests._cases import case
from tests.test_golden_oracle import check_against_gold, load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dropin():
    import torch

    assert torch.cuda.is_available(), "GPU tests need CUDA (no CPU fallback exists)"
    from oracle import pyoracle

    if not pyoracle.dropin_available():
        pytest.skip("oracle/_ref/libstmg_dropin.so not built (needs /root/reference; __graft_entry__.build())")
    return pyoracle.Ref(dropin=True)


def test_reference_optimise_runs_on_the_dropin(dropin):
    """The reference's optimise() with GPU solves: the same per-iteration V-cycle
    counts and statuses, theta and the final design as the unmodified reference."""
    from tests.golden.make_golden import OPT_SMALL

    gold = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "opt_small.npz")))
    o = dict(OPT_SMALL)
    r = dropin.optimise(o.pop("L"), o.pop("tT"), o.pop("n_el"), o.pop("n_t"), o.pop("mat"), **o)
    rec, want = r["records"], gold["records"]
    assert rec.shape == want.shape
    assert np.array_equal(rec[:, 4:8], want[:, 4:8])  # statuses and cycle counts
    np.testing.assert_allclose(rec[:, 0], want[:, 0], rtol=1e-9)  # theta
    np.testing.assert_allclose(rec[:, 1], want[:, 1], rtol=0, atol=1e-12)  # volume
    np.testing.assert_allclose(rec[:, 8:10], want[:, 8:10], rtol=1e-6)  # convergence factors
    assert np.max(np.abs(r["chi"] - gold["chi"])) <= 1e-9
    assert abs(r["theta"] - float(gold["theta"])) <= 1e-9 * abs(float(gold["theta"]))


@pytest.mark.parametrize("name", ["cfg0", "cfg1_mini", "cfg1_mini_adj", "cfg2_mini", "time_first", "cfg4_mini"])
def test_reference_mg_solve_runs_on_the_dropin(dropin, port, name):
    """build_hierarchy (+ transposed_hierarchy) + mg_solve through the reference's
    API against the reference's own solves of the same cases."""
    gold = load(name)
    cs = case(name)
    h = dropin.hierarchy(cs.L, cs.tT, cs.n_el, cs.n_t, cs.k, cs.c, gold["dirs"], method=cs.method,
                         adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat)
    assert h.n_levels == len(gold["dirs"]) + 1 and h.ndofs(0) == cs.n_dofs
    b = cs.rhs_vector(port)
    u, rep = h.solve(b, nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    check_against_gold(gold, u, rep.cycles, rep.status, rep.history, cs)


def test_dropin_keeps_the_reference_error_classes(dropin, port):
    """std::invalid_argument (size mismatch, bad options) surfaces as the harness's
    code 1, as from the unmodified reference (proj/src/multigrid.cpp:214-220)."""
    from oracle.pyoracle import OracleError

    cs = case("cfg0")
    h = dropin.hierarchy(cs.L, cs.tT, cs.n_el, cs.n_t, cs.k, cs.c, [0], method=cs.method)
    b = cs.rhs_vector(port)
    with pytest.raises(OracleError, match="rc=1"):
        h.solve(b, nu=-1)
    with pytest.raises(OracleError, match="rc=1"):
        h.solve(b, tol=0.0)
