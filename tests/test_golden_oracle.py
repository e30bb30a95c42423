"""The C oracle reproduces the committed reference fixtures (tests/golden),
which were produced by the unmodified reference (tests/golden/make_golden.py)."""
import os

import numpy as np
import pytest

from tests._cases import case

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["cfg0", "cfg1_mini", "cfg1_mini_adj", "cfg2_mini", "cfgD", "time_first", "cfg4_mini"]


def load(name):
    return dict(np.load(os.path.join(GOLD, f"{name}.npz")))


def check_against_gold(gold, u, cycles, status, history, cs, floor=1e-13):
    from tests._tol import histories_match

    assert cycles == int(gold["cycles"]) and status == int(gold["status"])
    assert histories_match(history, gold["history"], floor), floor
    if "u" in gold:
        scale = max(np.max(np.abs(gold["u"])), 1e-300)
        assert np.max(np.abs(u - gold["u"])) <= 1e-10 * scale
    else:
        s = gold["u_sample"]
        assert np.max(np.abs(u[::97] - s)) <= 1e-10 * max(np.max(np.abs(s)), 1e-300)
        ls = u.reshape(cs.n_t + 1, cs.n_el + 1).sum(axis=1)
        assert np.max(np.abs(ls - gold["level_sums"])) <= 1e-10 * max(np.max(np.abs(gold["level_sums"])), 1e-300)


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference_golden(port, name):
    gold = load(name)
    cs = case(name)
    dirs = cs.plan(port)
    assert np.array_equal(dirs, gold["dirs"])
    hp = port.hierarchy(cs.L, cs.tT, cs.n_el, cs.n_t, cs.k, cs.c, dirs, reassembly=cs.reassembly,
                        adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat)
    u, rep = hp.solve(cs.rhs_vector(port), nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    check_against_gold(gold, u, rep.cycles, rep.status, rep.history, cs)
