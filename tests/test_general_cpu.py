"""General coarse discretisations on the host (no GPU): the Galerkin R J P build,
bilinear / FullST level grids and transposition, pinned bitwise to the compiled
reference through tests/golden/general.npz.

The operator digests compare this library's host half of build_hierarchy
(stmg_level_stencil9_host, include/stmg_b200.h) with the reference's CSR level
operators (proj/src/multigrid.cpp:86-160, proj/src/sparse.cpp:121-162) re-laid
out as 9-point stencils.
"""
import os

import numpy as np
import pytest

from tests._cases import GENERAL_CASES, case
from tests._general import GOLDEN, csr_to_stencil9, digest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(HERE, "golden", GOLDEN))


@pytest.fixture(scope="module")
def S():
    from paper_2505_10168_b200 import stmg

    return stmg


def host_levels(S, cs):
    g = S.build_fine_grid(cs.L, cs.tT, cs.n_el, cs.n_t)
    g.k, g.c = cs.k, cs.c
    path = S.CoarseningPath([S.CoarseningDirection(int(d)) for d in cs.dirs])
    return [S.level_stencil9_host(g, cs.method, path, l, chi=cs.chi, mat=cs.mat, adjoint=cs.adjoint)
            for l in range(len(cs.dirs) + 1)]


@pytest.mark.parametrize("name", GENERAL_CASES)
def test_operators_match_reference_bitwise(S, gold, name):
    cs = case(name)
    for l, st in enumerate(host_levels(S, cs)):
        want = gold[f"{name}__op{l}"]
        got = [digest(st["v9"]), digest(st["mask"]), digest(st["inv_diag"])]
        assert got == list(want), f"{name} level {l}: (values, mask, 1/diag) digests differ"


def test_operators_against_live_reference(S, ref):
    """Same comparison on the full arrays, where the compiled reference exists."""
    for name in ("gen_cp", "gen_bp_uni", "gen_cp_xt_adj"):
        cs = case(name)
        h = ref.hierarchy(cs.L, cs.tT, cs.n_el, cs.n_t, cs.k, cs.c, cs.dirs, method=cs.method,
                          adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat)
        for l, st in enumerate(host_levels(S, cs)):
            rp, ci, v, inv = h.csr(l)
            V, M = csr_to_stencil9(rp, ci, v, st["n_el"], st["n_t"])
            assert np.array_equal(M, st["mask"])
            assert np.array_equal(V.view(np.uint64), st["v9"].view(np.uint64))
            assert np.array_equal(inv.view(np.uint64), st["inv_diag"].view(np.uint64))


def test_galerkin_levels_are_not_rediscretised(S):
    """A P level differs from the K level of the same grid (it is R J P)."""
    cs = case("gen_cp")
    p = host_levels(S, cs)
    cs.method = "CK"
    k = host_levels(S, cs)
    assert np.array_equal(p[0]["v9"], k[0]["v9"])  # the fine level is always assembled
    assert not np.array_equal(p[1]["v9"], k[1]["v9"])


def test_fullst_bilinear_rejected(S):
    """build_prolongation: combined coarsening is causal-only (proj/src/transfer.cpp:44-47)."""
    cs = case("gen_ck_xt")
    cs.method = "BK"
    with pytest.raises(ValueError, match="causal-only"):
        host_levels(S, cs)


@pytest.mark.parametrize("method", ["XK", "CQ", "C", "CKR"])
def test_parse_method_errors(S, method):
    """parse_method (proj/src/rediscretisation.cpp:19-38) raises invalid_argument."""
    cs = case("gen_cp")
    cs.method = method
    with pytest.raises(ValueError, match="parse_method"):
        host_levels(S, cs)
