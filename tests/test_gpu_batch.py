"""Concurrent independent solves (stmg_mg_solve_batch): each entry equals the
same solve run alone, bit for bit (u, history, cycles, status)."""
import numpy as np
import pytest

from tests._cases import case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as _t

    assert _t.cuda.is_available(), "GPU tests need CUDA (no CPU fallback exists)"
    return _t


@pytest.fixture(scope="module")
def S(torch):
    from paper_2505_10168_b200 import stmg

    return stmg


def build(S, cs, port):
    dirs = cs.plan(port)
    g = S.build_fine_grid(cs.L, cs.tT, cs.n_el, cs.n_t)
    g.k, g.c = cs.k, cs.c
    path = S.CoarseningPath([S.CoarseningDirection(int(d)) for d in dirs])
    h = S.build_hierarchy(g, cs.method, path, chi=cs.chi, mat=cs.mat)
    return S.transposed_hierarchy(h) if cs.adjoint else h


NAMES = ["cfg0", "cfg1_mini", "cfg1_mini_adj", "wide_coarsest", "time_first", "gen_cp", "gen_bk", "cfg4_mini"]


def test_batch_equals_individual_solves(torch, S, port):
    hs = [build(S, case(n), port) for n in NAMES]
    bs = [torch.from_numpy(case(n).rhs_vector(port)).cuda() for n in NAMES]
    opts = S.SolveOptions(nu=2, tol=1e-10, max_cycles=30)
    solo = []
    for h, b in zip(hs, bs):
        u = torch.zeros_like(b)
        solo.append((S.mg_solve(h, b, u, opts), u))
    us = [torch.zeros_like(b) for b in bs]
    reps = S.mg_solve_batch(hs, bs, us, opts)
    for (r1, u1), r2, u2, n in zip(solo, reps, us, NAMES):
        assert r1.cycles == r2.cycles and r1.status == r2.status, n
        assert r1.history == r2.history, n
        assert torch.equal(u1, u2), n


def test_batch_host_vectors_and_empty(torch, S, port):
    cs = case("cfg0")
    hs = [build(S, cs, port) for _ in range(3)]
    b = cs.rhs_vector(port)
    us = [np.zeros_like(b) for _ in hs]
    reps = S.mg_solve_batch(hs, [b] * 3, us, S.SolveOptions(nu=1, tol=1e-10))
    assert all(r.cycles == reps[0].cycles for r in reps)
    assert all(np.array_equal(u, us[0]) for u in us)
    assert S.mg_solve_batch([], [], [], S.SolveOptions()) == []


def test_batch_rejects_shared_workspace(torch, S, port):
    cs = case("cfg0")
    h = build(S, cs, port)
    ht = S.transposed_hierarchy(h)
    b = torch.from_numpy(cs.rhs_vector(port)).cuda()
    with pytest.raises(ValueError, match="share a workspace"):
        S.mg_solve_batch([h, ht], [b, b], [torch.zeros_like(b), torch.zeros_like(b)], S.SolveOptions())
    with pytest.raises(ValueError):
        S.mg_solve_batch([h, h], [b, b], [torch.zeros_like(b), torch.zeros_like(b)], S.SolveOptions())
