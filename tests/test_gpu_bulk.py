"""The bulk-copy pipelined fused pair (k_bulk: cp.async.bulk rows into an
mbarrier ring, persistent CTAs) against the register-staged pair k_lean2x2 and,
through whole solves, against the CPU oracle.  Bar: bit-identical."""
import os

import numpy as np
import pytest

from tests._cases import case

pytestmark = pytest.mark.gpu
PAD = 512  # tail padding the bulk-copy kernel needs (kVecPad)


@pytest.fixture(scope="module")
def torch():
    import torch as _t

    assert _t.cuda.is_available(), "GPU tests need CUDA (no CPU fallback exists)"
    return _t


@pytest.fixture(scope="module")
def S(torch):
    from paper_2505_10168_b200 import stmg

    return stmg


def hier(S, cs, port):
    dirs = cs.plan(port)
    g = S.build_fine_grid(cs.L, cs.tT, cs.n_el, cs.n_t)
    g.k, g.c = cs.k, cs.c
    path = S.CoarseningPath([S.CoarseningDirection(int(d)) for d in dirs])
    h = S.build_hierarchy(g, cs.method, path, chi=cs.chi, mat=cs.mat)
    return S.transposed_hierarchy(h) if cs.adjoint else h


@pytest.mark.parametrize("name", ["cfg1_mini", "cfg1_mini_adj", "wide_short", "cfg0", "tiny", "space_first"])
def test_bulk_pair_bitwise(torch, S, port, name):
    cs = case(name)
    h = hier(S, cs, port)
    rng = np.random.default_rng(5)
    for l, lv in enumerate(h.levels):
        n = lv.n_dofs
        f = torch.from_numpy(rng.standard_normal(n + PAD)).cuda()
        x0 = torch.from_numpy(rng.standard_normal(n + PAD)).cuda()
        xa, ya = x0.clone(), torch.zeros_like(x0)
        xb, yb = x0.clone(), torch.zeros_like(x0)
        h.sweep_kernels(l, f, xa, ya, 3, True)   # lean pairs: x -> y -> x -> y
        h.sweep_kernels(l, f, xb, yb, 3, 5)      # bulk pairs
        torch.cuda.synchronize()
        assert torch.equal(ya[:n], yb[:n]), f"level {l}"
        assert torch.equal(xa[:n], xb[:n]), f"level {l}"


@pytest.mark.parametrize("name", ["cfg1_mini", "cfg1_mini_adj", "cfg4_mini", "wide_coarsest_adj"])
def test_solves_with_bulk_pairs_match_oracle(torch, S, port, name, monkeypatch):
    from tests.test_gpu_parity import check_solve, port_hier

    monkeypatch.setenv("STMG_BULK_DOFS", "1")  # every level (read at hierarchy build)
    cs = case(name)
    h = hier(S, cs, port)
    b = cs.rhs_vector(port)
    bt = torch.from_numpy(b).cuda()
    ut = torch.zeros_like(bt)
    rep = S.mg_solve(h, bt, ut, S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles))
    u_p, rep_p = port_hier(port, cs).solve(b, nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    check_solve(rep, ut.cpu().numpy(), rep_p, u_p)
