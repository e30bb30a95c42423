"""GPU parity of the general coarse discretisations:
Galerkin (P) coarse operators, bilinear temporal transfers and FullST steps,
against outputs of the compiled reference (tests/golden/general.npz, made by
tests/golden/make_golden_general.py).

Bar: level operators, residuals, sweeps, restrictions and prolongations
bit-identical to the reference's CSR kernels; the exact coarsest solve within
1e-12 relative; whole solves with the same status and V-cycle count, histories
within 1e-10 relative (+ the fp64 floor of tests/_tol.py) and u within 1e-10
relative max-norm.
"""
import os

import numpy as np
import pytest

from tests._cases import GENERAL_CASES, case
from tests._general import GOLDEN, digest, level_inputs

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def torch():
    import torch as _t

    assert _t.cuda.is_available(), "GPU tests need CUDA (no CPU fallback exists)"
    return _t


@pytest.fixture(scope="module")
def S(torch):
    from paper_2505_10168_b200 import stmg

    return stmg


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(HERE, "golden", GOLDEN))


def gpu_hier(S, cs):
    g = S.build_fine_grid(cs.L, cs.tT, cs.n_el, cs.n_t)
    g.k, g.c = cs.k, cs.c
    path = S.CoarseningPath([S.CoarseningDirection(int(d)) for d in cs.dirs])
    h = S.build_hierarchy(g, cs.method, path, chi=cs.chi, mat=cs.mat)
    return S.transposed_hierarchy(h) if cs.adjoint else h


def ndofs(h):
    return [(lv.n_el + 1) * (lv.n_t + 1) for lv in h.levels]


@pytest.mark.parametrize("name", GENERAL_CASES)
def test_level_kernels_bitwise(torch, S, gold, name):
    cs = case(name)
    h = gpu_hier(S, cs)
    nds = ndofs(h)
    ins, fco = level_inputs(name, nds)
    dev = torch.device("cuda:0")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    for l, (x, f, xc) in enumerate(ins):
        st = h.level_stencil9(l)
        assert [digest(st["v9"]), digest(st["mask"]), digest(st["inv_diag"])] == \
            list(gold[f"{name}__op{l}"]), f"operator level {l}"
        want = list(gold[f"{name}__k{l}"])
        xt, ft = T(x), T(f)
        r = torch.empty_like(xt)
        h.residual(l, ft, xt, r)
        assert digest(r) == want[0], f"residual level {l}"
        xs = xt.clone()
        h.sweeps(l, ft, xs, 3)
        assert digest(xs) == want[1], f"sweeps level {l}"
        if xc is not None:
            fc = torch.empty(nds[l + 1], dtype=torch.float64, device=dev)
            h.restrict(l, r, fc)
            assert digest(fc) == want[2], f"restrict level {l}"
            fc2 = torch.empty_like(fc)
            h.restrict_residual(l, ft, xt, fc2)
            assert digest(fc2) == want[2], f"restrict_residual level {l}"
            xp = xt.clone()
            h.prolong_add(l, T(xc), xp)
            assert digest(xp) == want[3], f"prolong level {l}"
    x = torch.zeros(nds[-1], dtype=torch.float64, device=dev)
    h.coarsest_solve(T(fco), x)
    want = gold[f"{name}__coarsest"]
    assert np.max(np.abs(x.cpu().numpy() - want)) <= 1e-12 * np.max(np.abs(want))


@pytest.mark.parametrize("name", GENERAL_CASES)
def test_solve_parity(torch, S, port, gold, name):
    from tests._tol import histories_match

    cs = case(name)
    h = gpu_hier(S, cs)
    b = cs.rhs_vector(port)
    bt = torch.from_numpy(b).to("cuda:0")
    ut = torch.zeros_like(bt)
    rep = S.mg_solve(h, bt, ut, S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles))
    status, cycles, absn = (int(v) for v in gold[f"{name}__meta"])
    assert int(rep.status) == status and rep.cycles == cycles
    assert int(rep.absolute_norms) == absn
    hist = gold[f"{name}__history"]
    assert histories_match(rep.history, hist, 1e-13)
    u_ref = gold[f"{name}__u"]
    u = ut.cpu().numpy()
    assert np.max(np.abs(u - u_ref)) <= 1e-10 * np.max(np.abs(u_ref))


def test_general_solve_graph_counts(torch, S, port):
    """The captured V-cycle of a Galerkin + bilinear hierarchy launches the
    general kernels (one per sweep, residual + restriction, prolongation) and
    the block march, and repeated solves are deterministic."""
    cs = case("gen_bp_uni")
    h = gpu_hier(S, cs)
    b = torch.from_numpy(cs.rhs_vector(port)).to("cuda:0")
    u1, u2 = torch.zeros_like(b), torch.zeros_like(b)
    r1 = S.mg_solve(h, b, u1, S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=5))
    r2 = S.mg_solve(h, b, u2, S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=5))
    assert torch.equal(u1, u2) and list(r1.history) == list(r2.history)
    assert r1.kernel_launches == r2.kernel_launches > 5 * 10
