"""A stream of solves on one hierarchy with host vectors (stmg_mg_solve_stream): each
entry equals the same solve run alone through stmg_mg_solve / stmg_mg_solve_ex, bit
for bit (u, history, cycles, status), whatever the overlap of its copies with its
neighbours' solves."""
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


def rhs_family(b, count):
    """count distinct right-hand sides of one grid (scaled and sign-flipped rows of b)."""
    rng = np.random.default_rng(7)
    out = []
    for k in range(count):
        s = rng.uniform(0.25, 4.0, size=b.shape)
        out.append(b * s if k else b.copy())
    return out


@pytest.mark.parametrize("name", ["cfg0", "cfg1_mini", "cfg1_mini_adj", "time_first", "gen_cp"])
@pytest.mark.parametrize("zero_guess", [False, True])
@pytest.mark.parametrize("nu", [1, 2])
def test_stream_equals_individual_solves(torch, S, port, name, zero_guess, nu):
    cs = case(name)
    h = build(S, cs, port)
    bs = rhs_family(cs.rhs_vector(port), 5)
    opts = S.SolveOptions(nu=nu, tol=1e-10, max_cycles=12)
    rng = np.random.default_rng(3)
    starts = [np.zeros_like(bs[0]) if zero_guess else rng.standard_normal(bs[0].shape) * 1e-3 for _ in bs]
    solo = []
    for b, u0 in zip(bs, starts):
        u = u0.copy()
        solo.append((S.mg_solve(h, b, u, opts, zero_guess=zero_guess), u))
    # pinned host vectors: the copies of entries k - 1 / k + 1 overlap solve k
    pb = [torch.from_numpy(b).pin_memory() for b in bs]
    pu = [torch.from_numpy(u0.copy()).pin_memory() for u0 in starts]
    if zero_guess:  # u is output only: whatever it holds is not read
        for u in pu:
            u.fill_(float("nan"))
    reps = S.mg_solve_stream(h, pb, pu, opts, zero_guess=zero_guess)
    assert len(reps) == len(bs)
    for k, ((r1, u1), r2, u2) in enumerate(zip(solo, reps, pu)):
        assert r1.cycles == r2.cycles and r1.status == r2.status, k
        assert r1.history == r2.history, k
        assert np.array_equal(u1, u2.numpy()), k
    h.release_staging()
    # after the release the next stream allocates fresh slots; pageable vectors work too
    us = [u0.copy() for u0 in starts[:3]]
    reps = S.mg_solve_stream(h, bs[:3], us, opts, zero_guess=zero_guess)
    for (r1, u1), r2, u2 in zip(solo, reps, us):
        assert r1.history == r2.history and np.array_equal(u1, u2)


def test_stream_one_output_buffer_and_degenerate_counts(torch, S, port):
    cs = case("cfg0")
    h = build(S, cs, port)
    b = cs.rhs_vector(port)
    opts = S.SolveOptions(nu=1, tol=1e-10)
    ref = np.zeros_like(b)
    r0 = S.mg_solve(h, b, ref, opts, zero_guess=True)
    # the same pinned b uploaded every step, every result downloaded into one buffer
    pb = torch.from_numpy(b).pin_memory()
    pu = torch.zeros(b.size, dtype=torch.float64).pin_memory()
    reps = S.mg_solve_stream(h, [pb] * 6, [pu] * 6, opts, zero_guess=True)
    assert all(r.history == r0.history for r in reps)
    assert np.array_equal(pu.numpy(), ref)
    assert S.mg_solve_stream(h, [], [], opts) == []
    u1 = np.zeros_like(b)
    (r1,) = S.mg_solve_stream(h, [b], [u1], opts)  # count 1: the plain solve
    assert r1.history == r0.history and np.array_equal(u1, ref)
    # device vectors: nothing to overlap, the plain sequence of solves
    db = torch.from_numpy(b).cuda()
    dus = [torch.zeros_like(db) for _ in range(2)]
    reps = S.mg_solve_stream(h, [db, db], dus, opts)
    assert all(r.history == r0.history for r in reps)
    assert all(np.array_equal(u.cpu().numpy(), ref) for u in dus)


def test_stream_argument_errors(torch, S, port):
    cs = case("cfg0")
    h = build(S, cs, port)
    b = cs.rhs_vector(port)
    with pytest.raises(ValueError):
        S.mg_solve_stream(h, [b, b], [np.zeros_like(b)], S.SolveOptions())
    with pytest.raises(ValueError):
        S.mg_solve_stream(h, [b[:-1], b], [np.zeros_like(b), np.zeros_like(b)], S.SolveOptions())
    with pytest.raises(ValueError):  # the solve's own option checks apply to every entry
        S.mg_solve_stream(h, [b, b], [np.zeros_like(b), np.zeros_like(b)], S.SolveOptions(omega=-1.0))


def test_stream_on_a_hierarchy_and_its_transpose_sharing_one_workspace(torch, S, port):
    """The staging slots live in the workspace a hierarchy shares with its transpose: streams
    on J and on J^T alternate over the same slots, with a release in between."""
    cs = case("cfg1_mini")
    h = build(S, cs, port)
    ht = S.transposed_hierarchy(h)
    bs = rhs_family(cs.rhs_vector(port), 3)
    opts = S.SolveOptions(nu=1, tol=1e-10, max_cycles=8)
    want = {}
    for name, hh in (("J", h), ("JT", ht)):
        want[name] = []
        for b in bs:
            u = np.zeros_like(b)
            want[name].append((S.mg_solve(hh, b, u, opts, zero_guess=True), u))
    pb = [torch.from_numpy(b).pin_memory() for b in bs]
    for round_ in range(2):
        for name, hh in (("J", h), ("JT", ht)):
            pu = [torch.full((b.size,), float("nan"), dtype=torch.float64).pin_memory() for b in bs]
            reps = S.mg_solve_stream(hh, pb, pu, opts, zero_guess=True)
            for (r1, u1), r2, u2 in zip(want[name], reps, pu):
                assert r1.history == r2.history and np.array_equal(u1, u2.numpy()), (round_, name)
        h.release_staging()
