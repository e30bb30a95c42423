"""Time-slab multi-GPU path, validated on one GPU with the loopback transport:
all `world` ranks of the exact product code path (slab kernels, ghost
exchanges, all-reduced norms, gather / tail solve / broadcast) run in one
process, and must reproduce the single-domain solve: identical iterate
(bitwise), same cycle count, histories equal up to norm summation order."""
import numpy as np
import pytest

from tests._cases import case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import torch

    assert torch.cuda.is_available(), "GPU tests need CUDA (no CPU fallback exists)"
    from paper_2505_10168_b200 import stmg

    return stmg


def grid_path(S, cs, port):
    dirs = cs.plan(port)
    g = S.build_fine_grid(cs.L, cs.tT, cs.n_el, cs.n_t)
    g.k, g.c = cs.k, cs.c
    return g, S.CoarseningPath([S.CoarseningDirection(int(d)) for d in dirs])


@pytest.mark.parametrize("name,world", [("cfg1_mini", 2), ("cfg1_mini", 4), ("cfg1_mini_adj", 4),
                                        ("cfg4_mini", 8), ("cfgD", 2), ("cfg0_deep", 2), ("cfg2_mini", 4)])
def test_loopback_slabs_match_single_domain(S, port, name, world):
    cs = case(name)
    g, path = grid_path(S, cs, port)
    b = cs.rhs_vector(port)
    opts = S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    h = S.build_hierarchy(g, cs.method, path, chi=cs.chi, mat=cs.mat)
    if cs.adjoint:
        h = S.transposed_hierarchy(h)
    u1 = np.zeros_like(b)
    r1 = S.mg_solve(h, b, u1, opts)
    dh = S.build_dist_hierarchy(g, cs.method, path, world, adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat,
                                min_slab=8)
    assert dh.n_distributed >= 1
    u2 = np.zeros_like(b)
    r2 = S.mg_solve_dist(dh, b, u2, opts)
    assert dh.loop_on_device
    assert r2.cycles == r1.cycles and r2.status == r1.status
    assert np.array_equal(u1.view(np.uint64), u2.view(np.uint64))
    assert np.allclose(r2.history, r1.history, rtol=1e-12, atol=0)


@pytest.mark.parametrize("name,world", [("cfg1_mini", 2), ("cfg1_mini_adj", 4), ("cfg2_mini", 4)])
def test_slab_local_vectors_match_full_vectors(S, port, name, world):
    """stmg_dist_mg_solve_local: the caller holds only this process's level-0 rows
    of b and u (loopback: all ranks' rows, [row_lo, row_hi)); the library exchanges
    the right-hand side's ghost rows.  Bitwise the full-vector slab solve."""
    import torch

    cs = case(name)
    g, path = grid_path(S, cs, port)
    b = cs.rhs_vector(port)
    opts = S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    dh = S.build_dist_hierarchy(g, cs.method, path, world, adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat,
                                min_slab=8)
    u_full = np.zeros_like(b)
    r_full = S.mg_solve_dist(dh, b, u_full, opts)
    nn = cs.n_el + 1
    rows = slice(dh.row_lo * nn, dh.row_hi * nn)
    b_loc = torch.from_numpy(np.ascontiguousarray(b[rows])).cuda()
    u_loc = torch.zeros_like(b_loc)
    r_loc = S.mg_solve_dist_local(dh, b_loc, u_loc, opts)
    assert r_loc.cycles == r_full.cycles and r_loc.history == r_full.history
    assert np.array_equal(u_loc.cpu().numpy().view(np.uint64), u_full[rows].view(np.uint64))


def test_partition_rules(S):
    # cfg1 path x,x,x,t,x,t,t,x,t: n_t per level 4096 x4, 2048 x2, 1024, 512 x2, 256
    nts = [4096, 4096, 4096, 4096, 2048, 2048, 1024, 512, 512, 256]
    dirs = [0, 0, 0, 1, 0, 1, 1, 0, 1]
    lg, b = S.dist_partition(nts, dirs, 8, 16)
    assert lg == 9  # the coarsest level is always gathered
    assert list(b[0]) == [0, 512, 1024, 1536, 2048, 2560, 3072, 3584, 4097]
    assert list(b[3])[-1] == 4097 and b[4][1] == 256
    lg, _ = S.dist_partition(nts, dirs, 8, 128)
    assert lg == 7  # level 7 has 512/8 = 64 < 128 steps per slab
    lg, _ = S.dist_partition([30, 15], [1], 4, 8)
    assert lg == 0  # 30 steps do not split into 4 slabs


def test_nccl_transport_world1_matches_single_domain(S, port):
    """The NCCL transport itself (dlopen'ed libnccl, communicator init, NCCL
    calls captured in the V-cycle graph) on a one-rank communicator."""
    cs = case("cfg1_mini")
    g, path = grid_path(S, cs, port)
    b = cs.rhs_vector(port)
    opts = S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    h = S.build_hierarchy(g, cs.method, path)
    u1 = np.zeros_like(b)
    r1 = S.mg_solve(h, b, u1, opts)
    dh = S.build_dist_hierarchy(g, cs.method, path, 1, rank=0, nccl_id=S.nccl_unique_id(), min_slab=8)
    u2 = np.zeros_like(b)
    r2 = S.mg_solve_dist(dh, b, u2, opts)
    assert r2.cycles == r1.cycles
    assert np.array_equal(u1.view(np.uint64), u2.view(np.uint64))


def test_slab_storage_scales_with_world(S):
    """Each rank allocates only its slab (plus a few margin levels) of every
    distributed level vector, so the loopback process, which hosts all ranks,
    holds about one full-size copy whatever the world size (full-size rank
    vectors would grow linearly with it)."""
    n_el, n_t = 64, 2048
    g = S.build_fine_grid(1.0, 1.0, n_el, n_t)
    g.k, g.c = np.ones(n_el), np.ones(n_el)
    X, T = S.CoarseningDirection.SpaceX, S.CoarseningDirection.TimeT
    path = S.CoarseningPath([X, T, T, T])
    sizes = {}
    for world in (2, 8):
        dh = S.build_dist_hierarchy(g, "CK", path, world, min_slab=8)
        assert dh.n_distributed >= 1
        sizes[world] = dh.device_bytes
    vec_bytes = 8 * (n_el + 1) * (n_t + 1)
    # full-size rank storage would grow by at least 6 ranks x 3 level-0 vectors;
    # slab storage grows only by margins, padding and the small gathered level
    assert sizes[8] - sizes[2] < 0.15 * 6 * 3 * vec_bytes, sizes


@pytest.mark.parametrize("mode", ["1", "2"])
@pytest.mark.parametrize("name,world", [("cfg1_mini", 2), ("cfg1_mini_adj", 4), ("cfg4_mini", 8),
                                        ("cfg0_deep", 2)])
def test_p2p_transport_loopback_matches_single_domain(S, port, monkeypatch, name, world, mode):
    """Peer-memory ghost pulls behind the neighbour epoch barrier, all ranks in this
    process: bitwise the single-domain iterate, through graph replays and repeated
    solves (epochs keep counting).  STMG_DIST_P2P=1: every exchange is ONE cooperative
    grid over all ranks, each rank running the cross-process protocol unchanged (its
    block 0 posts, its blocks spin on the neighbours' posts), so the post / wait /
    epoch path races between ranks on the hardware.  STMG_DIST_P2P=2: the pre-posted
    form (all ranks signal, then all pull; the waits are already satisfied)."""
    cs = case(name)
    g, path = grid_path(S, cs, port)
    b = cs.rhs_vector(port)
    opts = S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    h = S.build_hierarchy(g, cs.method, path, chi=cs.chi, mat=cs.mat)
    if cs.adjoint:
        h = S.transposed_hierarchy(h)
    u1 = np.zeros_like(b)
    r1 = S.mg_solve(h, b, u1, opts)
    monkeypatch.setenv("STMG_DIST_P2P", mode)
    dh = S.build_dist_hierarchy(g, cs.method, path, world, adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat,
                                min_slab=8)
    assert dh.transport == "p2p"
    for _ in range(2):
        u2 = np.zeros_like(b)
        r2 = S.mg_solve_dist(dh, b, u2, opts)
        assert r2.cycles == r1.cycles and r2.status == r1.status
        assert np.array_equal(u1.view(np.uint64), u2.view(np.uint64))
        assert np.allclose(r2.history, r1.history, rtol=1e-12, atol=0)
    monkeypatch.delenv("STMG_DIST_P2P")
    assert S.build_dist_hierarchy(g, cs.method, path, world, adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat,
                                  min_slab=8).transport == "loopback"


def test_p2p_over_nccl_world1_gathers_handles_and_matches(S, port, monkeypatch):
    """STMG_DIST_P2P=1 on a real NCCL communicator: the CUDA IPC handles of
    every slab vector are all-gathered over NCCL (no neighbour to map in a
    world of one), and the solve equals the single-domain one bitwise."""
    cs = case("cfg1_mini")
    g, path = grid_path(S, cs, port)
    b = cs.rhs_vector(port)
    opts = S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    h = S.build_hierarchy(g, cs.method, path)
    u1 = np.zeros_like(b)
    r1 = S.mg_solve(h, b, u1, opts)
    monkeypatch.setenv("STMG_DIST_P2P", "1")
    dh = S.build_dist_hierarchy(g, cs.method, path, 1, rank=0, nccl_id=S.nccl_unique_id(), min_slab=8)
    assert dh.transport == "p2p"
    u2 = np.zeros_like(b)
    r2 = S.mg_solve_dist(dh, b, u2, opts)
    assert r2.cycles == r1.cycles
    assert np.array_equal(u1.view(np.uint64), u2.view(np.uint64))


@pytest.mark.parametrize("name,world", [("cfg1_mini", 2), ("cfg1_mini_adj", 4), ("cfg2_mini", 4), ("cfg4_mini", 8)])
def test_device_cycle_loop_equals_host_loop(S, port, monkeypatch, name, world):
    """The time-slab solve's cycle loop as one conditional WHILE graph (dist_loop:
    V-cycle with its ghost exchanges and gathered tail, all-reduced norm, bookkeeping
    kernel; the default in loopback) against the host loop with a norm read-back per
    cycle (STMG_DIST_DEVICE_LOOP=0): same cycles, status, history and iterate, bitwise;
    also for a solve that stops at max_cycles and one that diverges (cfg2_mini)."""
    cs = case(name)
    g, path = grid_path(S, cs, port)
    b = cs.rhs_vector(port)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("STMG_DIST_DEVICE_LOOP", mode)
        dh = S.build_dist_hierarchy(g, cs.method, path, world, adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat,
                                    min_slab=8)
        res = []
        for max_cycles in (cs.max_cycles, 3):
            u = np.zeros_like(b)
            r = S.mg_solve_dist(dh, b, u, S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=max_cycles))
            assert dh.loop_on_device == (mode == "1")
            res.append((r, u))
        out[mode] = res
    for (r1, u1), (r0, u0) in zip(out["1"], out["0"]):
        assert r1.cycles == r0.cycles and r1.status == r0.status
        assert r1.history == r0.history
        assert np.array_equal(u1.view(np.uint64), u0.view(np.uint64))


def test_device_cycle_loop_with_nccl_in_the_body_world1(S, port, monkeypatch):
    """STMG_DIST_DEVICE_LOOP=1 on a real NCCL communicator (world of one): the NCCL
    all-reduce, gather and broadcast are captured INSIDE the conditional WHILE body.
    Same result as the single-domain solve."""
    cs = case("cfg1_mini")
    g, path = grid_path(S, cs, port)
    b = cs.rhs_vector(port)
    opts = S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    h = S.build_hierarchy(g, cs.method, path)
    u1 = np.zeros_like(b)
    r1 = S.mg_solve(h, b, u1, opts)
    monkeypatch.setenv("STMG_DIST_DEVICE_LOOP", "1")
    dh = S.build_dist_hierarchy(g, cs.method, path, 1, rank=0, nccl_id=S.nccl_unique_id(), min_slab=8)
    assert dh.transport == "nccl"
    u2 = np.zeros_like(b)
    r2 = S.mg_solve_dist(dh, b, u2, opts)
    assert dh.loop_on_device
    assert r2.cycles == r1.cycles and r2.status == r1.status
    assert np.array_equal(u1.view(np.uint64), u2.view(np.uint64))
    assert np.allclose(r2.history, r1.history, rtol=1e-12, atol=0)


@pytest.mark.parametrize("p2p", ["0", "1"])
@pytest.mark.parametrize("loop", ["1", "0"])
@pytest.mark.parametrize("name,world", [("cfg1_mini", 2), ("cfg1_mini_adj", 2), ("cfg2_mini", 2), ("cfg4_mini", 2)])
def test_overlapped_ghost_exchange_is_bitwise(S, port, monkeypatch, name, world, loop, p2p):
    """STMG_DIST_OVERLAP: the ghost exchange of a pass runs on a forked side stream while
    every rank's kernel runs on the interior rows of its slab; the first and last 16 rows
    follow after the join (sweeps, fused pairs, restrictions; inside the captured V-cycle and
    inside the device loop's conditional body).  Same iterate as the single-domain solve."""
    cs = case(name)
    g, path = grid_path(S, cs, port)
    b = cs.rhs_vector(port)
    opts = S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=min(cs.max_cycles, 20))
    h = S.build_hierarchy(g, cs.method, path, chi=cs.chi, mat=cs.mat)
    if cs.adjoint:
        h = S.transposed_hierarchy(h)
    u1 = np.zeros_like(b)
    r1 = S.mg_solve(h, b, u1, opts)
    monkeypatch.setenv("STMG_DIST_OVERLAP", "1")
    monkeypatch.setenv("STMG_DIST_DEVICE_LOOP", loop)
    monkeypatch.setenv("STMG_DIST_P2P", p2p)  # 1: the cooperative all-ranks pull kernel on the side stream
    dh = S.build_dist_hierarchy(g, cs.method, path, world, adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat, min_slab=8)
    for _ in range(2):
        u2 = np.zeros_like(b)
        r2 = S.mg_solve_dist(dh, b, u2, opts)
        assert r2.cycles == r1.cycles and r2.status == r1.status
        assert np.array_equal(u1.view(np.uint64), u2.view(np.uint64))
    assert dh.split_passes > 0 and dh.loop_on_device == (loop == "1")
