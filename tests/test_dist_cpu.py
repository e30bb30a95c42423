"""Multi-process (gloo, world size 2 and 4) CPU test of the time-slab algorithm:
slab partition from the product's stmg_dist_partition, ghost-level exchange,
all-reduced norms, gather / tail solve / broadcast — on the oracle kernels —
must reproduce the single-domain oracle iterate bit for bit at every cycle."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from tests._cases import case


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    import torch.distributed as dist

    from oracle.pyoracle import Port
    from paper_2505_10168_b200 import stmg as S
    from tests._dist_sim import SlabSim

    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        port_ = Port()
        cs = case(name)
        dirs = cs.plan(port_)
        hp = port_.hierarchy(cs.L, cs.tT, cs.n_el, cs.n_t, cs.k, cs.c, dirs, reassembly=cs.reassembly,
                             adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat)
        shapes = [(ne, nt) for ne, nt, _ in hp.shapes]
        lg, bounds = S.dist_partition([nt for _, nt in shapes], [int(d) for d in dirs], world, 8)
        sim = SlabSim(hp, dirs, shapes, bounds, lg, rank, world, cs.nu)
        b = cs.rhs_vector(port_)
        x, hist, cycles, iterates = sim.solve(b, cs.tol, 12)
        lo, hi = int(bounds[0][rank]), int(bounds[0][rank + 1])
        # single-domain reference: the oracle's own mg_solve, cycle by cycle
        ok = True
        for k, it in enumerate(iterates, start=1):
            u_ref, _ = hp.solve(b, nu=cs.nu, tol=1e-300, max_cycles=k)
            nn = cs.n_el + 1
            a = it.reshape(-1, nn)[lo:hi]
            r = u_ref.reshape(-1, nn)[lo:hi]
            ok = ok and np.array_equal(a.view(np.uint64), r.view(np.uint64))
        u_ref, rep = hp.solve(b, nu=cs.nu, tol=cs.tol, max_cycles=12)
        hist_ok = np.allclose(hist, rep.history, rtol=1e-12, atol=0)
        q.put((rank, lg, ok, hist_ok, cycles == rep.cycles))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, -1, False, False, repr(e)))


@pytest.mark.parametrize("name,world", [("cfg1_mini", 2), ("cfg1_mini_adj", 2), ("cfg0_deep", 2),
                                        ("cfg4_mini", 4)])
def test_slab_algorithm_gloo(name, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, lg, ok, hist_ok, cyc_ok in res:
        assert lg >= 1, (rank, cyc_ok)
        assert ok, f"rank {rank}: slab iterate differs from the single-domain oracle"
        assert hist_ok and cyc_ok is True, (rank, hist_ok, cyc_ok)
