"""Multi-process CPU model of the peer-memory ghost exchange's epoch protocol
(k_p2p_pull in paper_2505_10168_b200/csrc/stmg_dist.cuh), world 2 and 4.

Each process owns a time slab of two ping-pong level vectors in shared memory
(as the product's xa / xb) and runs the product's schedule: exchange the
current vector's ghost levels, then compute the other vector from it.  An
exchange follows the device protocol exactly: e = completed + 1; post e into
both neighbours' flag slots; wait until both neighbours posted >= e; pull the
ghost rows straight out of the neighbours' vectors; record e as completed.
Random delays between steps let the ranks drift apart.  The protocol claims one
handshake per exchange suffices (a vector is rewritten only after a later
barrier, which needs the puller's next post), so the result must equal the
single-domain computation bit for bit.  No GPU, no product library."""
import multiprocessing as mp
import random
import time

import numpy as np
import pytest

NT, NN, STEPS, DEPTH = 64, 33, 40, 2


def _step(prev, cur, lo, hi):
    """Stand-in stencil pass (rows [lo, hi) of the output): reads rows n-2..n+1
    of the input, i.e. two ghost levels below and one above the slab."""
    out = cur.copy()
    for n in range(lo, hi):
        a = prev[n - 2] if n >= 2 else 0.0
        b = prev[n - 1] if n >= 1 else 0.0
        c = prev[n + 1] if n + 1 < NT else 0.0
        out[n] = 0.25 * a + 0.5 * b + 0.125 * prev[n] + 0.0625 * c + 1.0
    return out


def _reference():
    x = [np.zeros((NT, NN)), np.zeros((NT, NN))]
    x[0][:] = np.arange(NT * NN, dtype=np.float64).reshape(NT, NN) % 7
    cur = 0
    for _ in range(STEPS):
        x[1 - cur] = _step(x[cur], x[1 - cur], 0, NT)
        cur = 1 - cur
    return x[cur]


def _worker(g, world, bufs, flags, seed, out_q):
    rng = random.Random(seed * 100 + g)
    b = [g * NT // world for g in range(world + 1)]
    lo, hi = b[g], b[g + 1]
    vec = [np.frombuffer(bb.get_obj(), dtype=np.float64).reshape(world, NT, NN) for bb in bufs]
    fl = np.frombuffer(flags.get_obj(), dtype=np.int64).reshape(world, 3)
    mine = [v[g] for v in vec]

    def exchange(which):
        e = fl[g, 0] + 1
        if g > 0:
            fl[g - 1, 2] = e  # I am the left rank's right neighbour
        if g < world - 1:
            fl[g + 1, 1] = e
        t0 = time.time()
        while (g > 0 and fl[g, 1] < e) or (g < world - 1 and fl[g, 2] < e):
            if time.time() - t0 > 30:
                raise RuntimeError("p2p model: wait timed out")
            time.sleep(0)
        time.sleep(rng.random() * 1e-3)
        if g > 0:  # leading ghosts from the left rank's rows [lo - DEPTH, lo)
            mine[which][lo - DEPTH:lo] = vec[which][g - 1][lo - DEPTH:lo]
        if g < world - 1:  # trailing ghost from the right rank's row hi
            mine[which][hi:hi + 1] = vec[which][g + 1][hi:hi + 1]
        fl[g, 0] = e

    try:
        cur = 0
        for _ in range(STEPS):
            exchange(cur)
            time.sleep(rng.random() * 1e-3)
            new = _step(mine[cur], mine[1 - cur], lo, hi)
            mine[1 - cur][lo:hi] = new[lo:hi]  # in-place write of the other ping-pong vector
            cur = 1 - cur
        out_q.put((g, mine[cur][lo:hi].copy()))
    except Exception as ex:  # pragma: no cover - reported to the parent
        out_q.put((g, repr(ex)))


@pytest.mark.parametrize("world", [2, 4])
def test_p2p_epoch_protocol_model(world):
    ctx = mp.get_context("fork")
    init = np.arange(NT * NN, dtype=np.float64).reshape(NT, NN) % 7
    bufs = [ctx.Array("d", world * NT * NN) for _ in range(2)]
    a0 = np.frombuffer(bufs[0].get_obj(), dtype=np.float64).reshape(world, NT, NN)
    a0[:] = init  # every rank's copy starts from the same data (its own rows matter)
    flags = ctx.Array("q", world * 3)
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(g, world, bufs, flags, 7, q)) for g in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=30)
    want = _reference()
    b = [g * NT // world for g in range(world + 1)]
    for g in range(world):
        assert not isinstance(res[g], str), res[g]
        assert np.array_equal(res[g], want[b[g]:b[g + 1]]), g
