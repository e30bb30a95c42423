"""Shared helpers for the general coarse-discretisation parity tests
(Galerkin P, bilinear transfers, FullST).

The same seeded inputs are generated here (golden-fixture generation against
the compiled reference) and on the GPU box (tests/test_gpu_general.py), and
bitwise outputs are compared through SHA-256 digests of their bytes, so the
committed fixture stays small.
"""
from __future__ import annotations

import hashlib
import zlib

import numpy as np

GOLDEN = "general.npz"


def digest(a) -> str:
    if hasattr(a, "cpu"):
        a = a.cpu().numpy()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def special_values(rng, n):
    """Gaussian values salted with exact +0, -0 and powers of two."""
    v = rng.standard_normal(n)
    idx = rng.choice(n, size=max(1, n // 16), replace=False)
    v[idx[0::3]] = 0.0
    v[idx[1::3]] = -0.0
    v[idx[2::3]] = 2.0 ** rng.integers(-20, 20, size=idx[2::3].size)
    return v


def level_inputs(name: str, ndofs: list[int]):
    """Per level (x, f, xc) -- xc on the next coarser level, None on the last --
    then the coarsest right-hand side; one fixed stream per case."""
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    out = []
    for l, n in enumerate(ndofs):
        x = special_values(rng, n)
        f = special_values(rng, n)
        xc = special_values(rng, ndofs[l + 1]) if l + 1 < len(ndofs) else None
        out.append((x, f, xc))
    f_coarsest = rng.standard_normal(ndofs[-1])
    return out, f_coarsest


def csr_to_stencil9(rp, ci, v, n_el, n_t):
    """A reference CSR level operator as (v9[9, nd], mask[nd]) (slot 3(dn+1)+(di+1))."""
    nn = n_el + 1
    nd = nn * (n_t + 1)
    rows = np.repeat(np.arange(nd), np.diff(rp))
    n, i = np.divmod(rows, nn)
    n2, i2 = np.divmod(ci.astype(np.int64), nn)
    dn, di = n2 - n, i2 - i
    assert np.all(np.abs(dn) <= 1) and np.all(np.abs(di) <= 1)
    slot = 3 * (dn + 1) + (di + 1)
    V = np.zeros((9, nd))
    V[slot, rows] = v
    M = np.zeros(nd, np.uint16)
    np.bitwise_or.at(M, rows, (1 << slot).astype(np.uint16))
    return V, M
