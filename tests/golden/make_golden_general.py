"""Golden fixtures for the general coarse discretisations, from the UNMODIFIED
reference (oracle/_ref):  python tests/golden/make_golden_general.py

For every case in tests/_cases.GENERAL it records, computed by the reference:
  * each level operator's bytes digest (CSR re-laid out as a 9-point stencil);
  * digests of residual, 3 Jacobi sweeps, R r and x + P xc on seeded inputs
    (tests/_general.level_inputs);
  * the coarsest exact solve of a seeded right-hand side;
  * a full mg_solve from u = 0: status, cycles, history and u.
Writes tests/golden/general.npz.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Port, Ref  # noqa: E402
from tests._cases import GENERAL_CASES, case  # noqa: E402
from tests._general import GOLDEN, csr_to_stencil9, digest, level_inputs  # noqa: E402


def level_dims(cs):
    ne, nt = cs.n_el, cs.n_t
    out = [(ne, nt)]
    for d in cs.dirs:
        ne, nt = (ne // 2 if d != 1 else ne), (nt // 2 if d != 0 else nt)
        out.append((ne, nt))
    return out


def main():
    ref, port = Ref(), Port()
    out = {}
    for name in GENERAL_CASES:
        cs = case(name)
        h = ref.hierarchy(cs.L, cs.tT, cs.n_el, cs.n_t, cs.k, cs.c, cs.dirs, method=cs.method,
                          adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat)
        dims = level_dims(cs)
        nds = [h.ndofs(l) for l in range(h.n_levels)]
        ins, fco = level_inputs(name, nds)
        for l, (x, f, xc) in enumerate(ins):
            rp, ci, v, inv = h.csr(l)
            V, M = csr_to_stencil9(rp, ci, v, *dims[l])
            out[f"{name}__op{l}"] = np.array([digest(V), digest(M), digest(inv)])
            r = h.residual(l, f, x)
            ks = [digest(r), digest(h.sweeps(l, f, x, 3))]
            if xc is not None:
                ks += [digest(h.restrict(l, r)), digest(h.prolong_add(l, xc, x))]
            out[f"{name}__k{l}"] = np.array(ks)
        out[f"{name}__coarsest"] = h.coarsest(fco)
        b = cs.rhs_vector(port)
        u, rep = h.solve(b, nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
        out[f"{name}__u"] = u
        out[f"{name}__history"] = rep.history
        out[f"{name}__meta"] = np.array([rep.status, rep.cycles, int(rep.absolute_norms)])
        print(f"{name}: status {rep.status}, cycles {rep.cycles}, final {rep.history[-1]:.3e}")
    np.savez_compressed(os.path.join(HERE, GOLDEN), **out)


if __name__ == "__main__":
    main()
