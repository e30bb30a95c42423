"""Generate golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run here (where /root/reference exists):  python tests/golden/make_golden.py [--full]

Writes tests/golden/*.npz / *.json.  The GPU box has no /root/reference, so
GPU tests pin against these committed outputs of the reference itself.
Contents:
  plans.json            reference plan_coarsening paths + indicators for every
                        BASELINE config at full size (and the test cases)
  <case>.npz            history, cycles, status of a reference mg_solve and u
                        (u itself up to 40k DOFs, else u[::97] and per-level sums)
  cfg1_full.npz (--full) history, cycles, status and per-time-level sums of u
                        for BASELINE config 1 at full size (4.2 M DOFs)
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Port, Ref  # noqa: E402
from paper_2505_10168_b200 import configs as C  # noqa: E402
from tests._cases import case  # noqa: E402

GOLDEN_CASES = ["cfg0", "cfg1_mini", "cfg1_mini_adj", "cfg2_mini", "cfgD", "time_first", "cfg4_mini"]


def plans(ref):
    out = {}
    for name, cfg in (("cfg0", C.cfg0()), ("cfg1", C.cfg1()), ("cfg2", C.cfg2()), ("cfg4", C.cfg4())):
        dirs, ind = ref.plan(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t, cfg.k, cfg.c, cfg.n_levels,
                             lambda_crit=cfg.lambda_crit, strategy=cfg.strategy,
                             reassembly=cfg.reassembly, min_elements=cfg.min_elements, chi=cfg.chi,
                             mat=cfg.mat)
        out[name] = {"n_levels": cfg.n_levels, "strategy": cfg.strategy, "reassembly": cfg.reassembly,
                     "min_elements": cfg.min_elements, "dirs": [int(d) for d in dirs],
                     "indicators": [float(v).hex() for v in ind]}
    return out


def solve_case(ref, port, name):
    cs = case(name)
    dirs = cs.plan(port)
    b = cs.rhs_vector(port)
    h = ref.hierarchy(cs.L, cs.tT, cs.n_el, cs.n_t, cs.k, cs.c, dirs, method=cs.method,
                      adjoint=cs.adjoint, chi=cs.chi, mat=cs.mat)
    u, rep = h.solve(b, nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    out = dict(history=rep.history, cycles=rep.cycles, status=rep.status,
               dirs=np.asarray(dirs, np.int32))
    if u.size <= 40000:
        out["u"] = u
    else:  # keep fixtures small: a fixed strided sample and per-level sums
        out["u_sample"] = u[::97]
        out["level_sums"] = u.reshape(cs.n_t + 1, cs.n_el + 1).sum(axis=1)
    return out


def cfg1_full(ref, port):
    cfg = C.cfg1()
    dirs, _ = ref.plan(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t, cfg.k, cfg.c, cfg.n_levels,
                       strategy=cfg.strategy, reassembly=cfg.reassembly, chi=cfg.chi, mat=cfg.mat)
    b = ref.load_vector(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t, cfg.source_kind, cfg.source_params)
    h = ref.hierarchy(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t, cfg.k, cfg.c, dirs, method=cfg.method)
    t0 = time.time()
    u, rep = h.solve(b, nu=cfg.nu, tol=cfg.tol, max_cycles=cfg.max_cycles)
    secs = time.time() - t0
    U = u.reshape(cfg.n_t + 1, cfg.n_el + 1)
    return dict(history=rep.history, cycles=rep.cycles, status=rep.status,
                level_sums=U.sum(axis=1), level_max=np.abs(U).max(axis=1),
                node_sums=U.sum(axis=0), u_max=np.abs(u).max(), dirs=np.asarray(dirs, np.int32),
                ref_seconds=secs, ref_build_seconds=h.build_seconds)


OPT_SMALL = dict(L=1.0, tT=1.0, n_el=64, n_t=128, mat=(1e-3, 1.0, 1.0, 1.0, 3.0, 2.0), method="CR",
                 strategy=3, n_levels=6, max_iterations=8, nu=5, tol=1e-8, stable_iterations=100)


def opt_small(ref):
    o = dict(OPT_SMALL)
    r = ref.optimise(o.pop("L"), o.pop("tT"), o.pop("n_el"), o.pop("n_t"), o.pop("mat"), **o)
    return dict(chi=r["chi"], records=r["records"], theta=r["theta"])


def cfg1_adj_full(ref):
    """Adjoint solve (transposed hierarchy) on the full config-1 grid and design with the
    config-3 right-hand side (dx*dt at unmasked DOFs): the adjoint path at full size."""
    cfg = C.cfg1()
    dirs, _ = ref.plan(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t, cfg.k, cfg.c, cfg.n_levels,
                       strategy=cfg.strategy, reassembly=cfg.reassembly, chi=cfg.chi, mat=cfg.mat)
    c = C.adjoint_uniform_rhs(cfg.n_el, cfg.n_t, cfg.L, cfg.t_T)
    h = ref.hierarchy(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t, cfg.k, cfg.c, dirs, method=cfg.method, adjoint=True)
    lam, rep = h.solve(c, nu=cfg.nu, tol=cfg.tol, max_cycles=cfg.max_cycles)
    U = lam.reshape(cfg.n_t + 1, cfg.n_el + 1)
    return dict(history=rep.history, cycles=rep.cycles, status=rep.status, level_sums=U.sum(axis=1),
                level_max=np.abs(U).max(axis=1), node_sums=U.sum(axis=0), u_max=np.abs(lam).max(),
                dirs=np.asarray(dirs, np.int32), ref_seconds=rep.seconds)


def main():
    ref, port = Ref(), Port()
    if "--adj-only" in sys.argv:  # only the adjoint full-size fixture
        np.savez_compressed(os.path.join(HERE, "cfg1_adj_full.npz"), **cfg1_adj_full(ref))
        print("wrote cfg1_adj_full")
        return
    np.savez_compressed(os.path.join(HERE, "opt_small.npz"), **opt_small(ref))
    with open(os.path.join(HERE, "plans.json"), "w") as fh:
        json.dump(plans(ref), fh, indent=1)
    for name in GOLDEN_CASES:
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **solve_case(ref, port, name))
        print("wrote", name)
    if "--full" in sys.argv:
        np.savez_compressed(os.path.join(HERE, "cfg1_full.npz"), **cfg1_full(ref, port))
        print("wrote cfg1_full")
    if "--full" in sys.argv or "--adj" in sys.argv:
        np.savez_compressed(os.path.join(HERE, "cfg1_adj_full.npz"), **cfg1_adj_full(ref))
        print("wrote cfg1_adj_full")


if __name__ == "__main__":
    main()
