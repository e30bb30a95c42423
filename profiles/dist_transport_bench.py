"""Ghost-exchange transports of the time-slab path on ONE GPU (loopback: all
ranks in this process, run one after another): BASELINE config 1 solved to
1e-10 with world W in {2, 4, 8}, exchanges by device copies ("loopback") or by
the peer-memory pull kernels behind the epoch barrier ("p2p", STMG_DIST_P2P=1).
Every rank's kernels serialise on one GPU, so the time is W slabs of work plus
the exchange overhead; the difference between transports is the cost of the
exchange mechanism itself.  Also checks the iterates are bitwise equal.

    python profiles/dist_transport_bench.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np

    import bench
    from paper_2505_10168_b200 import configs as C
    from paper_2505_10168_b200 import stmg as S

    cfg = C.CONFIGS["cfg1"]()
    g = S.build_fine_grid(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t)
    g.k, g.c = cfg.k, cfg.c
    req = S.PlanRequest(n_levels=cfg.n_levels, lambda_crit=cfg.lambda_crit, strategy=S.PlanStrategy(cfg.strategy),
                        reassembly=S.ReassemblyMethod(cfg.reassembly), min_elements=cfg.min_elements,
                        chi=cfg.chi, mat=cfg.mat)
    path = S.plan_coarsening(g, req)
    b = bench.rhs_for(cfg, S, g)
    opts = S.SolveOptions(nu=cfg.nu, omega=cfg.omega, tol=cfg.tol, div_tol=cfg.div_tol, max_cycles=cfg.max_cycles)
    ref = None
    for world in (2, 4, 8):
        for tr in ("loopback", "p2p"):
            if tr == "p2p":
                os.environ["STMG_DIST_P2P"] = "1"
            else:
                os.environ.pop("STMG_DIST_P2P", None)
            dh = S.build_dist_hierarchy(g, cfg.method, path, world, chi=cfg.chi, mat=cfg.mat, min_slab=16)
            assert dh.transport == tr
            times = []
            for _ in range(4):
                u = np.zeros_like(b)
                t0 = time.perf_counter()
                r = S.mg_solve_dist(dh, b, u, opts)
                times.append(time.perf_counter() - t0)
            if ref is None:
                ref = u.copy()
            same = bool(np.array_equal(ref.view(np.uint64), u.view(np.uint64)))
            print(json.dumps({"world": world, "transport": tr, "cycles": r.cycles,
                              "solve_ms_best": round(1e3 * min(times[1:]), 3),
                              "bitwise_equal_to_world2_loopback": same, "n_distributed": dh.n_distributed}),
                  flush=True)
            del dh


if __name__ == "__main__":
    main()
