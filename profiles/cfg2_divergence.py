"""BASELINE config 2 convergence table: the reference algorithm's
behaviour on the i.i.d. 1e4-contrast design for smoothing nu and resolution
guard M, at full size on the GPU (--where gpu, 1.07e9 DOFs) or at reduced size
through the compiled reference itself (--where ref, default 1024 x 2048).

Each entry: the planned path, then mg_solve from u = 0 with the reference's
stop rule (tol 1e-10, div_tol 1e9) and at most --max-cycles V-cycles: status,
cycles, the convergence factor (r_N / r_0)^(1/N), the last relative residual.

    python profiles/cfg2_divergence.py --where gpu > profiles/round2_cfg2_divergence_gpu.jsonl
    python profiles/cfg2_divergence.py --where ref > profiles/round2_cfg2_divergence_ref.jsonl
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--where", default="gpu", choices=["gpu", "ref"])
    ap.add_argument("--n-el", type=int, default=None)
    ap.add_argument("--n-t", type=int, default=None)
    ap.add_argument("--nus", default="1,5,10,20")
    ap.add_argument("--guards", default="0,64,256,full")
    ap.add_argument("--max-cycles", type=int, default=20)
    ap.add_argument("--n-levels", type=int, default=18)
    a = ap.parse_args()
    from paper_2505_10168_b200 import configs as C

    kw = {}
    if a.where == "ref":
        kw = {"n_el": a.n_el or 1024, "n_t": a.n_t or 2048}
    elif a.n_el:
        kw = {"n_el": a.n_el, "n_t": a.n_t}
    base = C.cfg2(**kw)
    if a.where == "gpu":
        import torch

        from paper_2505_10168_b200 import stmg as S

        g = S.build_fine_grid(base.L, base.t_T, base.n_el, base.n_t)
        g.k, g.c = base.k, base.c
        b = torch.from_numpy(S.load_vector(g, kind=base.source_kind, params=base.source_params, masked=True)).cuda()
        u = torch.zeros_like(b)
    else:
        from oracle.pyoracle import Ref

        ref = Ref()
        b = ref.load_vector(base.L, base.t_T, base.n_el, base.n_t, base.source_kind, base.source_params)
    for gs in a.guards.split(","):
        M = base.n_el if gs == "full" else int(gs)
        if a.where == "gpu":
            path = None
            for nl in range(a.n_levels, 1, -1):  # the deepest plan the guard allows
                req = S.PlanRequest(n_levels=nl, strategy=S.PlanStrategy(base.strategy),
                                    reassembly=S.ReassemblyMethod(base.reassembly), min_elements=M)
                try:
                    path = S.plan_coarsening(g, req)
                    break
                except Exception:
                    continue
            if path is None:
                print(json.dumps({"M": M, "error": "no legal plan"}), flush=True)
                continue
            dirs = [int(d) for d in path.dirs]
            h = S.build_hierarchy(g, base.method, path)
        else:
            dirs = None
            for nl in range(a.n_levels, 1, -1):  # the deepest plan the guard allows
                try:
                    dirs, _ = ref.plan(base.L, base.t_T, base.n_el, base.n_t, base.k, base.c, nl,
                                       strategy=base.strategy, reassembly=base.reassembly, min_elements=M)
                    break
                except Exception:
                    continue
            if dirs is None:
                print(json.dumps({"M": M, "error": "no legal plan"}), flush=True)
                continue
            dirs = [int(d) for d in dirs]
            h = ref.hierarchy(base.L, base.t_T, base.n_el, base.n_t, base.k, base.c, dirs, method=base.method)
        path_s = ",".join("x" if d == 0 else "t" for d in dirs)
        for nu in (int(v) for v in a.nus.split(",")):
            t0 = time.perf_counter()
            if a.where == "gpu":
                u.zero_()
                rep = S.mg_solve(h, b, u, S.SolveOptions(nu=nu, tol=1e-10, max_cycles=a.max_cycles))
                status, cycles, factor, hist = S.status_name(rep.status), rep.cycles, rep.factor, rep.history
            else:
                _, rep = h.solve(b, nu=nu, tol=1e-10, max_cycles=a.max_cycles)
                status = {0: "converged", 1: "max-cycles", 2: "diverged"}[rep.status]
                cycles, factor, hist = rep.cycles, rep.factor, list(rep.history)
            print(json.dumps({"where": a.where, "grid": f"{base.n_el}x{base.n_t}", "M": M, "path": path_s,
                              "levels": len(dirs) + 1, "nu": nu, "status": status, "cycles": cycles,
                              "factor": factor, "last_rel_residual": hist[-1],
                              "seconds": round(time.perf_counter() - t0, 3)}), flush=True)


if __name__ == "__main__":
    main()
