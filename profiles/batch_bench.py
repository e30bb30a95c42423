"""Replica throughput: K independent solves of a small BASELINE-shaped problem
run one after another vs concurrently (stmg_mg_solve_batch, one stream each).
python profiles/batch_bench.py [--config cfg0 --replicas 32]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg0")
    ap.add_argument("--replicas", type=int, default=32)
    ap.add_argument("--n-levels", type=int, default=None)
    a = ap.parse_args()
    import torch

    from paper_2505_10168_b200 import configs as C
    from paper_2505_10168_b200 import stmg as S

    cfg = C.CONFIGS[a.config]()
    if a.n_levels:
        cfg.n_levels = a.n_levels
    g = S.build_fine_grid(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t)
    g.k, g.c = cfg.k, cfg.c
    path = S.plan_coarsening(g, S.PlanRequest(n_levels=cfg.n_levels, strategy=S.PlanStrategy(cfg.strategy),
                                              reassembly=S.ReassemblyMethod(cfg.reassembly),
                                              min_elements=cfg.min_elements, chi=cfg.chi, mat=cfg.mat))
    hs = [S.build_hierarchy(g, cfg.method, path, chi=cfg.chi, mat=cfg.mat) for _ in range(a.replicas)]
    b = S.load_vector_device(g, kind=cfg.source_kind, params=cfg.source_params)
    opts = S.SolveOptions(nu=cfg.nu, tol=cfg.tol, max_cycles=cfg.max_cycles)
    us = [torch.zeros_like(b) for _ in hs]
    S.mg_solve_batch(hs, [b] * len(hs), us, opts)  # warm-up (graph capture)
    for u in us:
        u.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for h, u in zip(hs, us):
        rep = S.mg_solve(h, b, u, opts)
    torch.cuda.synchronize()
    seq = time.perf_counter() - t0
    for u in us:
        u.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = S.mg_solve_batch(hs, [b] * len(hs), us, opts)
    torch.cuda.synchronize()
    bat = time.perf_counter() - t0
    print(json.dumps({"config": a.config, "replicas": a.replicas, "dofs": g.n_dofs(), "cycles": rep.cycles,
                      "sequential_s": seq, "batched_s": bat, "speedup": seq / bat,
                      "solves_per_s_batched": a.replicas / bat,
                      "same_cycles": all(r.cycles == rep.cycles for r in reps)}))


if __name__ == "__main__":
    main()
