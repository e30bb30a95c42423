"""Per-entry timings of a streamed sequence of config-2 solves (stmg_mg_solve_stream):
python profiles/stream_probe.py [--config cfg2] [--steps 8]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--steps", type=int, default=8)
    a = ap.parse_args()
    import torch

    from paper_2505_10168_b200 import configs as C
    from paper_2505_10168_b200 import stmg as S

    cfg = C.CONFIGS[a.config]()
    g = S.build_fine_grid(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t)
    g.k, g.c = cfg.k, cfg.c
    path = S.plan_coarsening(g, S.PlanRequest(n_levels=cfg.n_levels, strategy=S.PlanStrategy(cfg.strategy),
                                              reassembly=S.ReassemblyMethod(cfg.reassembly),
                                              min_elements=cfg.min_elements, chi=cfg.chi, mat=cfg.mat))
    h = S.build_hierarchy(g, cfg.method, path, chi=cfg.chi, mat=cfg.mat)
    b = torch.from_numpy(S.load_vector(g, kind=cfg.source_kind, params=cfg.source_params, masked=True)).pin_memory()
    u = torch.zeros_like(b).pin_memory()
    opts = S.SolveOptions(nu=cfg.nu, tol=cfg.tol, max_cycles=cfg.max_cycles)
    S.mg_solve_stream(h, [b] * 2, [u] * 2, opts, zero_guess=True)
    for k in (1, a.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rs = S.mg_solve_stream(h, [b] * k, [u] * k, opts, zero_guess=True) if k > 1 else [
            S.mg_solve(h, b, u, opts, zero_guess=True)]
        wall = time.perf_counter() - t0
        print(json.dumps({"steps": k, "wall_s": round(wall, 4), "per_step_s": round(wall / k, 4),
                          "entry_wall_s": [round(r.seconds, 4) for r in rs],
                          "entry_device_s": [round(r.device_seconds, 4) for r in rs]}))


if __name__ == "__main__":
    main()
