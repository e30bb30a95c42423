"""One STMG solve of a BASELINE config through the public API (target for
ncu launch lists): python profiles/solve_once.py --config cfg1 [--solves 1]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--solves", type=int, default=1)
    ap.add_argument("--n-levels", type=int, default=None)
    ap.add_argument("--nu", type=int, default=None)
    a = ap.parse_args()
    import torch

    from paper_2505_10168_b200 import configs as C
    from paper_2505_10168_b200 import stmg as S

    cfg = C.CONFIGS[a.config]()
    if a.n_levels:
        cfg.n_levels = a.n_levels
    if a.nu is not None:
        cfg.nu = a.nu
    g = S.build_fine_grid(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t)
    g.k, g.c = cfg.k, cfg.c
    path = S.plan_coarsening(g, S.PlanRequest(n_levels=cfg.n_levels, strategy=S.PlanStrategy(cfg.strategy),
                                              reassembly=S.ReassemblyMethod(cfg.reassembly),
                                              min_elements=cfg.min_elements, chi=cfg.chi, mat=cfg.mat))
    h = S.build_hierarchy(g, cfg.method, path, chi=cfg.chi, mat=cfg.mat)
    b = torch.from_numpy(S.load_vector(g, kind=cfg.source_kind, params=cfg.source_params, masked=True)).cuda()
    ap_prof = os.environ.get("STMG_PROFILE_LEVELS") == "1"
    for k in range(a.solves):
        if ap_prof and k == a.solves - 1:
            h.set_profiling(2)
        u = torch.zeros_like(b)
        rep = S.mg_solve(h, b, u, S.SolveOptions(nu=cfg.nu, tol=cfg.tol, max_cycles=cfg.max_cycles))
    print(f"{cfg.name} path={S.path_to_string(path)} cycles={rep.cycles} seconds={rep.seconds:.4f} "
          f"device_seconds={rep.device_seconds:.4f} launches={rep.kernel_launches}")
    prof = h.profile() if ap_prof else {}
    total = 0.0
    for l, lv in enumerate(h.levels):
        kinds = prof.get(l, {})
        t_l = sum(t for _, t in kinds.values())
        total += t_l
        desc = ", ".join(f"{k} {n}x{1e6 * t / n:.1f}us" for k, (n, t) in kinds.items())
        print(f"level {l}: {lv.n_el}x{lv.n_t} dofs={lv.n_dofs} in-graph {1e3 * t_l:.2f} ms  [{desc}]")
    if prof:
        print(f"sum of in-graph kernel time {1e3 * total:.2f} ms vs solve {1e3 * rep.device_seconds:.2f} ms")


if __name__ == "__main__":
    main()
