"""Same-process A/B of the V-cycle fusions (stmg_hierarchy_set_fusion) on a
BASELINE config: whole-solve device time per flag set, then one profiled solve
(every kernel timed by in-graph events) with the default fusions.

    python profiles/fusion_ab.py --config cfg2 [--solves 3] [--flags 0,1,2,3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--solves", type=int, default=3)
    ap.add_argument("--flags", default="0,1,2,3")
    ap.add_argument("--nu", type=int, default=None)
    ap.add_argument("--max-cycles", type=int, default=None)
    ap.add_argument("--profile", type=int, default=1)
    a = ap.parse_args()
    import torch

    from paper_2505_10168_b200 import configs as C
    from paper_2505_10168_b200 import stmg as S

    cfg = C.CONFIGS[a.config]()
    if a.nu is not None:
        cfg.nu = a.nu
    if a.max_cycles is not None:
        cfg.max_cycles = a.max_cycles
    g = S.build_fine_grid(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t)
    g.k, g.c = cfg.k, cfg.c
    path = S.plan_coarsening(g, S.PlanRequest(n_levels=cfg.n_levels, strategy=S.PlanStrategy(cfg.strategy),
                                              reassembly=S.ReassemblyMethod(cfg.reassembly),
                                              min_elements=cfg.min_elements, chi=cfg.chi, mat=cfg.mat))
    h = S.build_hierarchy(g, cfg.method, path, chi=cfg.chi, mat=cfg.mat)
    if cfg.adjoint:
        h = S.transposed_hierarchy(h)
    if cfg.rhs == "adjoint_uniform":
        bh = C.adjoint_uniform_rhs(cfg.n_el, cfg.n_t, cfg.L, cfg.t_T)
    else:
        bh = S.load_vector(g, kind=cfg.source_kind, params=cfg.source_params, masked=True)
    b = torch.from_numpy(bh).cuda()
    u = torch.zeros_like(b)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    opts = S.SolveOptions(nu=cfg.nu, tol=cfg.tol, max_cycles=cfg.max_cycles)
    out = {"config": cfg.name, "path": S.path_to_string(path), "ms": {}}
    flags = [int(f) for f in a.flags.split(",")]
    for rnd in range(2):  # two interleaved rounds against box drift
        for fl in flags:
            h.set_fusion(fl)
            for _ in range(2):
                u.zero_()
                S.mg_solve(h, b, u, opts)
            ts = []
            for _ in range(a.solves):
                flush.fill_(1.0)
                u.zero_()
                torch.cuda.synchronize()
                rep = S.mg_solve(h, b, u, opts)
                ts.append(rep.device_seconds * 1e3)
            out["ms"].setdefault(str(fl), []).extend(ts)
            out["cycles"] = rep.cycles
    out["ms_min"] = {k: min(v) for k, v in out["ms"].items()}
    print(json.dumps(out), flush=True)
    if a.profile:
        h.set_fusion(3)
        h.set_profiling(2)
        u.zero_()
        rep = S.mg_solve(h, b, u, opts)
        prof = h.profile()
        total = 0.0
        for l, lv in enumerate(h.levels):
            kinds = prof.get(l, {})
            t_l = sum(t for _, t in kinds.values())
            total += t_l
            desc = ", ".join(f"{k} {n}x{1e6 * t / n:.1f}us" for k, (n, t) in kinds.items())
            print(f"level {l}: {lv.n_el}x{lv.n_t} dofs={lv.n_dofs} in-graph {1e3 * t_l:.2f} ms  [{desc}]")
        np_, ns = rep.kernel_times.get("fine_norm_pass", (0, 0.0))
        if np_:
            print(f"level-0 norm passes {np_}x{1e3 * ns / np_:.3f} ms")
            total += ns
        print(f"sum of timed kernels {1e3 * total:.2f} ms vs profiled solve {1e3 * rep.device_seconds:.2f} ms")


if __name__ == "__main__":
    main()
