"""Per-kernel cost inside a CUDA graph, per level of a BASELINE hierarchy.

K back-to-back single sweeps (or fused pairs) of one level are captured into
one CUDA graph (the library launches on a torch capture stream) and the graph
is replayed; time / K is what one such kernel costs inside the V-cycle graph,
launch gaps included, with no event nodes.  Compare with the per-level
in-graph event breakdown of solve_once.py (which adds timer overhead).

    python profiles/launch_floor.py --config cfg1 --k 200
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--k", type=int, default=200)
    ap.add_argument("--reps", type=int, default=5)
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
    out = []
    for l, lv in enumerate(h.levels[:-1]):
        n = lv.n_dofs
        # 512 doubles of tail padding: the bulk-copy kernel (mode 5) rounds row copies out
        f = torch.randn(n + 512, dtype=torch.float64, device="cuda")
        x = torch.randn(n + 512, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        row = {"level": l, "n_el": lv.n_el, "n_t": lv.n_t, "dofs": n}
        for name, pairs in (("sweep_us", False), ("pair_us", True), ("bulk_pair_us", 5), ("deep3_us", 3),
                            ("deep4_us", 4)):
            row[name] = graph_time(h, lambda: h.sweep_kernels(l, f, x, y, a.k, pairs), a.k, a.reps)
        nc = h.levels[l + 1].n_dofs
        fc = torch.empty(nc, dtype=torch.float64, device="cuda")
        row["restrict_us"] = graph_time(h, lambda: [h.restrict_residual(l, f, x, fc) for _ in range(a.k)],
                                        a.k, a.reps)
        out.append(row)
        print(json.dumps(row), flush=True)
    lv = h.levels[-1]
    f = torch.randn(lv.n_dofs, dtype=torch.float64, device="cuda")
    x = torch.zeros_like(f)
    k = max(a.k // 10, 5)
    print(json.dumps({"level": len(h.levels) - 1, "n_el": lv.n_el, "n_t": lv.n_t, "dofs": lv.n_dofs,
                      "coarsest_us": graph_time(h, lambda: [h.coarsest_solve(f, x) for _ in range(k)], k,
                                                a.reps)}), flush=True)


def graph_time(h, body, k, reps):
    """us per launch of `body` (k launches) captured into one CUDA graph on the hierarchy stream."""
    import torch

    s = torch.cuda.Stream()
    h.set_stream(s)
    with torch.cuda.stream(s):
        body()
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        body()
    h.set_stream(None)
    graph.replay()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        e1.synchronize()
        t = e0.elapsed_time(e1) * 1e3 / k
        best = t if best is None else min(best, t)
    return round(best, 2)


if __name__ == "__main__":
    main()
