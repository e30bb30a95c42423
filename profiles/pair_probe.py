"""Fused-pair kernel probe (ncu target): one level of a BASELINE config, K
launches of the register-staged pair (mode 1) or the bulk-copy pair (mode 5).
python profiles/pair_probe.py --config cfg1 --level 0 --mode 5 --k 4"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--level", type=int, default=0)
    ap.add_argument("--mode", type=int, default=5)
    ap.add_argument("--k", type=int, default=4)
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
    n = h.levels[a.level].n_dofs
    f = torch.randn(n + 512, dtype=torch.float64, device="cuda")
    x = torch.randn(n + 512, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    h.sweep_kernels(a.level, f, x, y, a.k, a.mode)
    torch.cuda.synchronize()
    print("ok", n)


if __name__ == "__main__":
    main()
