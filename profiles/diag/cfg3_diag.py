"""Diagnostic: cfg3 (adjoint, 1.07e9 DOFs) GPU vs C oracle: histories, field
difference, and the coarsest exact solve alone (GPU march vs the oracle's
Thomas march) on the full-size hierarchy's coarsest level."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch

    from oracle.pyoracle import Port
    from paper_2505_10168_b200 import configs as C
    from paper_2505_10168_b200 import stmg as S

    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    cfg = C.CONFIGS[name]()
    port = Port()
    dirs, _ = port.plan(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t, cfg.k, cfg.c, cfg.n_levels, strategy=cfg.strategy,
                        reassembly=cfg.reassembly, min_elements=cfg.min_elements, chi=cfg.chi, mat=cfg.mat)
    g = S.build_fine_grid(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t)
    g.k, g.c = cfg.k, cfg.c
    h = S.build_hierarchy(g, cfg.method, S.CoarseningPath([S.CoarseningDirection(int(d)) for d in dirs]))
    if cfg.adjoint:
        h = S.transposed_hierarchy(h)
    hp = port.hierarchy(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t, cfg.k, cfg.c, dirs, reassembly=cfg.reassembly,
                        adjoint=cfg.adjoint, chi=cfg.chi, mat=cfg.mat)
    L = h.n_levels() - 1
    nc = hp.ndofs(L)
    rng = np.random.default_rng(1)
    f = rng.standard_normal(nc)
    xg = torch.zeros(nc, dtype=torch.float64, device="cuda")
    h.coarsest_solve(torch.from_numpy(f).cuda(), xg)
    xo = hp.coarsest(f)
    xg = xg.cpu().numpy()
    print("coarsest", hp.shapes[L], "rel max diff GPU vs oracle", np.max(np.abs(xg - xo)) / np.max(np.abs(xo)))
    b = C.adjoint_uniform_rhs(cfg.n_el, cfg.n_t, cfg.L, cfg.t_T) if cfg.rhs == "adjoint_uniform" else \
        port.load_vector(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t, cfg.source_kind, cfg.source_params)
    for mc in (1, 2, 3):
        bt = torch.from_numpy(b).cuda()
        ut = torch.zeros_like(bt)
        rep = S.mg_solve(h, bt, ut, S.SolveOptions(nu=cfg.nu, tol=cfg.tol, max_cycles=mc))
        u = ut.cpu().numpy()
        del bt, ut
        uo, repo = hp.solve(b, nu=cfg.nu, tol=cfg.tol, max_cycles=mc)
        print(f"cycles={mc} gpu hist {rep.history} oracle hist {list(repo.history)}")
        print("  rel hist diff", np.abs(np.asarray(rep.history) - repo.history) / np.abs(repo.history),
              "field rel max diff", np.max(np.abs(u - uo)) / np.max(np.abs(uo)))


if __name__ == "__main__":
    main()
