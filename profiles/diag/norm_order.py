"""Diagnostic: where does the cfg2/cfg3 first-cycle history spread between the
GPU and the C oracle come from?  After one V-cycle from u = 0 (fields agree to
~1e-15), the residual b - J u is evaluated once by the oracle (the reference's
row arithmetic) and its 2-norm summed three ways: the reference's sequential
4-lane order (or_norm2, proj/src/kernels/kernels.cpp:23-31), numpy's pairwise
sum, and an exact sum (math.fsum over per-chunk fsums).  The GPU reports the
same residual through a block tree."""
import math
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
    b = C.adjoint_uniform_rhs(cfg.n_el, cfg.n_t, cfg.L, cfg.t_T) if cfg.rhs == "adjoint_uniform" else \
        port.load_vector(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t, cfg.source_kind, cfg.source_params)
    bt = torch.from_numpy(b).cuda()
    ut = torch.zeros_like(bt)
    rep = S.mg_solve(h, bt, ut, S.SolveOptions(nu=cfg.nu, tol=cfg.tol, max_cycles=1))
    u = ut.cpu().numpy()
    del bt, ut
    nb_seq = port.norm2(b)
    r = hp.residual(0, b, u)
    seq = port.norm2(r) / nb_seq
    pair = float(np.linalg.norm(r)) / float(np.linalg.norm(b))
    sq = r * r
    exact_ss = math.fsum(math.fsum(sq[k:k + (1 << 24)].tolist()) for k in range(0, sq.size, 1 << 24))
    sqb = b * b
    exact_bb = math.fsum(math.fsum(sqb[k:k + (1 << 24)].tolist()) for k in range(0, sqb.size, 1 << 24))
    exact = math.sqrt(exact_ss) / math.sqrt(exact_bb)
    print(f"{name}: GPU history[1] {rep.history[1]!r}")
    print(f"  residual of the GPU iterate, reference 4-lane order {seq!r} rel to exact {seq / exact - 1:.3e}")
    print(f"  numpy pairwise {pair!r} rel to exact {pair / exact - 1:.3e}")
    print(f"  exact (fsum) {exact!r};  GPU rel to exact {rep.history[1] / exact - 1:.3e}")


if __name__ == "__main__":
    main()
