"""Time the exact coarsest solve of the cfg1 hierarchy (32 x 256 grid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_10168_b200 import configs as C  # noqa: E402
from paper_2505_10168_b200 import stmg as S  # noqa: E402

cfg = C.cfg1()
g = S.build_fine_grid(1, 1, cfg.n_el, cfg.n_t)
g.k, g.c = cfg.k, cfg.c
p = S.plan_coarsening(g, S.PlanRequest(n_levels=int(sys.argv[1]) if len(sys.argv) > 1 else 10,
                                       strategy=S.PlanStrategy.Contrast, reassembly=S.ReassemblyMethod.R))
h = S.build_hierarchy(g, "CR", p)
lv = h.levels[-1]
f = torch.rand(lv.n_dofs, dtype=torch.float64, device="cuda")
x = torch.zeros_like(f)
for _ in range(3):
    h.coarsest_solve(f, x)
t = time.perf_counter()
for _ in range(50):
    h.coarsest_solve(f, x)
print(f"coarsest {lv.n_el}x{lv.n_t}: {(time.perf_counter() - t) / 50 * 1e6:.1f} us per call (incl. launch + sync)")
