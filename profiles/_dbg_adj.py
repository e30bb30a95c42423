import sys, numpy as np, torch
sys.path.insert(0, '.')
from tests._cases import case
from tests.test_gpu_parity import gpu_hier, port_hier, special_values, bits
from oracle.pyoracle import Port
from paper_2505_10168_b200 import stmg as S
port = Port()
cs = case("cfg1_mini_adj")
h = gpu_hier(S, cs, port); h.set_march(1)
hp = port_hier(port, cs)
rng = np.random.default_rng(23)
l = 0
n = hp.ndofs(l)
x, f = special_values(rng, n), special_values(rng, n)
xt, ft = torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda()
y = torch.full_like(xt, np.nan)
h.sweep_kernels(l, ft, xt, y, 1, False, 0.5); torch.cuda.synchronize()
want = hp.sweeps(l, f, x, 1, 0.5)
bad = np.nonzero(bits(y) != bits(want))[0]
lv = h.levels[l]; nn = lv.n_el + 1
print("level", lv.n_el, lv.n_t, "bad", bad.size, "of", n)
rows = np.unique(bad // nn); cols = np.unique(bad % nn)
print("rows", rows[:20], rows[-5:], "cols", cols[:20], cols[-5:])
