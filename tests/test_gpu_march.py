"""The streaming fused pair (k_march2: each warp marches its strip through a
segment of rows, x / f of the next rows in a register queue; opt-in through
STMG_MARCH_DOFS, measured slower than k_lean2x2) against the tiled pair and,
through whole solves, against the CPU oracle.  Bar: bit-identical."""
import numpy as np
import pytest

from tests._cases import case
from tests.test_gpu_bulk import S, hier, torch  # noqa: F401  (fixtures)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["cfg1_mini", "cfg1_mini_adj", "wide_short", "cfg0", "tiny", "space_first"])
def test_march_pair_bitwise(torch, S, port, name, monkeypatch):
    cs = case(name)
    ha = hier(S, cs, port)
    monkeypatch.setenv("STMG_MARCH_DOFS", "1")  # every level (read at hierarchy build)
    hb = hier(S, cs, port)
    rng = np.random.default_rng(11)
    for l, lv in enumerate(ha.levels):
        n = lv.n_dofs
        f = torch.from_numpy(rng.standard_normal(n)).cuda()
        x0 = torch.from_numpy(rng.standard_normal(n)).cuda()
        xa, ya = x0.clone(), torch.zeros_like(x0)
        xb, yb = x0.clone(), torch.zeros_like(x0)
        ha.sweep_kernels(l, f, xa, ya, 3, True)  # tiled pairs: x -> y -> x -> y
        hb.sweep_kernels(l, f, xb, yb, 3, True)  # streaming pairs
        torch.cuda.synchronize()
        assert torch.equal(ya, yb), f"level {l}"
        assert torch.equal(xa, xb), f"level {l}"


@pytest.mark.parametrize("name", ["cfg1_mini", "cfg1_mini_adj", "cfg4_mini", "wide_coarsest_adj"])
def test_solves_with_march_pairs_match_oracle(torch, S, port, name, monkeypatch):
    from tests.test_gpu_parity import check_solve, port_hier

    monkeypatch.setenv("STMG_MARCH_DOFS", "1")
    cs = case(name)
    h = hier(S, cs, port)
    b = cs.rhs_vector(port)
    bt = torch.from_numpy(b).cuda()
    ut = torch.zeros_like(bt)
    rep = S.mg_solve(h, bt, ut, S.SolveOptions(nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles))
    u_p, rep_p = port_hier(port, cs).solve(b, nu=cs.nu, tol=cs.tol, max_cycles=cs.max_cycles)
    check_solve(rep, ut.cpu().numpy(), rep_p, u_p)
