"""One launch of each level-kernel form on one large level (the ncu target):
single sweep, fused pair, residual restriction (stored / virtual zero iterate),
fused prolong-sweep (stored / virtual), and the fine down-pass.  Default grid
16384 x 8192 (1.3e8 DOFs, 1.07 GB per vector, far beyond L2); x step.

    ncu --set full --clock-control none -o prof python profiles/kernel_probe.py
    python profiles/kernel_probe.py --time      (CUDA-event times, no profiler)
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-el", type=int, default=16384)
    ap.add_argument("--n-t", type=int, default=8192)
    ap.add_argument("--dir", type=int, default=0)
    ap.add_argument("--adjoint", action="store_true")
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--tiles", type=int, default=0, help="force 4- or 2-level time tiles (0: default tiling)")
    ap.add_argument("--only", default="", help="comma-separated subset of the forms")
    a = ap.parse_args()
    import torch

    from paper_2505_10168_b200 import configs as C
    from paper_2505_10168_b200 import stmg as S

    cfg = C.cfg2(n_el=a.n_el, n_t=a.n_t)
    g = S.build_fine_grid(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t)
    g.k, g.c = cfg.k, cfg.c
    path = S.CoarseningPath([S.CoarseningDirection(a.dir), S.CoarseningDirection.TimeT])
    h = S.build_hierarchy(g, cfg.method, path, chi=cfg.chi, mat=cfg.mat)
    if a.adjoint:
        h = S.transposed_hierarchy(h)
    if a.tiles:
        h.set_tiling(small_dofs=10 ** 15, tiny_dofs=10 ** 15 if a.tiles == 2 else 1)
    H = S.LevelHierarchy
    n0, n1 = h.levels[0].n_dofs, h.levels[1].n_dofs
    dev = torch.device("cuda:0")
    f = torch.randn(n0, dtype=torch.float64, device=dev)
    x = torch.randn(n0, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    fc = torch.empty(n1, dtype=torch.float64, device=dev)
    xc = torch.randn(n1, dtype=torch.float64, device=dev)
    w = torch.empty_like(x)
    torch.cuda.synchronize()
    forms = {
        "sweep": lambda: h.sweep_kernels(0, f, x, y, 1, False),
        "pair": lambda: h.sweep_kernels(0, f, x, y, 1, True),
        "restrict": lambda: h.restrict_residual(0, f, x, fc),
        "restrict_zero": lambda: h.fused_kernel(0, H.FUSED_ZERO_RESTRICT, f, fc=fc),
        "prolong_sweep_zero": lambda: h.fused_kernel(0, H.FUSED_ZERO_PROLONG_SWEEP, f, xc=xc, y=y),
        "down": lambda: h.fused_kernel(0, H.FUSED_FINE_DOWN, f, x=x, y=y, fc=fc),
        "norm_sweep": lambda: h.fused_kernel(0, H.FUSED_NORM_SWEEP, f, x=x, y=y),
        "prolong_sweep": lambda: h.fused_kernel(0, H.FUSED_PROLONG_SWEEP, f, x=x, xc=xc, y=y),
        "pair_zero": lambda: h.fused_kernel(0, H.FUSED_ZERO_PAIR, f, y=y),
        "up": lambda: h.fused_kernel(0, H.FUSED_FINE_UP, f, x=x, xc=xc, y=y, fc=w),
    }
    # algorithmic bytes per fine DOF (coarse vectors are half size: 4 B per fine DOF)
    bytes_per_dof = {"sweep": 24, "pair": 24, "restrict": 20, "restrict_zero": 12, "prolong_sweep_zero": 20,
                     "down": 28, "norm_sweep": 24, "pair_zero": 16, "prolong_sweep": 28, "up": 36}
    if a.only:
        forms = {k: v for k, v in forms.items() if k in a.only.split(",")}
    if not a.time:
        for fn in forms.values():
            fn()
        torch.cuda.synchronize()
        return
    out = {"grid": f"{a.n_el}x{a.n_t}", "dofs": n0, "dir": a.dir, "adjoint": a.adjoint, "tiles": a.tiles or 8}
    st = torch.cuda.current_stream()
    for name, fn in forms.items():
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = None
        for _ in range(a.reps):
            e0.record(st)
            fn()
            e1.record(st)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        out[name] = {"ms": round(best, 4), "GBps": round(bytes_per_dof[name] * n0 / best / 1e6, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
