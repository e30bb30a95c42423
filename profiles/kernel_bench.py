"""Kernel microbenchmark: fine-level Jacobi sweeps (and the other V-cycle
kernels) on a BASELINE-sized grid, timed with CUDA events on the hierarchy's
stream.  Used for the roofline numbers in profiles/*.md and as the target
command for ncu captures.

    python profiles/kernel_bench.py --n-el 16384 --n-t 65536 --sweeps 20
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
    ap.add_argument("--n-el", type=int, default=16384)
    ap.add_argument("--n-t", type=int, default=65536)
    ap.add_argument("--sweeps", type=int, default=20)
    ap.add_argument("--adjoint", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2505_10168_b200 import configs as C
    from paper_2505_10168_b200 import stmg as S

    cfg = C.CONFIGS[args.config](n_el=args.n_el, n_t=args.n_t)
    g = S.build_fine_grid(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t)
    g.k, g.c = cfg.k, cfg.c
    # one x step and one t step so that both transfer kernels exist
    path = S.CoarseningPath([S.CoarseningDirection.SpaceX, S.CoarseningDirection.TimeT])
    h = S.build_hierarchy(g, cfg.method, path, chi=cfg.chi, mat=cfg.mat)
    if args.adjoint:
        h = S.transposed_hierarchy(h)
    st = torch.cuda.Stream()
    h.set_stream(st)
    n0 = h.levels[0].n_dofs
    n1 = h.levels[1].n_dofs
    with torch.cuda.stream(st):
        f = torch.randn(n0, dtype=torch.float64, device="cuda")
        x = torch.randn(n0, dtype=torch.float64, device="cuda")
        fc = torch.empty(n1, dtype=torch.float64, device="cuda")
        xc = torch.randn(n1, dtype=torch.float64, device="cuda")
    st.synchronize()
    out = {"n_dofs": n0, "adjoint": args.adjoint}

    def timed(fn, reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        st.synchronize()
        best = None
        for _ in range(reps):
            e0.record(st)
            fn()
            e1.record(st)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        return best

    y = torch.empty_like(x)
    ms = timed(lambda: h.sweep_kernels(0, f, x, y, args.sweeps, False), args.reps)
    per = ms / args.sweeps
    out["sweep_ms"] = per
    out["sweep_GBps"] = 24.0 * n0 / (per * 1e-3) / 1e9
    out["sweep_dof_updates_per_s"] = n0 / (per * 1e-3)
    ms = timed(lambda: h.sweep_kernels(0, f, x, y, args.sweeps, True), args.reps)
    per = ms / args.sweeps
    out["sweep_pair_ms"] = per
    out["sweep_pair_GBps"] = 24.0 * n0 / (per * 1e-3) / 1e9
    out["sweep_pair_dof_updates_per_s"] = 2 * n0 / (per * 1e-3)
    ms = timed(lambda: h.sweep_kernels(0, f, x, y, args.sweeps, 5), args.reps)
    per = ms / args.sweeps
    out["bulk_pair_ms"] = per
    out["bulk_pair_GBps"] = 24.0 * n0 / (per * 1e-3) / 1e9
    out["bulk_pair_dof_updates_per_s"] = 2 * n0 / (per * 1e-3)
    ms = timed(lambda: h.restrict_residual(0, f, x, fc), args.reps)
    out["restrict_x_ms"] = ms
    out["restrict_x_GBps"] = (16.0 * n0 + 8.0 * n1) / (ms * 1e-3) / 1e9
    ms = timed(lambda: h.prolong_add(0, xc, x), args.reps)
    out["prolong_x_ms"] = ms
    out["prolong_x_GBps"] = (16.0 * n0 + 8.0 * n1) / (ms * 1e-3) / 1e9
    r = torch.empty_like(f)
    ms = timed(lambda: h.residual(0, f, x, r), args.reps)
    out["residual_ms"] = ms
    out["residual_GBps"] = 24.0 * n0 / (ms * 1e-3) / 1e9
    ms = timed(lambda: h.residual_norm(f, x), args.reps)
    out["resid_norm_ms"] = ms
    out["resid_norm_GBps"] = 16.0 * n0 / (ms * 1e-3) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
