"""objective_sensitivities on the GPU at BASELINE config 4's size (4096 x 16384):
k_sensitivities streams u and lambda once (2 x 537 MB).  Prints the call's
CUDA-event time and the kernel's achieved bandwidth; the ncu target for the
kernel's DRAM bytes.

    python profiles/sens_bench.py [--reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-el", type=int, default=4096)
    ap.add_argument("--n-t", type=int, default=16384)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_2505_10168_b200 import stmg as S

    n = (a.n_el + 1) * (a.n_t + 1)
    geom = S.build_fine_grid(1.0, 1.0, a.n_el, a.n_t)
    mat = (1e-3, 1.0, 1.0, 1.0, 3.0, 2.0)
    chi = np.random.default_rng(1).uniform(0.0, 1.0, a.n_el)
    u = torch.randn(n, dtype=torch.float64, device="cuda")
    lam = torch.randn(n, dtype=torch.float64, device="cuda")
    S.objective_sensitivities(geom, mat, chi, u, lam)
    best = None
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        S.objective_sensitivities(geom, mat, chi, u, lam)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    print(json.dumps({"grid": f"{a.n_el}x{a.n_t}", "bytes": 16 * n, "call_ms": best,
                      "achieved_GBps_call": 16 * n / best / 1e6}))


if __name__ == "__main__":
    main()
