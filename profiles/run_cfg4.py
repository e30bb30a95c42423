"""BASELINE config 4: the topology-optimisation loop at full size with GPU
STMG solves.  python profiles/run_cfg4.py [--iterations 50 --nu 20 --n-levels 14]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iterations", type=int, default=50)
    ap.add_argument("--nu", type=int, default=20)
    ap.add_argument("--n-levels", type=int, default=6)
    ap.add_argument("--n-el", type=int, default=4096)
    ap.add_argument("--n-t", type=int, default=16384)
    a = ap.parse_args()
    import torch

    from paper_2505_10168_b200 import stmg as S

    torch.zeros(1, device="cuda")  # CUDA context created before the timed optimise() call

    geom = S.build_fine_grid(1.0, 1.0, a.n_el, a.n_t)
    opts = S.OptimisationOptions(method="CR", strategy=S.PlanStrategy.DesignIndependent, n_levels=a.n_levels,
                                 max_iterations=a.iterations, stable_iterations=10 ** 6,
                                 solve=S.SolveOptions(nu=a.nu, tol=1e-8))
    res = S.optimise(geom, (1e-3, 1.0, 1.0, 1.0, 3.0, 2.0), opts)
    h = res.history
    out = {"config": "cfg4", "n_el": a.n_el, "n_t": a.n_t, "nu": a.nu, "n_levels": a.n_levels,
           "iterations": res.iterations, "total_seconds": res.seconds,
           "stmg_seconds": sum(r["primal_seconds"] + r["adjoint_seconds"] for r in h),
           "primal_cycles": [r["primal_cycles"] for r in h], "adjoint_cycles": [r["adjoint_cycles"] for r in h],
           "primal_seconds": [round(r["primal_seconds"], 5) for r in h],
           "adjoint_seconds": [round(r["adjoint_seconds"], 5) for r in h],
           "statuses": sorted({(r["primal_status"], r["adjoint_status"]) for r in h}),
           "theta_first_last": [h[0]["theta"], h[-1]["theta"]], "volume_last": h[-1]["volume"]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
