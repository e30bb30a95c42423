"""Generate the BASELINE config-4 golden at its configured size from the UNMODIFIED
reference (oracle/_ref): optimise() on 4096 x 16384, CR, DesignIndependent,
6 levels, nu = 20, tol 1e-8, warm starts, for the first ITER design iterations
(proj/src/optimisation.cpp:83-186).

Run here (where /root/reference exists; ~1 h on one core, ~25 GB RAM):
    python tests/golden/make_golden_cfg4.py [--iterations 2]
Writes tests/golden/cfg4_full.npz: the reference's per-iteration records
(theta, volume, constraint, change, statuses, primal/adjoint cycles and
factors, seconds), the final design chi and theta.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Ref  # noqa: E402

CFG4_FULL = dict(L=1.0, tT=1.0, n_el=4096, n_t=16384, mat=(1e-3, 1.0, 1.0, 1.0, 3.0, 2.0), method="CR",
                 strategy=3, n_levels=6, nu=20, tol=1e-8, stable_iterations=10 ** 6)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iterations", type=int, default=2)
    ap.add_argument("--out", default=os.path.join(HERE, "cfg4_full.npz"))
    a = ap.parse_args()
    o = dict(CFG4_FULL)
    t0 = time.time()
    r = Ref().optimise(o.pop("L"), o.pop("tT"), o.pop("n_el"), o.pop("n_t"), o.pop("mat"),
                       max_iterations=a.iterations, **o)
    wall = time.time() - t0
    np.savez_compressed(a.out, chi=r["chi"], records=r["records"], theta=r["theta"],
                        iterations=a.iterations, ref_wall_seconds=wall)
    print("wrote", a.out, "in", round(wall, 1), "s")
    print(r["records"])


if __name__ == "__main__":
    main()
