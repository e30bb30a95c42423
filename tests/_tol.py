"""Parity tolerances (BASELINE north_star: 1e-10 relative).

Per-cycle relative residual norms are compared as |h_a - h_b| <= 1e-10 h_b +
floor, with a fixed absolute floor (in units of ||b||):

* HIST_ABS = 1e-13 on the small cases (<= 1.3e5 DOFs);
* HIST_ABS_FULL = 1e-12 at BASELINE config 1's full size (4.2e6 DOFs).

Two exact coarsest solvers (the reference's sparse LU and the oracle's Thomas
march, or our parallel-in-time march) agree to ~1 ulp; that moves every later
residual b - J u by its fp64 evaluation noise, which grows with the grid.  The
floor is set from a measurement, not a bound: at full cfg1 size the C oracle and
the compiled reference -- the same algorithm, two exact coarsest solvers -- differ
by at most 4.4e-13 in any history entry (tests/test_gpu_scale.py re-measures it
on every run), so 1e-12 is the smallest floor both independent CPU
implementations pass.  Fields are compared as max|u_a - u_b| <= 1e-10 max|u_b|.
"""
import numpy as np

HIST_REL = 1e-10
HIST_ABS = 1e-13
HIST_ABS_FULL = 1e-12
FIELD_REL = 1e-10


def histories_match(h_got, h_want, floor: float = HIST_ABS) -> bool:
    h_got = np.asarray(h_got, np.float64)
    h_want = np.asarray(h_want, np.float64)
    return h_got.shape == h_want.shape and bool(
        np.all(np.abs(h_got - h_want) <= HIST_REL * np.abs(h_want) + floor))
