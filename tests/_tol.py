"""Parity tolerances (BASELINE north_star: 1e-10 relative).

Per-cycle residual norms are compared as |h_a - h_b| <= 1e-10 * h_b + tau with
tau = 16 eps ||J||_inf ||u||_2 / ||b||_2: the fp64 rounding floor of evaluating
b - J u in the reference's own arithmetic.  Two exact coarsest solvers (the
reference's sparse LU and our PCR march) differ by ~1 ulp, which moves every
later residual by about this floor; once h itself approaches the floor (the
last cycles before 1e-10) only the absolute floor is meaningful.  Fields are
compared as max|u_a - u_b| <= 1e-10 max|u_b|.
"""
import numpy as np

EPS = np.finfo(np.float64).eps
HIST_REL = 1e-10
FIELD_REL = 1e-10


def j_inf_norm(coeffs: dict, w: float) -> float:
    rows = sum(np.abs(coeffs[k]) for k in ("cur_m", "cur_0", "cur_p", "oth_m", "oth_0", "oth_p"))
    return float(max(np.max(rows), abs(w)))


def residual_floor(j_norm: float, u: np.ndarray, b: np.ndarray) -> float:
    nb = float(np.linalg.norm(b))
    if nb == 0.0:
        return 16 * EPS * j_norm * float(np.linalg.norm(u))
    return 16 * EPS * j_norm * float(np.linalg.norm(u)) / nb


def histories_match(h_got, h_want, floor: float) -> bool:
    h_got = np.asarray(h_got, np.float64)
    h_want = np.asarray(h_want, np.float64)
    return h_got.shape == h_want.shape and bool(
        np.all(np.abs(h_got - h_want) <= HIST_REL * np.abs(h_want) + floor))
