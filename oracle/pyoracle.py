"""TEST INFRASTRUCTURE — ctypes access to the two CPU checkers.

* ``Port``: oracle/liboracle_port.so, the plain-C restatement (stmg_oracle.c).
* ``Ref``:  oracle/_ref/libstmg_ref.so, the UNMODIFIED reference compiled from
  /root/reference/proj (see oracle/Makefile) behind oracle/ref_harness.cpp.
  ``Ref(dropin=True)`` loads oracle/_ref/libstmg_dropin.so instead: the same
  reference objects and harness with multigrid.o replaced by the B200 drop-in
  (paper_2505_10168_b200/dropin/multigrid_b200.cpp), i.e. the reference's own
  callers (optimise(), mg_solve) running on libstmg_b200.so.  Only the harness
  entry points that go through build_hierarchy / transposed_hierarchy / mg_solve /
  optimise are meaningful there (no host CSR operators exist in the drop-in).

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this module.  The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle_port.so")
REF_SO = os.path.join(HERE, "_ref", "libstmg_ref.so")
DROPIN_SO = os.path.join(HERE, "_ref", "libstmg_dropin.so")
REF_SRC = "/root/reference/proj"

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def build_port() -> str:
    """Compile the C restatement (needs only gcc; works on the GPU box too)."""
    src = os.path.join(HERE, "stmg_oracle.c")
    if not os.path.exists(PORT_SO) or os.path.getmtime(PORT_SO) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE, "port"])
    return PORT_SO


def build_ref() -> str | None:
    """Compile the reference in place (only possible where /root/reference exists),
    and the drop-in library over it when libstmg_b200.so is built."""
    if os.path.isdir(REF_SRC):
        subprocess.check_call(["make", "-s", "-j8", "-C", HERE, "ref"])
        if os.path.exists(os.path.join(os.path.dirname(HERE), "paper_2505_10168_b200", "libstmg_b200.so")):
            subprocess.check_call(["make", "-s", "-j8", "-C", HERE, "dropin", "acceptance"])
    return REF_SO if os.path.exists(REF_SO) else None


def dropin_available() -> bool:
    return os.path.exists(DROPIN_SO)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


@dataclass
class Report:
    status: int
    cycles: int
    factor: float
    absolute_norms: bool
    history: np.ndarray
    seconds: float = 0.0
    build_seconds: float = 0.0
    extra: dict = field(default_factory=dict)


class OracleError(RuntimeError):
    pass


class Port:
    """The C restatement."""

    def __init__(self):
        lib = C.CDLL(build_port())
        i64, f64, i32 = C.c_int64, C.c_double, C.c_int
        lib.or_last_error.restype = C.c_char_p
        lib.or_plan.argtypes = [f64, f64, i64, i64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                i32, f64, i32, i32, i64, _ip, C.c_void_p]
        lib.or_build.argtypes = [f64, f64, i64, i64, _dp, _dp, C.c_void_p, C.c_void_p, i32, i32,
                                 C.c_void_p, i32, C.POINTER(C.c_void_p)]
        lib.or_free.argtypes = [C.c_void_p]
        lib.or_n_levels.argtypes = [C.c_void_p]
        lib.or_level_shape.argtypes = [C.c_void_p, i32, C.POINTER(i64), C.POINTER(i64), C.POINTER(f64)]
        lib.or_level_coeffs.argtypes = [C.c_void_p, i32] + [_dp] * 7
        lib.or_residual.argtypes = [C.c_void_p, i32, _dp, _dp, _dp]
        lib.or_jacobi_sweeps.argtypes = [C.c_void_p, i32, _dp, _dp, i32, f64]
        lib.or_restrict.argtypes = [C.c_void_p, i32, _dp, _dp]
        lib.or_prolong_add.argtypes = [C.c_void_p, i32, _dp, _dp]
        lib.or_coarsest_solve.argtypes = [C.c_void_p, _dp, _dp]
        lib.or_norm2.argtypes = [_dp, i64]
        lib.or_norm2.restype = f64
        lib.or_set_norm_mode.argtypes = [i32]
        lib.or_mg_solve.argtypes = [C.c_void_p, _dp, _dp, i32, f64, f64, f64, i32, C.POINTER(i32),
                                    C.POINTER(i32), C.POINTER(f64), C.POINTER(i32), _dp, C.POINTER(i64)]
        lib.or_apply_design.argtypes = [_dp, i64, C.c_void_p, _dp, _dp]
        lib.or_load_vector.argtypes = [f64, f64, i64, i64, i32, _dp, i32, _dp]
        self.lib = lib

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(f"oracle rc={rc}: {self.lib.or_last_error().decode()}")

    @staticmethod
    def _mat(mat):
        if mat is None:
            return None
        return C.cast((C.c_double * 6)(*mat), C.c_void_p)

    def plan(self, L, tT, n_el, n_t, k, c, n_levels, lambda_crit=0.25, strategy=1, reassembly=0,
             min_elements=0, chi=None, mat=None):
        dirs = np.zeros(max(n_levels - 1, 1), np.int32)
        ind = np.zeros(max(n_levels - 1, 1), np.float64)
        kk = None if k is None else np.ascontiguousarray(k, np.float64)
        cc = None if c is None else np.ascontiguousarray(c, np.float64)
        ch = None if chi is None else np.ascontiguousarray(chi, np.float64)
        self._chk(self.lib.or_plan(L, tT, n_el, n_t,
                                   None if kk is None else kk.ctypes.data,
                                   None if cc is None else cc.ctypes.data,
                                   None if ch is None else ch.ctypes.data, self._mat(mat),
                                   n_levels, lambda_crit, strategy, reassembly, min_elements, dirs,
                                   ind.ctypes.data))
        return dirs[: n_levels - 1].copy(), ind[: n_levels - 1].copy()

    def hierarchy(self, L, tT, n_el, n_t, k, c, dirs, reassembly=2, adjoint=False, chi=None, mat=None):
        return PortHier(self, L, tT, n_el, n_t, k, c, dirs, reassembly, adjoint, chi, mat)

    def load_vector(self, L, tT, n_el, n_t, kind, params, masked=True):
        b = np.empty((n_t + 1) * (n_el + 1), np.float64)
        p = np.zeros(4, np.float64)
        p[: len(params)] = params
        self._chk(self.lib.or_load_vector(L, tT, n_el, n_t, kind, p, 1 if masked else 0, b))
        return b

    def apply_design(self, chi, mat):
        chi = np.ascontiguousarray(chi, np.float64)
        k = np.empty_like(chi)
        c = np.empty_like(chi)
        self._chk(self.lib.or_apply_design(chi, chi.size, self._mat(mat), k, c))
        return k, c

    def norm2(self, x):
        return self.lib.or_norm2(np.ascontiguousarray(x, np.float64), x.size)

    def set_norm_mode(self, pairwise: bool):
        """Residual norms of solve(): the reference's 4-lane order (False) or pairwise (True)."""
        self.lib.or_set_norm_mode(1 if pairwise else 0)


class PortHier:
    def __init__(self, port, L, tT, n_el, n_t, k, c, dirs, reassembly, adjoint, chi, mat):
        self.p = port
        lib = port.lib
        d = np.ascontiguousarray(dirs, np.int32)
        self._chi = None if chi is None else np.ascontiguousarray(chi, np.float64)
        h = C.c_void_p()
        port._chk(lib.or_build(L, tT, n_el, n_t, np.ascontiguousarray(k, np.float64),
                               np.ascontiguousarray(c, np.float64),
                               None if self._chi is None else self._chi.ctypes.data,
                               port._mat(mat), reassembly, d.size,
                               d.ctypes.data if d.size else None, 1 if adjoint else 0, C.byref(h)))
        self.h = h
        self.n_levels = lib.or_n_levels(h)
        self.shapes = []
        for l in range(self.n_levels):
            ne, nt, w = C.c_int64(), C.c_int64(), C.c_double()
            lib.or_level_shape(h, l, C.byref(ne), C.byref(nt), C.byref(w))
            self.shapes.append((ne.value, nt.value, w.value))

    def __del__(self):
        try:
            self.p.lib.or_free(self.h)
        except Exception:
            pass

    def ndofs(self, l):
        ne, nt, _ = self.shapes[l]
        return (ne + 1) * (nt + 1)

    def coeffs(self, l):
        nn = self.shapes[l][0] + 1
        arrs = [np.zeros(nn) for _ in range(7)]
        self.p._chk(self.p.lib.or_level_coeffs(self.h, l, *arrs))
        return dict(zip(["W", "D", "E", "SW", "S", "SE", "inv_diag"], arrs))

    def residual(self, l, f, x):
        r = np.empty(self.ndofs(l))
        self.p._chk(self.p.lib.or_residual(self.h, l, f, x, r))
        return r

    def sweeps(self, l, f, x, n, omega=0.5):
        x = np.array(x, np.float64, copy=True)
        self.p._chk(self.p.lib.or_jacobi_sweeps(self.h, l, f, x, n, omega))
        return x

    def restrict(self, l, r):
        fc = np.empty(self.ndofs(l + 1))
        self.p._chk(self.p.lib.or_restrict(self.h, l, r, fc))
        return fc

    def prolong_add(self, l, xc, x):
        x = np.array(x, np.float64, copy=True)
        self.p._chk(self.p.lib.or_prolong_add(self.h, l, xc, x))
        return x

    def coarsest(self, f):
        x = np.empty(self.ndofs(self.n_levels - 1))
        self.p._chk(self.p.lib.or_coarsest_solve(self.h, f, x))
        return x

    def solve(self, b, u=None, nu=1, omega=0.5, tol=1e-10, div_tol=1e9, max_cycles=100):
        u = np.zeros(self.ndofs(0)) if u is None else np.array(u, np.float64, copy=True)
        hist = np.zeros(max_cycles + 1)
        st, cy, ab = C.c_int(), C.c_int(), C.c_int()
        fa = C.c_double()
        nh = C.c_int64()
        self.p._chk(self.p.lib.or_mg_solve(self.h, np.ascontiguousarray(b, np.float64), u, nu, omega,
                                           tol, div_tol, max_cycles, C.byref(st), C.byref(cy),
                                           C.byref(fa), C.byref(ab), hist, C.byref(nh)))
        return u, Report(st.value, cy.value, fa.value, bool(ab.value), hist[: nh.value].copy())


class Ref:
    """The unmodified reference (requires oracle/_ref/libstmg_ref.so); dropin=True:
    the reference's callers over the B200 drop-in (oracle/_ref/libstmg_dropin.so)."""

    def __init__(self, dropin: bool = False):
        if not ref_available():
            build_ref()
        lib = C.CDLL(DROPIN_SO if dropin else REF_SO)
        f64, i32 = C.c_double, C.c_int
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_plan.argtypes = [f64, f64, i32, i32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 i32, f64, i32, i32, i32, _ip, C.c_void_p]
        lib.ref_hier_create.argtypes = [f64, f64, i32, i32, _dp, _dp, C.c_void_p, C.c_void_p,
                                        C.c_char_p, i32, C.c_void_p, i32, C.POINTER(C.c_void_p),
                                        C.POINTER(f64)]
        lib.ref_hier_free.argtypes = [C.c_void_p]
        lib.ref_hier_n_levels.argtypes = [C.c_void_p]
        lib.ref_hier_level_dofs.argtypes = [C.c_void_p, i32]
        lib.ref_hier_level_dofs.restype = C.c_longlong
        lib.ref_hier_level_nnz.argtypes = [C.c_void_p, i32]
        lib.ref_hier_level_nnz.restype = C.c_longlong
        lib.ref_hier_level_csr.argtypes = [C.c_void_p, i32, _ip, _ip, _dp, _dp]
        lib.ref_residual.argtypes = [C.c_void_p, i32, _dp, _dp, _dp]
        lib.ref_jacobi_sweeps.argtypes = [C.c_void_p, i32, _dp, _dp, i32, f64]
        lib.ref_restrict.argtypes = [C.c_void_p, i32, _dp, _dp]
        lib.ref_prolong_add.argtypes = [C.c_void_p, i32, _dp, _dp]
        lib.ref_coarsest_solve.argtypes = [C.c_void_p, _dp, _dp]
        lib.ref_mg_solve.argtypes = [C.c_void_p, _dp, _dp, i32, f64, f64, f64, i32, C.POINTER(i32),
                                     C.POINTER(i32), C.POINTER(f64), C.POINTER(i32), _dp,
                                     C.POINTER(i32), C.POINTER(f64)]
        lib.ref_load_vector.argtypes = [f64, f64, i32, i32, i32, _dp, i32, _dp]
        lib.ref_apply_design.argtypes = [_dp, i32, _dp, _dp, _dp]
        lib.ref_objective_sensitivities.argtypes = [f64, f64, i32, i32, _dp, _dp, _dp, _dp, _dp]
        lib.ref_norm2.argtypes = [_dp, C.c_longlong]
        lib.ref_norm2.restype = f64
        lib.ref_set_backend.argtypes = [i32]
        lib.ref_optimise.argtypes = [f64, f64, i32, i32, _dp, C.c_char_p, i32, i32, f64, i32, i32, f64, f64,
                                     f64, i32, f64, i32, i32, f64, f64, f64, i32, _dp, _dp,
                                     C.POINTER(i32), C.POINTER(f64), C.POINTER(i32), C.POINTER(f64)]
        self.lib = lib

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(f"reference rc={rc}: {self.lib.ref_last_error().decode()}")

    def plan(self, L, tT, n_el, n_t, k, c, n_levels, lambda_crit=0.25, strategy=1, reassembly=0,
             min_elements=0, chi=None, mat=None):
        dirs = np.zeros(max(n_levels - 1, 1), np.int32)
        ind = np.zeros(max(n_levels - 1, 1), np.float64)
        kk = None if k is None else np.ascontiguousarray(k, np.float64)
        cc = None if c is None else np.ascontiguousarray(c, np.float64)
        ch = None if chi is None else np.ascontiguousarray(chi, np.float64)
        m = None if mat is None else np.ascontiguousarray(mat, np.float64)
        self._chk(self.lib.ref_plan(L, tT, n_el, n_t,
                                    None if kk is None else kk.ctypes.data,
                                    None if cc is None else cc.ctypes.data,
                                    None if ch is None else ch.ctypes.data,
                                    None if m is None else m.ctypes.data,
                                    n_levels, lambda_crit, strategy, reassembly, min_elements, dirs,
                                    ind.ctypes.data))
        return dirs[: n_levels - 1].copy(), ind[: n_levels - 1].copy()

    def hierarchy(self, L, tT, n_el, n_t, k, c, dirs, method="CR", adjoint=False, chi=None, mat=None):
        return RefHier(self, L, tT, n_el, n_t, k, c, dirs, method, adjoint, chi, mat)

    def load_vector(self, L, tT, n_el, n_t, kind, params, masked=True):
        b = np.empty((n_t + 1) * (n_el + 1), np.float64)
        p = np.zeros(4, np.float64)
        p[: len(params)] = params
        self._chk(self.lib.ref_load_vector(L, tT, n_el, n_t, kind, p, 1 if masked else 0, b))
        return b

    def apply_design(self, chi, mat):
        chi = np.ascontiguousarray(chi, np.float64)
        k = np.empty_like(chi)
        c = np.empty_like(chi)
        self._chk(self.lib.ref_apply_design(chi, chi.size, np.ascontiguousarray(mat, np.float64), k, c))
        return k, c

    def norm2(self, x):
        return self.lib.ref_norm2(np.ascontiguousarray(x, np.float64), x.size)

    def objective_sensitivities(self, L, tT, n_el, n_t, mat, chi, u, lam):
        sens = np.empty(n_el)
        self._chk(self.lib.ref_objective_sensitivities(L, tT, n_el, n_t, np.ascontiguousarray(mat, np.float64),
                                                       np.ascontiguousarray(chi, np.float64),
                                                       np.ascontiguousarray(u, np.float64),
                                                       np.ascontiguousarray(lam, np.float64), sens))
        return sens

    def optimise(self, L, tT, n_el, n_t, mat, method="CR", strategy=3, n_levels=6, lambda_crit=0.25,
                 min_elements=0, warm_start=True, volume_limit=0.5, theta_ref=1e6, chi_init=0.5,
                 max_iterations=10, rel_change_tol=1e-3, stable_iterations=5, nu=20, omega=0.5,
                 tol=1e-9, div_tol=1e9, max_cycles=100):
        chi = np.zeros(n_el)
        rec = np.zeros(12 * max_iterations)
        nr, conv = C.c_int(), C.c_int()
        th, secs = C.c_double(), C.c_double()
        self._chk(self.lib.ref_optimise(L, tT, n_el, n_t, np.ascontiguousarray(mat, np.float64),
                                        method.encode(), strategy, n_levels, lambda_crit, min_elements,
                                        1 if warm_start else 0, volume_limit, theta_ref, chi_init,
                                        max_iterations, rel_change_tol, stable_iterations, nu, omega,
                                        tol, div_tol, max_cycles, chi, rec, C.byref(nr), C.byref(th),
                                        C.byref(conv), C.byref(secs)))
        return dict(chi=chi, records=rec[: 12 * nr.value].reshape(nr.value, 12), theta=th.value,
                    converged=bool(conv.value), seconds=secs.value)


class RefHier:
    def __init__(self, ref, L, tT, n_el, n_t, k, c, dirs, method, adjoint, chi, mat):
        self.r = ref
        d = np.ascontiguousarray(dirs, np.int32)
        ch = None if chi is None else np.ascontiguousarray(chi, np.float64)
        m = None if mat is None else np.ascontiguousarray(mat, np.float64)
        self._keep = (ch, m, d)
        h = C.c_void_p()
        bs = C.c_double()
        ref._chk(ref.lib.ref_hier_create(L, tT, n_el, n_t, np.ascontiguousarray(k, np.float64),
                                         np.ascontiguousarray(c, np.float64),
                                         None if ch is None else ch.ctypes.data,
                                         None if m is None else m.ctypes.data,
                                         method.encode(), d.size, d.ctypes.data if d.size else None,
                                         1 if adjoint else 0, C.byref(h), C.byref(bs)))
        self.h = h
        self.build_seconds = bs.value
        self.n_levels = ref.lib.ref_hier_n_levels(h)

    def __del__(self):
        try:
            self.r.lib.ref_hier_free(self.h)
        except Exception:
            pass

    def ndofs(self, l):
        return int(self.r.lib.ref_hier_level_dofs(self.h, l))

    def csr(self, l):
        n = self.ndofs(l)
        nnz = int(self.r.lib.ref_hier_level_nnz(self.h, l))
        rp = np.zeros(n + 1, np.int32)
        ci = np.zeros(nnz, np.int32)
        v = np.zeros(nnz)
        inv = np.zeros(n)
        self.r._chk(self.r.lib.ref_hier_level_csr(self.h, l, rp, ci, v, inv))
        return rp, ci, v, inv

    def residual(self, l, f, x):
        r = np.empty(self.ndofs(l))
        self.r._chk(self.r.lib.ref_residual(self.h, l, f, x, r))
        return r

    def sweeps(self, l, f, x, n, omega=0.5):
        x = np.array(x, np.float64, copy=True)
        self.r._chk(self.r.lib.ref_jacobi_sweeps(self.h, l, f, x, n, omega))
        return x

    def restrict(self, l, r):
        fc = np.empty(self.ndofs(l + 1))
        self.r._chk(self.r.lib.ref_restrict(self.h, l, r, fc))
        return fc

    def prolong_add(self, l, xc, x):
        x = np.array(x, np.float64, copy=True)
        self.r._chk(self.r.lib.ref_prolong_add(self.h, l, xc, x))
        return x

    def coarsest(self, f):
        x = np.empty(self.ndofs(self.n_levels - 1))
        self.r._chk(self.r.lib.ref_coarsest_solve(self.h, f, x))
        return x

    def solve(self, b, u=None, nu=1, omega=0.5, tol=1e-10, div_tol=1e9, max_cycles=100):
        u = np.zeros(self.ndofs(0)) if u is None else np.array(u, np.float64, copy=True)
        hist = np.zeros(max_cycles + 1)
        st, cy, ab, nh = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        fa, sec = C.c_double(), C.c_double()
        self.r._chk(self.r.lib.ref_mg_solve(self.h, np.ascontiguousarray(b, np.float64), u, nu, omega,
                                            tol, div_tol, max_cycles, C.byref(st), C.byref(cy),
                                            C.byref(fa), C.byref(ab), hist, C.byref(nh),
                                            C.byref(sec)))
        return u, Report(st.value, cy.value, fa.value, bool(ab.value), hist[: nh.value].copy(),
                         seconds=sec.value, build_seconds=self.build_seconds)
