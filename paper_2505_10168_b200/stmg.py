"""Python mirror of the reference's solver API over the stmg_b200 C ABI.

Names, argument meaning and error behaviour follow the reference's C++ API
(namespace ``stmg``; proj/include/stmg/*.hpp) so a caller of the reference
can switch to the B200 path:

    reference (C++)                         here
    build_fine_grid (mesh.hpp:62)           build_fine_grid
    apply_design (materials.hpp:48-49)      apply_design
    load_vector (assembly.hpp:54-56)        load_vector
    dof_is_masked (assembly.hpp:68)         dof_is_masked
    plan_coarsening (strategy.hpp:104-105)  plan_coarsening
    path_to_string (strategy.hpp:99)        path_to_string
    parse_method (rediscretisation.cpp:19-38)  (method strings C|B + K|D|R|P)
    build_hierarchy (multigrid.hpp:70-74)   build_hierarchy
    transposed_hierarchy (multigrid.hpp:77) transposed_hierarchy
    mg_solve (multigrid.hpp:107-108)        mg_solve
    SolveOptions / SolveReport / SolveStatus

Exceptions: std::invalid_argument -> ValueError, std::runtime_error ->
RuntimeError, std::out_of_range -> IndexError (STMG_EINVAL / ERUNTIME / ERANGE).

All compute runs in libstmg_b200.so on the GPU.  There is no CPU fallback:
importing this module without the built extension raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# STMG_LIB_PATH: benchmarking override (A/B builds); the in-tree build otherwise.
LIB_PATH = os.environ.get("STMG_LIB_PATH") or os.path.join(_HERE, "libstmg_b200.so")


class StmgCudaError(RuntimeError):
    pass


ABI_VERSION = 4  # include/stmg_b200.h STMG_ABI_VERSION (stmg_solve_report layout)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"stmg_b200 CUDA extension not built ({LIB_PATH} missing); run "
            "`python -c 'import __graft_entry__ as g; g.build()'` or paper_2505_10168_b200/build.py")
    lib = C.CDLL(LIB_PATH)
    i32, i64, f64, vp = C.c_int32, C.c_int64, C.c_double, C.c_void_p
    lib.stmg_last_error.restype = C.c_char_p
    lib.stmg_abi_version.restype = C.c_int
    if lib.stmg_abi_version() != ABI_VERSION:  # struct layouts below are this version's
        raise ImportError(f"{LIB_PATH} has C ABI version {lib.stmg_abi_version()}, this module needs "
                          f"{ABI_VERSION}: rebuild with paper_2505_10168_b200/build.py")
    sig = {
        "stmg_apply_design": [vp, i64, vp, vp, vp],
        "stmg_load_vector": [vp, i32, vp, i32, vp],
        "stmg_load_vector_cb": [vp, vp, vp, i32, vp],
        "stmg_load_vector_device": [vp, i32, vp, i32, vp, vp],
        "stmg_plan_coarsening": [vp, vp, vp, vp, vp, vp, vp, vp],
        "stmg_hierarchy_create": [vp, vp, vp, vp, vp, C.c_char_p, i32, vp, i32, C.POINTER(vp)],
        "stmg_hierarchy_transposed": [vp, C.POINTER(vp)],
        "stmg_hierarchy_n_levels": [vp, C.POINTER(i32)],
        "stmg_hierarchy_level_info": [vp, i32, C.POINTER(i64), C.POINTER(i64), C.POINTER(f64)],
        "stmg_hierarchy_level_coeffs": [vp, i32, vp, vp, vp, vp, vp, vp, vp],
        "stmg_hierarchy_device_bytes": [vp, C.POINTER(i64)],
        "stmg_hierarchy_level_stencil9": [vp, i32, vp, vp, vp],
        "stmg_level_stencil9_host": [vp, vp, vp, vp, vp, C.c_char_p, i32, vp, i32, i32, vp, vp, vp],
        "stmg_hierarchy_set_stream": [vp, vp],
        "stmg_hierarchy_set_profiling": [vp, i32],
        "stmg_hierarchy_profile": [vp, i32, i32, C.POINTER(i64), C.POINTER(f64)],
        "stmg_mg_solve": [vp, vp, vp, vp, vp, vp, i32],
        "stmg_mg_solve_ex": [vp, vp, vp, vp, i32, vp, vp, i32],
        "stmg_mg_solve_batch": [i32, vp, vp, vp, vp, vp, vp, i32],
        "stmg_mg_solve_stream": [vp, i32, vp, vp, vp, i32, vp, vp, i32],
        "stmg_hierarchy_release_staging": [vp],
        "stmg_level_sweeps": [vp, i32, vp, vp, i32, f64],
        "stmg_level_residual": [vp, i32, vp, vp, vp],
        "stmg_level_sweep_kernels": [vp, i32, vp, vp, vp, i32, i32, f64],
        "stmg_level_restrict_residual": [vp, i32, vp, vp, vp],
        "stmg_level_restrict": [vp, i32, vp, vp],
        "stmg_level_prolong_add": [vp, i32, vp, vp],
        "stmg_coarsest_solve": [vp, vp, vp],
        "stmg_residual_norm": [vp, vp, vp, C.POINTER(f64)],
        "stmg_norm2": [vp, vp, i64, C.POINTER(f64)],
        "stmg_synchronize": [vp],
        "stmg_hierarchy_set_tiling": [vp, i64, i64],
        "stmg_hierarchy_set_fusion": [vp, i32],
        "stmg_objective_sensitivities": [vp, vp, vp, vp, vp, vp, i32],
        "stmg_level_fused": [vp, i32, i32, vp, vp, vp, vp, vp, f64, C.POINTER(f64)],
        "stmg_dist_partition": [i32, vp, vp, i32, i64, C.POINTER(i32), vp],
        "stmg_optimise": [vp, vp, i32, vp, vp, C.POINTER(i32), C.POINTER(f64), C.POINTER(i32),
                          C.POINTER(f64), vp],
        "stmg_dist_nccl_unique_id": [vp, i32],
        "stmg_dist_create": [vp, vp, vp, vp, vp, C.c_char_p, i32, vp, i32, i32, i32, vp, i32, i64,
                             C.POINTER(vp)],
        "stmg_dist_loop_on_device": [vp, C.POINTER(i32)],
        "stmg_dist_split_passes": [vp, C.POINTER(i64)],
        "stmg_dist_info": [vp, C.POINTER(i32), C.POINTER(i64), C.POINTER(i64), C.POINTER(i32),
                           C.POINTER(i64)],
        "stmg_dist_mg_solve": [vp, vp, vp, vp, vp, vp, i32],
        "stmg_dist_mg_solve_local": [vp, vp, vp, vp, vp, vp, i32],
        "stmg_dist_transport": [vp, C.c_char_p, i32],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.stmg_hierarchy_destroy.argtypes = [vp]
    lib.stmg_hierarchy_destroy.restype = None
    lib.stmg_dist_destroy.argtypes = [vp]
    lib.stmg_dist_destroy.restype = None
    return lib


_lib = _load()

STMG_OK, STMG_EINVAL, STMG_ERUNTIME, STMG_ERANGE, STMG_ECUDA, STMG_ENOMEM = range(6)


def _check(rc: int):
    if rc == STMG_OK:
        return
    msg = _lib.stmg_last_error().decode(errors="replace")
    if rc == STMG_EINVAL:
        raise ValueError(msg)
    if rc == STMG_ERANGE:
        raise IndexError(msg)
    if rc == STMG_ENOMEM:
        raise MemoryError(msg)
    if rc == STMG_ECUDA:
        raise StmgCudaError(msg)
    raise RuntimeError(msg)


# ---- C structs (include/stmg_b200.h) -------------------------------------------------
class _Grid(C.Structure):
    _fields_ = [("L", C.c_double), ("t_T", C.c_double), ("n_el", C.c_int64), ("n_t", C.c_int64)]


class _Mat(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("k_ins", "k_con", "c_ins", "c_con", "p_k", "p_c")]


class _PlanReq(C.Structure):
    _fields_ = [("n_levels", C.c_int32), ("lambda_crit", C.c_double), ("strategy", C.c_int32),
                ("reassembly", C.c_int32), ("min_elements", C.c_int64)]


class _SolveOpts(C.Structure):
    _fields_ = [("nu", C.c_int32), ("omega", C.c_double), ("tol", C.c_double),
                ("div_tol", C.c_double), ("max_cycles", C.c_int32)]


class _OptOpts(C.Structure):
    _fields_ = [("mat", _Mat), ("method", C.c_char * 4), ("strategy", C.c_int32), ("n_levels", C.c_int32),
                ("lambda_crit", C.c_double), ("min_elements", C.c_int64), ("warm_start", C.c_int32),
                ("volume_limit", C.c_double), ("theta_ref", C.c_double), ("chi_init", C.c_double),
                ("max_iterations", C.c_int32), ("rel_change_tol", C.c_double),
                ("stable_iterations", C.c_int32), ("solve", _SolveOpts), ("mma_x_min", C.c_double),
                ("mma_x_max", C.c_double), ("mma_move_limit", C.c_double), ("mma_asym_init", C.c_double),
                ("mma_asym_shrink", C.c_double), ("mma_asym_grow", C.c_double)]


class _IterRec(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("theta", C.c_double), ("volume", C.c_double),
                ("constraint", C.c_double), ("change", C.c_double), ("primal_status", C.c_int32),
                ("adjoint_status", C.c_int32), ("primal_cycles", C.c_int32), ("adjoint_cycles", C.c_int32),
                ("primal_factor", C.c_double), ("adjoint_factor", C.c_double),
                ("primal_seconds", C.c_double), ("adjoint_seconds", C.c_double), ("path", C.c_char * 96)]


class _SolveRep(C.Structure):
    _fields_ = [("status", C.c_int32), ("cycles", C.c_int32), ("factor", C.c_double),
                ("absolute_norms", C.c_int32), ("n_history", C.c_int32), ("seconds", C.c_double),
                ("device_seconds", C.c_double), ("smoother_dof_updates", C.c_double),
                ("kernel_launches", C.c_int64), ("fine_sweeps", C.c_int64),
                ("fine_sweep_seconds", C.c_double), ("fine_restricts", C.c_int64),
                ("fine_restrict_seconds", C.c_double), ("fine_prolong_sweeps", C.c_int64),
                ("fine_prolong_sweep_seconds", C.c_double), ("fine_sweep_pairs", C.c_int64),
                ("fine_sweep_pair_seconds", C.c_double), ("fine_norm_passes", C.c_int64),
                ("fine_norm_pass_seconds", C.c_double), ("fine_ups", C.c_int64), ("fine_up_seconds", C.c_double)]


# ---- enums ---------------------------------------------------------------------------
class CoarseningDirection(enum.IntEnum):
    SpaceX = 0
    TimeT = 1
    FullST = 2


class ReassemblyMethod(enum.IntEnum):
    K = 0
    D = 1
    R = 2
    P = 3


class PlanStrategy(enum.IntEnum):
    Uniform = 0
    Contrast = 1
    Resolution = 2
    DesignIndependent = 3


class SolveStatus(enum.IntEnum):
    Converged = 0
    MaxCycles = 1
    Diverged = 2


def direction_name(d) -> str:
    return {0: "x", 1: "t", 2: "xt"}[int(d)]


def status_name(s) -> str:
    return {0: "converged", 1: "max-cycles", 2: "diverged"}[int(s)]


# ---- value types -----------------------------------------------------------------------
@dataclass
class MaterialPair:
    k_ins: float = 0.0
    k_con: float = 0.0
    c_ins: float = 0.0
    c_con: float = 0.0
    p_k: float = 3.0
    p_c: float = 2.0

    def _c(self) -> _Mat:
        return _Mat(self.k_ins, self.k_con, self.c_ins, self.c_con, self.p_k, self.p_c)

    @classmethod
    def of(cls, m) -> "MaterialPair":
        return m if isinstance(m, MaterialPair) else cls(*m)


@dataclass
class SpaceTimeGrid:
    """proj/include/stmg/mesh.hpp:27-59"""
    L: float
    t_T: float
    n_el: int
    n_t: int
    k: Optional[np.ndarray] = None
    c: Optional[np.ndarray] = None

    @property
    def dx(self) -> float:
        return self.L / self.n_el

    @property
    def dt(self) -> float:
        return self.t_T / self.n_t

    def n_nodes(self) -> int:
        return self.n_el + 1

    def n_times(self) -> int:
        return self.n_t + 1

    def n_dofs(self) -> int:
        return self.n_times() * self.n_nodes()

    def flatten(self, n: int, i: int) -> int:
        return n * self.n_nodes() + i

    def unflatten(self, flat: int):
        return divmod(flat, self.n_nodes())

    def element_centre(self, e: int) -> float:
        return (e + 0.5) * self.dx

    def has_materials(self) -> bool:
        return self.k is not None and self.c is not None and len(self.k) == self.n_el == len(self.c)

    def _c(self) -> _Grid:
        return _Grid(float(self.L), float(self.t_T), int(self.n_el), int(self.n_t))


def build_fine_grid(L: float, t_T: float, n_el: int, n_t: int) -> SpaceTimeGrid:
    if L <= 0.0 or t_T <= 0.0:
        raise ValueError("build_fine_grid: non-positive extent")
    if n_el <= 0 or n_t <= 0:
        raise ValueError("build_fine_grid: non-positive count")
    return SpaceTimeGrid(float(L), float(t_T), int(n_el), int(n_t))


def _f64(a, n: Optional[int] = None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and a.size != n:
        raise ValueError("size mismatch")
    return a


def _ptr(a) -> int:
    """Data pointer of a float64 contiguous numpy array or torch tensor (None -> null)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
            raise ValueError("expected a C-contiguous float64 array")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        import torch

        if a.dtype != torch.float64 or not a.is_contiguous():
            raise ValueError("expected a contiguous float64 tensor")
        return a.data_ptr()
    raise TypeError(f"unsupported array type {type(a)}")


def _numel(a) -> int:
    return a.size if isinstance(a, np.ndarray) else a.numel()


def apply_design(chi, mat) -> tuple[np.ndarray, np.ndarray]:
    """k(chi), c(chi) per element (proj/src/materials.cpp:27-50)."""
    chi = _f64(chi)
    k = np.empty_like(chi)
    c = np.empty_like(chi)
    m = MaterialPair.of(mat)._c()
    _check(_lib.stmg_apply_design(chi.ctypes.data, chi.size, C.byref(m), k.ctypes.data, c.ctypes.data))
    return k, c


_SOURCE_FN = C.CFUNCTYPE(C.c_double, C.c_double, C.c_double, C.c_void_p)


def load_vector(g: SpaceTimeGrid, q: Optional[Callable[[float, float], float]] = None, *,
                kind: Optional[int] = None, params: Sequence[float] = (), masked: bool = False,
                out: Optional[np.ndarray] = None) -> np.ndarray:
    """All-at-once load vector (proj/src/assembly.cpp:65-83).

    Either a Python callable q(x, t) (the std::function overload; slow, for
    small grids) or a preset source ``kind`` (configs.py) evaluated natively.
    With kind=None and q=None the reference's heat_load_value is used
    (proj/src/assembly.cpp:80-83).  masked=True zeroes the fixed DOFs as
    assemble_system does (proj/src/assembly.cpp:128-130).
    """
    b = out if out is not None else np.empty(g.n_dofs(), np.float64)
    if b.size != g.n_dofs() or b.dtype != np.float64:
        raise ValueError("load_vector: output size mismatch")
    gc = g._c()
    if q is not None:
        cb = _SOURCE_FN(lambda x, t, _ctx: float(q(x, t)))
        _check(_lib.stmg_load_vector_cb(C.byref(gc), cb, None, 1 if masked else 0, b.ctypes.data))
        return b
    if kind is None:
        kind = 3
    p = (C.c_double * 4)(*list(params)[:4])
    _check(_lib.stmg_load_vector(C.byref(gc), int(kind), p, 1 if masked else 0, b.ctypes.data))
    return b


def load_vector_device(g: SpaceTimeGrid, *, kind: int = 3, params=(), masked: bool = True, out=None,
                       stream=None):
    """load_vector for a preset source ``kind``, evaluated by a CUDA kernel into a
    float64 torch tensor on the GPU (``out`` or a new tensor on cuda:0); kinds 0/1
    bit-identical to load_vector, kinds 2/3 within a few ulp (device sin/cos)."""
    import torch

    b = out if out is not None else torch.empty(g.n_dofs(), dtype=torch.float64, device="cuda:0")
    if b.numel() != g.n_dofs() or b.dtype != torch.float64 or not b.is_cuda or not b.is_contiguous():
        raise ValueError("load_vector_device: out must be a contiguous float64 CUDA tensor of n_dofs")
    gc = g._c()
    p = (C.c_double * 4)(*list(params)[:4])
    s = stream if stream is not None else torch.cuda.current_stream(b.device).cuda_stream
    _check(_lib.stmg_load_vector_device(C.byref(gc), int(kind), p, 1 if masked else 0, b.data_ptr(),
                                        C.c_void_p(s)))
    return b


def dof_is_masked(g: SpaceTimeGrid, flat: int) -> bool:
    n, i = g.unflatten(flat)
    return n == 0 or i == 0


@dataclass
class PlanRequest:
    """proj/include/stmg/strategy.hpp:76-86"""
    n_levels: int = 2
    lambda_crit: float = 0.25
    strategy: PlanStrategy = PlanStrategy.Contrast
    reassembly: ReassemblyMethod = ReassemblyMethod.K
    min_elements: int = 0
    chi: Optional[np.ndarray] = None
    mat: Optional[MaterialPair] = None


@dataclass
class CoarseningPath:
    """proj/include/stmg/strategy.hpp:88-96"""
    dirs: list = field(default_factory=list)
    indicator_at_decision: list = field(default_factory=list)
    strategy: PlanStrategy = PlanStrategy.Contrast
    lambda_crit: float = 0.25
    min_elements: int = 0

    def n_levels(self) -> int:
        return len(self.dirs) + 1


def path_to_string(path: CoarseningPath) -> str:
    return ",".join(direction_name(d) for d in path.dirs)


def plan_coarsening(fine: SpaceTimeGrid, req: PlanRequest) -> CoarseningPath:
    n = max(req.n_levels - 1, 0)
    dirs = np.zeros(max(n, 1), np.int32)
    ind = np.zeros(max(n, 1), np.float64)
    k = None if fine.k is None else _f64(fine.k, fine.n_el)
    c = None if fine.c is None else _f64(fine.c, fine.n_el)
    chi = None if req.chi is None else _f64(req.chi, fine.n_el)
    mat = None if req.mat is None else MaterialPair.of(req.mat)._c()
    pr = _PlanReq(int(req.n_levels), float(req.lambda_crit), int(req.strategy), int(req.reassembly),
                  int(req.min_elements))
    gc = fine._c()
    _check(_lib.stmg_plan_coarsening(C.byref(gc), None if k is None else k.ctypes.data,
                                     None if c is None else c.ctypes.data,
                                     None if chi is None else chi.ctypes.data,
                                     None if mat is None else C.byref(mat), C.byref(pr),
                                     dirs.ctypes.data, ind.ctypes.data))
    return CoarseningPath([CoarseningDirection(int(d)) for d in dirs[:n]], [float(v) for v in ind[:n]],
                          PlanStrategy(req.strategy), float(req.lambda_crit), int(req.min_elements))


@dataclass
class SolveOptions:
    """proj/include/stmg/multigrid.hpp:83-89"""
    nu: int = 5
    omega: float = 0.5
    tol: float = 1e-9
    div_tol: float = 1e9
    max_cycles: int = 100


@dataclass
class SolveReport:
    """proj/include/stmg/multigrid.hpp:91-102 (+ device timing and work counters)"""
    status: SolveStatus = SolveStatus.MaxCycles
    cycles: int = 0
    factor: float = 1.0
    history: list = field(default_factory=list)
    absolute_norms: bool = False
    seconds: float = 0.0
    device_seconds: float = 0.0
    smoother_dof_updates: float = 0.0
    kernel_launches: int = 0
    kernel_times: dict = field(default_factory=dict)  # profiling: kind -> (launches, seconds)


@dataclass
class LevelInfo:
    n_el: int
    n_t: int
    w_diri: float

    @property
    def n_dofs(self) -> int:
        return (self.n_el + 1) * (self.n_t + 1)


class LevelHierarchy:
    """Device-resident hierarchy (proj/include/stmg/multigrid.hpp:51-65).

    Owns the C handle; level operators, transfers and the coarsest exact solver
    live on the GPU.  A hierarchy and its transpose share vector workspaces and
    must not be solved concurrently (the reference never does,
    proj/src/optimisation.cpp:132-139).
    """

    def __init__(self, handle: C.c_void_p, path: Optional[CoarseningPath], method: str, device: int,
                 adjoint: bool = False, parent: Optional["LevelHierarchy"] = None):
        self._h = handle
        self.path = path
        self.method = method
        self.device = device
        self.adjoint = adjoint
        self._parent = parent  # keeps the shared workspace owner alive
        n = C.c_int32()
        _check(_lib.stmg_hierarchy_n_levels(self._h, C.byref(n)))
        self._n_levels = n.value
        self.levels = []
        for l in range(self._n_levels):
            ne, nt, w = C.c_int64(), C.c_int64(), C.c_double()
            _check(_lib.stmg_hierarchy_level_info(self._h, l, C.byref(ne), C.byref(nt), C.byref(w)))
            self.levels.append(LevelInfo(ne.value, nt.value, w.value))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.stmg_hierarchy_destroy(h)
            self._h = None

    def close(self):
        self.__del__()

    @property
    def handle(self):
        return self._h


    def n_levels(self) -> int:
        return self._n_levels

    def device_bytes(self) -> int:
        b = C.c_int64()
        _check(_lib.stmg_hierarchy_device_bytes(self._h, C.byref(b)))
        return b.value

    def release_staging(self) -> None:
        """Free the device (b, u) slots mg_solve_stream keeps between calls."""
        _check(_lib.stmg_hierarchy_release_staging(self._h))

    def level_coeffs(self, l: int) -> dict:
        nn = self.levels[l].n_el + 1
        arrs = [np.zeros(nn) for _ in range(7)]
        _check(_lib.stmg_hierarchy_level_coeffs(self._h, l, *[a.ctypes.data for a in arrs]))
        return dict(zip(["cur_m", "cur_0", "cur_p", "oth_m", "oth_0", "oth_p", "inv_diag"], arrs))

    def level_stencil9(self, l: int) -> dict:
        """Level l's operator as a 9-point stencil (any level, Galerkin included)."""
        lv = self.levels[l]
        nd = (lv.n_el + 1) * (lv.n_t + 1)
        v9, mask, inv = np.zeros(9 * nd), np.zeros(nd, np.uint16), np.zeros(nd)
        _check(_lib.stmg_hierarchy_level_stencil9(self._h, l, v9.ctypes.data, mask.ctypes.data,
                                                  inv.ctypes.data))
        return dict(v9=v9.reshape(9, nd), mask=mask, inv_diag=inv)

    # -- level kernels on device vectors (torch tensors on this hierarchy's device) --
    def sweeps(self, l, f, x, n, omega=0.5):
        _check(_lib.stmg_level_sweeps(self._h, l, _ptr(f), _ptr(x), int(n), float(omega)))

    def sweep_kernels(self, l, f, x, y, launches, fused_pairs=False, omega=0.5):
        """Benchmark form (asynchronous): ping-pong x <-> y for `launches` launches of a
        single sweep (False / 0), a fused pair (True / 1) or a fused 3- / 4-sweep pass (3, 4)."""
        _check(_lib.stmg_level_sweep_kernels(self._h, l, _ptr(f), _ptr(x), _ptr(y), int(launches),
                                             int(fused_pairs), float(omega)))

    def residual(self, l, f, x, r):
        _check(_lib.stmg_level_residual(self._h, l, _ptr(f), _ptr(x), _ptr(r)))

    def restrict_residual(self, l, f, x, fc):
        _check(_lib.stmg_level_restrict_residual(self._h, l, _ptr(f), _ptr(x), _ptr(fc)))

    def restrict(self, l, r, fc):
        _check(_lib.stmg_level_restrict(self._h, l, _ptr(r), _ptr(fc)))

    def prolong_add(self, l, xc, x):
        _check(_lib.stmg_level_prolong_add(self._h, l, _ptr(xc), _ptr(x)))

    def coarsest_solve(self, f, x):
        _check(_lib.stmg_coarsest_solve(self._h, _ptr(f), _ptr(x)))

    def residual_norm(self, f, x) -> float:
        v = C.c_double()
        _check(_lib.stmg_residual_norm(self._h, _ptr(f), _ptr(x), C.byref(v)))
        return v.value

    def norm2(self, x) -> float:
        v = C.c_double()
        _check(_lib.stmg_norm2(self._h, _ptr(x), _numel(x), C.byref(v)))
        return v.value

    def synchronize(self):
        _check(_lib.stmg_synchronize(self._h))

    def set_stream(self, stream):
        """Run on a caller stream (a torch.cuda.Stream, a raw cudaStream_t int, or None)."""
        raw = getattr(stream, "cuda_stream", stream)
        _check(_lib.stmg_hierarchy_set_stream(self._h, C.c_void_p(raw) if raw else None))

    def set_tiling(self, small_dofs=0, tiny_dofs=0):
        """Per-handle time-tile thresholds (stmg_hierarchy_set_tiling; 0 = defaults)."""
        _check(_lib.stmg_hierarchy_set_tiling(self._h, int(small_dofs), int(tiny_dofs)))

    FUSE_VIRTUAL_ZERO, FUSE_FINE_DOWN, FUSE_FINE_UP, FUSE_ALL, FUSE_DEFAULT = 1, 2, 4, 7, 5

    def set_fusion(self, flags=5):
        """V-cycle fusions (stmg_hierarchy_set_fusion): bit-identical, traffic differs."""
        _check(_lib.stmg_hierarchy_set_fusion(self._h, int(flags)))

    (FUSED_ZERO_SWEEP, FUSED_ZERO_PAIR, FUSED_ZERO_RESTRICT, FUSED_ZERO_PROLONG_SWEEP, FUSED_FINE_DOWN,
     FUSED_NORM_SWEEP, FUSED_PROLONG_SWEEP, FUSED_FINE_UP) = range(8)

    def fused_kernel(self, l, kind, f, x=None, xc=None, y=None, fc=None, omega=0.5):
        """stmg_level_fused on device tensors; returns ||f - J x||^2 for FUSED_FINE_DOWN."""
        nrm = C.c_double(0.0)
        _check(_lib.stmg_level_fused(self._h, int(l), int(kind), _ptr(f), _ptr(x), _ptr(xc), _ptr(y), _ptr(fc),
                                     float(omega), C.byref(nrm)))
        return nrm.value

    def set_profiling(self, on=True):
        """True / 1: finest-level kernels; 2: every kernel (see stmg_b200.h)."""
        _check(_lib.stmg_hierarchy_set_profiling(self._h, int(on)))

    PROFILE_KINDS = ("sweep", "restrict", "prolong_sweep", "sweep_pair", "sweep_from_zero", "coarsest")

    def profile(self) -> dict:
        """{level: {kind: (launches, seconds)}} accumulated over profiled solves."""
        out = {}
        for l in range(self._n_levels):
            d = {}
            for kind, name in enumerate(self.PROFILE_KINDS):
                n, t = C.c_int64(), C.c_double()
                _check(_lib.stmg_hierarchy_profile(self._h, l, kind, C.byref(n), C.byref(t)))
                if n.value:
                    d[name] = (n.value, t.value)
            out[l] = d
        return out


def build_hierarchy(fine: SpaceTimeGrid, method, path: CoarseningPath, chi=None, mat=None,
                    device: int = 0) -> LevelHierarchy:
    """proj/src/multigrid.cpp:86-143: method "CK"/"CD"/"CR"/"CP" (causal) or "BK"/"BD"/"BR"/"BP"
    (bilinear temporal transfers); path directions x, t or xt (FullST, causal only)."""
    if not fine.has_materials():
        raise ValueError("build_hierarchy: fine grid has no materials")
    name = method if isinstance(method, str) else str(method)
    k = _f64(fine.k, fine.n_el)
    c = _f64(fine.c, fine.n_el)
    chi_a = None if chi is None else _f64(chi.chi if hasattr(chi, "chi") else chi, fine.n_el)
    m = None if mat is None else MaterialPair.of(mat)._c()
    dirs = np.array([int(d) for d in path.dirs], np.int32)
    h = C.c_void_p()
    gc = fine._c()
    _check(_lib.stmg_hierarchy_create(C.byref(gc), k.ctypes.data, c.ctypes.data,
                                      None if chi_a is None else chi_a.ctypes.data,
                                      None if m is None else C.byref(m), name.encode(), dirs.size,
                                      dirs.ctypes.data if dirs.size else None, int(device),
                                      C.byref(h)))
    return LevelHierarchy(h, path, name, device)


def level_stencil9_host(fine: SpaceTimeGrid, method, path: CoarseningPath, level: int, chi=None,
                        mat=None, adjoint: bool = False) -> dict:
    """build_hierarchy's host half only (no GPU): level `level`'s operator as a
    9-point stencil, transposed when `adjoint` (see include/stmg_b200.h)."""
    if not fine.has_materials():
        raise ValueError("build_hierarchy: fine grid has no materials")
    k = _f64(fine.k, fine.n_el)
    c = _f64(fine.c, fine.n_el)
    chi_a = None if chi is None else _f64(chi.chi if hasattr(chi, "chi") else chi, fine.n_el)
    m = None if mat is None else MaterialPair.of(mat)._c()
    dirs = np.array([int(d) for d in path.dirs], np.int32)
    ne, nt = fine.n_el, fine.n_t
    for d in dirs[:level]:
        ne, nt = (ne // 2 if d != 1 else ne), (nt // 2 if d != 0 else nt)
    nd = (ne + 1) * (nt + 1)
    v9, mask, inv = np.zeros(9 * nd), np.zeros(nd, np.uint16), np.zeros(nd)
    gc = fine._c()
    _check(_lib.stmg_level_stencil9_host(C.byref(gc), k.ctypes.data, c.ctypes.data,
                                         None if chi_a is None else chi_a.ctypes.data,
                                         None if m is None else C.byref(m), str(method).encode(),
                                         dirs.size, dirs.ctypes.data if dirs.size else None,
                                         int(level), 1 if adjoint else 0, v9.ctypes.data,
                                         mask.ctypes.data, inv.ctypes.data))
    return dict(v9=v9.reshape(9, nd), mask=mask, inv_diag=inv, n_el=ne, n_t=nt)


def transposed_hierarchy(h: LevelHierarchy) -> LevelHierarchy:
    """proj/src/multigrid.cpp:145-160"""
    out = C.c_void_p()
    _check(_lib.stmg_hierarchy_transposed(h.handle, C.byref(out)))
    return LevelHierarchy(out, h.path, h.method, h.device, adjoint=not h.adjoint, parent=h)


def mg_solve(h: LevelHierarchy, b, u, opts: Optional[SolveOptions] = None, zero_guess: bool = False) -> SolveReport:
    """V-cycle solve of J u = b from the caller's u (warm start), u updated in place.

    b and u may be numpy arrays (host) or torch tensors (host, pinned or on the
    hierarchy's GPU); proj/src/multigrid.cpp:212-279.  zero_guess: start from zero, u is
    output only (stmg_mg_solve_ex, STMG_SOLVE_ZERO_GUESS): a host u is not uploaded.
    """
    o = opts or SolveOptions()
    n = h.levels[0].n_dofs
    if _numel(b) != n or _numel(u) != n:
        raise ValueError("mg_solve: vector size mismatch")
    hist = np.zeros(max(o.max_cycles, 0) + 1, np.float64)
    rep = _SolveRep()
    co = _SolveOpts(int(o.nu), float(o.omega), float(o.tol), float(o.div_tol), int(o.max_cycles))
    if zero_guess:
        _check(_lib.stmg_mg_solve_ex(h.handle, _ptr(b), _ptr(u), C.byref(co), 1, C.byref(rep), hist.ctypes.data,
                                     hist.size))
    else:
        _check(_lib.stmg_mg_solve(h.handle, _ptr(b), _ptr(u), C.byref(co), C.byref(rep), hist.ctypes.data,
                                  hist.size))
    kt = {}
    if rep.fine_sweeps or rep.fine_restricts or rep.fine_prolong_sweeps or rep.fine_sweep_pairs:
        kt = {"fine_sweep": (rep.fine_sweeps, rep.fine_sweep_seconds),
              "fine_sweep_pair": (rep.fine_sweep_pairs, rep.fine_sweep_pair_seconds),
              "fine_restrict": (rep.fine_restricts, rep.fine_restrict_seconds),
              "fine_prolong_sweep": (rep.fine_prolong_sweeps, rep.fine_prolong_sweep_seconds),
              "fine_norm_pass": (rep.fine_norm_passes, rep.fine_norm_pass_seconds),
              "fine_up": (rep.fine_ups, rep.fine_up_seconds)}
    return SolveReport(SolveStatus(rep.status), rep.cycles, rep.factor,
                       [float(v) for v in hist[: rep.n_history]], bool(rep.absolute_norms),
                       rep.seconds, rep.device_seconds, rep.smoother_dof_updates, rep.kernel_launches,
                       kt)


def mg_solve_batch(hs: Sequence[LevelHierarchy], bs, us, opts: Optional[SolveOptions] = None) -> list:
    """Independent solves run concurrently (each hierarchy on its own stream / GPU):
    entry i is mg_solve(hs[i], bs[i], us[i], opts).  Hierarchies must not share a
    workspace (a hierarchy and its transpose do)."""
    o = opts or SolveOptions()
    k = len(hs)
    if len(bs) != k or len(us) != k:
        raise ValueError("mg_solve_batch: hs, bs and us differ in length")
    for h, b, u in zip(hs, bs, us):
        n = h.levels[0].n_dofs
        if _numel(b) != n or _numel(u) != n:
            raise ValueError("mg_solve_batch: vector size mismatch")
    cap = max(o.max_cycles, 0) + 1
    hist = np.zeros((max(k, 1), cap), np.float64)
    reps = (_SolveRep * max(k, 1))()
    co = _SolveOpts(int(o.nu), float(o.omega), float(o.tol), float(o.div_tol), int(o.max_cycles))
    H = (C.c_void_p * max(k, 1))(*[h.handle.value for h in hs])
    B = (C.c_void_p * max(k, 1))(*[_ptr(b) for b in bs])
    U = (C.c_void_p * max(k, 1))(*[_ptr(u) for u in us])
    P = (C.c_void_p * max(k, 1))(*[hist[i].ctypes.data for i in range(k)])
    _check(_lib.stmg_mg_solve_batch(k, H, B, U, C.byref(co), reps, P, cap))
    out = []
    for i in range(k):
        r = reps[i]
        out.append(SolveReport(SolveStatus(r.status), r.cycles, r.factor, [float(v) for v in hist[i, : r.n_history]],
                               bool(r.absolute_norms), r.seconds, r.device_seconds, r.smoother_dof_updates,
                               r.kernel_launches))
    return out


def mg_solve_stream(h: LevelHierarchy, bs, us, opts: Optional[SolveOptions] = None, zero_guess: bool = False) -> list:
    """A stream of solves on one hierarchy with host vectors (stmg_mg_solve_stream):
    entry k is mg_solve(h, bs[k], us[k], opts, zero_guess), in order, bit-identical; the
    upload of entry k + 1 and the download of entry k - 1 overlap solve k (pinned host
    vectors).  h.release_staging() frees the two device (b, u) slots it keeps."""
    o = opts or SolveOptions()
    k = len(bs)
    if len(us) != k:
        raise ValueError("mg_solve_stream: bs and us differ in length")
    n = h.levels[0].n_dofs
    for b, u in zip(bs, us):
        if _numel(b) != n or _numel(u) != n:
            raise ValueError("mg_solve_stream: vector size mismatch")
    cap = max(o.max_cycles, 0) + 1
    hist = np.zeros((max(k, 1), cap), np.float64)
    reps = (_SolveRep * max(k, 1))()
    co = _SolveOpts(int(o.nu), float(o.omega), float(o.tol), float(o.div_tol), int(o.max_cycles))
    B = (C.c_void_p * max(k, 1))(*[_ptr(b) for b in bs])
    U = (C.c_void_p * max(k, 1))(*[_ptr(u) for u in us])
    P = (C.c_void_p * max(k, 1))(*[hist[i].ctypes.data for i in range(k)])
    _check(_lib.stmg_mg_solve_stream(h.handle, k, B, U, C.byref(co), 1 if zero_guess else 0, reps, P, cap))
    out = []
    for i in range(k):
        r = reps[i]
        out.append(SolveReport(SolveStatus(r.status), r.cycles, r.factor, [float(v) for v in hist[i, : r.n_history]],
                               bool(r.absolute_norms), r.seconds, r.device_seconds, r.smoother_dof_updates,
                               r.kernel_launches))
    return out


# ---- topology optimisation (BASELINE config 4; proj/src/optimisation.cpp:83-186) -----
@dataclass
class OptimisationOptions:
    """proj/include/stmg/optimisation.hpp:59-75 (+ MmaOptions, mma.hpp:23-30)."""
    method: str = "CR"
    strategy: PlanStrategy = PlanStrategy.Contrast
    n_levels: int = 6
    lambda_crit: float = 0.25
    min_elements: int = 0
    warm_start: bool = True
    volume_limit: float = 0.5
    theta_ref: float = 1e6
    chi_init: float = 0.5
    max_iterations: int = 500
    rel_change_tol: float = 1e-3
    stable_iterations: int = 5
    solve: SolveOptions = field(default_factory=lambda: SolveOptions(nu=20))
    mma_x_min: float = 0.0
    mma_x_max: float = 1.0
    mma_move_limit: float = 0.2
    mma_asym_init: float = 0.5
    mma_asym_shrink: float = 0.7
    mma_asym_grow: float = 1.2


@dataclass
class OptimisationResult:
    chi: np.ndarray
    theta: float
    converged: bool
    iterations: int
    history: list
    seconds: float
    design_history: Optional[np.ndarray] = None  # row i: the design evaluated at iteration i + 1


def objective_sensitivities(geom: SpaceTimeGrid, mat, chi, u, lam, device: int = 0) -> np.ndarray:
    """proj/src/optimisation.cpp:34-73 on the GPU (u, lam host arrays or device tensors)."""
    n = (geom.n_el + 1) * (geom.n_t + 1)
    if _numel(u) != n or _numel(lam) != n:
        raise ValueError("objective_sensitivities: state size mismatch")
    chi_a = _f64(chi.chi if hasattr(chi, "chi") else chi, geom.n_el)
    sens = np.zeros(geom.n_el)
    gc = geom._c()
    m = MaterialPair.of(mat)._c()
    _check(_lib.stmg_objective_sensitivities(C.byref(gc), C.byref(m), chi_a.ctypes.data, _ptr(u), _ptr(lam),
                                             sens.ctypes.data, int(device)))
    return sens


def optimise(geom: SpaceTimeGrid, mat, opts: Optional[OptimisationOptions] = None,
             device: int = 0) -> OptimisationResult:
    o = opts or OptimisationOptions()
    so = o.solve
    co = _OptOpts(MaterialPair.of(mat)._c(), o.method.encode(), int(o.strategy), int(o.n_levels),
                  float(o.lambda_crit), int(o.min_elements), 1 if o.warm_start else 0,
                  float(o.volume_limit), float(o.theta_ref), float(o.chi_init), int(o.max_iterations),
                  float(o.rel_change_tol), int(o.stable_iterations),
                  _SolveOpts(int(so.nu), float(so.omega), float(so.tol), float(so.div_tol), int(so.max_cycles)),
                  o.mma_x_min, o.mma_x_max, o.mma_move_limit, o.mma_asym_init, o.mma_asym_shrink,
                  o.mma_asym_grow)
    chi = np.zeros(geom.n_el)
    recs = (_IterRec * int(o.max_iterations))()
    designs = np.zeros((int(o.max_iterations), geom.n_el))
    nr, conv = C.c_int32(), C.c_int32()
    th, secs = C.c_double(), C.c_double()
    gc = geom._c()
    _check(_lib.stmg_optimise(C.byref(gc), C.byref(co), int(device), chi.ctypes.data, recs, C.byref(nr),
                              C.byref(th), C.byref(conv), C.byref(secs), designs.ctypes.data))
    hist = []
    for i in range(nr.value):
        d = {f: getattr(recs[i], f) for f, _ in _IterRec._fields_}
        d["path"] = d["path"].decode()
        hist.append(d)
    return OptimisationResult(chi, th.value, bool(conv.value), nr.value, hist, secs.value,
                              designs[: nr.value].copy())


# ---- time-slab multi-GPU ------------------------------------------
def dist_partition(n_t_per_level: Sequence[int], dirs: Sequence[int], world: int,
                   min_slab: int = 16) -> tuple[int, np.ndarray]:
    """(number of distributed levels Lg, bounds[Lg, world+1]) of the time-slab split."""
    nts = np.ascontiguousarray(n_t_per_level, np.int64)
    d = np.ascontiguousarray(list(dirs) if len(dirs) else [0], np.int32)
    lg = C.c_int32()
    bounds = np.zeros(nts.size * (world + 1), np.int64)
    _check(_lib.stmg_dist_partition(nts.size, nts.ctypes.data, d.ctypes.data, int(world),
                                    int(min_slab), C.byref(lg), bounds.ctypes.data))
    return lg.value, bounds[: lg.value * (world + 1)].reshape(lg.value, world + 1)


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(_lib.stmg_dist_nccl_unique_id(buf, 128))
    return bytes(buf)


class DistHierarchy:
    """Time-slab distributed hierarchy (include/stmg_b200.h, stmg_dist_*)."""

    def __init__(self, handle, levels, world, rank):
        self._h = handle
        self.levels = levels
        self.world = world
        self.rank = rank
        lg, lo, hi, nl, db = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int32(), C.c_int64()
        _check(_lib.stmg_dist_info(self._h, C.byref(lg), C.byref(lo), C.byref(hi), C.byref(nl), C.byref(db)))
        self.n_distributed = lg.value
        self.row_lo, self.row_hi, self.n_local, self.device_bytes = lo.value, hi.value, nl.value, db.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.stmg_dist_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def split_passes(self) -> int:
        """Passes captured with the ghost exchange overlapping interior rows (STMG_DIST_OVERLAP)."""
        v = C.c_int64(0)
        _check(_lib.stmg_dist_split_passes(self._h, C.byref(v)))
        return int(v.value)

    @property
    def loop_on_device(self) -> bool:
        """The last solve's cycle loop ran as one device graph (stmg_dist_loop_on_device)."""
        v = C.c_int32(0)
        _check(_lib.stmg_dist_loop_on_device(self._h, C.byref(v)))
        return bool(v.value)

    @property
    def transport(self) -> str:
        """Ghost-exchange transport: "nccl", "loopback" or "p2p" (STMG_DIST_P2P=1)."""
        buf = C.create_string_buffer(32)
        _check(_lib.stmg_dist_transport(self._h, buf, 32))
        return buf.value.decode()


def build_dist_hierarchy(fine: SpaceTimeGrid, method, path: CoarseningPath, world: int, rank: int = 0,
                         nccl_id: Optional[bytes] = None, device: int = 0, adjoint: bool = False,
                         chi=None, mat=None, min_slab: int = 16) -> DistHierarchy:
    """Distributed (time-slab) hierarchy.  nccl_id=None: loopback (all ranks in this process)."""
    if not fine.has_materials():
        raise ValueError("build_hierarchy: fine grid has no materials")
    k = _f64(fine.k, fine.n_el)
    c = _f64(fine.c, fine.n_el)
    chi_a = None if chi is None else _f64(chi, fine.n_el)
    m = None if mat is None else MaterialPair.of(mat)._c()
    dirs = np.array([int(d) for d in path.dirs], np.int32)
    idbuf = None if nccl_id is None else (C.c_char * 128).from_buffer_copy(nccl_id)
    h = C.c_void_p()
    gc = fine._c()
    _check(_lib.stmg_dist_create(C.byref(gc), k.ctypes.data, c.ctypes.data,
                                 None if chi_a is None else chi_a.ctypes.data,
                                 None if m is None else C.byref(m), str(method).encode(), dirs.size,
                                 dirs.ctypes.data if dirs.size else None, 1 if adjoint else 0,
                                 int(world), int(rank), idbuf, int(device), int(min_slab), C.byref(h)))
    levels = []
    ne, nt = fine.n_el, fine.n_t
    levels.append(LevelInfo(ne, nt, 0.0))
    for d in dirs:
        if d == 0:
            ne //= 2
        else:
            nt //= 2
        levels.append(LevelInfo(ne, nt, 0.0))
    return DistHierarchy(h, levels, world, rank)


def mg_solve_dist(h: DistHierarchy, b, u, opts: Optional[SolveOptions] = None) -> SolveReport:
    """Distributed solve; b, u full-size; u receives this process's slab rows (loopback: all)."""
    o = opts or SolveOptions()
    n = h.levels[0].n_dofs
    if _numel(b) != n or _numel(u) != n:
        raise ValueError("mg_solve: vector size mismatch")
    hist = np.zeros(max(o.max_cycles, 0) + 1, np.float64)
    rep = _SolveRep()
    co = _SolveOpts(int(o.nu), float(o.omega), float(o.tol), float(o.div_tol), int(o.max_cycles))
    _check(_lib.stmg_dist_mg_solve(h.handle, _ptr(b), _ptr(u), C.byref(co), C.byref(rep),
                                   hist.ctypes.data, hist.size))
    return SolveReport(SolveStatus(rep.status), rep.cycles, rep.factor,
                       [float(v) for v in hist[: rep.n_history]], bool(rep.absolute_norms),
                       rep.seconds, rep.device_seconds, rep.smoother_dof_updates, rep.kernel_launches)


def mg_solve_dist_local(h: DistHierarchy, b_local, u_local, opts: Optional[SolveOptions] = None) -> SolveReport:
    """Distributed solve on slab-local vectors: this process's level-0 rows
    [h.row_lo, h.row_hi) only (stmg_dist_mg_solve_local); memory scales as 1/W."""
    o = opts or SolveOptions()
    n = (h.row_hi - h.row_lo) * (h.levels[0].n_el + 1)
    if _numel(b_local) != n or _numel(u_local) != n:
        raise ValueError("mg_solve: vector size mismatch")
    hist = np.zeros(max(o.max_cycles, 0) + 1, np.float64)
    rep = _SolveRep()
    co = _SolveOpts(int(o.nu), float(o.omega), float(o.tol), float(o.div_tol), int(o.max_cycles))
    _check(_lib.stmg_dist_mg_solve_local(h.handle, _ptr(b_local), _ptr(u_local), C.byref(co), C.byref(rep),
                                         hist.ctypes.data, hist.size))
    return SolveReport(SolveStatus(rep.status), rep.cycles, rep.factor,
                       [float(v) for v in hist[: rep.n_history]], bool(rep.absolute_norms),
                       rep.seconds, rep.device_seconds, rep.smoother_dof_updates, rep.kernel_launches)



def abi_version() -> int:
    return _lib.stmg_abi_version()
