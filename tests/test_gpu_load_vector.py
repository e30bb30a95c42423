"""Device-side right-hand side: load_vector
(proj/src/assembly.cpp:65-83) evaluated by a CUDA kernel, against the host
restatement (itself pinned bitwise to the oracle and the reference,
tests/test_capi_cpu.py).  Kinds without transcendentals are bit-identical;
sin / cos sources agree to a few ulp of the vector's max-norm (CUDA's fp64
sin/cos vs glibc; heat_load_value's 1 + cos(.) cancels near its zeros, so the
error is absolute, not relative per entry)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ULP_TOL = 4 * np.finfo(np.float64).eps


@pytest.fixture(scope="module")
def torch():
    import torch as _t

    assert _t.cuda.is_available(), "GPU tests need CUDA (no CPU fallback exists)"
    return _t


@pytest.fixture(scope="module")
def S(torch):
    from paper_2505_10168_b200 import stmg

    return stmg


SOURCES = [(0, (1.0,)), (1, (1.0, 0.1)), (2, (0.5, 8.0, 0.05)), (3, ())]


@pytest.mark.parametrize("kind,params", SOURCES)
@pytest.mark.parametrize("ne,nt,masked", [(16, 8, True), (1024, 33, True), (37, 5, False), (1, 3, True)])
def test_device_matches_host(torch, S, kind, params, ne, nt, masked):
    g = S.build_fine_grid(1.0, 2.0, ne, nt)
    h = S.load_vector(g, kind=kind, params=params, masked=masked)
    d = S.load_vector_device(g, kind=kind, params=params, masked=masked).cpu().numpy()
    if kind in (0, 1):
        assert np.array_equal(d.view(np.uint64), h.view(np.uint64))
    else:
        assert np.max(np.abs(d - h)) <= ULP_TOL * np.max(np.abs(h))


def test_cfg2_source_on_full_width_window(torch, S):
    """The cfg2 source (modulated box, BASELINE configs[2]) at the full 16384-node
    width over a 256-level window, whose dt equals the full grid's."""
    from paper_2505_10168_b200 import configs as C

    cfg = C.cfg2(n_el=16384, n_t=256)
    g = S.build_fine_grid(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t)
    h = S.load_vector(g, kind=cfg.source_kind, params=cfg.source_params, masked=True)
    d = S.load_vector_device(g, kind=cfg.source_kind, params=cfg.source_params).cpu().numpy()
    assert np.max(np.abs(d - h)) <= ULP_TOL * np.max(np.abs(h))
    assert np.count_nonzero(d) == np.count_nonzero(h)


def test_rejects_host_memory(torch, S):
    g = S.build_fine_grid(1.0, 1.0, 4, 4)
    gc = g._c()
    b = np.zeros(g.n_dofs())
    import ctypes as C

    p = (C.c_double * 4)(1.0, 0, 0, 0)
    rc = S._lib.stmg_load_vector_device(C.byref(gc), 0, p, 1, b.ctypes.data, None)
    assert rc == S.STMG_EINVAL
