"""The C-ABI library (no GPU needed): it loads, exports every symbol that
include/stmg_b200.h declares, and its host-side setup functions reproduce the
reference bit for bit (via the oracle restatement and the golden plans)."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stmg_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(stmg_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    from paper_2505_10168_b200 import stmg

    lib = ctypes.CDLL(stmg.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a_only():
    import subprocess

    from paper_2505_10168_b200 import stmg

    out = subprocess.run(["cuobjdump", "--list-elf", stmg.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def test_apply_design_and_load_vector_match_oracle(port):
    from paper_2505_10168_b200 import stmg as S

    chi = np.linspace(0, 1, 257)
    mat = (1e-3, 1.0, 1.0, 2.0, 3.0, 2.0)
    k, c = S.apply_design(chi, mat)
    kp, cp = port.apply_design(chi, mat)
    assert np.array_equal(bits(k), bits(kp)) and np.array_equal(bits(c), bits(cp))
    for kind, params in ((0, (1.0,)), (1, (1.0, 0.1)), (2, (0.5, 8.0, 0.05)), (3, ())):
        for ne, nt in ((16, 8), (1024, 33)):
            g = S.build_fine_grid(1.0, 1.0, ne, nt)
            b = S.load_vector(g, kind=kind, params=params, masked=True)
            assert np.array_equal(bits(b), bits(port.load_vector(1.0, 1.0, ne, nt, kind, params)))


def test_load_vector_callback_matches_preset():
    from paper_2505_10168_b200 import stmg as S

    g = S.build_fine_grid(4.0, 2.0, 4, 2)
    b = S.load_vector(g, lambda x, t: 1.0)
    # proj/tests/test_assembly.cpp:72-85: q dx/2 per element-node, none at t = 0
    np.testing.assert_array_equal(b[:5], 0.0)
    np.testing.assert_allclose(b[5:10], [0.5, 1.0, 1.0, 1.0, 0.5])
    bp = S.load_vector(g, kind=0, params=(1.0,))
    assert np.array_equal(bits(b), bits(bp))


def test_plans_match_reference_golden():
    from paper_2505_10168_b200 import configs as C
    from paper_2505_10168_b200 import stmg as S

    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "plans.json")))
    for name, want in gold.items():
        cfg = C.CONFIGS[name]()
        g = S.build_fine_grid(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t)
        g.k, g.c = cfg.k, cfg.c
        req = S.PlanRequest(n_levels=want["n_levels"], strategy=S.PlanStrategy(want["strategy"]),
                            reassembly=S.ReassemblyMethod(want["reassembly"]),
                            min_elements=want["min_elements"], chi=cfg.chi, mat=cfg.mat)
        p = S.plan_coarsening(g, req)
        assert [int(d) for d in p.dirs] == want["dirs"], name
        assert [float(v).hex() for v in p.indicator_at_decision] == want["indicators"], name


def test_planner_known_answers():
    """proj/tests/test_strategy.cpp:93-110, 163-189."""
    from paper_2505_10168_b200 import stmg as S

    g = S.build_fine_grid(1.0, 1.0, 16, 16)
    g.k, g.c = np.ones(16), np.ones(16)
    p = S.plan_coarsening(g, S.PlanRequest(n_levels=6, strategy=S.PlanStrategy.Uniform))
    assert S.path_to_string(p) == "x,x,x,x,t"
    assert p.indicator_at_decision == [16.0, 4.0, 1.0, 0.25, 0.0625]
    g8 = S.build_fine_grid(1.0, 1.0, 8, 8)
    g8.k, g8.c = np.ones(8), np.ones(8)
    p = S.plan_coarsening(g8, S.PlanRequest(n_levels=4, strategy=S.PlanStrategy.Resolution, min_elements=8))
    assert S.path_to_string(p) == "t,t,t"
    with pytest.raises(RuntimeError):  # std::runtime_error: forced time step impossible
        S.plan_coarsening(g8, S.PlanRequest(n_levels=5, strategy=S.PlanStrategy.Resolution, min_elements=8))
    p = S.plan_coarsening(g8, S.PlanRequest(n_levels=4, strategy=S.PlanStrategy.Resolution, min_elements=2))
    assert S.path_to_string(p) == "x,x,t" and p.indicator_at_decision == [8.0, 2.0, 0.5]
    with pytest.raises(ValueError):  # std::invalid_argument
        S.plan_coarsening(g8, S.PlanRequest(n_levels=0))
    # R reassembly: harmonic mean gives the smaller coarse indicator (test_strategy.cpp:127-133)
    g4 = S.build_fine_grid(1.0, 1.0, 4, 16)
    g4.k, g4.c = np.array([1.0, 4.0, 1.0, 4.0]), np.ones(4)
    p = S.plan_coarsening(g4, S.PlanRequest(n_levels=3, reassembly=S.ReassemblyMethod.R))
    assert S.path_to_string(p) == "x,x" and p.indicator_at_decision == [2.0, 0.4]


def test_design_independent_plan_and_validation():
    from paper_2505_10168_b200 import stmg as S

    g = S.build_fine_grid(0.1, 10.0, 16, 16)
    mat = (0.197, 214.0, 1.67e6, 2.41e6, 3.0, 2.0)
    p = S.plan_coarsening(g, S.PlanRequest(n_levels=3, strategy=S.PlanStrategy.DesignIndependent, mat=mat))
    assert S.path_to_string(p) == "t,t"  # proj/tests/test_strategy.cpp:191-212
    with pytest.raises(ValueError):
        S.plan_coarsening(g, S.PlanRequest(n_levels=3, strategy=S.PlanStrategy.DesignIndependent,
                                           mat=(0.5, 1.0, 0.5, 1.0, 3.0, 2.0)))


def test_errors_map_to_reference_exception_classes():
    from paper_2505_10168_b200 import stmg as S

    with pytest.raises(ValueError):
        S.build_fine_grid(0.0, 1.0, 4, 4)
    with pytest.raises(ValueError):
        S.apply_design(np.array([1.5]), (1, 1, 1, 1, 3, 2))
    g = S.build_fine_grid(1.0, 1.0, 4, 4)
    with pytest.raises(ValueError):  # no materials
        S.build_hierarchy(g, "CK", S.CoarseningPath([]))
    g.k, g.c = np.ones(4), np.ones(4)
    with pytest.raises(ValueError):  # FullST is causal-only (proj/src/transfer.cpp:44-47)
        S.build_hierarchy(g, "BK", S.CoarseningPath([S.CoarseningDirection.FullST]))
    with pytest.raises(ValueError):
        S.build_hierarchy(g, "XX", S.CoarseningPath([]))


def test_no_silent_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2505_10168_b200 import stmg as S

    g = S.build_fine_grid(1.0, 1.0, 4, 4)
    g.k, g.c = np.ones(4), np.ones(4)
    with pytest.raises(S.StmgCudaError):
        S.build_hierarchy(g, "CK", S.CoarseningPath([]))


def test_dist_create_argument_errors_before_device_work():
    from paper_2505_10168_b200 import stmg as S

    g = S.build_fine_grid(1.0, 1.0, 8, 8)
    g.k, g.c = np.ones(8), np.ones(8)
    with pytest.raises(ValueError):  # time slabs take causal K/D/R only: rejected in the C layer, no device touched
        S.build_dist_hierarchy(g, "CP", S.CoarseningPath([S.CoarseningDirection(0)]), world=1, rank=0)


def test_abi_version_matches_header():
    """The ctypes struct layouts in stmg.py belong to one C ABI version: the header's."""
    import re

    from paper_2505_10168_b200 import stmg as S

    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "stmg_b200.h")).read()
    v = int(re.search(r"#define STMG_ABI_VERSION (\d+)", hdr).group(1))
    assert S.ABI_VERSION == v == S.abi_version()
