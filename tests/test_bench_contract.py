"""bench.py's output contract: exactly one JSON line on stdout with the keys the
driver reads, for the reference arm (CPU, a tiny time-truncated sample) and for
the GPU arm (BASELINE config 1, one timed step)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def run_bench(*args, timeout=600):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, p.stdout[-3000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libstmg_ref.so")) and \
            not os.path.exists(os.path.join(ROOT, "oracle", "liboracle_port.so")):
        pytest.skip("oracle libraries not built (run __graft_entry__.build())")
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "1", "--cpu-sample-nt", "16",
                  "--ref-cores", "2", timeout=300)
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "cfg2" and d["config"]["n_t"] == 65536 and d["config"]["sample_n_t"] == 16
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["cores"] == 2 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["cpu_baseline"]["nproc"] >= 1 and "cpu_model" in d["cpu_baseline"]


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = run_bench("--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--cfg1", "0", "--profile-steps", "1",
                  timeout=900)
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["config"]["workload"] == "cfg2" and d["dtype"] == "f64" and d["n_gpus"] == 1
    assert d["config"]["dofs"] == 16385 * 65537
    # the reference's own stopping rule: Diverged after 3 V-cycles (the C oracle at full
    # size, tests/test_gpu_scale.py; the reference at reduced size, tests/golden/cfg2_mini.npz)
    assert d["cycles"] == 3 and d["status"] == "diverged"
    assert d["value"] > 0 and d["gpu_launches"] > 0
    # headline e2e: b uploaded, u output only (zero initial guess flag); in/out u beside it
    assert d["e2e"]["h2d_bytes_per_step"] == 8 * d["config"]["dofs"]
    assert d["e2e"]["d2h_bytes_per_step"] == 8 * d["config"]["dofs"]
    assert d["e2e"]["inout_u"]["h2d_bytes_per_step"] == 16 * d["config"]["dofs"]
    assert d["e2e"]["value"] > d["e2e"]["inout_u"]["value"] > 0
    # streamed e2e (copies overlap the neighbouring solves) with the one-solve figure beside it
    assert d["e2e"]["steps"] >= 2 and "stmg_mg_solve_stream" in d["e2e"]["mode"]
    assert d["e2e"]["value"] >= 0.9 * d["e2e"]["single"]["value"] > d["e2e"]["inout_u"]["value"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    assert "sm_mhz" in d["clocks"]
