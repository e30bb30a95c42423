#!/usr/bin/env python
"""Benchmark: STMG solve on B200 (BASELINE metric: space-time DOF smoother
updates/s; STMG solve time).

Workload (N = 1): BASELINE configs[2], the largest single-GPU config:
cfg2 = 16384 x 65536 (1.07e9 space-time DOFs, 8.6 GB per vector), CR,
Resolution planner (M = 256), 18 levels, V(1,1), run under the reference's
own stopping rule (tol 1e-10, div_tol 1e9, proj/src/multigrid.cpp:260-273):
the i.i.d. 1e4-contrast design makes the reference algorithm diverge, and both
the reference (tests/golden/cfg2_mini.npz) and this build stop with Diverged
after the same V-cycles (3 at full size).  A step is one such solve.

* `value`: smoother DOF updates per second (sum over non-coarsest levels of
  2 nu N_l per cycle) with b and u resident in HBM, CUDA events on the solve's
  stream, max over ranks.  Inputs exceed L2 (3 x 8.6 GB), so no flush is needed.
* `e2e`: the same solve through the C ABI with pinned HOST b and u: h2d of b and d2h
  of u inside the timed region (stmg_mg_solve_ex with STMG_SOLVE_ZERO_GUESS: the
  workload starts from u = 0, so u is output only).  `e2e.value` is the throughput of a
  stream of such solves on one hierarchy (stmg_mg_solve_stream: every step uploads its b
  and downloads its u, step k's copies overlap its neighbours' solves; fill and drain
  timed) -- the figure the reference arm's batch of concurrent CPU solves compares
  with; `e2e.single` is one solve alone (upload + solve + download in sequence) and
  `e2e.inout_u` the reference signature's in/out u (u uploaded too).
* `roofline`: the level-0 kernel with the largest share of the profiled solves
  (in-graph CUDA events), algorithmic bytes per launch / its launch time.
* `cpu_baseline`: the compiled reference (oracle/_ref) on one host core, on a
  bounded sample of the same workload (the cfg2 grid truncated in time).
* `cfg1`: BASELINE config 1 (1024 x 4096, V(5,5), to 1e-10) as an extra key.

Launch: python bench.py [--gpus N --steps K --warmup W --config cfg2]
        torchrun --nproc-per-node N bench.py --gpus N ...   (N > 1: time slabs, strong scaling)
        python bench.py --impl reference ...                (reference CPU arm)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "space-time DOF smoother updates/s; STMG solve time to 1e-10 rel residual"
UNIT = "DOF-updates/s"
# algorithmic HBM bytes per fine DOF of the level-0 kernels
KERNEL_BYTES = {
    "fine_norm_pass": 24,      # residual norm + first sweep: read u, f; write u'
    "fine_sweep": 24,          # read u, f; write u'
    "fine_sweep_pair": 24,     # two sweeps in one pass: read u, f; write u''
    "fine_restrict": 20,       # read u, f; write f_c (half size: 4 B per fine DOF)
    "fine_prolong_sweep": 28,  # read u, f, x_c (4 B per fine DOF); write u'
    "fine_up": 36,             # prolongation + post-sweep + norm + next pre-sweep: read u, f, x_c; write u', u''
}
KERNEL_NAMES = {
    "fine_norm_pass": "k_lean2<sweep, norm> (residual norm + speculative first sweep)",
    "fine_sweep": "k_lean2<sweep>",
    "fine_sweep_pair": "k_lean2x2 (two fused Jacobi sweeps)",
    "fine_restrict": "k_restrict2 (residual + restriction)",
    "fine_prolong_sweep": "k_lean2<sweep, ProlongLoad> (prolongation + first post-sweep)",
    "fine_up": "k_up (prolongation + post-sweep + residual norm + next cycle's first sweep)",
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def host_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def bench_config(name: str, args):
    """The workload and its pinned solver parameters."""
    from paper_2505_10168_b200 import configs as C

    kw = {}
    if args.n_el:
        kw["n_el"] = args.n_el
    if args.n_t:
        kw["n_t"] = args.n_t
    cfg = C.CONFIGS[name](**kw)
    if args.nu is not None:
        cfg.nu = args.nu
    if args.n_levels is not None:
        cfg.n_levels = args.n_levels
    if args.min_elements is not None:
        cfg.min_elements = args.min_elements
    if args.max_cycles is not None:
        cfg.max_cycles = args.max_cycles
    return cfg


def rhs_for(cfg, S, g):
    from paper_2505_10168_b200 import configs as C

    if cfg.rhs == "adjoint_uniform":
        return C.adjoint_uniform_rhs(cfg.n_el, cfg.n_t, cfg.L, cfg.t_T)
    return S.load_vector(g, kind=cfg.source_kind, params=cfg.source_params, masked=True)


def plan_for(S, cfg, g):
    req = S.PlanRequest(n_levels=cfg.n_levels, lambda_crit=cfg.lambda_crit, strategy=S.PlanStrategy(cfg.strategy),
                        reassembly=S.ReassemblyMethod(cfg.reassembly), min_elements=cfg.min_elements,
                        chi=cfg.chi, mat=cfg.mat)
    return S.plan_coarsening(g, req)


class ClockSampler:
    """SM clocks / throttle reasons sampled DURING the timed region (the recipe's
    nvidia-smi clocks line, read through NVML so the first sample is taken
    synchronously on entry and the poll period, 5 ms, resolves a ~250 ms region).
    Falls back to `nvidia-smi -lms 50` when NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.sm, self.mx, self.reasons = [], [], set()
        self.source = None
        self._stop = threading.Event()
        self._thread = None
        self._proc = None
        self._path = None

    def _nvml_handle(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        p = torch.cuda.get_device_properties(self.device)
        try:
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(int(self.device))

    def _sample(self, nv, h):
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
        self.mx.append(float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)))
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        for name, const in self.REASONS:
            if bits & getattr(nv, const):
                self.reasons.add(name)

    def __enter__(self):
        try:
            nv, h = self._nvml_handle()
            self._sample(nv, h)
            self.source = "nvml"

            def loop():
                while not self._stop.wait(0.005):
                    self._sample(nv, h)

            self._thread = threading.Thread(target=loop, daemon=True)
            self._thread.start()
        except Exception:
            self.source = "nvidia-smi"
            fd, self._path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            try:
                idx = int(self.device) if not hasattr(self.device, "index") else int(self.device.index or 0)
                self._proc = subprocess.Popen(
                    ["nvidia-smi", f"--id={idx}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits", "-lms", "50"],
                    stdout=open(self._path, "w"), stderr=subprocess.DEVNULL)
            except Exception:
                self._proc = None
        return self

    def __exit__(self, *a):
        if self._thread:
            self._stop.set()
            self._thread.join(timeout=5)
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
        if self._path and os.path.exists(self._path):
            with open(self._path) as fh:
                for line in fh:
                    parts = [q.strip() for q in line.split(",")]
                    if len(parts) < 9:
                        continue
                    try:
                        self.sm.append(float(parts[1]))
                        self.mx.append(float(parts[2]))
                    except ValueError:
                        continue
                    for (name, _), v in zip(self.REASONS, parts[5:9]):
                        if v.lower() == "active":
                            self.reasons.add(name)
            os.unlink(self._path)

    def summary(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": sorted(self.reasons),
               "samples": len(self.sm), "source": self.source}
        if self.sm:
            out.update(sm_mhz=statistics.median(self.sm), sm_max_mhz=max(self.mx))
        return out


def truncated_sample(cfg, sample_nt: int, dirs):
    """Bounded CPU sample of a workload: the same grid and design truncated to
    sample_nt time steps (same dt), coarsened along the workload's own path for
    as long as the truncated grid allows it."""
    import copy

    s = copy.copy(cfg)
    s.t_T = cfg.t_T * sample_nt / cfg.n_t
    s.n_t = sample_nt
    ne, nt, pre = s.n_el, s.n_t, []
    for d in dirs:
        d = int(d)
        if (d == 0 and (ne < 2 or ne % 2)) or (d == 1 and (nt < 4 or nt % 2)):
            break
        pre.append(d)
        if d == 0:
            ne //= 2
        else:
            nt //= 2
    return s, pre


def per_cycle_updates(s, dirs, nu):
    """Smoother DOF updates of one V(nu, nu) cycle: 2 nu N_l over the non-coarsest levels."""
    ne, nt, total = s.n_el, s.n_t, 0.0
    for d in dirs:
        total += 2 * nu * (ne + 1) * (nt + 1)
        if int(d) == 0:
            ne //= 2
        else:
            nt //= 2
    return total


def sample_rhs(s, lib):
    from paper_2505_10168_b200 import configs as C

    if s.rhs == "adjoint_uniform":
        return C.adjoint_uniform_rhs(s.n_el, s.n_t, s.L, s.t_T)
    return lib.load_vector(s.L, s.t_T, s.n_el, s.n_t, s.source_kind, s.source_params)


def run_cpu_sample(cfg, sample_nt: int, dirs):
    """The compiled reference (oracle/_ref; the C port if it is absent) on the
    truncated sample: hierarchy built outside the timed region, one solve."""
    from oracle import pyoracle

    s, pre = truncated_sample(cfg, sample_nt, dirs)
    if pyoracle.ref_available():
        lib, kind = pyoracle.Ref(), "reference"
        h = lib.hierarchy(s.L, s.t_T, s.n_el, s.n_t, s.k, s.c, pre, method=s.method, adjoint=s.adjoint,
                          chi=s.chi, mat=s.mat)
    else:
        lib, kind = pyoracle.Port(), "port"
        h = lib.hierarchy(s.L, s.t_T, s.n_el, s.n_t, s.k, s.c, pre, reassembly=s.reassembly, adjoint=s.adjoint,
                          chi=s.chi, mat=s.mat)
    b = sample_rhs(s, lib)
    t0 = time.perf_counter()
    u, rep = h.solve(b, nu=s.nu, omega=s.omega, tol=s.tol, div_tol=s.div_tol, max_cycles=s.max_cycles)
    wall = time.perf_counter() - t0
    secs = rep.seconds if rep.seconds > 0 else wall
    return {"kind": kind, "updates": per_cycle_updates(s, pre, s.nu) * rep.cycles, "seconds": secs,
            "cycles": rep.cycles, "status": rep.status, "dofs": (s.n_el + 1) * (s.n_t + 1), "n_t": s.n_t,
            "levels": len(pre) + 1}


def _ref_worker(conn, config, argd, sample_nt, dirs):
    """--impl reference worker: one single-threaded reference solve per request
    on the bounded sample; the hierarchy is built once, before the timed steps."""
    try:
        from oracle import pyoracle

        cfg = bench_config(config, argparse.Namespace(**argd))
        s, pre = truncated_sample(cfg, sample_nt, dirs)
        ref = pyoracle.Ref()
        h = ref.hierarchy(s.L, s.t_T, s.n_el, s.n_t, s.k, s.c, pre, method=s.method, adjoint=s.adjoint,
                          chi=s.chi, mat=s.mat)
        b = sample_rhs(s, ref)
        upc = per_cycle_updates(s, pre, s.nu)
        conn.send(("ready", (s.n_el + 1) * (s.n_t + 1), len(pre) + 1))
        while True:
            if conn.recv() == "stop":
                break
            u, rep = h.solve(b, nu=s.nu, omega=s.omega, tol=s.tol, div_tol=s.div_tol, max_cycles=s.max_cycles)
            conn.send((upc * rep.cycles, rep.seconds, rep.cycles, int(rep.status)))
    except Exception as e:  # reported by the parent
        conn.send(("error", repr(e)))


def planned_dirs(cfg):
    """The GPU arm's coarsening path, planned by the product's planner on the host
    (pinned bitwise to the reference planner, tests/test_capi_cpu.py)."""
    from paper_2505_10168_b200 import stmg as S

    g = S.build_fine_grid(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t)
    g.k, g.c = cfg.k, cfg.c
    return [int(d) for d in plan_for(S, cfg, g).dirs]


def reference_arm(args):
    """--impl reference: the reference's own CPU path on all host cores.  The
    reference is single-threaded (no threads in proj/src), so each core runs one
    reference solve of the bounded sample per step; a step ends when every core
    is done.  value = all cores' smoother DOF updates / summed step wall time."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import multiprocessing as mp

    cfg = bench_config(args.config, args)
    dirs = planned_dirs(cfg)
    cores = max(1, min(os.cpu_count() or 1, args.ref_cores))
    sample_nt = min(args.cpu_sample_nt, cfg.n_t)
    ctx = mp.get_context("spawn")
    pipes, procs = [], []
    for _ in range(cores):
        a, b_ = ctx.Pipe()
        p = ctx.Process(target=_ref_worker, args=(b_, args.config, vars(args), sample_nt, dirs), daemon=True)
        p.start()
        pipes.append(a)
        procs.append(p)
    t_build = time.perf_counter()
    info = [c.recv() for c in pipes]
    t_build = time.perf_counter() - t_build
    for m in info:
        if m[0] != "ready":
            raise RuntimeError(f"reference worker failed: {m[1]}")
    dofs, levels = info[0][1], info[0][2]
    upd = wall = 0.0
    last = None
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        for c in pipes:
            c.send("go")
        res = [c.recv() for c in pipes]
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            upd += sum(r[0] for r in res)
            wall += dt
            last = res[0]
    for c in pipes:
        c.send("stop")
    for p in procs:
        p.join(timeout=30)
    value = upd / wall if wall > 0 else 0.0
    status = {0: "converged", 1: "max_cycles", 2: "diverged"}.get(last[3], str(last[3])) if last else None
    sample = (f"{cores} concurrent single-threaded reference solves, each of {cfg.name} truncated to "
              f"n_t={sample_nt} ({dofs} DOFs, {levels} levels along the GPU arm's path, nu={cfg.nu}, "
              f"{last[2] if last else 0} V-cycles to {status}); hierarchies built once before the timed steps "
              f"({t_build:.1f} s)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / max(args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE shapes)",
        "config": {"workload": cfg.name, "n_el": cfg.n_el, "n_t": cfg.n_t, "dofs": (cfg.n_el + 1) * (cfg.n_t + 1),
                   "method": cfg.method, "strategy": int(cfg.strategy), "n_levels": cfg.n_levels,
                   "min_elements": cfg.min_elements, "nu": cfg.nu, "tol": cfg.tol, "div_tol": cfg.div_tol,
                   "parallelism": f"{cores} host cores, one single-threaded reference solve each",
                   "adjoint": cfg.adjoint, "sample_n_t": sample_nt, "sample_dofs": dofs},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample,
                         **host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "solve_seconds_sample": last[1] if last else None,
    }
    print(json.dumps(line), flush=True)
    return 0


def kernel_table(prof_reps, n0, hbm):
    """Level-0 kernels of the profiled solves: launches, mean launch time and the
    algorithmic bandwidth (KERNEL_BYTES x fine DOFs per launch / mean time)."""
    kt = {}
    for key, bpd in KERNEL_BYTES.items():
        c, secs = 0, 0.0
        for r in prof_reps:
            cc, ss = r.kernel_times.get(key, (0, 0.0))
            c += cc
            secs += ss
        if c:
            avg = secs / c
            ach = bpd * n0 / avg / 1e9
            kt[key] = {"launches": c, "avg_ms": 1e3 * avg, "total_ms": 1e3 * secs, "bytes_per_dof": bpd,
                       "achieved_GBps": ach, "frac": ach / hbm}
    return kt


def ncu_traffic(config_name, kernel_key):
    """DRAM bytes per launch of the roofline kernel from the committed ncu --set full
    capture of the same workload (profiles/round2_ncu_<config>.json), or None."""
    path = os.path.join(ROOT, "profiles", f"round2_ncu_{config_name}.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        k = d["kernels"][kernel_key]
        return float(k["dram_bytes_read"]) + float(k["dram_bytes_write"]), os.path.relpath(path, ROOT)
    except Exception:
        return None, None


def cfg1_extra(S, torch, dev, args):
    """BASELINE config 1 (4.2e6 DOFs, V(5,5), 10 levels) to 1e-10 from u = 0, b and u
    in HBM, L2 flushed before each solve; the reference's full-grid solve time of the
    same problem is the committed golden's (tests/golden/cfg1_full.npz, one core)."""
    import numpy as np

    from paper_2505_10168_b200 import configs as C

    cfg = C.cfg1()
    g = S.build_fine_grid(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t)
    g.k, g.c = cfg.k, cfg.c
    path = plan_for(S, cfg, g)
    h = S.build_hierarchy(g, cfg.method, path, chi=cfg.chi, mat=cfg.mat, device=dev.index or 0)
    st = torch.cuda.Stream(device=dev)
    h.set_stream(st)
    b = torch.from_numpy(rhs_for(cfg, S, g)).to(dev)
    u = torch.zeros_like(b)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    opts = S.SolveOptions(nu=cfg.nu, omega=cfg.omega, tol=cfg.tol, div_tol=cfg.div_tol, max_cycles=cfg.max_cycles)
    ts, reps = [], []
    for k in range(args.cfg1_warmup + args.cfg1_steps):
        with torch.cuda.stream(st):
            flush.fill_(1.0)
            u.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        rep = S.mg_solve(h, b, u, opts, zero_guess=True)
        e1.record(st)
        e1.synchronize()
        if k >= args.cfg1_warmup:
            ts.append(e0.elapsed_time(e1))
            reps.append(rep)
    ms = sum(ts) / len(ts)
    out = {"grid": "1024x4096", "dofs": (cfg.n_el + 1) * (cfg.n_t + 1), "nu": cfg.nu, "n_levels": cfg.n_levels,
           "solves": len(ts), "solve_ms": ms, "cycles": reps[-1].cycles,
           "status": S.status_name(reps[-1].status), "final_rel_residual": reps[-1].history[-1],
           "value": reps[-1].smoother_dof_updates / (ms * 1e-3), "l2": "flushed (256 MB write) before each solve"}
    try:
        gold = np.load(os.path.join(ROOT, "tests", "golden", "cfg1_full.npz"))
        out["reference_full_grid"] = {"cycles": int(gold["cycles"]), "solve_seconds": float(gold["ref_seconds"]),
                                      "cores": 1, "where": "builder container (tests/golden/make_golden.py --full)"}
    except Exception:
        pass
    return out


def cfg3_extra(S, torch, dev, h, cfg, stream, steps=2, warmup=1):
    """BASELINE config 3: the adjoint solve on the config-2 grid and design (J^T, the
    transposed hierarchy shares config 2's workspace), right-hand side dJ/dT of the
    time- and space-integrated temperature, from lambda = 0, b and lambda in HBM."""
    from paper_2505_10168_b200 import configs as C

    ht = S.transposed_hierarchy(h)
    ht.set_stream(stream)
    with torch.cuda.stream(stream):
        b = torch.from_numpy(C.adjoint_uniform_rhs(cfg.n_el, cfg.n_t, cfg.L, cfg.t_T)).to(dev)
        lam = torch.empty_like(b)
    opts = S.SolveOptions(nu=cfg.nu, omega=cfg.omega, tol=cfg.tol, div_tol=cfg.div_tol, max_cycles=cfg.max_cycles)
    ts, rep = [], None
    for k in range(warmup + steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rep = S.mg_solve(ht, b, lam, opts, zero_guess=True)
        e1.record(stream)
        e1.synchronize()
        if k >= warmup:
            ts.append(e0.elapsed_time(e1))
    ms = sum(ts) / len(ts)
    return {"grid": f"{cfg.n_el}x{cfg.n_t}", "dofs": (cfg.n_el + 1) * (cfg.n_t + 1), "adjoint": True, "solves": len(ts),
            "solve_ms": ms, "cycles": rep.cycles, "status": S.status_name(rep.status), "history": rep.history,
            "value": rep.smoother_dof_updates / (ms * 1e-3),
            "note": "same coarsening path and stop rule as config 2 (the reference algorithm diverges on this design)"}


def cfg4_extra(S, torch, iterations=50):
    """BASELINE config 4: the 50-iteration topology-optimisation loop at 4096 x 16384
    (nu = 20, tol 1e-8, warm-started, DesignIndependent, 6 levels): forward and adjoint
    STMG solves and the sensitivities on the GPU, the MMA design update on the host."""
    geom = S.build_fine_grid(1.0, 1.0, 4096, 16384)
    opts = S.OptimisationOptions(method="CR", strategy=S.PlanStrategy.DesignIndependent, n_levels=6,
                                 max_iterations=iterations, stable_iterations=10 ** 6,
                                 solve=S.SolveOptions(nu=20, tol=1e-8))
    res = S.optimise(geom, (1e-3, 1.0, 1.0, 1.0, 3.0, 2.0), opts)
    hst = res.history
    return {"grid": "4096x16384", "iterations": res.iterations, "total_seconds": res.seconds,
            "stmg_seconds": sum(r["primal_seconds"] + r["adjoint_seconds"] for r in hst),
            "primal_cycles": [r["primal_cycles"] for r in hst], "adjoint_cycles": [r["adjoint_cycles"] for r in hst],
            "statuses": sorted({(r["primal_status"], r["adjoint_status"]) for r in hst}),
            "theta_first_last": [hst[0]["theta"], hst[-1]["theta"]], "volume_last": hst[-1]["volume"],
            "reference": "iterations 1-2: 6/6 and 5/5 primal/adjoint cycles (tests/golden/cfg4_full.npz; "
                         "546 s + 524 s per solve on one core)"}


def e2e_stream(S, torch, h, bh, uh, opts, stream, dev, K, e2e):
    """Streamed e2e: K solves through stmg_mg_solve_stream, every step uploading its b and
    downloading its u; updates e2e in place (value, mode, single)."""
    S.mg_solve_stream(h, [bh] * 2, [uh] * 2, opts, zero_guess=True)  # slots + graphs (untimed)
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    rs = S.mg_solve_stream(h, [bh] * K, [uh] * K, opts, zero_guess=True)
    e1.record(stream)
    e1.synchronize()
    wall = time.perf_counter() - t0
    ms = e0.elapsed_time(e1)
    h.release_staging()
    single = {k_: e2e[k_] for k_ in ("value", "solve_seconds")}
    e2e.update({
        "value": sum(r.smoother_dof_updates for r in rs) / (ms * 1e-3),
        "solve_seconds": ms * 1e-3 / K, "wall_seconds_per_step": wall / K, "steps": K,
        "mode": f"stream of {K} solves on one hierarchy (stmg_mg_solve_stream): each step uploads its b "
                "from pinned host memory and downloads its u; the copies of steps k - 1 / k + 1 overlap "
                "solve k (two device slots); pipeline fill and drain are inside the timed region",
        "single": single})


def main():
    # NCCL_DEBUG=VERSION (set on some images) prints a banner on stdout at
    # communicator creation; the bench prints exactly one JSON line there
    if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
        os.environ["NCCL_DEBUG"] = "WARN"
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nu", type=int, default=None)
    ap.add_argument("--n-levels", type=int, default=None)
    ap.add_argument("--min-elements", type=int, default=None)
    ap.add_argument("--max-cycles", type=int, default=None)
    ap.add_argument("--n-el", type=int, default=None)
    ap.add_argument("--n-t", type=int, default=None)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--e2e-stream-steps", type=int, default=8,
                    help="solves in the streamed e2e measurement (0/1: skip; e2e.value is then the one-solve figure)")
    ap.add_argument("--cpu-sample-nt", type=int, default=512)
    ap.add_argument("--ref-cores", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=2,
                    help="extra solves with in-graph kernel timers (roofline), after the timed steps")
    ap.add_argument("--cfg1", type=int, default=1, help="also time BASELINE config 1 (extra key)")
    ap.add_argument("--cfg3", type=int, default=1, help="also time BASELINE config 3 (adjoint, extra key)")
    ap.add_argument("--cfg4", type=int, default=1, help="also run BASELINE config 4 (optimisation loop, extra key)")
    ap.add_argument("--cfg1-steps", type=int, default=5)
    ap.add_argument("--cfg1-warmup", type=int, default=3)
    ap.add_argument("--dist", action="store_true",
                    help="use the time-slab (NCCL) path even at N=1 (smoke test of that path)")
    args = ap.parse_args()

    if args.impl == "reference":
        return reference_arm(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2505_10168_b200 import stmg as S

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    cfg = bench_config(args.config, args)
    g = S.build_fine_grid(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t)
    g.k, g.c = cfg.k, cfg.c
    path = plan_for(S, cfg, g)
    t_build = time.perf_counter()
    dh = None
    if world > 1 or args.dist:
        # time slabs over NCCL: rank 0 makes the NCCL id, torch.distributed ships it
        obj = [S.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        dh = S.build_dist_hierarchy(g, cfg.method, path, world, rank=rank, nccl_id=obj[0], device=local,
                                    adjoint=cfg.adjoint, chi=cfg.chi, mat=cfg.mat, min_slab=16)
        h = None
    else:
        h = S.build_hierarchy(g, cfg.method, path, chi=cfg.chi, mat=cfg.mat, device=local)
        if cfg.adjoint:
            h = S.transposed_hierarchy(h)
    t_build = time.perf_counter() - t_build
    b_host = rhs_for(cfg, S, g)
    n0 = (cfg.n_el + 1) * (cfg.n_t + 1)
    if dh is not None:  # slab-local vectors: this process's level-0 rows only (memory ~ 1/W)
        nn_ = cfg.n_el + 1
        b_host = np.ascontiguousarray(b_host[dh.row_lo * nn_: dh.row_hi * nn_])
    n = b_host.size
    stream = torch.cuda.Stream(device=dev)
    if h is not None:
        h.set_stream(stream)
    opts = S.SolveOptions(nu=cfg.nu, omega=cfg.omega, tol=cfg.tol, div_tol=cfg.div_tol, max_cycles=cfg.max_cycles)
    with torch.cuda.stream(stream):
        b_dev = torch.from_numpy(b_host).to(dev)
        u_dev = torch.zeros_like(b_dev)
    stream.synchronize()
    l2_note = ("inputs larger than L2 (b, u, u' = 3 x {:.1f} GB)".format(8 * n0 / 1e9) if 24 * n0 > 126e6 else
               "L2 flushed (256 MB write) before every timed step")
    flush = None if 24 * n0 > 126e6 else torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)

    def solve_on(bv, uv, zero_guess=False):
        if dh is not None:
            stream.synchronize()
            return S.mg_solve_dist_local(dh, bv, uv, opts)
        return S.mg_solve(h, bv, uv, opts, zero_guess=zero_guess)

    def timed_solves(count):
        reps, ms = [], []
        for _ in range(count):
            with torch.cuda.stream(stream):
                if flush is not None:
                    flush.fill_(1.0)
                if dh is not None:
                    u_dev.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            # a solve from u = 0: STMG_SOLVE_ZERO_GUESS (u is output only)
            reps.append(solve_on(b_dev, u_dev, zero_guess=dh is None))
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        return reps, ms

    timed_solves(args.warmup)
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev) as clk:
        reps, step_ms = timed_solves(args.steps)
    torch.cuda.synchronize(dev)
    barrier()
    clocks = clk.summary()
    t_max = max_over_ranks(sum(step_ms))
    updates = sum(r.smoother_dof_updates for r in reps)
    if world > 1:
        uu = torch.tensor([updates], dtype=torch.float64, device=dev)
        dist.all_reduce(uu, op=dist.ReduceOp.SUM)
        updates = float(uu.item())
    value = updates / (t_max * 1e-3)
    last = reps[-1]
    hbm, peak_kind = peaks()

    # Kernel-level timing (roofline): further solves with CUDA event nodes around
    # the level-0 kernels inside the graph (host cycle loop).  Kept out of the
    # timed steps: each event node adds launch-gap overhead.
    kt, prof_ms = {}, []
    if h is not None and args.profile_steps > 0:
        h.set_profiling(True)
        timed_solves(1)  # capture the profiled graph
        prof_reps, prof_ms = timed_solves(args.profile_steps)
        h.set_profiling(False)
        kt = kernel_table(prof_reps, n0, hbm)
    roofline = None
    if kt:
        key = max(kt, key=lambda k_: kt[k_]["total_ms"])
        k = kt[key]
        traffic, tsrc = ncu_traffic(cfg.name, key)
        roofline = {"bound": "hbm", "achieved": k["achieved_GBps"], "peak": hbm, "unit": "GB/s",
                    "frac": k["frac"], "traffic": traffic, "traffic_source": tsrc,
                    "kernel": f"{KERNEL_NAMES[key]}, level 0 of the {cfg.name} solve (in-graph CUDA events)",
                    "kernel_key": key, "algorithmic_bytes_per_launch": k["bytes_per_dof"] * n0,
                    "algorithmic_bytes_per_dof": k["bytes_per_dof"], "avg_launch_ms": k["avg_ms"],
                    "launches_timed": k["launches"], "peak_source": peak_kind}
        if key == "fine_up":
            roofline["note"] = ("k_up is the fusion of the prolong-sweep (28 B/DOF, 0.88 of peak alone) and the norm "
                                "pass (24 B/DOF, 0.83): it moves 36 B/DOF instead of 52, is instruction-bound (ncu: "
                                "54 % issue slots, 124 registers) and runs at the 1 kW power cap inside the solve; the "
                                "timed span includes the fixed-order sum of its norm partials")
        # all level-0 kernels together: algorithmic bytes of one cycle's level-0 passes over their time
        l0 = [v for v in kt.values() if isinstance(v, dict)]
        l0_bytes = sum(v["bytes_per_dof"] * n0 * v["launches"] for v in l0)
        l0_secs = sum(v["total_ms"] for v in l0) * 1e-3
        if l0_secs > 0:
            roofline["level0"] = {"bytes_per_dof_per_cycle": sum(v["bytes_per_dof"] for v in l0),
                                  "achieved": l0_bytes / l0_secs / 1e9, "frac": l0_bytes / l0_secs / 1e9 / hbm,
                                  "kernels": sorted(k_ for k_, v in kt.items() if isinstance(v, dict))}
        kt["profiled_steps"] = len(prof_ms)
        kt["profiled_ms_per_step"] = sum(prof_ms) / len(prof_ms)
        kt["level0_share_of_step"] = sum(v["total_ms"] for v in kt.values() if isinstance(v, dict)) / max(
            sum(prof_ms), 1e-9)

    # e2e through the C ABI with pinned host buffers (copies inside the timed region).
    # The workload is a solve from u = 0, so the headline e2e passes STMG_SOLVE_ZERO_GUESS
    # (stmg_mg_solve_ex): b is uploaded, u is output only and downloaded.  The reference
    # signature's in/out u (a warm start: u uploaded too) is timed beside it (e2e.inout_u).
    e2e = None
    if args.e2e_steps > 0:
        bh = torch.from_numpy(b_host).pin_memory()
        uh = torch.zeros(n, dtype=torch.float64).pin_memory()

        def e2e_run(zero_guess):
            tot_ms, tot_upd = 0.0, 0.0
            for _ in range(args.e2e_steps):
                uh.zero_()
                torch.cuda.synchronize(dev)
                barrier()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                r = S.mg_solve(h, bh, uh, opts, zero_guess=True) if zero_guess else solve_on(bh, uh)
                e1.record(stream)
                e1.synchronize()
                tot_ms += e0.elapsed_time(e1)
                tot_upd += r.smoother_dof_updates
            tot_ms = max_over_ranks(tot_ms)
            if world > 1:
                uu = torch.tensor([tot_upd], dtype=torch.float64, device=dev)
                dist.all_reduce(uu, op=dist.ReduceOp.SUM)
                tot_upd = float(uu.item())
            return tot_upd / (tot_ms * 1e-3), tot_ms * 1e-3 / args.e2e_steps

        nbytes = n
        if world > 1:  # every rank copies its own slab rows
            nb = torch.tensor([float(n)], dtype=torch.float64, device=dev)
            dist.all_reduce(nb, op=dist.ReduceOp.SUM)
            nbytes = int(nb.item())
        v_io, s_io = e2e_run(False)
        if h is not None:
            v_z, s_z = e2e_run(True)
            e2e = {"value": v_z, "unit": UNIT, "h2d_bytes_per_step": 8 * nbytes, "d2h_bytes_per_step": 8 * nbytes,
                   "solve_seconds": s_z, "initial_guess": "zero (STMG_SOLVE_ZERO_GUESS: u is output only)",
                   "inout_u": {"value": v_io, "solve_seconds": s_io, "h2d_bytes_per_step": 16 * nbytes,
                               "d2h_bytes_per_step": 8 * nbytes}}
        else:
            e2e = {"value": v_io, "unit": UNIT, "h2d_bytes_per_step": 16 * nbytes,
                   "d2h_bytes_per_step": 8 * nbytes, "solve_seconds": s_io}
        # A stream of solves through stmg_mg_solve_stream (one hierarchy, host vectors): every
        # step still uploads its b and downloads its u, but step k's copies overlap its
        # neighbours' solves.  This is the throughput figure the reference arm's batch of
        # concurrent CPU solves compares with; the one-solve latency stays in e2e.single.
        if h is not None and world == 1 and args.e2e_stream_steps > 1:
            try:
                e2e_stream(S, torch, h, bh, uh, opts, stream, dev, args.e2e_stream_steps, e2e)
            except Exception as e:  # e2e.value stays the one-solve figure
                e2e["stream_error"] = repr(e)

    cpu = None
    dev_bytes = h.device_bytes() if h is not None else dh.device_bytes
    cfg1 = cfg3 = cfg4 = None
    if rank == 0 and world == 1:
        if args.cfg3 and cfg.name == "cfg2" and h is not None:
            try:
                del b_dev, u_dev
                b_dev = u_dev = None
                torch.cuda.empty_cache()
                cfg3 = cfg3_extra(S, torch, dev, h, cfg, stream)
            except Exception as e:  # an extra key, never required
                cfg3 = {"error": repr(e)}
        if (args.cfg1 and cfg.name != "cfg1") or args.cfg4:
            b_dev = u_dev = None
            h = None  # release the config-2 hierarchy (60 GB) before the other configs
            torch.cuda.empty_cache()
        if args.cfg1 and cfg.name != "cfg1":
            try:
                cfg1 = cfg1_extra(S, torch, dev, args)
            except Exception as e:  # an extra key, never required
                cfg1 = {"error": repr(e)}
        if args.cfg4 and cfg.name == "cfg2":
            try:
                cfg4 = cfg4_extra(S, torch)
            except Exception as e:  # an extra key, never required
                cfg4 = {"error": repr(e)}
        if not args.no_cpu_baseline:
            try:
                res = run_cpu_sample(cfg, args.cpu_sample_nt, [int(d) for d in path.dirs])
                cpu = {"value": res["updates"] / res["seconds"] if res["seconds"] > 0 else None,
                       "unit": UNIT, "cores": 1, "kind": res["kind"],
                       "sample": f"{cfg.name} truncated to n_t={res['n_t']} ({res['dofs']} DOFs, {res['levels']} "
                                 f"levels along the GPU arm's path), one solve after an untimed hierarchy build, "
                                 f"{res['cycles']} V-cycles to status {res['status']}, {res['seconds']:.2f} s on "
                                 f"1 core", **host_info()}
            except Exception as e:  # the baseline is reported, never required
                cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / max(args.steps, 1), "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded mt19937_64 designs, BASELINE shapes)",
            "config": {"workload": cfg.name, "n_el": cfg.n_el, "n_t": cfg.n_t, "dofs": n0,
                       "method": cfg.method, "strategy": int(cfg.strategy), "n_levels": cfg.n_levels,
                       "min_elements": cfg.min_elements, "nu": cfg.nu, "tol": cfg.tol, "div_tol": cfg.div_tol,
                       "max_cycles": cfg.max_cycles, "path": S.path_to_string(path),
                       "stop_rule": "the reference's (proj/src/multigrid.cpp:260-273): converged below tol, "
                                    "diverged above div_tol",
                       "parallelism": (f"time-slabs{world} (NCCL, {dh.n_distributed} distributed levels)"
                                       if dh is not None else "single"),
                       "l2": l2_note, "adjoint": cfg.adjoint},
            "solve_seconds": t_max * 1e-3 / max(args.steps, 1), "cycles": last.cycles,
            "status": S.status_name(last.status), "history": last.history,
            "gpu_launches": int(sum(r.kernel_launches for r in reps)),
            "roofline": roofline, "kernels": kt, "e2e": e2e, "cpu_baseline": cpu, "clocks": clocks,
            "cfg1": cfg1, "cfg3": cfg3, "cfg4": cfg4, "build_seconds": t_build,
            "device_bytes": dev_bytes,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
