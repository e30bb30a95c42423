#!/usr/bin/env python
"""Benchmark: STMG solve on B200 (BASELINE metric: space-time DOF smoother
updates/s; STMG solve time to the config's relative-residual tolerance).

A step is one complete STMG solve (cold start u = 0) of the configured
workload through the public C ABI.  `value` is whole-job smoother DOF updates
per second with b already resident in HBM; `e2e` is the same metric through
the C ABI with pinned HOST buffers (h2d of b and u, d2h of u inside the timed
region).  `roofline` is the fine-level Jacobi sweep kernel (24 B per DOF
update: read u, read f, write u'), timed by CUDA events recorded inside the
V-cycle graph during the timed steps.  `cpu_baseline` is the compiled
reference (oracle/_ref) timed on a bounded, time-truncated sample of the same
workload on one host core.

Launch: python bench.py [--gpus N --steps K --warmup W --config cfg2]
        torchrun --nproc-per-node N bench.py --gpus N ...   (N > 1)
        python bench.py --impl reference ...                (reference CPU arm)
"""
from __future__ import annotations

import argparse
import json
import math
import os
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


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def bench_config(name: str, args):
    """The workload and its pinned solver parameters (Appendix B of SURVEY)."""
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


def cpu_sample_config(cfg, sample_nt: int):
    """Bounded CPU sample: the same config truncated to sample_nt time steps."""
    from paper_2505_10168_b200 import configs as C

    import copy

    s = copy.copy(cfg)
    s.n_t = sample_nt
    return s


def run_cpu_sample(cfg, sample_nt: int, prefer_ref: bool = True):
    """Reference (oracle/_ref) or the C port on a time-truncated sample; returns dict."""
    import numpy as np

    from oracle import pyoracle

    s = cpu_sample_config(cfg, sample_nt)
    port = pyoracle.Port()
    dirs, _ = port.plan(s.L, s.t_T, s.n_el, s.n_t, s.k, s.c, s.n_levels, strategy=s.strategy,
                        reassembly=s.reassembly, min_elements=s.min_elements, chi=s.chi, mat=s.mat)
    if s.rhs == "adjoint_uniform":
        from paper_2505_10168_b200 import configs as C

        b = C.adjoint_uniform_rhs(s.n_el, s.n_t, s.L, s.t_T)
    else:
        b = port.load_vector(s.L, s.t_T, s.n_el, s.n_t, s.source_kind, s.source_params)
    kind = "port"
    if prefer_ref and pyoracle.ref_available():
        ref = pyoracle.Ref()
        dirs_r, _ = ref.plan(s.L, s.t_T, s.n_el, s.n_t, s.k, s.c, s.n_levels, strategy=s.strategy,
                             reassembly=s.reassembly, min_elements=s.min_elements, chi=s.chi,
                             mat=s.mat)
        h = ref.hierarchy(s.L, s.t_T, s.n_el, s.n_t, s.k, s.c, dirs_r, method=s.method,
                          adjoint=s.adjoint, chi=s.chi, mat=s.mat)
        kind = "reference"
        dirs = dirs_r
    else:
        h = port.hierarchy(s.L, s.t_T, s.n_el, s.n_t, s.k, s.c, dirs, reassembly=s.reassembly,
                           adjoint=s.adjoint, chi=s.chi, mat=s.mat)
    t0 = time.perf_counter()
    u, rep = h.solve(b, nu=s.nu, tol=s.tol, max_cycles=s.max_cycles)
    wall = time.perf_counter() - t0
    secs = rep.seconds if rep.seconds > 0 else wall
    # smoother DOF updates of this solve: sum over non-coarsest levels of 2 nu N_l per cycle
    ne, nt = s.n_el, s.n_t
    per_cycle = 0.0
    for d in dirs:
        per_cycle += 2 * s.nu * (ne + 1) * (nt + 1)
        if int(d) == 0:
            ne //= 2
        else:
            nt //= 2
    updates = per_cycle * rep.cycles
    return {"kind": kind, "updates": updates, "seconds": secs, "cycles": rep.cycles,
            "status": rep.status, "dofs": (s.n_el + 1) * (s.n_t + 1), "n_t": s.n_t,
            "build_seconds": getattr(rep, "build_seconds", 0.0)}


def hbm_scale_sweep(S, torch, dev, hbm_peak, n_el=16384, n_t=65536, sweeps=10):
    """Fine-level Jacobi sweep on the cfg2 grid (1.07e9 DOFs, 8.6 GB per vector,
    far beyond L2): algorithmic 24 B per DOF update over CUDA-event time."""
    from paper_2505_10168_b200 import configs as C

    try:
        cfg = C.cfg2(n_el=n_el, n_t=n_t)
        g = S.build_fine_grid(cfg.L, cfg.t_T, n_el, n_t)
        g.k, g.c = cfg.k, cfg.c
        h2 = S.build_hierarchy(g, cfg.method, S.CoarseningPath([]), device=dev.index or 0)
        st = torch.cuda.Stream(device=dev)
        h2.set_stream(st)
        n0 = (n_el + 1) * (n_t + 1)
        with torch.cuda.stream(st):
            f = torch.rand(n0, dtype=torch.float64, device=dev)
            x = torch.rand(n0, dtype=torch.float64, device=dev)
            y = torch.empty_like(x)
        out = {"grid": f"{n_el}x{n_t}", "dofs": n0, "peak": hbm_peak, "unit": "GB/s",
               "bytes_per_launch": 24 * n0}
        for label, pairs in (("single_sweep", False), ("fused_two_sweeps", True)):
            h2.sweep_kernels(0, f, x, y, 2, pairs)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            h2.sweep_kernels(0, f, x, y, sweeps, pairs)
            e1.record(st)
            e1.synchronize()
            ms = e0.elapsed_time(e1) / sweeps
            achieved = 24.0 * n0 / (ms * 1e-3) / 1e9
            out[label] = {"avg_launch_ms": ms, "achieved": achieved, "frac": achieved / hbm_peak,
                          "dof_updates_per_s": (2 if pairs else 1) * n0 / (ms * 1e-3)}
        out["achieved"] = out["single_sweep"]["achieved"]
        out["frac"] = out["single_sweep"]["frac"]
        out["avg_launch_ms"] = out["single_sweep"]["avg_launch_ms"]
        del f, x, y, h2
        torch.cuda.empty_cache()
        return out
    except Exception as e:  # reported, never required
        return {"error": str(e)}


def reference_arm(args):
    """--impl reference: the reference's own CPU path on all host cores (one
    single-threaded reference solve per core, the reference has no threads)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import multiprocessing as mp

    cfg = bench_config(args.config, args)
    cores = min(os.cpu_count() or 1, args.ref_cores)
    sample_nt = args.cpu_sample_nt
    ctx = mp.get_context("spawn")
    vals = []
    info = None
    with ctx.Pool(cores) as pool:
        for step in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            res = pool.starmap(_ref_worker, [(args.config, vars(args), sample_nt)] * cores)
            wall = time.perf_counter() - t0
            if step >= args.warmup:
                upd = sum(r["updates"] for r in res)
                vals.append((upd, wall, max(r["seconds"] for r in res)))
                info = res[0]
    upd = sum(v[0] for v in vals)
    wall = sum(v[1] for v in vals)
    value = upd / wall if wall > 0 else 0.0
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / max(args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE shapes)",
        # the same workload as the GPU arm; each step is a bounded sample of it
        # (the time-truncated grid below), the metric is a rate
        "config": {"workload": cfg.name, "n_el": cfg.n_el, "n_t": cfg.n_t,
                   "dofs": (cfg.n_el + 1) * (cfg.n_t + 1), "method": cfg.method,
                   "strategy": int(cfg.strategy), "n_levels": cfg.n_levels,
                   "min_elements": cfg.min_elements, "nu": cfg.nu, "tol": cfg.tol,
                   "parallelism": f"{cores} host cores, one single-threaded reference solve each",
                   "adjoint": cfg.adjoint, "sample_n_t": sample_nt},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": info["kind"] if info else "port",
                         "sample": f"{cores} concurrent single-threaded solves of {cfg.name} truncated to "
                                   f"n_t={sample_nt} ({info['dofs'] if info else 0} DOFs, "
                                   f"{info['cycles'] if info else 0} V-cycles each)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "solve_seconds_sample": info["seconds"] if info else None,
    }
    print(json.dumps(line), flush=True)
    return 0


def _ref_worker(config, argd, sample_nt):
    ns = argparse.Namespace(**argd)
    cfg = bench_config(config, ns)
    return run_cpu_sample(cfg, sample_nt, prefer_ref=True)


def main():
    # NCCL_DEBUG=VERSION (set on some images) prints a banner on stdout at
    # communicator creation; the bench prints exactly one JSON line there
    if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
        os.environ["NCCL_DEBUG"] = "WARN"
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nu", type=int, default=None)
    ap.add_argument("--n-levels", type=int, default=None)
    ap.add_argument("--min-elements", type=int, default=None)
    ap.add_argument("--max-cycles", type=int, default=None)
    ap.add_argument("--n-el", type=int, default=None)
    ap.add_argument("--n-t", type=int, default=None)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--cpu-sample-nt", type=int, default=512)
    ap.add_argument("--ref-cores", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--hbm-roofline", type=int, default=1)
    ap.add_argument("--profile-steps", type=int, default=3,
                    help="extra solves with in-graph kernel timers (roofline), after the timed steps")
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

    cfg = bench_config(args.config, args)
    if world > 1 and args.config == "cfg1":
        from paper_2505_10168_b200 import configs as Cf

        nu_, nl_ = cfg.nu, cfg.n_levels
        cfg = Cf.cfg1_weak(world)
        cfg.nu, cfg.n_levels = nu_, nl_
    g = S.build_fine_grid(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t)
    g.k, g.c = cfg.k, cfg.c
    req = S.PlanRequest(n_levels=cfg.n_levels, lambda_crit=cfg.lambda_crit,
                        strategy=S.PlanStrategy(cfg.strategy),
                        reassembly=S.ReassemblyMethod(cfg.reassembly), min_elements=cfg.min_elements,
                        chi=cfg.chi, mat=cfg.mat)
    path = S.plan_coarsening(g, req)
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
    n = b_host.size
    stream = torch.cuda.Stream(device=dev)
    if h is not None:
        h.set_stream(stream)
    opts = S.SolveOptions(nu=cfg.nu, omega=cfg.omega, tol=cfg.tol, div_tol=cfg.div_tol,
                          max_cycles=cfg.max_cycles)
    with torch.cuda.stream(stream):
        b_dev = torch.from_numpy(b_host).to(dev)
        u_dev = torch.zeros_like(b_dev)
    stream.synchronize()

    def solve_on(bv, uv):
        if dh is not None:
            stream.synchronize()
            return S.mg_solve_dist(dh, bv, uv, opts)
        return S.mg_solve(h, bv, uv, opts)

    def one_solve():
        with torch.cuda.stream(stream):
            u_dev.zero_()
        return solve_on(b_dev, u_dev)

    for _ in range(args.warmup):
        rep = one_solve()
    # L2 flush buffer (> 126 MB L2): written between timed steps, outside the events
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    reps = []
    step_ms = []
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
                u_dev.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            reps.append(solve_on(b_dev, u_dev))
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize(dev)
    barrier()
    # Kernel-level timing (roofline): the same solves again with CUDA event
    # nodes around the fine-level kernels inside the graph.  Kept out of the
    # timed steps above: each event node adds launch-gap overhead (~10 us per
    # bracketed kernel when every level is profiled).
    prof_reps, prof_ms = [], []
    if h is not None and args.profile_steps > 0:
        h.set_profiling(True)
        one_solve()  # capture the profiled graph
        for _ in range(args.profile_steps):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
                u_dev.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            prof_reps.append(solve_on(b_dev, u_dev))
            e1.record(stream)
            e1.synchronize()
            prof_ms.append(e0.elapsed_time(e1))
        h.set_profiling(False)
    ms = sum(step_ms)
    updates = sum(r.smoother_dof_updates for r in reps)
    t_max = ms
    upd_total = updates
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
        uu = torch.tensor([updates], dtype=torch.float64, device=dev)
        dist.all_reduce(uu, op=dist.ReduceOp.SUM)
        upd_total = float(uu.item())
    value = upd_total / (t_max * 1e-3)
    last = reps[-1]

    # roofline: the dominant fine-level kernel from in-graph CUDA events.  The
    # fused two-sweep kernel (temporal blocking) moves 24 B/DOF (read u, f;
    # write u'') for two DOF updates; a single sweep 24 B/DOF for one.
    n0 = (cfg.n_el + 1) * (cfg.n_t + 1)
    hbm, peak_kind = peaks()

    def tot(key):
        c, t_ = 0, 0.0
        for r in prof_reps:
            cc, ss = r.kernel_times.get(key, (0, 0.0))
            c += cc
            t_ += ss
        return c, t_

    roofline = None
    pairs, pair_s = tot("fine_sweep_pair")
    singles, single_s = tot("fine_sweep")
    if pairs or singles:
        use_pair = pair_s >= single_s
        cnt, secs = (pairs, pair_s) if use_pair else (singles, single_s)
        avg = secs / cnt
        achieved = 24.0 * n0 / avg / 1e9
        # DRAM bytes per launch of the same kernel at this size from the committed
        # `ncu --set full` capture (profiles/round1.md, session 4: k_lean2x2<0,4,4,1>,
        # grid (10, 1025) x 128 threads): 67.297 MB read + 8.578 MB written; ncu
        # replays cold-cache, so this is the L2-miss traffic of an isolated launch,
        # an upper bound for the in-solve one
        traffic = (67.296768e6 + 8.578304e6) if (use_pair and n0 == 1025 * 4097) else None
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                    "frac": achieved / hbm, "traffic": traffic,
                    "traffic_source": ("ncu --set full, profiles/round1.md (cold-cache replay)"
                                       if traffic else None),
                    "kernel": ("k_lean2x2 (two fused Jacobi sweeps, fine level, in-graph CUDA events)"
                               if use_pair else "k_lean2<sweep> (fine level, in-graph CUDA events)"),
                    "algorithmic_bytes_per_launch": 24 * n0, "dof_updates_per_launch": (2 if use_pair else 1) * n0,
                    "avg_launch_ms": avg * 1e3, "launches_timed": cnt, "peak_source": peak_kind}
    kt = {}
    for key in ("fine_sweep", "fine_sweep_pair", "fine_restrict", "fine_prolong_sweep"):
        c, s_ = 0, 0.0
        for r in prof_reps:
            cc, ss = r.kernel_times.get(key, (0, 0.0))
            c += cc
            s_ += ss
        if c:
            kt[key] = {"launches": c, "avg_ms": 1e3 * s_ / c}
    step_ms_avg = t_max / max(args.steps, 1)
    if kt:
        kt["profiled_steps"] = len(prof_ms)
        kt["profiled_ms_per_step"] = sum(prof_ms) / len(prof_ms)
        kt["fine_share_of_step"] = sum(v["launches"] * v["avg_ms"] for v in kt.values()
                                       if isinstance(v, dict)) / max(sum(prof_ms), 1e-9)

    # e2e through the C ABI with pinned host buffers
    e2e = None
    if args.e2e_steps > 0:
        bh = torch.from_numpy(b_host).pin_memory()
        uh = torch.zeros(n, dtype=torch.float64).pin_memory()
        tot_ms, tot_upd = 0.0, 0.0
        for _ in range(args.e2e_steps):
            uh.zero_()
            torch.cuda.synchronize(dev)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = solve_on(bh, uh)
            e1.record(stream)
            e1.synchronize()
            tot_ms += e0.elapsed_time(e1)
            tot_upd += r.smoother_dof_updates
        if world > 1:
            tt = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tot_ms = float(tt.item())
            uu = torch.tensor([tot_upd], dtype=torch.float64, device=dev)
            dist.all_reduce(uu, op=dist.ReduceOp.SUM)
            tot_upd = float(uu.item())
        e2e = {"value": tot_upd / (tot_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 16 * n * world,
               "d2h_bytes_per_step": 8 * n * world, "solve_seconds": tot_ms * 1e-3 / args.e2e_steps}

    hbm_scale = None
    if rank == 0 and args.hbm_roofline:
        hbm_scale = hbm_scale_sweep(S, torch, dev, hbm)
        if hbm_scale is not None and roofline is not None:
            roofline["hbm_scale_cfg2_sweep"] = hbm_scale
        elif hbm_scale is not None and "achieved" in hbm_scale:
            # distributed solves carry no in-graph event timers: report the same kernel at HBM scale
            roofline = {"bound": "hbm", "achieved": hbm_scale["achieved"], "peak": hbm, "unit": "GB/s",
                        "frac": hbm_scale["frac"], "traffic": None,
                        "kernel": "k_lean2<sweep> on the cfg2 grid (in-graph timers off for slab solves)",
                        "algorithmic_bytes_per_launch": 24 * hbm_scale["dofs"],
                        "avg_launch_ms": hbm_scale["avg_launch_ms"], "peak_source": peak_kind,
                        "hbm_scale_cfg2_sweep": hbm_scale}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            res = run_cpu_sample(cfg, args.cpu_sample_nt, prefer_ref=True)
            cpu = {"value": res["updates"] / res["seconds"] if res["seconds"] > 0 else None,
                   "unit": UNIT, "cores": 1, "kind": res["kind"],
                   "sample": f"{cfg.name} truncated to n_t={res['n_t']} ({res['dofs']} DOFs), one full "
                             f"solve, {res['cycles']} V-cycles, {res['seconds']:.2f} s on 1 core"}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    clocks = clk.summary()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms_avg, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded mt19937_64 designs, BASELINE shapes)",
            "config": {"workload": cfg.name, "n_el": cfg.n_el, "n_t": cfg.n_t, "dofs": n0,
                       "method": cfg.method, "strategy": int(cfg.strategy), "n_levels": cfg.n_levels,
                       "min_elements": cfg.min_elements, "nu": cfg.nu, "tol": cfg.tol,
                       "path": S.path_to_string(path),
                       "parallelism": (f"time-slabs{world} (NCCL, {dh.n_distributed} distributed levels)"
                                       if dh is not None else "single"),
                       "l2": ("inputs larger than L2" if n0 * 8 * 3 > 126e6 else
                              "L2 flushed (256 MB write) before every timed step"),
                       "adjoint": cfg.adjoint},
            "solve_seconds": step_ms_avg * 1e-3, "cycles": last.cycles, "status": S.status_name(last.status),
            "final_rel_residual": last.history[-1], "gpu_launches": int(sum(r.kernel_launches for r in reps)),
            "roofline": roofline, "kernels": kt, "e2e": e2e, "cpu_baseline": cpu, "clocks": clocks,
            "build_seconds": t_build, "device_bytes": h.device_bytes() if h is not None else dh.device_bytes,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
