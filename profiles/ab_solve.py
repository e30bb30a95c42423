"""Same-box A/B of whole-solve time under environment variants.

Each variant runs in its own process with its own environment (e.g.
STMG_LIB_PATH=<an A/B build of libstmg_b200.so>); variants are interleaved over --rounds so that box drift hits all
of them alike.  Per process: --warmup untimed solves, then --solves timed solves
(L2 flushed before each, CUDA-event device time from the solve report).

    python profiles/ab_solve.py --config cfg1 \
        --variant base= --variant new=STMG_LIB_PATH=/tmp/ab/libstmg_b200.so
"""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(config, warmup, solves, n_levels):
    import torch

    from paper_2505_10168_b200 import configs as C
    from paper_2505_10168_b200 import stmg as S

    cfg = C.CONFIGS[config]()
    if n_levels:
        cfg.n_levels = n_levels
    g = S.build_fine_grid(cfg.L, cfg.t_T, cfg.n_el, cfg.n_t)
    g.k, g.c = cfg.k, cfg.c
    path = S.plan_coarsening(g, S.PlanRequest(n_levels=cfg.n_levels, strategy=S.PlanStrategy(cfg.strategy),
                                              reassembly=S.ReassemblyMethod(cfg.reassembly),
                                              min_elements=cfg.min_elements, chi=cfg.chi, mat=cfg.mat))
    h = S.build_hierarchy(g, cfg.method, path, chi=cfg.chi, mat=cfg.mat)
    b = torch.from_numpy(S.load_vector(g, kind=cfg.source_kind, params=cfg.source_params, masked=True)).cuda()
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    opts = S.SolveOptions(nu=cfg.nu, tol=cfg.tol, max_cycles=cfg.max_cycles)
    ts, cyc = [], None
    for k in range(warmup + solves):
        u = torch.zeros_like(b)
        flush.fill_(float(k))
        torch.cuda.synchronize()
        rep = S.mg_solve(h, b, u, opts)
        cyc = rep.cycles
        if k >= warmup:
            ts.append(rep.device_seconds * 1e3)
    print(json.dumps({"ms": ts, "cycles": cyc}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--variant", action="append", default=[],
                    help="name=K1=V1,K2=V2 (empty after '=' for the defaults)")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--solves", type=int, default=5)
    ap.add_argument("--n-levels", type=int, default=None)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        child(a.config, a.warmup, a.solves, a.n_levels)
        return
    variants = []
    for v in a.variant or ["base="]:
        name, _, spec = v.partition("=")
        env = dict(kv.split("=", 1) for kv in spec.split(",") if kv)
        variants.append((name, env))
    res = {n: [] for n, _ in variants}
    cycles = {}
    for _ in range(a.rounds):
        for name, env in variants:
            cmd = [sys.executable, os.path.abspath(__file__), "--child", "--config", a.config,
                   "--warmup", str(a.warmup), "--solves", str(a.solves)]
            if a.n_levels:
                cmd += ["--n-levels", str(a.n_levels)]
            p = subprocess.run(cmd, env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
            if p.returncode != 0:
                print(f"{name}: rc={p.returncode}\n{p.stderr[-2000:]}", flush=True)
                continue
            d = json.loads(p.stdout.strip().splitlines()[-1])
            res[name] += d["ms"]
            cycles[name] = d["cycles"]
    for name, _ in variants:
        ms = res[name]
        if ms:
            print(json.dumps({"variant": name, "median_ms": statistics.median(ms), "min_ms": min(ms),
                              "n": len(ms), "cycles": cycles.get(name)}), flush=True)


if __name__ == "__main__":
    main()
