"""Summarise ncu captures into profiles/*.md tables (run here, no GPU needed).

  python profiles/summarize.py report <file.ncu-rep>      key metrics per kernel
  python profiles/summarize.py launches <launches.csv>    per-kernel time shares
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size"]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {k: hdr.index(k) for k in KEYS if k in hdr}
    print("| kernel | " + " | ".join(KEYS) + " |")
    print("|---" * (len(KEYS) + 1) + "|")
    for r in rows[2:]:
        name = re.sub(r"\(.*", "", r[hdr.index("Kernel Name")])[:70]
        vals = [f"{r[idx[k]]} {units[idx[k]]}".strip() if k in idx else "-" for k in KEYS]
        print(f"| {name} | " + " | ".join(vals) + " |")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for d in data:
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("stmgb::", "")
        key = f"{name[:64]} grid={d.get('Grid Size', '')}"
        v = float(d["Metric Value"]) * scale.get(d["Metric Unit"], 1e-3)
        tot[key] += v
        cnt[key] += 1
    grand = sum(tot.values())
    print(f"{len(data)} launches, {grand / 1e3:.2f} ms total (serialised, cold-cache)\n")
    print("| share | total us | launches | avg us | kernel |")
    print("|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:30]:
        print(f"| {100 * v / grand:5.1f}% | {v:10.1f} | {cnt[k]} | {v / cnt[k]:8.2f} | {k} |")


if __name__ == "__main__":
    {"report": report, "launches": launches}[sys.argv[1]](sys.argv[2])
