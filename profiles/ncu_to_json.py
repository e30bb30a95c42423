"""Per-kernel DRAM bytes and durations from `ncu --set full` captures of the
full-size level-0 kernels (profiles/kernel_probe.py --n-t 65536 on the cfg2
grid, 1.07e9 DOFs) into profiles/round2_ncu_cfg2.json, keyed like bench.py's
kernel table so the bench line's roofline.traffic is the measured DRAM traffic.

    python profiles/ncu_to_json.py gpurun_out/probe_cfg2.ncu-rep gpurun_out/probe_cfg2b.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {  # demangled-name prefix -> bench.py kernel key (a trailing level-width parameter may follow)
    "k_lean2<0, 0, 1, 8, 3, unnamed>::PlainLoad": "fine_norm_pass",
    "k_lean2<0, 0, 0, 8, 3, unnamed>::PlainLoad": "fine_sweep",
    "k_lean2x2<0, 8, 3, 0": "fine_sweep_pair",
    "k_restrict2<0, 0, 8, 3, 0": "fine_restrict",
    "k_restrict2<0, 0, 16, 2, 0": "fine_restrict",
    "k_restrict2<0, 0, 16, 3, 1": "zero_restrict",
    "k_lean2<0, 0, 0, 8, 4, unnamed>::ProlongOn<0, unnamed>::ZeroLoad>": "zero_prolong_sweep",
    "k_lean2<0, 0, 0, 8, 3, unnamed>::ProlongOn<0, unnamed>::PlainLoad>": "fine_prolong_sweep",
    "k_up<0, 8, unnamed>::ProlongOn<0, unnamed>::PlainLoad>": "fine_up",
}
METRICS = "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"


def main():
    path = os.path.join(ROOT, "profiles", "round2_ncu_cfg2.json")
    out = {"source": "ncu --set full --clock-control none, profiles/kernel_probe.py --n-t 65536 "
                     "(cfg2 level 0: 16384 x 65536, 1.07e9 DOFs)", "kernels": {}}
    if os.path.exists(path):  # later captures update single kernels
        with open(path) as fh:
            out["kernels"] = json.load(fh).get("kernels", {})
    for rep in sys.argv[1:]:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base", "--metrics", METRICS],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        hdr = rows[0]
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            for frag, key in KEYS.items():
                if frag in d["Kernel Name"]:
                    out["kernels"][key] = {"kernel": d["Kernel Name"][:120],
                                           "duration_ms": float(d["gpu__time_duration.sum"]) * 1e-6,
                                           "dram_bytes_read": float(d["dram__bytes_read.sum"]),
                                           "dram_bytes_write": float(d["dram__bytes_write.sum"])}
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
