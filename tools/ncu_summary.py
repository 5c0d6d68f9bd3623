"""Summarise ncu captures for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py full  <report.ncu-rep> [algorithmic_bytes]
  python tools/ncu_summary.py launches <launches.csv>
  python tools/ncu_summary.py alg <plain run log>   (algorithmic bytes of one launch)
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_lg_throttle",
        "smsp__pcsamp_warps_issue_stalled_drain",
        "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def full(rep, alg=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{vals[i]} {units[i]}".strip()
        tr = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(k)
            tr += float(vals[i].replace(",", "")) * SCALE.get(units[i], 1)
        d["dram_traffic_bytes"] = tr
        if alg:
            d["algorithmic_bytes"] = float(alg)
            d["traffic_over_algorithmic"] = round(tr / float(alg), 4)
        out.append(d)
    print(json.dumps(out, indent=1))


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, n = defaultdict(float), defaultdict(int)
    mult = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[1:]:
        k = r[ki].split("(")[0]
        tot[k] += float(r[vi].replace(",", "")) * mult.get(r[ui], 1.0)
        n[k] += 1
    total = sum(tot.values())
    res = [{"kernel": k, "launches": n[k], "avg_us": round(tot[k] / n[k], 1),
            "share": round(tot[k] / total, 4)} for k in sorted(tot, key=tot.get, reverse=True)]
    print(json.dumps(res, indent=1))


def alg(plain_log, key=None):
    """Per-launch algorithmic bytes from a tools/ncu_targets.py or
    tools/bench_raw.py JSON line (prints nothing when absent)."""
    for line in open(plain_log):
        if line.startswith("{"):
            d = json.loads(line)
            keys = [key] if key else ["algorithmic_bytes_per_launch",
                                      "algorithmic_bytes_per_unit", "algorithmic_bytes"]
            for k in keys:
                if k in d:
                    print(int(d[k]))
                    return


if __name__ == "__main__":
    {"full": full, "launches": launches, "alg": alg}[sys.argv[1]](*sys.argv[2:])
