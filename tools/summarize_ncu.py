"""Summarise ncu reports into profiles/ (tracked).

  python tools/summarize_ncu.py full <report.ncu-rep> <out.json>
      per-kernel key metrics of a --set full capture (+ ncu_traffic.json for bench.py)
  python tools/summarize_ncu.py launches <launches.csv> <out.json>
      per-kernel-name count / total / share of a gpu__time_duration launch list
"""

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_registers",
    "sm__cycles_elapsed.avg.per_second",
    "dram__cycles_elapsed.avg.per_second",
]


def full(rep, out):
    text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        rec = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                v = r[hdr.index(k)].replace(",", "")
                try:
                    rec[k] = float(v)
                except ValueError:
                    rec[k] = v
                rec[k + ".unit"] = units[hdr.index(k)]
        kernels.append(rec)
    with open(out, "w") as fh:
        json.dump({"report": rep, "kernels": kernels}, fh, indent=1)
    print(json.dumps(kernels, indent=1)[:3000])


def launches(path, out):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1 :]:
        if len(r) != len(hdr) or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[hdr.index("Kernel Name")].split("(")[0]
        val = float(r[hdr.index("Metric Value")].replace(",", ""))
        unit = r[hdr.index("Metric Unit")]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
        agg[name][0] += 1
        agg[name][1] += val * scale
    total = sum(v[1] for v in agg.values())
    summary = {k: {"launches": v[0], "total_us": v[1], "mean_us": v[1] / v[0], "share": v[1] / total}
               for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}
    with open(out, "w") as fh:
        json.dump({"source": path, "kernels": summary, "total_us": total}, fh, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
