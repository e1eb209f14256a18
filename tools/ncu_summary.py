#!/usr/bin/env python
"""Summarise ncu output for profiles/.

  tools/ncu_summary.py launches <launches.csv> [<cmd>]   per-kernel launch list (share of time)
  tools/ncu_summary.py full <prof.ncu-rep>                key metrics of a --set full capture
"""
import collections
import csv
import io
import subprocess
import sys

FULL_KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
]


def to_us(v, unit):
    return v / 1000.0 if unit in ("ns", "nsecond") else v * 1000.0 if unit in ("ms", "msecond") else v


def launches(path, cmd=""):
    agg = collections.defaultdict(list)
    hdr = None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = to_us(float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
                agg[d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")].append(v)
    prod = {k: v for k, v in agg.items() if not k.split("::")[-1].startswith("synth_")}
    tot = sum(sum(v) for v in prod.values()) or 1.0
    out = []
    if cmd:
        out.append(f"# ncu launch list of: {cmd}")
    out.append("# ncu times are cold-cache and serialised (each launch replayed): compare SHARES, not absolutes.")
    out.append("# share = of the path's kernels (synth_* = synthetic input generation, outside the timed region)")
    out.append("kernel,launches,total_us,mean_us,share")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        share = f"{sum(v) / tot:.3f}" if k in prod else "nan"
        out.append(f"{k.split('::')[-1]},{len(v)},{sum(v):.1f},{sum(v) / len(v):.2f},{share}")
    return "\n".join(out)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        out.append("----")
        out.append(f"  Kernel Name = {v[hdr.index('Kernel Name')]}")
        for k in FULL_KEYS:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"  {k} [{units[i]}] = {v[i]}")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""))
    else:
        print(full(sys.argv[2]))
