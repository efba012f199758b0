"""Summarise ncu captures for profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py launches <launches.csv>            # per-kernel share of a step
    python tools/ncu_summary.py report <file.ncu-rep> [alg_bytes]  # key metrics of one capture
    python tools/ncu_summary.py raw <file.raw.csv> [alg_bytes]     # same, from `ncu -i .. --page raw --csv`
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_registers",
    "lts__t_bytes.sum",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_lg_throttle",
]

UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "byte": 1.0, "usecond": 1e-6, "msecond": 1e-3,
        "nsecond": 1e-9, "second": 1.0, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0}


def report(path, alg_bytes=None, raw_csv=None):
    out = raw_csv if raw_csv is not None else subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                                                             capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, r = rows[0], rows[1], rows[2]
    res = {"kernel": r[h.index("Kernel Name")]}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            v = r[i].replace(",", "")
            try:
                val = float(v) * UNIT.get(units[i], 1.0)
            except ValueError:
                val = v
            res[k] = val
    if "dram__bytes_read.sum" in res:
        res["dram_bytes_total"] = res["dram__bytes_read.sum"] + res.get("dram__bytes_write.sum", 0.0)
        if alg_bytes:
            res["alg_bytes"] = float(alg_bytes)
            res["traffic_over_alg"] = res["dram_bytes_total"] / float(alg_bytes)
    if "gpu__time_duration.sum" in res and "dram_bytes_total" in res:
        res["dram_GBps"] = res["dram_bytes_total"] / res["gpu__time_duration.sum"] / 1e9  # duration in seconds
    return res


def launches(path):
    """Per-kernel totals of a `--metrics gpu__time_duration.sum[,dram__bytes_*]` launch list."""
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.find('"ID"'):])))
    tot, cnt, dram, seen = {}, {}, {}, set()
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
        if r["Metric Name"] == "gpu__time_duration.sum":
            tot[name] = tot.get(name, 0.0) + v * 1e6
            if r["ID"] not in seen:
                seen.add(r["ID"])
                cnt[name] = cnt.get(name, 0) + 1
        elif r["Metric Name"].startswith("dram__bytes"):
            dram[name] = dram.get(name, 0.0) + v
    all_us = sum(tot.values())
    return {k: {"launches": cnt[k], "us_total": round(v, 1), "share": round(v / all_us, 4),
                **({"dram_GB": round(dram[k] / 1e9, 3), "dram_GBps": round(dram[k] / (v * 1e-6) / 1e9, 1)}
                   if k in dram else {})}
            for k, v in sorted(tot.items(), key=lambda kv: -kv[1])}


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    elif sys.argv[1] == "raw":
        print(json.dumps(report(None, sys.argv[3] if len(sys.argv) > 3 else None, open(sys.argv[2]).read()), indent=1))
    else:
        print(json.dumps(report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None), indent=1))
