"""Summarise a profile_round.sh output directory into profiles/<round>/ (no GPU needed).

    python tools/summarize_r02.py gpurun_out/r02prof profiles/r02

Writes launches_share.json (per-kernel share of the bench step from the ncu launch
list), kernels.json (key metrics of every full capture with DRAM traffic over the
kernel's algorithmic bytes) and kernels.md (the same as tables).
"""
import csv
import json
import os
import sys
from collections import defaultdict

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
        "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0}

# configs of the step (bench.py): config 5 HODLR, config 4 HSS
N5, B5, P5, K5, M5 = 1 << 24, 256, 16, 1, 1
N4, B4, P4, K4, M4 = 1 << 22, 128, 15, 32, 32


def alg_bytes_c5(kind):
    if kind == "vt_gemv":  # every level's V once, X once, t out (small)
        return 8 * (P5 * N5 * K5 + N5 * M5)
    return 8 * (N5 * B5 + P5 * N5 * K5 + 2 * N5 * M5)  # leaf pass: D, every level's U, X, Y


def c4_blocks(l):
    return (1 << l) * K4 * M4 * 8  # the x / y blocks of level l


def alg_bytes_c4(kind, idx):
    kk = K4 * K4 * 8
    if kind == "vt_batched":
        return 8 * (N4 * K4 + N4 * M4) + c4_blocks(P4)
    if kind == "up":  # launch idx 0..3 = levels 14..11: W of the level, children x in, x out
        l = P4 - 1 - idx
        return (1 << l) * 2 * kk + c4_blocks(l + 1) + c4_blocks(l)
    if kind == "down":  # idx 0..4 = levels 11..15: R and cores of the parents, x of the level, y parent, y out
        l = 11 + idx
        return (1 << (l - 1)) * 4 * kk + c4_blocks(l) + c4_blocks(l - 1) + c4_blocks(l)
    if kind == "down2":  # idx = first level l of the fused pair (l, l+1): R and cores of both levels' parents,
        l = idx           # x of both levels, y of level l-1 in, y of level l+1 out (y_l stays in shared memory)
        return ((1 << (l - 1)) + (1 << l)) * 4 * kk + c4_blocks(l) + 2 * c4_blocks(l + 1) + c4_blocks(l - 1)
    if kind == "leaf":
        return 8 * (N4 * B4 + N4 * K4 + 2 * N4 * M4) + c4_blocks(P4)
    return None


def read_raw(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {}
        for k in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                  "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                  "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
                  "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"):
            if k not in h:
                continue
            i = h.index(k)
            v = r[i]
            try:
                d[k] = float(v.replace(",", "")) * UNIT.get(units[i], 1.0)
            except ValueError:
                d[k] = v
        out.append(d)
    return out


def main(src, dst):
    os.makedirs(dst, exist_ok=True)
    # ---- launch list of the bench step
    per = defaultdict(lambda: {"launches": 0, "time_s": 0.0, "dram_bytes": 0.0})
    for r in csv.DictReader(l for l in open(os.path.join(src, "launches.csv")) if not l.startswith("==")):
        name, metric, unit, val = r["Kernel Name"], r["Metric Name"], r["Metric Unit"], r["Metric Value"]
        v = float(val.replace(",", "")) * UNIT.get(unit, 1.0)
        e = per[name.split("(")[0].replace("void ", "")]
        if metric == "gpu__time_duration.sum":
            e["launches"] += 1
            e["time_s"] += v
        elif metric.startswith("dram__bytes"):
            e["dram_bytes"] += v
    tot = sum(e["time_s"] for e in per.values())
    share = {k: {"launches": e["launches"], "share": round(e["time_s"] / tot, 4),
                 "dram_GBps": round(e["dram_bytes"] / e["time_s"] / 1e9, 1) if e["time_s"] else None}
             for k, e in sorted(per.items(), key=lambda kv: -kv[1]["time_s"])}
    json.dump({"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                         "--clock-control none over `bench.py --steps 2 --warmup 3 --no-sweep --no-parity "
                         "--no-cpu-baseline` (every libhm launch incl. warm-up and e2e calls; cold-cache, serialised)",
               "kernels": share}, open(os.path.join(dst, "launches_share.json"), "w"), indent=1)
    # ---- full captures
    caps = []
    for cfg, path in (("c5", "c5.raw.csv"), ("c4", "c4.raw.csv")):
        up = down = 0
        dl = 11  # next downsweep level (config 4: pair launch on 11, then hss_down_two on 12-13 and 14-15)
        for d in read_raw(os.path.join(src, path)):
            name = d["Kernel Name"]
            if cfg == "c5":
                kind = "vt_gemv" if "vt_gemv" in name else "leaf"
                alg = alg_bytes_c5(kind)
            elif "vt_batched" in name:
                kind, alg = "vt_batched", alg_bytes_c4("vt_batched", 0)
            elif "up_stage" in name or "up_pair" in name:
                kind, alg = f"up level {P4 - 1 - up}", alg_bytes_c4("up", up)
                up += 1
            elif "down_two" in name:
                kind, alg = f"down levels {dl}-{dl + 1} (one launch)", alg_bytes_c4("down2", dl)
                dl += 2
            elif "down_pair" in name or "down_stage" in name:
                kind, alg = f"down level {dl}", alg_bytes_c4("down", dl - 11)
                dl += 1
            elif "sweep" in name:
                kind, alg = "sweep (levels 1..10)", None
            elif "tree_flow" in name:
                kind, alg = "levels 10..1 up + 1..10 down (dataflow)", None
            else:
                kind, alg = "leaf", alg_bytes_c4("leaf", 0)
            t = d["gpu__time_duration.sum"]
            dram = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
            caps.append({"config": cfg, "kernel": name.split("(")[0].replace("void ", ""), "role": kind,
                         "us": round(t * 1e6, 1), "dram_bytes": dram, "alg_bytes": alg,
                         "traffic_over_alg": round(dram / alg, 3) if alg else None,
                         "dram_TBps": round(dram / t / 1e12, 2),
                         "tensor_pipe_pct": round(d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0.0), 1),
                         "warps_active_pct": round(d.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0.0), 1),
                         "regs": d.get("launch__registers_per_thread")})
    json.dump(caps, open(os.path.join(dst, "kernels.json"), "w"), indent=1)
    lines = ["| config | kernel | role | µs | DRAM TB/s | traffic / alg | tensor pipe % | warps active % | regs |",
             "|---|---|---|---|---|---|---|---|---|"]
    for c in caps:
        lines.append(f"| {c['config']} | `{c['kernel']}` | {c['role']} | {c['us']} | {c['dram_TBps']} | "
                     f"{c['traffic_over_alg'] if c['traffic_over_alg'] is not None else '—'} | {c['tensor_pipe_pct']} | "
                     f"{c['warps_active_pct']} | {int(c['regs']) if c['regs'] else ''} |")
    lines += ["", "| kernel (bench step launch list) | launches | share of libhm time | DRAM GB/s |", "|---|---|---|---|"]
    for k, e in share.items():
        lines.append(f"| `{k}` | {e['launches']} | {100 * e['share']:.1f}% | {e['dram_GBps']} |")
    open(os.path.join(dst, "kernels.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
