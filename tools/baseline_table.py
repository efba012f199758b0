"""Print BASELINE.md §5's results table from a bench.py JSON line and the oracle table.

    python tools/baseline_table.py profiles/r02/bench.json profiles/r02_cpu_table.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import hodlr_bytes, hodlr_flops, hss_bytes, hss_flops  # noqa: E402

READ_STREAM = 7185.1


def main(bench_path, table_path):
    d = json.loads(open(bench_path).read().strip().splitlines()[-1])
    t = {(r["config"], r["nrhs"]): r for r in json.load(open(table_path))["rows"]}
    peak = d["roofline"]["peak"]
    sw, par = d["sweep"], d["parity"]
    fp64 = 37.0

    def row(cfg, m, us, nb, fl, rel, note=""):
        gbs = nb / (us * 1e-6) / 1e9
        tf = fl / (us * 1e-6) / 1e12
        o = t[(cfg, m)]
        frac = f" ({tf / fp64:.2f} of {fp64} TF DMMA)" if tf > 5 else ""
        return (f"| {cfg} | {m} | 1 | {us:.1f}{note} | {gbs:.0f} | {100 * gbs / peak:.1f} | "
                f"{100 * gbs / READ_STREAM:.1f} | {tf * 1e3:.0f}{frac} | — | {rel:.1e} | "
                f"{o['s_1thr']:.4g} | {o['s_16thr']:.4g} |")

    out = [row("C1", 1, sw["c1_us_graph"], hodlr_bytes(1024, 64, 4, 8, 1), hodlr_flops(1024, 64, 4, 8, 1),
               par["c1"]["relerr_vs_oracle"], " (graph)"),
           row("C2", 16, sw["c2_us_graph"], hss_bytes(4096, 64, 6, 16, 16), hss_flops(4096, 64, 6, 16, 16),
               par["c2"]["relerr_vs_oracle"], " (graph)")]
    for m in (1, 8, 64):
        out.append(row("C3", m, sw[f"c3_m{m}"]["ms"] * 1e3, hodlr_bytes(1 << 20, 256, 12, 16, m),
                       hodlr_flops(1 << 20, 256, 12, 16, m), par[f"c3_m{m}"]["relerr_vs_oracle"]))
    out.append(row("C4", 32, d["per_config"]["c4_hss"]["ms"] * 1e3, hss_bytes(1 << 22, 128, 15, 32, 32),
                   hss_flops(1 << 22, 128, 15, 32, 32), par["c4"]["relerr_vs_oracle"]))
    out.append(row("C5", 1, d["per_config"]["c5_hodlr"]["ms"] * 1e3, hodlr_bytes(1 << 24, 256, 16, 1, 1),
                   hodlr_flops(1 << 24, 256, 16, 1, 1), par["c5"]["relerr_vs_oracle"]))
    print("\n".join(out))


if __name__ == "__main__":
    main(*sys.argv[1:3])
