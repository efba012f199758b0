#!/usr/bin/env python
"""Benchmark: HODLR/HSS fp64 matvec GB/s and % of the HBM roofline on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c5+c4]

One STEP = one pass of the whole hot path: one HODLR
matvec on BASELINE config 5 (inverse 1D Laplacian, n = 2^24, leaf 256, 16 levels,
rank 1, nrhs 1) and one HSS matvec on BASELINE config 4 (n = 2^22, leaf 128,
15 levels, rank 32, nrhs 32) — the two configs BASELINE.json quotes "at 1/2/4/8
B200" — with generators and X resident in HBM. `value` = algorithmic bytes
(every generator once + X once + Y once) of all steps on all ranks
/ device time of the timed region (max over ranks). Inputs (49 GB/step) are far
larger than the 126 MB L2, so no flush is needed between steps.

Prints ONE JSON line on rank 0. `--impl reference` times the CPU oracle (the
slow, plain C reference of oracle/) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import hm_inputs  # noqa: E402

METRIC = "HODLR/HSS fp64 matvec GB/s and % of HBM roofline vs nrhs, at 1/2/4/8 B200"


# ------------------------------------------------------------- workloads --

def hodlr_bytes(n, b, p, k, m):
    """8 (n b + 2 p n k + 2 n m)."""
    return 8 * (n * b + 2 * p * n * k + 2 * n * m)


def hodlr_flops(n, b, p, k, m):
    return 2 * n * m * (b + 2 * p * k)


def hss_bytes(n, b, p, k, m):
    """8 (n b + 2 n k + 4 (2^p - 2) k^2 + 2 (2^p - 1) k^2 + 2 n m)."""
    return 8 * (n * b + 2 * n * k + 4 * ((1 << p) - 2) * k * k + 2 * ((1 << p) - 1) * k * k + 2 * n * m)


def hss_flops(n, b, p, k, m):
    return 2 * n * m * (b + 2 * k) + 8 * ((1 << p) - 2) * k * k * m + 4 * ((1 << p) - 1) * k * k * m


READ_STREAM_GBS = 7185.1  # measured read-only fp64 stream on this pool's B200 (tools/fp64_peaks.cu)
FP64_PEAK_TFLOPS = 37.0  # measured DMMA (mma.sync f64) peak on this pool's B200, tools/fp64_peaks.cu
C5 = hm_inputs.CONFIGS[5]
C4 = hm_inputs.CONFIGS[4]
M5, M4 = 1, 32


def step_bytes():
    return hodlr_bytes(C5.n, C5.leaf, C5.levels, C5.k, M5) + hss_bytes(C4.n, C4.leaf, C4.levels, C4.k, M4)


def hss_attainable_ms(n, b, p, k, m, copy_gbs):
    """Config 4's attainable time: every phase at what the machine
    measurably delivers for it — the leaf pass (D X + U y: 2 n m (b + k) flops over
    its physical bytes) at the read-stream + DMMA ridge for its intensity
    (profiles/r02/fp64_peaks_ridge.json, interpolated between 4 and 6 flop/B),
    Step 1 (V, X read, leaf x written) at the read stream, the tree levels
    (W, R, B and the coefficient blocks they read and write) at the copy figure."""
    blk = k * m
    leaf_flops = 2.0 * n * m * (b + k)
    leaf_bytes = 8.0 * (n * b + n * k + 2 * n * m + (1 << p) * blk)
    inten = leaf_flops / leaf_bytes
    t = min(max((inten - 4.0) / 2.0, 0.0), 1.0)
    ridge_tf = 27.85 + t * (32.83 - 27.85)
    step1_bytes = 8.0 * (n * k + n * m + (1 << p) * blk)
    nodes = (1 << (p + 1)) - 2  # coefficient blocks of levels 1..p
    gen = 8.0 * (2 * ((1 << p) - 2) * 2 * k * k + ((1 << p) - 1) * 2 * k * k)
    coef = 8.0 * blk * ((nodes - 2) + (nodes - (1 << p)) + nodes + (nodes - (1 << p)) + nodes)
    ms = leaf_flops / (ridge_tf * 1e12) * 1e3 + step1_bytes / (READ_STREAM_GBS * 1e9) * 1e3 \
        + (gen + coef) / (copy_gbs * 1e9) * 1e3
    return ms


def leaf_apply_c5_bytes(n, b, p, k, m):
    """Algorithmic bytes of one HODLR leaf-pass (leaf_gemv) launch: D + every level's U + X + Y."""
    return 8 * (n * b + p * n * k + 2 * n * m)


# ------------------------------------------------------------------ peaks --

def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def committed_traffic(kernel, workload):
    """dram bytes per launch from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        e = t.get(workload, {}).get(kernel)
        return None if e is None else float(e)
    except Exception:
        return None


# ---------------------------------------------------------------- clocks --

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(prefix="hm_clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    sm.append(float(parts[0]))
                    smax = float(parts[1])
                except ValueError:
                    continue
                for nm, v in zip(names, parts[3:7]):
                    if v.lower() == "active":
                        reasons.add(nm)
        finally:
            try:
                os.unlink(self.path)
            except OSError:
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------- our implementation --

class Workload:
    """Device-resident generators for the step (rank-local shard when N > 1)."""

    def __init__(self, torch, device, seed):
        self.torch = torch
        self.device = device
        # config 5: closed-form inverse Laplacian filled on the device (no host round trip)
        self.h5 = hm_inputs.hodlr_inverse_laplacian(C5.n, C5.levels, xp=torch, device=device)
        g = torch.Generator(device=device)
        g.manual_seed(seed)
        self.X5 = torch.randn(C5.n, M5, dtype=torch.float64, device=device, generator=g)
        self.Y5 = torch.empty_like(self.X5)
        # config 4: orthonormalised Gaussian generators drawn on the device
        self.s4 = hm_inputs.device_hss_random(C4.n, C4.levels, C4.k, seed + 1, device)
        self.X4 = torch.randn(C4.n, M4, dtype=torch.float64, device=device, generator=g)
        self.Y4 = torch.empty_like(self.X4)
        import paper_1909_07909_b200 as hm
        self.hm = hm
        self.ws5 = torch.empty(hm.hm_hodlr_workspace_bytes(C5.n, C5.levels, C5.leaf, self.h5.ranks, M5),
                               dtype=torch.uint8, device=device)
        self.ws4 = torch.empty(hm.hm_hss_workspace_bytes(C4.n, C4.levels, C4.leaf, C4.k, M4), dtype=torch.uint8,
                               device=device)
        # end-to-end: pinned host X / Y, the library copies them through its own
        # workspace. Four lanes (stream + workspaces + host buffers) so that step
        # i+1's host-to-device copies overlap step i's kernels and device-to-host
        # copies (separate copy engines) — every step still moves its own X in
        # and its own Y out. Bound: 1.2 GB each way per step over PCIe, measured
        # 55.5 GB/s one way, 45.6 GB/s each way when both run (tools/pcie_bw.py)
        # -> >= 26 ms per step, 1.87 TB/s of algorithmic bytes.
        self.lanes = []
        for _ in range(int(os.environ.get("HM_E2E_LANES", "4"))):
            ln = {"stream": torch.cuda.Stream(device=device),
                  "X5h": self.X5.cpu().pin_memory(), "X4h": self.X4.cpu().pin_memory()}
            ln["Y5h"] = torch.empty_like(ln["X5h"]).pin_memory()
            ln["Y4h"] = torch.empty_like(ln["X4h"]).pin_memory()
            ln["ws5"] = torch.empty(hm.hm_hodlr_workspace_bytes(C5.n, C5.levels, C5.leaf, self.h5.ranks, M5,
                                                                hm.HM_WS_HOSTIO), dtype=torch.uint8, device=device)
            ln["ws4"] = torch.empty(hm.hm_hss_workspace_bytes(C4.n, C4.levels, C4.leaf, C4.k, M4, hm.HM_WS_HOSTIO),
                                    dtype=torch.uint8, device=device)
            self.lanes.append(ln)
        self.launches = 0

    def step(self):
        hm, h, s = self.hm, self.h5, self.s4
        hm.hodlr_matvec(C5.n, C5.levels, C5.leaf, h.ranks, h.D, h.U, h.V, self.X5, self.Y5, self.ws5)
        self.launches += hm.last_launch_count()
        hm.hss_matvec(C4.n, C4.levels, C4.leaf, C4.k, s.D, s.U, s.V, s.R, s.W, s.B, self.X4, self.Y4, self.ws4)
        self.launches += hm.last_launch_count()

    def step_e2e(self, i=0):
        hm, h, s = self.hm, self.h5, self.s4
        ln = self.lanes[i % len(self.lanes)]
        st = ln["stream"]
        hm.hodlr_matvec_hostio(C5.n, C5.levels, C5.leaf, h.ranks, h.D, h.U, h.V, ln["X5h"], ln["Y5h"], ln["ws5"],
                               stream=st)
        hm.hss_matvec_hostio(C4.n, C4.levels, C4.leaf, C4.k, s.D, s.U, s.V, s.R, s.W, s.B, ln["X4h"], ln["Y4h"],
                             ln["ws4"], stream=st)

    def e2e_begin(self, ev):
        for ln in self.lanes:
            ln["stream"].wait_event(ev)

    def e2e_end(self, torch):
        cur = torch.cuda.current_stream()
        for ln in self.lanes:
            cur.wait_stream(ln["stream"])

    def h2d_d2h_bytes(self):
        return 8 * (C5.n * M5 + C4.n * M4), 8 * (C5.n * M5 + C4.n * M4)

    calls = ("c5", "c4")  # matvec calls per step (launch-trace labels)
    rows5 = C5.n
    rows4 = C4.n


class DistWorkload:
    """Rank r of P: the shards of include/hm.h "multi-GPU" (rows of node (q, r) and its
    subtree), filled on this rank's GPU; one libhm call per product, the allgather
    inside libhm (NCCL communicator, hm_comm_*)."""

    calls = ("c5", "c4")  # one traced call per product

    def __init__(self, torch, device, seed, P, r):
        import paper_1909_07909_b200 as hm
        from paper_1909_07909_b200 import dist as hd
        self.torch, self.device, self.hm, self.hd, self.P, self.r = torch, device, hm, hd, P, r
        self.comm = hd.Comm.from_group()
        n5, p5, b5 = C5.n, C5.levels, C5.leaf
        lpr = (1 << p5) // P
        nl5 = n5 // P
        self.rows5 = nl5
        # only this rank's rows / subtree are generated (shard-local fill)
        self.D5 = hm_inputs.inverse_laplacian_leaf_blocks(n5, p5, leaves=range(r * lpr, (r + 1) * lpr), xp=torch,
                                                          device=device)
        self.ranks5 = [1] * p5
        self.U5, self.V5 = hm_inputs.inverse_laplacian_factors(n5, p5, xp=torch, device=device,
                                                               rows=(r * nl5, (r + 1) * nl5))
        g = torch.Generator(device=device)
        g.manual_seed(seed + r)
        self.X5 = torch.randn(nl5, M5, dtype=torch.float64, device=device, generator=g)
        self.Y5 = torch.empty_like(self.X5)
        self.sh4 = hm_inputs.device_hss_shard(C4.n, C4.levels, C4.k, seed + 1, device, P, r)
        nl4 = C4.n // P
        self.rows4 = nl4
        self.X4 = torch.randn(nl4, M4, dtype=torch.float64, device=device, generator=g)
        self.Y4 = torch.empty_like(self.X4)
        self.ws5 = torch.empty(hd.hodlr_dist_workspace_bytes(n5, p5, b5, self.ranks5, M5, P), dtype=torch.uint8,
                               device=device)
        self.ws4 = torch.empty(hd.hss_dist_workspace_bytes(C4.n, C4.levels, C4.leaf, C4.k, M4, P), dtype=torch.uint8,
                               device=device)
        self.X5h = self.X5.cpu().pin_memory()
        self.Y5h = torch.empty_like(self.X5h).pin_memory()
        self.X4h = self.X4.cpu().pin_memory()
        self.Y4h = torch.empty_like(self.X4h).pin_memory()
        self.launches = 0

    def step(self):
        hd = self.hd
        hd.hodlr_matvec_dist(self.comm, C5.n, C5.levels, C5.leaf, self.ranks5, self.D5, self.U5, self.V5, self.X5,
                             self.Y5, ws=self.ws5)
        hd.hss_matvec_dist(self.comm, C4.n, C4.levels, C4.leaf, C4.k, self.sh4, self.X4, self.Y4, ws=self.ws4)

    def e2e_begin(self, ev):
        pass

    def e2e_end(self, torch):
        pass

    def step_e2e(self, i=0):
        self.X5.copy_(self.X5h, non_blocking=True)
        self.X4.copy_(self.X4h, non_blocking=True)
        self.step()
        self.Y5h.copy_(self.Y5, non_blocking=True)
        self.Y4h.copy_(self.Y4, non_blocking=True)

    def h2d_d2h_bytes(self):
        return 8 * (self.X5.numel() + self.X4.numel()), 8 * (self.Y5.numel() + self.Y4.numel())

    def close(self):
        self.comm.close()


# ------------------------------------------------------ nrhs / ops sweep --

def _c4_leaf_roofline(per, steps, wl):
    d = per.get("c4:leaf_mma")
    if not d or d[0] == 0:
        return None
    rows = getattr(wl, "rows4", C4.n)
    flops = 2.0 * rows * M4 * (C4.leaf + C4.k)
    avg_ms = d[1] / d[0]
    tf = flops / (avg_ms * 1e-3) / 1e12
    # context: what the read stream and the DMMA pipe deliver TOGETHER at this
    # arithmetic intensity (tools/fp64_peaks.cu ridge kernel, sustained 3 s per
    # point, profiles/r02/fp64_peaks_ridge.json), interpolated between the measured
    # 4 and 6 flop/byte points; the kernel's physical bytes: D, U, X, Y, y
    phys = 8.0 * rows * (C4.leaf + C4.k + 2 * M4) + 8.0 * (rows // C4.leaf) * C4.k * M4
    inten = flops / phys
    r4, r6 = (6961.9, 27.85), (5472.0, 32.83)  # (read GB/s, DMMA TF/s) at 4 and 6 flop/byte
    t = min(max((inten - 4.0) / 2.0, 0.0), 1.0)
    ridge_tf = r4[1] + t * (r6[1] - r4[1])
    return {"bound": "tensor (fp64 DMMA)", "kernel": "leaf_mma_kernel<2,4,1,4> (config-4 leaf pass: D_i X_i + U_i y_i)",
            "achieved": _fin(tf, 2), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": _fin(tf / FP64_PEAK_TFLOPS, 4),
            "peak_kind": "measured DMMA (tools/fp64_peaks.cu, profiles/r01_next/fp64_peaks_mix.json)",
            "alg_flops_per_launch": flops, "avg_launch_ms": _fin(avg_ms, 4),
            "ridge_context": {"flop_per_byte": _fin(inten, 2), "dmma_tflops_at_this_intensity": _fin(ridge_tf, 2),
                              "frac": _fin(tf / ridge_tf, 4),
                              "source": "profiles/r02/fp64_peaks_ridge.json: a 128-bit read stream with KD DMMAs per "
                                        "4 loads, sustained; read and DMMA delivered together"}}


def _fin(x, nd):
    """round(x, nd), or None when x is not finite (strict JSON has no NaN)."""
    import math
    return round(x, nd) if isinstance(x, (int, float)) and math.isfinite(x) else None


def _graph_us(torch, f, calls=20, replays=20):
    """Device us per call with `calls` calls captured in one CUDA graph (the
    latency of a small, L2-resident product without host launch overhead)."""
    try:
        f()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            for _ in range(calls):
                f()
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(replays):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        return round(e0.elapsed_time(e1) * 1e3 / (calls * replays), 2)
    except Exception as e:  # report, do not fail the bench line
        return f"graph capture failed: {type(e).__name__}: {e}"[:200]


def _cold_us(torch, f, reps=30):
    """Device us of ONE call with a cold L2: a 256 MB scratch buffer (> the 126 MB L2)
    is written before every call; CUDA events around the call only; median."""
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=torch.cuda.current_device())
    f()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        scratch.fill_(1)
        a.record()
        f()
        b.record()
    torch.cuda.synchronize()
    del scratch
    return round(statistics.median(a.elapsed_time(b) for a, b in ev) * 1e3, 2)


def _time_call(torch, f, reps, warm=2):
    """Device ms per call: CUDA events on the current stream around `reps` calls."""
    for _ in range(warm):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def sweep(torch, device, wl, peak, parity=True):
    """Secondary measurements (not part of `value`): the metric "vs nrhs" on config 3
    (m = 1, 8, 64), the small configs 1-2 (latency-bound, L2-resident: us per call), the
    adjoint products, the ||A||_2 estimate (f2), hss2hodlr (f3) and
    general-tree / per-level-rank products (f4). Inputs drawn on the device."""
    hm = wl.hm
    out = {}

    def gbs(nbytes, ms):
        return round(nbytes / (ms * 1e-3) / 1e9, 1)

    g = torch.Generator(device=device)
    g.manual_seed(hm_inputs.MASTER_SEED + 7)
    # config 3: HODLR n = 2^20, leaf 256, 12 levels, k = 16, nrhs 1 / 8 / 64, A X and A^T X
    c3 = hm_inputs.CONFIGS[3]
    h3 = hm_inputs.device_hodlr_random(c3.n, c3.levels, [c3.k] * c3.levels, hm_inputs.MASTER_SEED + 3, device)
    if parity:
        import oracle
        oracle.set_num_threads(os.cpu_count() or 1)
        h3h = [t.cpu().numpy() for t in (h3.D, h3.U, h3.V)]
    for m in c3.nrhs:
        X = torch.randn(c3.n, m, dtype=torch.float64, device=device, generator=g)
        Y = torch.empty_like(X)
        ws = torch.empty(hm.hm_hodlr_workspace_bytes(c3.n, c3.levels, c3.leaf, h3.ranks, m), dtype=torch.uint8,
                         device=device)
        nb = hodlr_bytes(c3.n, c3.leaf, c3.levels, c3.k, m)
        fl = hodlr_flops(c3.n, c3.leaf, c3.levels, c3.k, m)
        for nm, fn in (("", hm.hodlr_matvec), ("^T", hm.hodlr_matvec_t)):
            ms = _time_call(torch, lambda: fn(c3.n, c3.levels, c3.leaf, h3.ranks, h3.D, h3.U, h3.V, X, Y, ws), 10)
            out[f"c3_m{m}{nm}"] = {"ms": round(ms, 4), "GB/s": gbs(nb, ms), "frac_hbm": round(nb / (ms * 1e-3) / 1e9 / peak, 4),
                                   "fp64_TFLOP/s": round(fl / (ms * 1e-3) / 1e12, 2),
                                   "frac_fp64": round(fl / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, 4),
                                   "matvecs/s": round(1e3 / ms, 1), "column_matvecs/s": round(m * 1e3 / ms, 1)}
            if parity:  # every row of this product vs the oracle on the same bytes
                ref = oracle.hodlr_matvec if nm == "" else oracle.hodlr_matvec_t
                Yr = ref(c3.n, c3.levels, h3.ranks, *h3h, X.cpu().numpy())
                out[f"c3_m{m}{nm}"]["parity"] = {"relerr_vs_oracle": _relerr(Y.cpu().numpy(), Yr), "rows": c3.n}
        del X, Y, ws
    # per-level ranks on the config-3 tree (f4): one V^T X pass per distinct
    # rank (tuned kernel where the rank fits it, vt_contract otherwise), one leaf pass
    for tag, m, rk in (("16/8", 8, [16 if l % 2 else 8 for l in range(c3.levels)]),
                       ("32/16", 8, [32 if l % 2 else 16 for l in range(c3.levels)]),
                       ("16/8/4/2", 1, [16 >> (l % 4) for l in range(c3.levels)])):
        hv = hm_inputs.device_hodlr_random(c3.n, c3.levels, rk, hm_inputs.MASTER_SEED + 5, device)
        X = torch.randn(c3.n, m, dtype=torch.float64, device=device, generator=g)
        Y = torch.empty_like(X)
        ws = torch.empty(hm.hm_hodlr_workspace_bytes(c3.n, c3.levels, c3.leaf, rk, m), dtype=torch.uint8,
                         device=device)
        nb = 8 * (c3.n * c3.leaf + 2 * sum(rk) * c3.n + 2 * c3.n * m)
        hm.hm_profile_collect()
        hm.hm_profile_enable(True)
        hm.hodlr_matvec(c3.n, c3.levels, c3.leaf, rk, hv.D, hv.U, hv.V, X, Y, ws)
        torch.cuda.synchronize()
        hm.hm_profile_enable(False)
        kern = sorted({t[0] for t in hm.hm_profile_collect()})
        ms = _time_call(torch, lambda: hm.hodlr_matvec(c3.n, c3.levels, c3.leaf, rk, hv.D, hv.U, hv.V, X, Y, ws), 5)
        out[f"c3_m{m}_per_level_ranks_{tag}"] = {"ms": round(ms, 4), "GB/s": gbs(nb, ms),
                                                 "frac_hbm": round(nb / (ms * 1e-3) / 1e9 / peak, 4),
                                                 "ranks": f"{tag} by level", "kernels": kern}
        del hv, X, Y, ws
    del h3
    if parity:
        del h3h
    # general cluster tree (f4) at the config-3 scale: ragged leaves of
    # 128..384 rows (config-3 mean 256), k = 16 on every level; general-tree kernels
    rng = np.random.default_rng(hm_inputs.MASTER_SEED + 9)
    nl = 1 << c3.levels
    sizes = rng.integers(128, 385, size=nl)
    c_end = np.cumsum(sizes).astype(np.int64)
    ng = int(c_end[-1])
    Dg = torch.randn(int((sizes.astype(np.int64) ** 2).sum()), dtype=torch.float64, device=device, generator=g)
    Ug = torch.randn(c3.levels * ng * c3.k, dtype=torch.float64, device=device, generator=g)
    Vg = torch.randn(c3.levels * ng * c3.k, dtype=torch.float64, device=device, generator=g)
    rk = [c3.k] * c3.levels
    for m in (1, 8):
        X = torch.randn(ng, m, dtype=torch.float64, device=device, generator=g)
        Y = torch.empty_like(X)
        ws = torch.empty(hm.hm_hodlr_general_workspace_bytes(ng, c3.levels, c_end, rk, m), dtype=torch.uint8,
                         device=device)
        nb = 8 * (int((sizes.astype(np.int64) ** 2).sum()) + 2 * c3.levels * ng * c3.k + 2 * ng * m)
        ms = _time_call(torch, lambda: hm.hodlr_matvec_general(ng, c3.levels, c_end, rk, Dg, Ug, Vg, X, 0, Y, ws), 5)
        out[f"c3_ragged_m{m}"] = {"ms": round(ms, 4), "GB/s": gbs(nb, ms),
                                  "frac_hbm": round(nb / (ms * 1e-3) / 1e9 / peak, 4),
                                  "tree": f"{nl} leaves of 128..384 rows, n = {ng}, k = {c3.k}",
                                  "path": "general-tree kernels"}
        del X, Y, ws
    del Dg, Ug, Vg
    # config 5 and 4 adjoints on the bench's own generators
    h, s4 = wl.h5, wl.s4
    ms = _time_call(torch, lambda: hm.hodlr_matvec_t(C5.n, C5.levels, C5.leaf, h.ranks, h.D, h.U, h.V, wl.X5, wl.Y5,
                                                     wl.ws5), 5)
    b5 = hodlr_bytes(C5.n, C5.leaf, C5.levels, C5.k, M5)
    out["c5^T"] = {"ms": round(ms, 4), "GB/s": gbs(b5, ms), "frac_hbm": round(b5 / (ms * 1e-3) / 1e9 / peak, 4)}
    ms = _time_call(torch, lambda: hm.hss_matvec_t(C4.n, C4.levels, C4.leaf, C4.k, s4.D, s4.U, s4.V, s4.R, s4.W, s4.B,
                                                   wl.X4, wl.Y4, wl.ws4), 5)
    b4 = hss_bytes(C4.n, C4.leaf, C4.levels, C4.k, M4)
    out["c4^T"] = {"ms": round(ms, 4), "GB/s": gbs(b4, ms), "frac_hbm": round(b4 / (ms * 1e-3) / 1e9 / peak, 4)}
    # HSS vs nrhs: config 4's generators with 1 and 8 columns (the step runs 32)
    for m in (1, 8):
        X = torch.randn(C4.n, m, dtype=torch.float64, device=device, generator=g)
        Y = torch.empty_like(X)
        ws = torch.empty(hm.hm_hss_workspace_bytes(C4.n, C4.levels, C4.leaf, C4.k, m), dtype=torch.uint8,
                         device=device)
        ms = _time_call(torch, lambda: hm.hss_matvec(C4.n, C4.levels, C4.leaf, C4.k, s4.D, s4.U, s4.V, s4.R, s4.W,
                                                     s4.B, X, Y, ws), 5)
        nb, fl = hss_bytes(C4.n, C4.leaf, C4.levels, C4.k, m), hss_flops(C4.n, C4.leaf, C4.levels, C4.k, m)
        out[f"c4_m{m}"] = {"ms": round(ms, 4), "GB/s": gbs(nb, ms), "frac_hbm": round(nb / (ms * 1e-3) / 1e9 / peak, 4),
                           "fp64_TFLOP/s": round(fl / (ms * 1e-3) / 1e12, 2), "matvecs/s": round(1e3 / ms, 1),
                           "column_matvecs/s": round(m * 1e3 / ms, 1)}
        del X, Y, ws
    # HSS with per-level and per-node ranks (f4) on a 13-level tree (n = 2^20,
    # leaf 128, nrhs 16), host-generated; every row vs the oracle
    nr, pr, br, mr = 1 << 20, 13, 128, 16
    lr = [32] * 4 + [24] * 4 + [16] * 5
    kn = np.array([16 + (7 * i + l) % 17 for l in range(1, pr + 1) for i in range(1 << l)], dtype=np.int32)
    Xr = hm_inputs.rhs(nr, mr, cid=60)
    Xd = torch.from_numpy(Xr).to(device)
    for tag, gen, wsq, call, ref in (
            ("hss_per_level_ranks", lambda: hm_inputs.hss_random_ranked(nr, pr, lr, cid=60),
             lambda: hm.hm_hss_ranked_workspace_bytes(nr, pr, br, lr, mr),
             lambda g, Y, w: hm.hss_matvec_ranked(nr, pr, br, lr, *g, Xd, Y=Y, workspace=w),
             lambda hh: __import__("oracle").hss_matvec_ranked(nr, pr, lr, hh.D, hh.U, hh.V, hh.R, hh.W, hh.B, Xr)),
            ("hss_per_node_ranks", lambda: hm_inputs.hss_random_noderanked(nr, pr, kn, cid=61),
             lambda: hm.hm_hss_noderanked_workspace_bytes(nr, pr, br, kn, mr),
             lambda g, Y, w: hm.hss_matvec_noderanked(nr, pr, br, kn, *g, Xd, Y=Y, workspace=w),
             lambda hh: __import__("oracle").hss_matvec_noderanked(nr, pr, kn, hh.D, hh.U, hh.V, hh.R, hh.W, hh.B, Xr))):
        hr = gen()
        gr = [torch.from_numpy(a).to(device) for a in (hr.D, hr.U, hr.V, hr.R, hr.W, hr.B)]
        Y = torch.empty_like(Xd)
        wr = torch.empty(wsq(), dtype=torch.uint8, device=device)  # the caller's workspace, reused
        ms = _time_call(torch, lambda: call(gr, Y, wr), 5)
        nb = 8 * (sum(a.numel() for a in gr) + 2 * nr * mr)
        out[tag] = {"ms": round(ms, 4), "GB/s": gbs(nb, ms), "frac_hbm": round(nb / (ms * 1e-3) / 1e9 / peak, 4),
                    "tree": f"n=2^20, leaf {br}, {pr} levels, nrhs {mr}",
                    "ranks": "32 x4, 24 x4, 16 x5 by level" if "level" in tag else "16..32 per node"}
        if parity:
            out[tag]["parity"] = {"relerr_vs_oracle": _relerr(Y.cpu().numpy(), ref(hr)), "rows": nr}
        del gr, Y, hr, wr
    del Xd
    # ||A||_2 of config 5 (power method on A A^*, 10 steps = 20 products)
    x0 = wl.X5[:, 0].contiguous()
    wsn = torch.empty(hm.hm_hodlr_norm2_workspace_bytes(C5.n, C5.levels, C5.leaf, h.ranks), dtype=torch.uint8,
                      device=device)
    est = torch.zeros(1, dtype=torch.float64, device=device)
    ms = _time_call(torch, lambda: hm.hodlr_norm2_est(C5.n, C5.levels, C5.leaf, h.ranks, h.D, h.U, h.V, x0, 10, est,
                                                      wsn), 2, warm=1)
    exact = 1.0 / (4.0 * np.sin(np.pi / (2 * (C5.n + 1))) ** 2)
    out["c5_norm2_est"] = {"ms": round(ms, 3), "iters": 10, "ms_per_product": round(ms / 20, 4),
                           "GB/s": gbs(20 * b5, ms), "rel_err_vs_closed_form": float(abs(est.item() - exact) / exact)}
    del wsn
    # hss2hodlr on config 4: bytes = generators read + 2 p n k doubles written
    Uh = torch.empty(C4.levels * C4.n * C4.k, dtype=torch.float64, device=device)
    Vh = torch.empty_like(Uh)
    ms = _time_call(torch, lambda: hm.hss_to_hodlr(C4.n, C4.levels, C4.leaf, C4.k, s4.U, s4.V, s4.R, s4.W, s4.B, Uh,
                                                   Vh), 3, warm=1)
    nbc = 8 * (2 * C4.n * C4.k + 2 * C4.levels * C4.n * C4.k + 4 * ((1 << C4.levels) - 2) * C4.k ** 2
               + 2 * ((1 << C4.levels) - 1) * C4.k ** 2)
    flc = 3 * 2 * C4.levels * C4.n * C4.k ** 2  # U S, U R, V W per row and level (upper bound: level 1 has no R/W)
    out["c4_hss2hodlr"] = {"ms": round(ms, 3), "GB/s": gbs(nbc, ms), "fp64_TFLOP/s": round(flc / (ms * 1e-3) / 1e12, 2),
                           "bytes": "U,V,R,W,B read + Uh,Vh (levels x n x k) written"}
    del Uh, Vh
    torch.cuda.empty_cache()
    # small configs: latency (us per call, L2-resident)
    c1, c2 = hm_inputs.CONFIGS[1], hm_inputs.CONFIGS[2]
    h1 = hm_inputs.device_hodlr_random(c1.n, c1.levels, [c1.k] * c1.levels, hm_inputs.MASTER_SEED + 1, device)
    X = torch.randn(c1.n, 1, dtype=torch.float64, device=device, generator=g)
    Y = torch.empty_like(X)
    ws = torch.empty(hm.hm_hodlr_workspace_bytes(c1.n, c1.levels, c1.leaf, h1.ranks, 1), dtype=torch.uint8,
                     device=device)
    ms = _time_call(torch, lambda: hm.hodlr_matvec(c1.n, c1.levels, c1.leaf, h1.ranks, h1.D, h1.U, h1.V, X, Y, ws), 200)
    out["c1_us"] = round(ms * 1e3, 2)
    out["c1_us_cold_l2"] = _cold_us(torch, lambda: hm.hodlr_matvec(c1.n, c1.levels, c1.leaf, h1.ranks, h1.D, h1.U,
                                                                  h1.V, X, Y, ws))
    out["c1_us_graph"] = _graph_us(torch, lambda: hm.hodlr_matvec(c1.n, c1.levels, c1.leaf, h1.ranks, h1.D, h1.U, h1.V,
                                                                  X, Y, ws))
    if parity:
        hm.hodlr_matvec(c1.n, c1.levels, c1.leaf, h1.ranks, h1.D, h1.U, h1.V, X, Y, ws)
        torch.cuda.synchronize()
        Yr = oracle.hodlr_matvec(c1.n, c1.levels, h1.ranks, h1.D.cpu().numpy(), h1.U.cpu().numpy(),
                                 h1.V.cpu().numpy(), X.cpu().numpy())
        out["c1"] = {"us": out["c1_us"], "parity": {"relerr_vs_oracle": _relerr(Y.cpu().numpy(), Yr), "rows": c1.n}}
    s2 = hm_inputs.device_hss_random(c2.n, c2.levels, c2.k, hm_inputs.MASTER_SEED + 2, device)
    X = torch.randn(c2.n, 16, dtype=torch.float64, device=device, generator=g)
    Y = torch.empty_like(X)
    ws = torch.empty(hm.hm_hss_workspace_bytes(c2.n, c2.levels, c2.leaf, c2.k, 16), dtype=torch.uint8, device=device)
    ms = _time_call(torch, lambda: hm.hss_matvec(c2.n, c2.levels, c2.leaf, c2.k, s2.D, s2.U, s2.V, s2.R, s2.W, s2.B, X,
                                                 Y, ws), 200)
    out["c2_us"] = round(ms * 1e3, 2)
    out["c2_us_cold_l2"] = _cold_us(torch, lambda: hm.hss_matvec(c2.n, c2.levels, c2.leaf, c2.k, s2.D, s2.U, s2.V,
                                                                s2.R, s2.W, s2.B, X, Y, ws))
    out["c2_us_graph"] = _graph_us(torch, lambda: hm.hss_matvec(c2.n, c2.levels, c2.leaf, c2.k, s2.D, s2.U, s2.V, s2.R,
                                                                s2.W, s2.B, X, Y, ws))
    if parity:
        hm.hss_matvec(c2.n, c2.levels, c2.leaf, c2.k, s2.D, s2.U, s2.V, s2.R, s2.W, s2.B, X, Y, ws)
        torch.cuda.synchronize()
        g2 = [t.cpu().numpy() for t in (s2.D, s2.U, s2.V, s2.R, s2.W, s2.B)]
        Yr = oracle.hss_matvec(c2.n, c2.levels, c2.k, *g2, X.cpu().numpy())
        out["c2"] = {"us": out["c2_us"], "parity": {"relerr_vs_oracle": _relerr(Y.cpu().numpy(), Yr), "rows": c2.n}}
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    # HM_BENCH_DIST=1: the multi-GPU workload even at N = 1 (a one-rank process
    # group), to exercise the distributed path on a single GPU
    use_dist = world > 1 or os.environ.get("HM_BENCH_DIST") == "1"
    if use_dist:
        dist.init_process_group("nccl", device_id=device)
    from paper_1909_07909_b200 import build as hm_build
    if rank == 0:
        hm_build.build()
    if world > 1:
        dist.barrier()

    if use_dist:
        wl = DistWorkload(torch, device, hm_inputs.MASTER_SEED, world, rank)
    else:
        wl = Workload(torch, device, seed=hm_inputs.MASTER_SEED)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        wl.step()
    torch.cuda.synchronize()
    wl.hm.hm_profile_collect()  # discard anything traced so far

    sampler = ClockSampler(local)
    sampler.start()
    wl.launches = 0
    wl.hm.hm_profile_enable(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        wl.step()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wl.hm.hm_profile_enable(False)
    ms = e0.elapsed_time(e1)
    if world > 1:  # max over ranks
        t = torch.tensor([ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clocks = sampler.stop()
    trace = wl.hm.hm_profile_collect()
    launches = len(trace)  # every traced record is one of libhm's kernel launches in the timed region

    # end-to-end (host X in, host Y out through the C-ABI hostio calls)
    for i in range(2):
        wl.step_e2e(i)
    torch.cuda.synchronize()
    # enough steps that the 4-lane copy/compute pipeline runs mostly in steady state
    # (the first step's copy in and the last step's copy out overlap nothing)
    e2 = int(os.environ.get("HM_E2E_STEPS", max(30, args.steps)))
    if world > 1:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    wl.e2e_begin(f0)
    for i in range(e2):
        wl.step_e2e(i)
    wl.e2e_end(torch)
    f1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = f0.elapsed_time(f1)
    if world > 1:
        t = torch.tensor([ms_e2e], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())

    # per-kernel device time from the trace: call 2j = HODLR (config 5), 2j+1 = HSS (config 4)
    per = {}
    ncall = len(wl.calls)
    for name, call, t in trace:
        key = wl.calls[call % ncall] + ":" + name
        d = per.setdefault(key, [0, 0.0])
        d[0] += 1
        d[1] += t
    step_ms = ms / args.steps
    # strong scaling: the P ranks together process ONE global C5 + C4 problem per
    # step (each rank holds n / P rows), so the job's bytes per step are
    # step_bytes() whatever P is
    total_bytes = step_bytes() * args.steps
    value = total_bytes / (ms * 1e-3) / 1e9
    peak, peak_kind = load_peaks()
    dom = per.get("c5:leaf_gemv", [1, float("nan")])
    dom_avg_ms = dom[1] / dom[0]
    dom_bytes = leaf_apply_c5_bytes(wl.rows5, C5.leaf, C5.levels, C5.k, M5)
    achieved = dom_bytes / (dom_avg_ms * 1e-3) / 1e9
    c5_ms = sum(v[1] for k_, v in per.items() if k_.startswith("c5:")) / args.steps
    c4_ms = sum(v[1] for k_, v in per.items() if k_.startswith("c4:")) / args.steps
    b5 = hodlr_bytes(C5.n, C5.leaf, C5.levels, C5.k, M5)
    b4 = hss_bytes(C4.n, C4.leaf, C4.levels, C4.k, M4)
    f4 = hss_flops(C4.n, C4.leaf, C4.levels, C4.k, M4)
    h2d, d2h = wl.h2d_d2h_bytes()  # this rank's copies; the job's = P times (equal shards)
    h2d, d2h = h2d * world, d2h * world
    out = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(step_ms, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded; config 5 closed-form inverse Laplacian, config 4 orthonormalised Gaussians)",
        "config": {
            "workload": "c5+c4: HODLR config 5 (n=2^24, leaf 256, 16 levels, k=1, nrhs=1) + HSS config 4 "
                        "(n=2^22, leaf 128, 15 levels, k=32, nrhs=32) per step",
            "step_alg_bytes": step_bytes(),
            "l2": "inputs 49 GB/step >> 126 MB L2; no flush needed",
            "seed": hm_inputs.MASTER_SEED,
            "parallelism": f"rows split by the top log2({world}) tree levels" if world > 1 else "single GPU",
        },
        "roofline": {
            "bound": "hbm",
            "kernel": "leaf_gemv_kernel<K=1> (config-5 leaf pass: D_i X_i + sum_l U_l t_l, all leaves, Y written once)",
            "achieved": _fin(achieved, 1),
            "peak": peak,
            "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured" else peak_kind,
            "unit": "GB/s",
            "frac": _fin(achieved / peak, 4),
            "traffic": committed_traffic("leaf_gemv", "c5"),
            "alg_bytes_per_launch": dom_bytes,
            "avg_launch_ms": _fin(dom_avg_ms, 4),
            "share_of_step": _fin(dom[1] / args.steps / step_ms, 4),
            # context: the kernel is 99.7% reads, so a read+write copy figure is not its ceiling
            "read_stream_peak": READ_STREAM_GBS,
            "frac_of_read_stream": _fin(achieved / READ_STREAM_GBS, 4),
            "read_stream_source": "tools/fp64_peaks.cu read-only stream, profiles/r01_next/fp64_peaks_mix.json",
        },
        # the second-largest kernel, config 4's leaf pass, is bound by the fp64
        # tensor pipe: its algorithmic flops 2 n m (b + k) per launch over its
        # average launch time, against the measured DMMA peak
        "roofline_c4_leaf": _c4_leaf_roofline(per, args.steps, wl),
        "per_config": {
            "c5_hodlr": {"ms": round(c5_ms, 4), "GB/s": round(b5 / (c5_ms * 1e-3) / 1e9, 1),
                         "frac_hbm": round(b5 / (c5_ms * 1e-3) / 1e9 / peak, 4),
                         "matvecs/s": round(1e3 / c5_ms, 1), "column_matvecs/s": round(M5 * 1e3 / c5_ms, 1)},
            "c4_hss": {"ms": round(c4_ms, 4), "GB/s": round(b4 / (c4_ms * 1e-3) / 1e9, 1),
                       "frac_hbm": round(b4 / (c4_ms * 1e-3) / 1e9 / peak, 4),
                       "fp64_TFLOP/s": round(f4 / (c4_ms * 1e-3) / 1e12, 2),
                       "frac_fp64": round(f4 / (c4_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, 4),
                       "fp64_peak": f"{FP64_PEAK_TFLOPS} TFLOP/s measured DMMA (profiles/r01_next/fp64_peaks_mix.json)",
                       "matvecs/s": round(1e3 / c4_ms, 1), "column_matvecs/s": round(M4 * 1e3 / c4_ms, 1),
                       "attainable_ms": round(hss_attainable_ms(C4.n, C4.leaf, C4.levels, C4.k, M4, peak), 4),
                       "frac_attainable": round(hss_attainable_ms(C4.n, C4.leaf, C4.levels, C4.k, M4, peak) / c4_ms, 4),
                       "attainable_note": "leaf pass at the measured read+DMMA ridge, Step 1 at the read stream, "
                                          "tree levels at the copy figure (DESIGN.md §11)"},
        },
        "kernels": {k_: {"launches_per_step": v[0] // args.steps, "ms_per_step": round(v[1] / args.steps, 4)}
                    for k_, v in sorted(per.items())},
        "e2e": {"value": round(step_bytes() * e2 / (ms_e2e * 1e-3) / 1e9, 2), "unit": "GB/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "note": "hodlr_matvec_hostio + hss_matvec_hostio: pinned host X in, host Y out, every step; "
                        f"consecutive steps rotate over {len(getattr(wl, "lanes", [0]))} streams so copies overlap kernels; "
                        f"{e2} steps timed; PCIe bound (pinned, both directions at once, measured 45.6 GB/s "
                        "each way) ~1.87 TB/s",
                "steps": e2},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if not use_dist and not args.no_parity:
        # every row of the timed step's Y vs the oracle on the same inputs (copied to
        # the host); the same oracle runs, timed, are the cpu_baseline
        par, cpu = parity_and_cpu(torch, wl, args.no_cpu_baseline)
        out["parity"] = par
        if cpu is not None:
            out["cpu_baseline"] = cpu
    if not use_dist and not args.no_sweep:
        out["sweep"] = sweep(torch, device, wl, peak, parity=not args.no_parity)
        if "parity" in out:  # configs 1-3 (sweep) beside 4-5 (the step): all five configs
            out["parity"].update({k_: v["parity"] for k_, v in out["sweep"].items()
                                  if isinstance(v, dict) and "parity" in v})
            out["parity"]["all_within_tol"] = all(
                v.get("relerr_vs_oracle", 0.0) <= out["parity"]["tol"] for v in out["parity"].values()
                if isinstance(v, dict))
    if use_dist:
        out["per_config"]["note"] = "per-rank device time (rank 0's launch trace)"
        out["roofline"]["kernel"] += f" — rank 0's shard (1/{world} of the rows)"
        out["parity"] = {"note": "the distributed product's parity is checked by tests/test_dist_*.py "
                                 "(emulated ranks vs the oracle, P = 1 NCCL vs the single-GPU product)"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if use_dist:
        wl.close()
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------ CPU oracle --
#
# The oracle (oracle/, plain C, the method written out from the paper) is the
# reported CPU baseline and the --impl reference arm. It is run
# as it stands; only its OpenMP thread count is chosen (results are bitwise
# independent of it).

def host_info():
    model, mem = "?", None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                mem = round(int(line.split()[1]) / 1024 / 1024, 1)
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "host_ram_gib": mem}


def _relerr(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _tridiag_residual(Y, X):
    TY = 2 * Y
    TY[1:] -= Y[:-1]
    TY[:-1] -= Y[1:]
    normT = 2 + 2 * np.cos(np.pi / (Y.shape[0] + 1))
    return float(np.linalg.norm(TY - X) / (normT * np.linalg.norm(Y) + np.linalg.norm(X)))


def parity_and_cpu(torch, wl, no_cpu=False, reps=3):
    """Every row of the timed step's outputs (configs 5 and 4, full size) against the
    oracle on the same input bytes, copied to the host; the oracle runs are timed
    (all host cores, median of `reps`) and reported as cpu_baseline."""
    import oracle
    oracle.build()
    h, s4 = wl.h5, wl.s4
    wl.step()
    torch.cuda.synchronize()
    host = lambda t: t.cpu().numpy()  # noqa: E731
    X5, Y5, X4, Y4 = host(wl.X5), host(wl.Y5), host(wl.X4), host(wl.Y4)
    D5, U5, V5 = host(h.D), host(h.U), host(h.V)
    g4 = {a: host(getattr(s4, a)) for a in ("D", "U", "V", "R", "W", "B")}
    oracle.set_num_threads(os.cpu_count() or 1)
    cores = oracle.num_threads()
    t5, t4 = [], []
    for _ in range(1 if no_cpu else reps):
        t0 = time.perf_counter()
        Yr5 = oracle.hodlr_matvec(C5.n, C5.levels, h.ranks, D5, U5, V5, X5)
        t5.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        Yr4 = oracle.hss_matvec(C4.n, C4.levels, C4.k, g4["D"], g4["U"], g4["V"], g4["R"], g4["W"], g4["B"], X4)
        t4.append(time.perf_counter() - t0)
    tol = 1e-12
    par = {"tol": tol, "metric": "||Y_gpu - Y_oracle||_F / ||Y_oracle||_F over every row (north_star)",
           "c5": {"relerr_vs_oracle": _relerr(Y5, Yr5),
                  "relerr_vs_closed_form": _relerr(Y5, oracle.laplacian_inverse_apply(X5)),
                  "tridiag_residual": _tridiag_residual(Y5, X5), "rows": C5.n},
           "c4": {"relerr_vs_oracle": _relerr(Y4, Yr4), "rows": C4.n, "nrhs": M4}}
    par["all_within_tol"] = par["c5"]["relerr_vs_oracle"] <= tol and par["c4"]["relerr_vs_oracle"] <= tol
    del D5, U5, V5, g4
    if no_cpu:
        return par, None
    m5, m4 = statistics.median(t5), statistics.median(t4)
    cpu = {"value": round(step_bytes() / (m5 + m4) / 1e9, 3), "unit": "GB/s", "cores": cores, "kind": "oracle",
           "sample": "the full timed workload (config 5 n=2^24 + config 4 n=2^22, nrhs 32) on the same input bytes "
                     f"as the GPU step, median of {reps}",
           "per_config_s": {"c5": round(m5, 3), "c4": round(m4, 3)}, **host_info()}
    table = os.path.join(ROOT, "profiles", "r02_cpu_table.json")
    if os.path.exists(table):
        cpu["per_config_table"] = "profiles/r02_cpu_table.json (bench.py --cpu-table: every config, 1 thread and " \
                                  "all cores, median of 3, full sizes)"
    return par, cpu


def host_workload():
    """The step's inputs generated on the host (hm_inputs), full size: config 5 from the
    closed form, config 4 orthonormalised Gaussians; X iid N(0,1)."""
    h = hm_inputs.hodlr_inverse_laplacian(C5.n, C5.levels)
    X5 = hm_inputs.rhs(C5.n, M5, cid=5)
    s = hm_inputs.hss_random(C4.n, C4.levels, C4.k, cid=4)
    X4 = hm_inputs.rhs(C4.n, M4, cid=4)
    return h, X5, s, X4


def run_reference(args):
    """The reference arm: the oracle on the host cores, the SAME workload as ours (one
    step = config 5 + config 4 at full size), all host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    oracle.build()
    oracle.set_num_threads(os.cpu_count() or 1)
    t_gen = time.perf_counter()
    h, X5, s, X4 = host_workload()
    t_gen = time.perf_counter() - t_gen

    def run():
        oracle.hodlr_matvec(C5.n, C5.levels, h.ranks, h.D, h.U, h.V, X5)
        oracle.hss_matvec(C4.n, C4.levels, C4.k, s.D, s.U, s.V, s.R, s.W, s.B, X4)

    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    el = sum(times)
    value = step_bytes() * args.steps / el / 1e9
    cores = oracle.num_threads()
    desc = ("oracle (oracle/hm_oracle.c) on the full step: HODLR config 5 (n=2^24, leaf 256, 16 levels, k=1, "
            "nrhs=1) + HSS config 4 (n=2^22, leaf 128, 15 levels, k=32, nrhs=32), host-generated inputs")
    out = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GB/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(el / args.steps * 1e3, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded; config 5 closed-form inverse Laplacian, config 4 orthonormalised Gaussians)",
        "config": {"workload": "c5+c4: HODLR config 5 (n=2^24, leaf 256, 16 levels, k=1, nrhs=1) + HSS config 4 "
                               "(n=2^22, leaf 128, 15 levels, k=32, nrhs=32) per step",
                   "step_alg_bytes": step_bytes(), "same_config": True,
                   "input_generation_s": round(t_gen, 1)},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "sample": desc + f"; {args.steps} steps, median step {statistics.median(times):.2f} s",
                         **host_info()},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def cpu_table(path, reps=3):
    """the oracle per config at full size, 1 thread and all host cores,
    median of `reps` (input generation excluded), with the host's CPU model and core count."""
    import oracle
    oracle.build()
    allc = os.cpu_count() or 1
    rows = []

    def timed(f, threads):
        oracle.set_num_threads(threads)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            f()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts)

    def add(cfg, nrhs, nbytes, flops, f):
        row = {"config": cfg, "nrhs": nrhs, "alg_bytes": nbytes, "gflop": round(flops / 1e9, 3)}
        for th in (1, allc):
            t = timed(f, th)
            row[f"s_{th}thr"] = float(f"{t:.4g}")
            row[f"GB/s_{th}thr"] = round(nbytes / t / 1e9, 3)
        rows.append(row)
        print(json.dumps(row), flush=True)

    c = hm_inputs.CONFIGS
    for cid in (1, 3):
        cfg = c[cid]
        h = hm_inputs.hodlr_random(cfg.n, cfg.levels, [cfg.k] * cfg.levels, cid=cid)
        for m in cfg.nrhs:
            X = hm_inputs.rhs(cfg.n, m, cid=cid)
            add(f"C{cid}", m, hodlr_bytes(cfg.n, cfg.leaf, cfg.levels, cfg.k, m),
                hodlr_flops(cfg.n, cfg.leaf, cfg.levels, cfg.k, m),
                lambda: oracle.hodlr_matvec(cfg.n, cfg.levels, h.ranks, h.D, h.U, h.V, X))
        del h
    for cid in (2, 4):
        cfg = c[cid]
        sh = hm_inputs.hss_random(cfg.n, cfg.levels, cfg.k, cid=cid)
        for m in cfg.nrhs:
            X = hm_inputs.rhs(cfg.n, m, cid=cid)
            add(f"C{cid}", m, hss_bytes(cfg.n, cfg.leaf, cfg.levels, cfg.k, m),
                hss_flops(cfg.n, cfg.leaf, cfg.levels, cfg.k, m),
                lambda: oracle.hss_matvec(cfg.n, cfg.levels, cfg.k, sh.D, sh.U, sh.V, sh.R, sh.W, sh.B, X))
        del sh
    cfg = c[5]
    h = hm_inputs.hodlr_inverse_laplacian(cfg.n, cfg.levels)
    X = hm_inputs.rhs(cfg.n, 1, cid=5)
    add("C5", 1, hodlr_bytes(cfg.n, cfg.leaf, cfg.levels, cfg.k, 1), hodlr_flops(cfg.n, cfg.leaf, cfg.levels, cfg.k, 1),
        lambda: oracle.hodlr_matvec(cfg.n, cfg.levels, h.ranks, h.D, h.U, h.V, X))
    out = {"what": "oracle/hm_oracle.c timed per BASELINE.json config at full size (BASELINE.md §4)",
           "reps": reps, "statistic": "median", "threads": [1, allc], "rows": rows,
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), **host_info()}
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({"written": path}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the secondary nrhs / ops sweep")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle comparison of the timed outputs")
    ap.add_argument("--cpu-table", metavar="PATH", help="time the oracle per config (BASELINE.md §4: 1 thread and "
                    "all cores, median of 3, full sizes) and write the JSON table to PATH; no GPU work")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.cpu_table:
        cpu_table(args.cpu_table)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
