"""Device timeline of one rank's distributed product: does the exchange overlap
the leaf pass? (development tool, not the bench contract.)

    python tools/overlap_timeline.py [--out profiles/r02/overlap_timeline.json]
                                     [--link-delay-us 20] [--P 8] [--rank 3]

This pool's boxes hold one GPU and NCCL rejects two ranks on one device, so the
P-rank exchange is EMULATED on one GPU, with rank r's libhm calls exactly as
the one-call hodlr_matvec_dist issues them (hm_hodlr.cu):

  caller stream s : _begin (top-level partials) | _local (subtree V^T X, leaf
                    pass without the top levels) | wait | _end (combine +
                    top-level epilogue)
  exchange        : after _begin, on a second stream: an optional modelled
                    link latency (torch.cuda._sleep, --link-delay-us), then
                    the gathered buffer (the P ranks' send slots) delivered by
                    one real NCCL allgather on libhm's one-rank communicator
                    (its own stream, traced as "nccl_allgather").

Before each traced step the caller stream gets a short spin (HOST_LEAD_US), so
the host has enqueued the whole step before the device reaches it: the
timeline then shows the device-side ordering of the two streams (what the
events allow to overlap), not this Python driver's enqueue latency.

Every record comes from libhm's launch trace (hm_profile_timeline: CUDA events
on the launching stream, start times on one device timeline). The same is done
for HSS (config-4 tree), whose schedule is deliberately NOT overlapped (every
local step after Step 1 needs the exchanged block): its timeline shows the
wait.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import hm_inputs  # noqa: E402
import paper_1909_07909_b200 as hm  # noqa: E402
from paper_1909_07909_b200 import dist as hd  # noqa: E402

CLK_HZ = 1.965e9  # B200 max SM clock: cycles of the modelled link latency
HOST_LEAD_US = 400.0


def _lead(s):
    with torch.cuda.stream(s):
        torch.cuda._sleep(int(HOST_LEAD_US * 1e-6 * CLK_HZ))


def _exchange(comm, allsends, gathered, side, s, delay_us):
    """One collective call, as the one-call product issues (a one-rank allgather of
    the P ranks' concatenated send buffers delivers the same gathered bytes)."""
    side.wait_stream(s)
    with torch.cuda.stream(side):
        if delay_us > 0:
            torch.cuda._sleep(int(delay_us * 1e-6 * CLK_HZ))
        comm.allgather(allsends, recv=gathered, stream=side)


def _records(tr, phases):
    out = []
    for name, call, t0, ms in tr:
        ph = "exchange" if name == "nccl_allgather" else phases.get(call, "?")
        out.append({"name": name, "phase": ph, "start_us": round(1e3 * t0, 2), "end_us": round(1e3 * (t0 + ms), 2)})
    return out


def _overlap(recs, pred):
    ex = [r for r in recs if r["phase"] == "exchange"]
    if not ex:
        return {}
    a, b = min(r["start_us"] for r in ex), max(r["end_us"] for r in ex)
    ov = sum(max(0.0, min(b, r["end_us"]) - max(a, r["start_us"])) for r in recs if pred(r))
    return {"exchange_window_us": [a, b], "window_us": round(b - a, 2), "caller_kernel_us_inside_window": round(ov, 2)}


def hodlr(comm, P, rank, delay_us, reps):
    cfg = hm_inputs.CONFIGS[5]
    n, p, b = cfg.n, cfg.levels, cfg.leaf
    dev = torch.device("cuda:0")
    h = hm_inputs.hodlr_inverse_laplacian(n, p, xp=torch, device=dev)
    X = torch.randn(n, 1, dtype=torch.float64, device=dev)
    nl = n // P
    sends, shards = [], {}
    for r in range(P):
        Dl, Ul, Vl = hd.hodlr_shard(n, p, b, h.ranks, h.D, h.U, h.V, P, r)
        Xl = X[r * nl:(r + 1) * nl].contiguous()
        wsb, sd = hd.hodlr_dist_sizes(n, p, b, h.ranks, 1, P, r)
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        send = torch.empty(sd, dtype=torch.float64, device=dev)
        hd.hodlr_matvec_dist_begin(n, p, b, h.ranks, P, r, Vl, Xl, send, ws)
        sends.append(send)
        if r == rank:
            shards = dict(D=Dl.contiguous(), U=Ul.contiguous(), V=Vl.contiguous(), X=Xl, ws=ws)
    gathered = torch.empty(P * sd, dtype=torch.float64, device=dev)
    allsends = torch.cat(sends)  # rank r's slot is rewritten by its _begin every step
    Yl = torch.empty_like(shards["X"])
    s, side = torch.cuda.Stream(), torch.cuda.Stream()
    sh = shards

    def step():
        _lead(s)
        with torch.cuda.stream(s):
            hd.hodlr_matvec_dist_begin(n, p, b, h.ranks, P, rank, sh["V"], sh["X"], allsends[rank * sd:(rank + 1) * sd],
                                       sh["ws"], stream=s)
            _exchange(comm, allsends, gathered, side, s, delay_us)
            hd.hodlr_matvec_dist_local(n, p, b, h.ranks, P, rank, sh["D"], sh["U"], sh["V"], sh["X"], Yl, sh["ws"],
                                       stream=s)
            s.wait_stream(side)
            hd.hodlr_matvec_dist_end(n, p, b, h.ranks, P, rank, sh["D"], sh["U"], sh["X"], gathered, Yl, sh["ws"],
                                     stream=s)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    runs = []
    for _ in range(reps):
        hm.hm_profile_collect()
        hm.hm_profile_enable(True)
        step()
        torch.cuda.synchronize()
        hm.hm_profile_enable(False)
        recs = _records(hm.hm_profile_timeline(), {0: "begin", 1: "local", 2: "end"})
        runs.append(recs)
    # parity of the emulated rank against the single-GPU product's rows
    Y1 = hm.hodlr_matvec(n, p, b, h.ranks, h.D, h.U, h.V, X)
    torch.cuda.synchronize()
    err = float((Yl - Y1[rank * nl:(rank + 1) * nl]).norm() / Y1[rank * nl:(rank + 1) * nl].norm())
    recs = runs[-1]
    return {
        "product": "hodlr_matvec_dist schedule (overlapped: leaf pass before the exchange's result, top-level epilogue)",
        "config": f"config 5 (n = 2^24, leaf 256, 16 levels, k = 1, nrhs = 1), P = {P}, rank {rank} "
                  f"({nl} rows), exchange = {P} x {sd} doubles",
        "rel_err_vs_single_gpu_rows": err,
        "overlap": _overlap(recs, lambda r: r["phase"] == "local"),
        "timeline": recs,
    }


def hss(comm, P, rank, delay_us, reps):
    cfg = hm_inputs.CONFIGS[4]
    n, p, b, k, m = cfg.n, cfg.levels, cfg.leaf, cfg.k, cfg.nrhs[0]
    dev = torch.device("cuda:0")
    g = hm_inputs.device_hss_random(n, p, k, 7, dev)
    X = torch.randn(n, m, dtype=torch.float64, device=dev)
    nl = n // P
    sends, mine = [], None
    for r in range(P):
        shd = {kk: v.contiguous() for kk, v in hd.hss_shard(n, p, b, k, g.D, g.U, g.V, g.R, g.W, g.B, P, r).items()}
        Xl = X[r * nl:(r + 1) * nl].contiguous()
        wsb, sd = hd.hss_dist_sizes(n, p, b, k, m, P, r)
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        send = torch.empty(sd, dtype=torch.float64, device=dev)
        hd.hss_matvec_dist_begin(n, p, b, k, P, r, shd, Xl, send, ws)
        sends.append(send)
        if r == rank:
            mine = (shd, Xl, ws)
        else:
            del shd
    shd, Xl, ws = mine
    gathered = torch.empty(P * sd, dtype=torch.float64, device=dev)
    allsends = torch.cat(sends)
    Yl = torch.empty_like(Xl)
    s, side = torch.cuda.Stream(), torch.cuda.Stream()

    def step():
        _lead(s)
        with torch.cuda.stream(s):
            hd.hss_matvec_dist_begin(n, p, b, k, P, rank, shd, Xl, allsends[rank * sd:(rank + 1) * sd], ws, stream=s)
            _exchange(comm, allsends, gathered, side, s, delay_us)
            s.wait_stream(side)
            hd.hss_matvec_dist_end(n, p, b, k, P, rank, shd, Xl, gathered, Yl, ws, stream=s)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    for _ in range(reps):
        hm.hm_profile_collect()
        hm.hm_profile_enable(True)
        step()
        torch.cuda.synchronize()
        hm.hm_profile_enable(False)
        recs = _records(hm.hm_profile_timeline(), {0: "begin", 1: "end"})
    Y1 = hm.hss_matvec(n, p, b, k, g.D, g.U, g.V, g.R, g.W, g.B, X)
    torch.cuda.synchronize()
    ref = Y1[rank * nl:(rank + 1) * nl]
    err = float((Yl - ref).norm() / ref.norm())
    return {
        "product": "hss_matvec_dist schedule (not overlapped: every local step after Step 1 needs the exchanged block)",
        "config": f"config 4 (n = 2^22, leaf 128, 15 levels, k = 32, nrhs = 32), P = {P}, rank {rank}, "
                  f"exchange = {P} x {sd} doubles",
        "rel_err_vs_single_gpu_rows": err,
        "overlap": _overlap(recs, lambda r: r["phase"] != "exchange"),
        "timeline": recs,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "overlap_timeline.json"))
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--rank", type=int, default=3)
    ap.add_argument("--link-delay-us", type=float, default=20.0)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    hm.load()
    comm = hd.Comm(1, 0, hd.unique_id())
    try:
        res = {
            "what": "one rank of a P-rank distributed product on one GPU; exchange emulated by P one-rank NCCL "
                    "allgathers on libhm's communicator stream after a modelled link latency (tools/overlap_timeline.py)",
            "link_delay_us": a.link_delay_us,
            "hodlr": hodlr(comm, a.P, a.rank, a.link_delay_us, a.reps),
            "hss": hss(comm, a.P, a.rank, a.link_delay_us, a.reps),
        }
    finally:
        comm.close()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    for key in ("hodlr", "hss"):
        r = res[key]
        print(key, r["overlap"], "err", r["rel_err_vs_single_gpu_rows"])
        for t in r["timeline"]:
            print(f"  {t['phase']:9s} {t['name']:40s} {t['start_us']:10.2f} {t['end_us']:10.2f}")


if __name__ == "__main__":
    main()
