"""Per-kernel timing of single configs (development tool, not the bench contract).

    python tools/kbench.py c5 c4 c3m1 c3m8 c3m64 c2 c1 c4m1 c4m8 hs:20:14:32:1 [--reps N]

A trailing "t" (c5t, c4t, c3m8t, ...) times the adjoint product A^T X instead.

Inputs drawn on the device; prints per-kernel device ms (launch trace of
libhm) and the config's algorithmic GB/s.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import hm_inputs  # noqa: E402
import paper_1909_07909_b200 as hm  # noqa: E402
from bench import hodlr_bytes, hss_bytes, hss_flops, hodlr_flops  # noqa: E402


def run(name, reps):
    dev = torch.device("cuda:0")
    adj = name.endswith("t")
    if adj:
        name = name[:-1]
    if name.startswith("cr"):  # ragged config-3-scale tree (general-tree kernels), e.g. cr1, cr8
        import numpy as np
        cfg = hm_inputs.CONFIGS[3]
        m = int(name[2:])
        rng = np.random.default_rng(9)
        sizes = rng.integers(128, 385, size=1 << cfg.levels)
        c = np.cumsum(sizes).astype(np.int64)
        n = int(c[-1])
        D = torch.randn(int((sizes.astype(np.int64) ** 2).sum()), dtype=torch.float64, device=dev)
        U = torch.randn(cfg.levels * n * cfg.k, dtype=torch.float64, device=dev)
        V = torch.randn(cfg.levels * n * cfg.k, dtype=torch.float64, device=dev)
        X = torch.randn(n, m, dtype=torch.float64, device=dev)
        Y = torch.empty_like(X)
        rk = [cfg.k] * cfg.levels
        ws = torch.empty(hm.hm_hodlr_general_workspace_bytes(n, cfg.levels, c, rk, m), dtype=torch.uint8, device=dev)
        f = lambda: hm.hodlr_matvec_general(n, cfg.levels, c, rk, D, U, V, X, 1 if adj else 0, Y, ws)
        nbytes = 8 * (D.numel() + U.numel() + V.numel() + 2 * n * m)
        flops = 2 * m * (D.numel() + U.numel() + V.numel())
    elif name.split(":")[0] in ("hpl", "hpn"):  # HSS with per-level / per-node ranks (the bench sweep's trees); hpl:1 = nrhs 1
        import numpy as np
        nr, pr, br, m = 1 << 20, 13, 128, 16
        if ":" in name:
            name, m = name.split(":")[0], int(name.split(":")[1])
        if name == "hpl":
            lr = [32] * 4 + [24] * 4 + [16] * 5
            hr = hm_inputs.hss_random_ranked(nr, pr, lr, cid=60)
            wsb = hm.hm_hss_ranked_workspace_bytes(nr, pr, br, lr, m)
        else:
            lr = np.array([16 + (7 * i + l) % 17 for l in range(1, pr + 1) for i in range(1 << l)], dtype=np.int32)
            hr = hm_inputs.hss_random_noderanked(nr, pr, lr, cid=61)
            wsb = hm.hm_hss_noderanked_workspace_bytes(nr, pr, br, lr, m)
        g = [torch.from_numpy(a).to(dev) for a in (hr.D, hr.U, hr.V, hr.R, hr.W, hr.B)]
        X = torch.randn(nr, m, dtype=torch.float64, device=dev)
        Y = torch.empty_like(X)
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        mv = hm.hss_matvec_ranked if name == "hpl" else hm.hss_matvec_noderanked
        f = lambda: mv(nr, pr, br, lr, *g, X, Y=Y, workspace=ws)
        nbytes = 8 * (sum(a.numel() for a in g) + 2 * nr * m)
        flops = 2 * m * sum(a.numel() for a in g)
    elif name.startswith("c3") or name in ("c5", "c1"):
        cfg = hm_inputs.CONFIGS[{"c1": 1, "c5": 5}.get(name, 3)]
        m = int(name[3:]) if name.startswith("c3m") else 1
        if cfg.laplacian:
            h = hm_inputs.hodlr_inverse_laplacian(cfg.n, cfg.levels, xp=torch, device=dev)
        else:
            h = hm_inputs.device_hodlr_random(cfg.n, cfg.levels, [cfg.k] * cfg.levels, 7, dev)
        X = torch.randn(cfg.n, m, dtype=torch.float64, device=dev)
        Y = torch.empty_like(X)
        ws = torch.empty(hm.hm_hodlr_workspace_bytes(cfg.n, cfg.levels, cfg.leaf, h.ranks, m), dtype=torch.uint8,
                         device=dev)
        mv = hm.hodlr_matvec_t if adj else hm.hodlr_matvec
        f = lambda: mv(cfg.n, cfg.levels, cfg.leaf, h.ranks, h.D, h.U, h.V, X, Y, ws)
        nbytes = hodlr_bytes(cfg.n, cfg.leaf, cfg.levels, cfg.k, m)
        flops = hodlr_flops(cfg.n, cfg.leaf, cfg.levels, cfg.k, m)
    elif name.startswith("hs:"):  # hs:<log2 n>:<levels>:<k>:<nrhs> — any uniform HSS tree (leaf = n >> levels)
        ln, p_, k_, m = (int(v) for v in name.split(":")[1:])
        n_, b_ = 1 << ln, (1 << ln) >> p_
        s = hm_inputs.device_hss_random(n_, p_, k_, 7, dev)
        X = torch.randn(n_, m, dtype=torch.float64, device=dev)
        Y = torch.empty_like(X)
        ws = torch.empty(hm.hm_hss_workspace_bytes(n_, p_, b_, k_, m), dtype=torch.uint8, device=dev)
        mv = hm.hss_matvec_t if adj else hm.hss_matvec
        f = lambda: mv(n_, p_, b_, k_, s.D, s.U, s.V, s.R, s.W, s.B, X, Y, ws)
        nbytes = hss_bytes(n_, b_, p_, k_, m)
        flops = hss_flops(n_, b_, p_, k_, m)
    else:
        cfg = hm_inputs.CONFIGS[{"c2": 2, "c4": 4}[name[:2]]]
        m = int(name[3:]) if name[2:3] == "m" else cfg.nrhs[0]  # c4m8: config 4 with 8 columns
        s = hm_inputs.device_hss_random(cfg.n, cfg.levels, cfg.k, 7, dev)
        X = torch.randn(cfg.n, m, dtype=torch.float64, device=dev)
        Y = torch.empty_like(X)
        ws = torch.empty(hm.hm_hss_workspace_bytes(cfg.n, cfg.levels, cfg.leaf, cfg.k, m), dtype=torch.uint8,
                         device=dev)
        mv = hm.hss_matvec_t if adj else hm.hss_matvec
        f = lambda: mv(cfg.n, cfg.levels, cfg.leaf, cfg.k, s.D, s.U, s.V, s.R, s.W, s.B, X, Y, ws)
        nbytes = hss_bytes(cfg.n, cfg.leaf, cfg.levels, cfg.k, m)
        flops = hss_flops(cfg.n, cfg.leaf, cfg.levels, cfg.k, m)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    hm.hm_profile_collect()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    plain = e0.elapsed_time(e1) / reps
    hm.hm_profile_enable(True)
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    hm.hm_profile_enable(False)
    tr = hm.hm_profile_collect()
    per = {}
    for nm, call, ms in tr:
        per.setdefault(nm, []).append(ms)
    print(f"== {name}{'^T' if adj else ''}: {plain * 1e3:.1f} us/call  {nbytes / plain / 1e6:.0f} GB/s  "
          f"{flops / plain / 1e9:.2f} TFLOP/s")
    for nm, v in per.items():
        cnt = len(v) // reps
        tot = sum(v) / reps
        print(f"   {nm:<18} x{cnt:<3} {tot * 1e3:9.1f} us")
    if "--levels" in sys.argv:
        calls = [t for t in tr if t[1] == 0]
        print("   " + " ".join(f"{n[:6]}:{ms * 1e3:.1f}" for n, _, ms in calls))
    del X, Y, ws
    torch.cuda.empty_cache()


if __name__ == "__main__":
    reps = 10
    names = [a for a in sys.argv[1:] if not a.startswith("--")]
    if "--reps" in sys.argv:
        reps = int(sys.argv[sys.argv.index("--reps") + 1])
        names = [a for a in names if not a.isdigit()]
    for nm in names:
        run(nm, reps)
