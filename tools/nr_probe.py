"""Probe: per-node-rank HSS call, kernel times vs wall time (development tool)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import hm_inputs  # noqa: E402
import paper_1909_07909_b200 as hm  # noqa: E402

nr, pr, br, mr = 1 << 20, 13, 128, 16
kn = np.array([16 + (7 * i + l) % 17 for l in range(1, pr + 1) for i in range(1 << l)], dtype=np.int32)
h = hm_inputs.hss_random_noderanked(nr, pr, kn, cid=61)
g = [torch.from_numpy(a).cuda() for a in (h.D, h.U, h.V, h.R, h.W, h.B)]
X = torch.randn(nr, mr, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
ws = torch.empty(hm.hm_hss_noderanked_workspace_bytes(nr, pr, br, kn, mr), dtype=torch.uint8, device="cuda")
if "--bench-state" in sys.argv:  # the bench's process state: big pinned host buffers, small tables in the ring
    pin = [torch.empty(1 << 27, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    big = torch.empty(40 << 30, dtype=torch.uint8, device="cuda")
    import numpy as np
    c = np.cumsum(np.full(1 << 10, 300, dtype=np.int64))
    n2 = int(c[-1])
    Dg = torch.randn(int((300 ** 2) * (1 << 10)), dtype=torch.float64, device="cuda")
    Ug = torch.randn(10 * n2 * 16, dtype=torch.float64, device="cuda")
    Xg = torch.randn(n2, 8, dtype=torch.float64, device="cuda")
    for _ in range(4):
        hm.hodlr_matvec_general(n2, 10, c, [16] * 10, Dg, Ug, Ug, Xg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for it in range(8):
        t0 = time.perf_counter()
        e0.record()
        hm.hss_matvec_noderanked(nr, pr, br, kn, *g, X, Y=Y, workspace=ws)
        e1.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        print(f"  call {it}: host {1e3 * (t1 - t0):8.2f} ms, device {e0.elapsed_time(e1):8.2f} ms")
for _ in range(3):
    hm.hss_matvec_noderanked(nr, pr, br, kn, *g, X, Y=Y, workspace=ws)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    hm.hss_matvec_noderanked(nr, pr, br, kn, *g, X, Y=Y, workspace=ws)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e3*(t1-t0)/5:.2f} ms/call, wall {1e3*(t2-t0)/5:.2f} ms/call, ws {ws.numel()/1e6:.0f} MB")
hm.hm_profile_collect()
hm.hm_profile_enable(True)
hm.hss_matvec_noderanked(nr, pr, br, kn, *g, X, Y=Y, workspace=ws)
torch.cuda.synchronize()
hm.hm_profile_enable(False)
for name, call, ms in hm.hm_profile_collect():
    print(f"  {name:<24} {ms*1e3:9.1f} us")
