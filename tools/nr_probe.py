"""Probe: per-node-rank HSS call, kernel times vs wall time (development tool)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import hm_inputs  # noqa: E402
import paper_1909_07909_b200 as hm  # noqa: E402

nr, pr, br, mr = 1 << 20, 13, 128, 16
kn = [16 + (7 * i + l) % 17 for l in range(1, pr + 1) for i in range(1 << l)]
h = hm_inputs.hss_random_noderanked(nr, pr, kn, cid=61)
g = [torch.from_numpy(a).cuda() for a in (h.D, h.U, h.V, h.R, h.W, h.B)]
X = torch.randn(nr, mr, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
ws = torch.empty(hm.hm_hss_noderanked_workspace_bytes(nr, pr, br, kn, mr), dtype=torch.uint8, device="cuda")
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
