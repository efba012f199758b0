"""cuBLAS DGEMM 8192^3 (torch.matmul float64) burst (best of 10) and sustained (4 s) — fp64 library peak."""
import json, time, torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
best = 1e30
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c = a @ b; e1.record(); e1.synchronize()
    best = min(best, e0.elapsed_time(e1))
t0 = time.time(); cnt = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    c = a @ b; cnt += 1
    if cnt % 8 == 0: torch.cuda.synchronize()
e1.record(); e1.synchronize()
sus = e0.elapsed_time(e1) / cnt
fl = 2.0 * n ** 3
print(json.dumps({"dgemm_tflops_burst": fl / best / 1e9, "dgemm_tflops_sustained": fl / sus / 1e9}))
