import sys, torch
sys.path.insert(0, '.')
import hm_inputs, paper_1909_07909_b200 as hm
c = hm_inputs.CONFIGS[4]
s = hm_inputs.device_hss_random(c.n, c.levels, c.k, 4, torch.device('cuda:0'))
Uh = torch.empty(c.levels * c.n * c.k, dtype=torch.float64, device='cuda'); Vh = torch.empty_like(Uh)
for _ in range(2): hm.hss_to_hodlr(c.n, c.levels, c.leaf, c.k, s.U, s.V, s.R, s.W, s.B, Uh, Vh)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(3): hm.hss_to_hodlr(c.n, c.levels, c.leaf, c.k, s.U, s.V, s.R, s.W, s.B, Uh, Vh)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
nb = 8 * (2 * c.n * c.k + 2 * c.levels * c.n * c.k)
print(f"hss2hodlr c4: {ms:.3f} ms  {nb/ms/1e6:.0f} GB/s  {387e9/ms/1e9:.1f} TFLOP/s-ish")
