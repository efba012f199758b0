import sys, numpy as np, torch
sys.path.insert(0, '.')
import hm_inputs, oracle, paper_1909_07909_b200 as hm
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
def run(n, b, p, k, m, only=None, zeroD=False):
    h = hm_inputs.hodlr_random(n, p, [k]*p, cid=11)
    if zeroD: h.D[:] = 0
    if only is not None:
        for l in range(1, p+1):
            if l != only: h.U[h.level_slice(l)] = 0
    X = hm_inputs.rhs(n, m, cid=11)
    Y = hm.hodlr_matvec(n, p, b, h.ranks, dev(h.D), dev(h.U), dev(h.V), dev(X)).cpu().numpy()
    Yr = oracle.hodlr_matvec(n, p, h.ranks, h.D, h.U, h.V, X)
    e = np.linalg.norm(Y-Yr)/np.linalg.norm(Yr)
    colerr = [float(np.linalg.norm(Y[:,c]-Yr[:,c])/np.linalg.norm(Yr[:,c])) for c in range(m)]
    print(n,b,p,k,m,'only',only,'zeroD',zeroD,'err %.2e'%e, 'bad cols', [c for c in range(m) if colerr[c]>1e-12])
for m in (1, 8, 15, 16, 17, 32):
    run(512, 64, 3, 5, m)
run(512,64,3,5,17,zeroD=True)
for l in (1,2,3): run(512,64,3,5,17,only=l,zeroD=True)
run(64,64,0,0,17)
run(512,64,3,0,17)
