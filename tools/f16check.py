import numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
from paper_2510_16028_b200 import bounds as B
from oracle import bounds as OB
rng = np.random.default_rng(0)
for (M, K, N, tb) in [(128,128,128,False),(129,300,131,False),(300,17,1000,True),(256,4096,256,False),(2048,128,640,True),(64,12288,96,False),(7,33,5,True)]:
    a = rng.standard_normal((M, K)).astype(np.float32)
    b = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    ref = OB.matmul_bound(a, b, OB.FpModel(), transpose_b=tb)
    c = OB.FpModel().reduction_const(2*K-1)
    for f64 in (True, False):
        got = B.abs_gemm_bound(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), c, tb, eps_f64=f64, path=2).cpu().numpy().astype(np.float64)
        r = got / ref - 1
        print((M,K,N,tb,f64), "min", r.min(), "max", r.max(), "below", int((got < ref).sum()))
# subnormal-half probe: tiny entries
a = np.ones((128, 64), np.float32); a[:, 1:] = 2.0**-30  # scaled: max->2^14, tiny 2^-16 -> subnormal hi
b = np.ones((64, 128), np.float32); b[0, :] = 0.0
ref = OB.matmul_bound(a, b, OB.FpModel())
got = B.abs_gemm_bound(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), 1.0, path=2).cpu().numpy()
print("subnormal probe ratio", (got/ref).min(), (got/ref).max())
