"""One abs-GEMM bound call at a Qwen3-8B shape (for ncu captures of k_absgemm_tc*).

    python tools/tc_probe.py M K N [reps]      plain A[M,K] @ B[K,N]
    python tools/tc_probe.py scores [reps]     32 heads of q[2048,128] @ k[2048,128]^T
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_16028_b200.bounds import FpModel, abs_gemm_bound  # noqa: E402

args = sys.argv[1:]
if args and args[0] == "scores":
    A = torch.randn((32, 2048, 128), device="cuda")
    B = torch.randn((32, 2048, 128), device="cuda")
    tb, K = True, 128
    reps = int(args[1]) if len(args) > 1 else 3
else:
    M, K, N = (int(v) for v in args[:3]) if len(args) >= 3 else (2048, 4096, 12288)
    reps = int(args[3]) if len(args) >= 4 else 3
    A = torch.randn((M, K), device="cuda")
    B = torch.randn((K, N), device="cuda")
    tb = False
c = FpModel().reduction_const(2 * K - 1)
for _ in range(reps):
    abs_gemm_bound(A, B, c, tb, eps_f64=False, path=1, cache_b=not tb)
torch.cuda.synchronize()
print("ok")
