"""One abs-GEMM bound call at a Qwen3-8B shape (for ncu captures of k_absgemm_tc*).

    python tools/tc_probe.py [M K N] [reps]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_16028_b200.bounds import FpModel, abs_gemm_bound  # noqa: E402

M, K, N = (int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (2048, 4096, 12288)
reps = int(sys.argv[4]) if len(sys.argv) >= 5 else 3
A = torch.randn((M, K), device="cuda")
B = torch.randn((K, N), device="cuda")
c = FpModel().reduction_const(2 * K - 1)
for _ in range(reps):
    abs_gemm_bound(A, B, c, False, eps_f64=False, path=1, cache_b=True)
torch.cuda.synchronize()
print("ok")
