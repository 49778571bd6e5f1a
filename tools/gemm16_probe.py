"""Launch one f16 abs-GEMM bound per Qwen shape (for an ncu launch list)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_16028_b200.bounds import FpModel, abs_gemm_bound  # noqa: E402

dev = torch.device("cuda")
torch.manual_seed(0)
S, NH = 2048, 32
c = FpModel().reduction_const(255)
q = torch.randn((NH, S, 128), device=dev)
k = torch.randn((NH, S, 128), device=dev)
p = torch.softmax(torch.randn((NH, S, S), device=dev) * 3, -1)
v = torch.randn((NH, S, 128), device=dev)
x = torch.randn((S, 4096), device=dev)
w = torch.randn((4096, 4096), device=dev)
for path in (1, 2):
    for _ in range(2):
        abs_gemm_bound(q, k, c, True, eps_f64=False, path=path)
        abs_gemm_bound(p, v, c, False, eps_f64=False, path=path)
        abs_gemm_bound(x, w, c, False, eps_f64=False, path=path, cache_b=True)
torch.cuda.synchronize()
print("ok")
