"""Probe: the FP16 abs-GEMM (path 2, FP32 eps) on the four Qwen3-8B projection
shapes of one layer, with and without the linear u|y| term; prints per-shape
ms / TFLOP/s and the per-layer sum.  python tools/gemm_layer_probe.py"""
import sys, json, torch
sys.path.insert(0, '.')
from paper_2510_16028_b200.bounds import abs_gemm_bound, FpModel
def timeit(fn, reps=20, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
m = FpModel()
for withy in (False, True):
    tot = 0.0
    for (M, K, N, w) in ((2048, 4096, 4096, 2), (2048, 4096, 1024, 2), (2048, 4096, 12288, 2), (2048, 12288, 4096, 1)):
        A = torch.randn((M, K), device='cuda'); B = torch.randn((K, N), device='cuda')
        Y = A @ B if withy else None
        c = m.reduction_const(2 * K - 1)
        ms = timeit(lambda: abs_gemm_bound(A, B, c, False, y=Y, u=2.0 ** -24, eps_f64=False, path=2, cache_b=True))
        tot += w * ms
        print(json.dumps({"y": withy, "M": M, "K": K, "N": N, "ms": round(ms, 4), "tflops": round(2 * M * N * K / ms / 1e9, 1)}))
    print(json.dumps({"y": withy, "layer_ms": round(tot, 4)}))
