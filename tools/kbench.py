"""Per-kernel microbenchmarks at Qwen3-8B shapes (CUDA events, warm L2 excluded by
using tensors >> L2).  Prints one JSON line per kernel with achieved GB/s or TFLOP/s.

    python tools/kbench.py [--only check,commit,softmax,gemm_tc,gemm_ffma,split,layernorm]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2510_16028_b200 import _lib  # noqa: E402
from paper_2510_16028_b200.bounds import (FpModel, abs_gemm_bound, layernorm_device,  # noqa: E402
                                          softmax_device, tf32_split)
from paper_2510_16028_b200.commitments import commit_tensors  # noqa: E402
from paper_2510_16028_b200.dispute import check_node  # noqa: E402
from paper_2510_16028_b200.executor import inject_drift  # noqa: E402

PEAK_HBM = json.load(open(Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json")).get(
    "hbm_gbs", 6650.0) if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else 6650.0


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def calltime(fn, reps=10, warm=3):
    """Sum of the library calls' event-timed durations (excludes Python-side
    preparation between calls, e.g. per-tensor verdict specs)."""
    from paper_2510_16028_b200 import _lib
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    store = {}
    _lib.set_timer(store, lambda n, a: 0.0, torch.cuda.current_stream())
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    _lib.set_timer(None, None, None)
    return sum(sum(v["ms"]) for v in store.values()) / reps


def report(name, ms, bytes_=None, flops=None, **kw):
    d = {"kernel": name, "ms": round(ms, 4)}
    if bytes_:
        d["GB/s"] = round(bytes_ / ms / 1e6, 1)
        d["frac_hbm"] = round(bytes_ / ms / 1e6 / PEAK_HBM, 3)
    if flops:
        d["TFLOP/s"] = round(flops / ms / 1e9, 2)
    d.update(kw)
    print(json.dumps(d), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    only = set(a.only.split(",")) if a.only else None
    want = lambda k: only is None or k in only  # noqa: E731
    dev = torch.device("cuda")
    torch.manual_seed(0)
    S, H, I, NH = 2048, 4096, 12288, 32
    model = FpModel()

    if want("check"):
        for shape in ((NH, S, S), (S, I), (S, H)):
            y = torch.randn(shape, device=dev)
            yc = inject_drift(y, 1, 16)
            eps = torch.rand(shape, device=dev)
            tau = np.linspace(1e-9, 1e-3, 23)
            n = y.numel()
            report("check_scaled", timeit(lambda: check_node(y, yc, ("scaled", 2 ** -24), tau, tau),
                                          a.reps), 8 * n, shape=list(shape))
            report("check_f32eps", timeit(lambda: check_node(y, yc, eps, tau, tau), a.reps),
                   12 * n, shape=list(shape))
    if want("commit"):
        for alg in ("keccak256", "sha256"):
            ts = [torch.randn((NH, S, S), device=dev)]
            nb = sum(t.numel() * 4 for t in ts)
            report(f"commit_{alg}", timeit(lambda: commit_tensors(ts, 4096, alg), a.reps), nb,
                   bytes_committed=nb)
            ts = [torch.randn((S, H), device=dev) for _ in range(20)]
            nb = sum(t.numel() * 4 for t in ts)
            report(f"commit_{alg}_batch20x33MB", timeit(lambda: commit_tensors(ts, 4096, alg),
                                                        a.reps), nb)
    if want("commitcheck"):
        from paper_2510_16028_b200.dispute import commit_check_nodes
        ys = [torch.randn((NH, S, S), device=dev)] + [torch.randn((S, H), device=dev)
                                                      for _ in range(8)]
        ycs = [inject_drift(y, 1, 16) if i % 2 == 0 else y.clone() for i, y in enumerate(ys)]
        nb = sum(t.numel() * 4 for t in ys)
        tau = np.linspace(1e-9, 1e-3, 23)
        eps = [("scaled", 2 ** -23)] * len(ys)
        taus = [(tau, tau)] * len(ys)
        report("commit_check_keccak", timeit(lambda: commit_check_nodes(ycs, ys, eps, taus, 4096,
                                                                         "keccak256"), a.reps), nb)
        report("commit_only_keccak", timeit(lambda: commit_tensors(ycs, 4096, "keccak256"),
                                            a.reps), nb)
        # every tensor drifting, FP32 eps tensors (GEMM / conv outputs)
        ycs2 = [inject_drift(y, 1, 16) for y in ys]
        eps2 = [(y.abs() * 2 ** -20).float() for y in ys]
        report("commit_check_keccak_alldrift_epsT",
               timeit(lambda: commit_check_nodes(ycs2, ys, eps2, taus, 4096, "keccak256"), a.reps),
               nb)
        ycs3 = [y.clone() for y in ys]
        report("commit_check_keccak_nodrift_epsT",
               timeit(lambda: commit_check_nodes(ycs3, ys, eps2, taus, 4096, "keccak256"), a.reps),
               nb)
        # many small tensors (UNet-like: 1M-element node outputs)
        sm = [torch.randn(1 << 20, device=dev) for _ in range(256)]
        smc = [inject_drift(y, 1, 16) for y in sm]
        report("commit_check_keccak_256x4MB",
               timeit(lambda: commit_check_nodes(smc, sm, [("scaled", 2 ** -23)] * 256,
                                                 [(tau, tau)] * 256, 4096, "keccak256"), a.reps),
               256 * 4 << 20)
        report("commit_check_keccak_256x4MB_calls",
               calltime(lambda: commit_check_nodes(smc, sm, [("scaled", 2 ** -23)] * 256,
                                                   [(tau, tau)] * 256, 4096, "keccak256"), a.reps),
               256 * 4 << 20)
        report("commit_only_keccak_256x4MB", timeit(lambda: commit_tensors(smc, 4096, "keccak256"),
                                                    a.reps), 256 * 4 << 20)
        inf = np.full(23, np.inf)
        report("commit_check_keccak_256x4MB_inf_tau",
               timeit(lambda: commit_check_nodes(smc, sm, [("scaled", 2 ** -23)] * 256,
                                                 [(inf, inf)] * 256, 4096, "keccak256"), a.reps),
               256 * 4 << 20)
        big = [torch.cat(sm)]
        bigc = [torch.cat(smc)]
        report("commit_check_keccak_1x1GB",
               timeit(lambda: commit_check_nodes(bigc, big, [("scaled", 2 ** -23)],
                                                 [(tau, tau)], 4096, "keccak256"), a.reps),
               256 * 4 << 20)
    if want("softmax"):
        x = torch.randn((NH, S, S), device=dev) * 3
        n = x.numel()
        report("softmax_bound_f32eps", timeit(lambda: softmax_device(x, -1, model, False), a.reps),
               12 * n)
    if want("reduce"):
        from paper_2510_16028_b200.bounds import reduce_device
        for shape in ((S, H), (S * NH, 128), (S * 8, 128)):
            x = torch.randn(shape, device=dev)
            report("mean_bound_f64eps", timeit(lambda: reduce_device("mean", x, -1, model, True),
                                               a.reps), 4 * x.numel() + 8 * shape[0],
                   shape=list(shape))
    if want("unary"):  # the SiLU of the MLP gate (2048 x 12288)
        from paper_2510_16028_b200.engine import unary
        x = torch.randn((S, I), device=dev)
        report("unary_silu_fp64", timeit(lambda: unary("silu", x), a.reps), 8 * x.numel())
    if want("drift"):
        x = torch.randn((NH, S, S), device=dev)
        report("inject_drift", timeit(lambda: inject_drift(x, 1, 16), a.reps), 8 * x.numel())
    if want("layernorm"):
        x = torch.randn((S, H), device=dev)
        report("layernorm_bound_f32eps", timeit(lambda: layernorm_device(x, -1, 1e-6, model, False),
                                                a.reps), 12 * x.numel())
    if want("split"):
        x = torch.randn((S, I), device=dev)
        report("tf32_split", timeit(lambda: tf32_split(x, S, I, False, False), a.reps),
               12 * x.numel())
        from paper_2510_16028_b200.bounds import f16_split
        for shp in ((NH * S, S), (S, H), (S, I)):  # probs (ctx A operand), x, act
            xs = torch.rand(shp, device=dev)
            report(f"f16_split_{shp[0]}x{shp[1]}",
                   timeit(lambda: f16_split(xs, shp[0], shp[1], False, False), a.reps),
                   8 * xs.numel())
            del xs
    for path, tag in ((1, "gemm_tc"), (2, "gemm_tc16"), (0, "gemm_ffma")):
        if want(tag):
            shapes = [(S, H, H), (S, H, I), (S, I, H)]
            if want("gemm_all"):  # every Qwen3-8B GEMM shape: k/v, scores, ctx, lm_head
                shapes += [(S, H, 1024), ("scores",), ("ctx",), (S, H, 151936)]
            for shp in shapes:
                if shp == ("scores",):  # q @ k^T, 32 heads, K = 128
                    A = torch.randn((NH, S, 128), device=dev)
                    B = torch.randn((NH, S, 128), device=dev)
                    tb, fl, K = True, 2.0 * NH * S * S * 128, 128
                elif shp == ("ctx",):  # p @ v, 32 heads, K = S
                    A = torch.rand((NH, S, S), device=dev)
                    B = torch.randn((NH, S, 128), device=dev)
                    tb, fl, K = False, 2.0 * NH * S * S * 128, S
                else:
                    M, K, N = shp
                    A = torch.randn((M, K), device=dev)
                    B = torch.randn((K, N), device=dev)
                    tb, fl = False, 2.0 * M * N * K
                c = model.reduction_const(2 * K - 1)
                cb = not (shp in (("scores",), ("ctx",)))
                abs_gemm_bound(A, B, c, tb, eps_f64=False, path=path, cache_b=cb)
                ms = timeit(lambda: abs_gemm_bound(A, B, c, tb, eps_f64=False, path=path,
                                                   cache_b=cb), a.reps)
                if path == 2:  # the f16 split of the activation operand alone
                    from paper_2510_16028_b200.bounds import f16_split
                    rows, KK = A.shape[-2], A.shape[-1]
                    ms_s = timeit(lambda: f16_split(A, rows, KK, False, False), a.reps)
                    report(tag, ms, flops=fl, shape=list(shp), split_ms=round(ms_s, 4))
                else:
                    report(tag, ms, flops=fl, shape=list(shp))
                del A, B
            if want("sgemm") or only is None:
                A = torch.randn((S, H), device=dev)
                B = torch.randn((H, I), device=dev)
                torch.backends.cuda.matmul.allow_tf32 = False
                report("cublas_sgemm_fp32", timeit(lambda: A @ B, a.reps), flops=2.0 * S * H * I)


if __name__ == "__main__":
    main()
