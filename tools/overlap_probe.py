"""Probe: how much of the Keccak commit hides under the forward's SGEMMs.

Times, with CUDA events, (a) a chain of Qwen-shaped cuBLAS FP32 GEMMs alone,
(b) a fused commit+check of a fixed byte volume alone, (c) both launched
concurrently on two streams, and reports the hidden fraction
(a + b - c) / min(a, b).  Variants: NAO_COMMIT_CTAS caps, stream priorities.

    python tools/overlap_probe.py [--gb 8] [--reps 3]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gb", type=float, default=8.0)
    ap.add_argument("--gemms", type=int, default=24)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--gemm", choices=["sgemm", "absgemm"], default="sgemm",
                    help="main-stream chain: cuBLAS FP32 GEMMs or the FP16-split abs-GEMM bound")
    args = ap.parse_args()
    from paper_2510_16028_b200 import _lib
    from paper_2510_16028_b200.commitments import commit_tensors
    torch.backends.cuda.matmul.allow_tf32 = False
    dev = torch.device("cuda")
    # SGEMM chain: gate/up-shaped (2048 x 4096 @ 4096 x 12288), ~206 GFLOP each
    x = torch.randn(2048, 4096, device=dev)
    w = torch.randn(4096, 12288, device=dev) / 64
    outs = [torch.empty(2048, 12288, device=dev) for _ in range(2)]
    # commit payload: claimed + local tensors of 64 MB each
    n_t = max(1, int(args.gb * (1 << 30) // (64 << 20)))
    claimed = [torch.randn(16 << 20, device=dev) for _ in range(n_t)]
    local = [c.clone() for c in claimed]
    spec = torch.frombuffer(bytearray(_lib.verdict_spec([50.0], [float("inf")], [float("inf")],
                                                         1e-12)), dtype=torch.uint8).to(dev)
    recs = torch.zeros((n_t, _lib.CHECK_RESULT_BYTES), dtype=torch.uint8, device=dev)
    checks = [_lib.CheckDesc(local[i].data_ptr(), None, spec.data_ptr(), recs[i].data_ptr(),
                             2.0 ** -23, 1.0, _lib.EPS_SCALED_LOCAL, 0, None, 0)
              for i in range(n_t)]

    if args.gemm == "absgemm":
        from paper_2510_16028_b200.bounds import abs_gemm_bound
        abs_gemm_bound(x, w, 1e-6, eps_f64=False, path=_lib.GEMM_TC_F16X3, cache_b=True)

    def gemms():
        for i in range(args.gemms):
            if args.gemm == "absgemm":
                abs_gemm_bound(x, w, 1e-6, eps_f64=False, path=_lib.GEMM_TC_F16X3, cache_b=True)
            else:
                torch.matmul(x, w, out=outs[i & 1])

    def commit():
        for lo in range(0, n_t, 16):
            commit_tensors(claimed[lo:lo + 16], 4096, "keccak256", checks=checks[lo:lo + 16])

    def timed(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    res = {}
    for prio_name, prio in (("equal", 0), ("main_high", -1)):
        s_main = torch.cuda.Stream(dev, priority=prio)
        s_side = torch.cuda.Stream(dev, priority=0)

        def both():
            cur = torch.cuda.current_stream()
            s_main.wait_stream(cur)
            s_side.wait_stream(cur)
            with torch.cuda.stream(s_main):
                gemms()
            with torch.cuda.stream(s_side):
                commit()
            cur.wait_stream(s_main)
            cur.wait_stream(s_side)

        for _ in range(2):  # warm-up
            gemms(); commit(); both()
        a = min(timed(gemms) for _ in range(args.reps))
        b = min(timed(commit) for _ in range(args.reps))
        c = min(timed(both) for _ in range(args.reps))
        res[prio_name] = {"gemm_ms": round(a, 2), "commit_ms": round(b, 2), "both_ms": round(c, 2),
                          "hidden_frac": round((a + b - c) / min(a, b), 3),
                          "commit_GBps": round(n_t * 64 / 1024 / (b / 1e3), 1),
                          "gemm_TFLOPs": round(args.gemms * 2 * 2048 * 4096 * 12288 / a / 1e9, 1)}
    res["ctas"] = os.environ.get("NAO_COMMIT_CTAS", "default")
    res["gemm"] = args.gemm
    res["lib"] = os.environ.get("NAO_LIB_PATH", "default")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
