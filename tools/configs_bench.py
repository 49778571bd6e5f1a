"""Overhead of the verified forward on the other BASELINE.json configs (the
headline Qwen3-8B line is bench.py's).  Same protocol as bench.py on one GPU:
plain forward (cuBLAS/cuDNN FP32, TF32 off) vs the streaming verifier
(bounds + check + exact percentile verdict + Keccak-256 chunked commit) with
the proposer harness (+-1-ulp drift on reduction nodes, one planted fault)
inside the timed region; thresholds calibrated on the device (alpha 3).

    python tools/configs_bench.py [--configs mlp,gpt2,resnet18,unet] [--steps 5]

Prints one JSON line per config.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
# many distinct large tensor sizes per step (node outputs, bounds, splits):
# expandable segments keep the caching allocator from fragmenting into
# cudaMalloc retries (device syncs) on the UNet-sized graphs
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

import torch  # noqa: E402


def _build(name):
    from paper_2510_16028_b200 import lowerings as L
    if name == "mlp":
        return L.build_mlp(seed=0, batch=64), "fc1", "2-layer MLP 784-256-10 FP32 batch 64"
    if name == "gpt2":
        return (L.build_decoder(L.GPT2_SMALL, seed=0), "l5_fc",
                "GPT-2 small FP32 seq 1024 batch 8")
    if name == "resnet18":
        return (L.build_resnet18(batch=32, side=224), "layer3.0.conv2",
                "ResNet-18 FP32 batch 32 224x224")
    if name == "unet":  # the 8-GPU batch-sharded config: one sample per GPU
        return (L.build_unet(dataclasses.replace(L.SD15_UNET, batch=1)), "down1.res0.conv2",
                "SD-1.5 UNet-shaped FP32 step, 64x64 latent, batch 8 over 8 GPUs "
                "(per-GPU shard: batch 1)")
    if name == "unet8":  # the whole batch on one GPU
        return (L.build_unet(L.SD15_UNET), "down1.res0.conv2",
                "SD-1.5 UNet-shaped FP32 step, 64x64 latent, batch 8 on one GPU")
    raise ValueError(name)


def run_config(name, steps, warmup, drift_period=16, profile=False, flush_mb=2048, graphs=0):
    from paper_2510_16028_b200.calibration import (PERCENTILE_GRID, OpThresholds, ThresholdSet,
                                                   error_profiles_device)
    from paper_2510_16028_b200.dispute import CheckRecord
    from paper_2510_16028_b200.executor import (NodeStats, StreamingVerifier, drift_claim,
                                                plain_forward)
    from paper_2510_16028_b200.tensor import Rng
    spec, fault, label = _build(name)
    g = spec.graph
    x = spec.make_inputs(Rng(2024))
    dev = torch.device("cuda")

    env = {}

    def calib_fn(node, y):
        yc = drift_claim(node, y, seed=11, period=max(1, drift_period // 4))
        if y.numel():
            pa, pr = error_profiles_device(y, yc)
            env[node.name] = (pa, pr)
        return yc

    StreamingVerifier(g, None, thresholds=None).run(x, calib_fn)
    torch.cuda.synchronize()
    th = ThresholdSet(alpha=3.0, epsilon=1e-12, grid=PERCENTILE_GRID,
                      ops=[OpThresholds(n, 3.0 * a.cpu().numpy(), 3.0 * r.cpu().numpy())
                           for n, (a, r) in env.items()])
    sv = StreamingVerifier(g, None, thresholds=th, max_lag=4, flush_bytes=flush_mb << 20,
                           missing_thresholds="inf")  # empty nodes were not calibrated

    def claimed(node, y):
        return drift_claim(node, y, 1, drift_period, fault)

    graphed = {}
    host = {}

    def plain():
        if "plain" in graphed:
            return graphed["plain"].replay()
        return plain_forward(g, x, dev)

    def ver():
        if "ver" in graphed:
            return graphed["ver"].replay()
        return sv.run(x, claimed)

    def timed(fn, key):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h0 = time.perf_counter()
        for _ in range(steps):
            out = fn()
            del out
        host[key] = (time.perf_counter() - h0) * 1e3 / steps
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    stats = NodeStats()
    _, recs = sv.run(x, claimed, stats=stats)
    plain_forward(g, x, dev)
    torch.cuda.synchronize()
    if graphs:
        from paper_2510_16028_b200.executor import GraphedRun
        graphed["plain"] = GraphedRun.record_plain(g, x, dev, 0, None, None, seg_nodes=graphs)
        graphed["ver"] = sv.capture(x, claimed, seg_nodes=graphs)
    t_plain = timed(plain, "plain")
    if t_plain * steps < 500.0:  # short steps: time >= ~0.5 s of work
        steps = int(500.0 / max(t_plain, 1e-3)) + 1
        t_plain = timed(plain, "plain")
    t_ver = timed(ver, "verified")
    _, recs = ver()
    torch.cuda.synchronize()
    if profile:  # top device kernels of one verified step (torch.profiler / CUPTI)
        from torch.profiler import ProfilerActivity
        from torch.profiler import profile as tprof
        with tprof(activities=[ProfilerActivity.CUDA]) as prof:
            ver()
            torch.cuda.synchronize()
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30),
              file=sys.stderr, flush=True)
    names = [n.name for n in g.nodes]
    flagged = []
    for i in range(len(names)):
        r = CheckRecord(recs[i]).host()
        if r["n_violations"] or r["threshold_exceeded"]:
            flagged.append(names[i])
    return {"config": label, "nodes": g.n_nodes, "plain_fwd_ms": round(t_plain, 3),
            "verified_fwd_ms": round(t_ver, 3),
            "overhead_pct": round(100.0 * (t_ver - t_plain) / t_plain, 1),
            "committed_gb_per_step": round(stats.bytes_committed / 1e9, 3),
            "gemm_tflop_per_step": round(stats.gemm_flops / 1e12, 3),
            "host_enqueue_ms": {k: round(v, 2) for k, v in host.items()},
            "mem_peak_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1),
            "mem_reserved_gb": round(torch.cuda.memory_reserved() / 1e9, 1),
            "mem_peak_reserved_gb": round(torch.cuda.max_memory_reserved() / 1e9, 1),
            "device_free_total_gb": [round(v / 1e9, 1) for v in torch.cuda.mem_get_info()],
            "alloc_retries": torch.cuda.memory_stats().get("num_alloc_retries", 0),
            "cuda_mallocs": torch.cuda.memory_stats().get("num_device_alloc", 0),
            "dispatch": f"cuda graphs ({graphs}-node segments)" if graphs else "eager",
            "flagged_nodes": flagged, "planted_fault": fault, "steps": steps,
            "warmup": warmup}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="mlp,gpt2,resnet18,unet")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--graphs", type=int, default=0, metavar="SEG")
    ap.add_argument("--flush-mb", default="2048", help="comma list: commit batch sizes to try")
    a = ap.parse_args()
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    # autotuned cuDNN algorithms for the conv values of both arms (the default
    # heuristics pick slow FP32 algorithms for some batch-1 UNet shapes)
    torch.backends.cudnn.benchmark = True
    torch.cuda.set_stream(torch.cuda.Stream(priority=-1))
    for name in a.configs.split(","):
        for fmb in (int(v) for v in a.flush_mb.split(",")):
            t0 = time.perf_counter()
            line = run_config(name, a.steps, a.warmup, profile=a.profile, flush_mb=fmb,
                              graphs=a.graphs)
            line["flush_mb"] = fmb
            line["wall_s"] = round(time.perf_counter() - t0, 1)
            print(json.dumps(line), flush=True)
            torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats()


if __name__ == "__main__":
    main()
