"""Host-side (Python) profile of the streaming verifier's per-node enqueue
path: cProfile over eager verified forwards of a few Qwen3-8B-shaped layers.

    python tools/host_profile.py [--layers 2] [--reps 3]
"""
import argparse
import cProfile
import dataclasses
import io
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--sort", default="tottime")
    a = ap.parse_args()
    from paper_2510_16028_b200.executor import StreamingVerifier, drift_claim
    from paper_2510_16028_b200.lowerings import QWEN3_8B, build_decoder
    from paper_2510_16028_b200.tensor import Rng
    torch.backends.cuda.matmul.allow_tf32 = False
    spec = build_decoder(dataclasses.replace(QWEN3_8B, seq=2048), seed=0, layers=a.layers)
    ids = spec.make_inputs(Rng(1))
    sv = StreamingVerifier(spec.graph, None, max_lag=4)
    cl = lambda node, y: drift_claim(node, y, 1, 16, None)  # noqa: E731
    for _ in range(2):
        sv.run(ids, cl)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(a.reps):
        sv.run(ids, cl)
    pr.disable()
    torch.cuda.synchronize()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats(a.sort).print_stats(45)
    print(f"nodes per run: {spec.graph.n_nodes}")
    print(s.getvalue())


if __name__ == "__main__":
    main()
