"""Check: a GPT-2-style decoder (LayerNorm, biases, GELU, no RoPE / GQA) and a
Qwen-style one verified eagerly and replayed as CUDA graphs with the
verifier's side streams give identical roots / records (run under
compute-sanitizer to locate an invalid access).

    python tools/graph_stream_check.py [--seq 256] [--batch 2] [--seg 96]
"""

from __future__ import annotations

import argparse
import dataclasses
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=256)
    ap.add_argument("--batch", type=int, default=2)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--seg", type=int, default=96)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--vocab", type=int, default=1000)
    ap.add_argument("--main-priority", type=int, default=None,
                    help="run on a fresh stream of this priority (bench.py does, -1)")
    a = ap.parse_args()
    if a.main_priority is not None:
        torch.cuda.set_stream(torch.cuda.Stream(priority=a.main_priority))
    from paper_2510_16028_b200 import lowerings as L
    from paper_2510_16028_b200.bounds import FpModel
    from paper_2510_16028_b200.executor import StreamingVerifier, drift_claim
    from paper_2510_16028_b200.tensor import Rng
    shape = dataclasses.replace(L.GPT2_SMALL, layers=a.layers, seq=a.seq, batch=a.batch,
                                vocab=a.vocab)
    spec = L.build_decoder(shape, seed=3)
    g = spec.graph
    ids = spec.make_inputs(Rng(5))

    def claimed_fn(node, y):
        return drift_claim(node, y, 1, 16, "l1_fc")

    ref = StreamingVerifier(g, FpModel(), hash_alg="keccak256", overlap=False)
    r0, c0 = ref.run(ids, claimed_fn)
    r0, c0 = r0.clone(), c0.clone()
    sv = StreamingVerifier(g, FpModel(), hash_alg="keccak256", bound_stream=True)
    r1, c1 = sv.run(ids, claimed_fn)
    torch.cuda.synchronize()
    print("eager equal:", torch.equal(r1, r0), torch.equal(c1, c0), flush=True)
    gr = sv.capture(ids, claimed_fn, seg_nodes=a.seg)
    for i in range(a.reps):
        r2, c2 = gr.replay()
        torch.cuda.synchronize()
        print(f"replay {i} equal:", torch.equal(r2, r0), torch.equal(c2, c0), flush=True)


if __name__ == "__main__":
    main()
