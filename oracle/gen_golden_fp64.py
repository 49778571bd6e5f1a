"""ORACLE -- TEST INFRASTRUCTURE ONLY.  Golden vectors of the reference's FP64
oracle path -- apply_op(node, args64, None, fp64=True) (engine.py:220-285), the
leaf route's theoretical recheck (dispute.py:648-656) -- from the UNMODIFIED
reference (/root/reference/pkg/src/fpverify) on small seeded FP32 inputs:
matmul (plain, transpose_b, batched), linear, softmax, layernorm, sum, mean
and the intrinsics.

    python oracle/gen_golden_fp64.py     # writes tests/golden/ref_fp64.npz

Nothing here is imported at test time.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True  # never write into /root/reference
REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "ref_fp64.npz"

CASES = [
    # tag, kind, attrs, input shapes, input scale
    ("matmul", "matmul", {}, [(7, 33), (33, 5)], 1.0),
    ("matmul_tb", "matmul", {"transpose_b": 1}, [(6, 40), (9, 40)], 1.0),
    ("matmul_batched", "matmul", {}, [(3, 5, 70), (3, 70, 4)], 1.0),
    ("linear", "linear", {}, [(8, 50), (50, 12), (12,)], 1.0),
    ("softmax", "softmax", {"axis": -1}, [(9, 31)], 4.0),
    ("softmax_axis0", "softmax", {"axis": 0}, [(17, 6)], 4.0),
    ("layernorm", "layernorm", {"axis": -1, "eps": 1e-5}, [(10, 40)], 3.0),
    ("sum", "sum", {"axis": -1}, [(11, 77)], 1.0),
    ("mean", "mean", {"axis": 0}, [(23, 9)], 1.0),
    ("exp", "exp", {}, [(300,)], 4.0),
    ("tanh", "tanh", {}, [(300,)], 4.0),
    ("silu", "silu", {}, [(300,)], 6.0),
    ("gelu", "gelu", {}, [(300,)], 2.0),
]


class _Node:
    def __init__(self, kind, attrs):
        self.kind, self.attrs = kind, attrs

    def attr(self, k, d=None):
        return self.attrs.get(k, d)


def main():
    sys.path.insert(0, REF_SRC)
    from fpverify import engine
    rng = np.random.default_rng(2026)
    out = {}
    for tag, kind, attrs, shapes, scale in CASES:
        ins = [(rng.standard_normal(s) * scale).astype(np.float32) for s in shapes]
        args64 = [a.astype(np.float64) for a in ins]
        y = engine.apply_op(_Node(kind, attrs), args64, None, fp64=True)
        for i, a in enumerate(ins):
            out[f"{tag}/in{i}"] = a
        out[f"{tag}/y"] = np.asarray(y, dtype=np.float64)
        out[f"{tag}/kind"] = np.array(kind)
        out[f"{tag}/attrs"] = np.array(repr(attrs))
    np.savez(OUT, **out)
    print(f"wrote {OUT} ({len(CASES)} cases)")


if __name__ == "__main__":
    main()
