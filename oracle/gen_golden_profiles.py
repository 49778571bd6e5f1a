"""ORACLE -- TEST INFRASTRUCTURE ONLY.  Golden vectors for the reference's
non-sequential device profiles: the UNMODIFIED
reference (/root/reference/pkg/src/fpverify, engine.py:75-113 reduction
orders, engine.py:157-213 matmul / softmax / layernorm parts, bounds.py:176-218
op_bound) run in the build container on small seeded inputs.

    python oracle/gen_golden_profiles.py     # writes tests/golden/ref_profiles.npz

Nothing here is imported at test time.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True  # never write into /root/reference
REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "ref_profiles.npz"

# (tag, reduction, block_size, perm_seed, fma)
PROFILES = [
    ("pair", "pairwise", 32, 0, False),
    ("blk32", "blocked", 32, 0, False),
    ("blk7", "blocked", 7, 0, False),
    ("perm7", "permuted", 32, 7, False),
    ("perm3fma", "permuted", 32, 3, True),
    ("pairfma", "pairwise", 32, 0, True),
]
RED_N = (1, 2, 3, 5, 8, 33, 100, 257, 1000)


class _Node:
    def __init__(self, kind, attrs):
        self.kind, self.attrs = kind, attrs

    def attr(self, k, d=None):
        return self.attrs.get(k, d)


def main():
    sys.path.insert(0, REF_SRC)
    from fpverify import bounds as B
    from fpverify.engine import DeviceProfile, matmul_op, reduce_last_axis

    rng = np.random.default_rng(2510)
    out = {}
    model = B.FpModel()
    for tag, red, blk, seed, fma in PROFILES:
        p = DeviceProfile(tag, red, block_size=blk, perm_seed=seed, fma=fma)
        for n in RED_N:
            x = (rng.standard_normal((3, n)) * 10.0 ** rng.integers(-3, 4, size=(3, n))).astype(
                np.float32)
            out[f"{tag}/reduce/{n}/x"] = x
            out[f"{tag}/reduce/{n}/y"] = reduce_last_axis(x, p)
        for (m, k, nn, tb) in ((4, 37, 6, False), (3, 64, 5, True), (2, 129, 3, False)):
            a = rng.standard_normal((m, k)).astype(np.float32)
            b = rng.standard_normal((nn, k) if tb else (k, nn)).astype(np.float32)
            key = f"{tag}/matmul/{m}x{k}x{nn}x{int(tb)}"
            out[key + "/a"], out[key + "/b"] = a, b
            out[key + "/y"] = matmul_op(a, b, p, transpose_b=tb)
            y, eps = B.op_bound(_Node("matmul", {"transpose_b": int(tb)}), [a, b], model, p)
            out[key + "/eps"] = eps
        for kind, shape, attrs in (("softmax", (4, 129), {"axis": -1}),
                                   ("softmax", (1, 2048), {"axis": -1}),
                                   ("layernorm", (4, 96), {"axis": -1, "eps": 1e-5}),
                                   ("layernorm", (2, 1000), {"axis": -1, "eps": 1e-6}),
                                   ("sum", (5, 77), {"axis": -1}),
                                   ("mean", (5, 300), {"axis": -1})):
            x = (rng.standard_normal(shape) * 3 + 0.5).astype(np.float32)
            key = f"{tag}/{kind}/{shape[0]}x{shape[1]}"
            y, eps = B.op_bound(_Node(kind, attrs), [x], model, p)
            out[key + "/x"], out[key + "/y"], out[key + "/eps"] = x, y, eps
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
