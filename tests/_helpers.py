"""Shared test helpers (importable as `_helpers`; pytest puts tests/ on sys.path)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def op_cases(ref_ops):
    tags = sorted({k.split("/")[0] for k in ref_ops})
    out = {}
    for t in tags:
        ins = []
        i = 0
        while f"{t}/in{i}" in ref_ops:
            ins.append(ref_ops[f"{t}/in{i}"])
            i += 1
        out[t] = (ins, ref_ops[f"{t}/y"], ref_ops[f"{t}/eps"])
    return out


# node descriptions for the single-op golden cases (oracle/gen_golden.py section 2)
OP_SPECS = {
    "softmax_prob": ("softmax", {"axis": -1}, "prob", False),
    "softmax_det": ("softmax", {"axis": -1}, "det", False),
    "softmax_axis0": ("softmax", {"axis": 0}, "prob", False),
    "softmax_n1": ("softmax", {"axis": -1}, "det", False),
    "layernorm_prob": ("layernorm", {"axis": -1, "eps": 1e-5}, "prob", False),
    "layernorm_det": ("layernorm", {"axis": -1, "eps": 1e-3}, "det", False),
    "sum_prob": ("sum", {"axis": -1}, "prob", False),
    "sum_axis0": ("sum", {"axis": 0}, "det", False),
    "mean_prob": ("mean", {"axis": 1}, "prob", False),
    "matmul_prob": ("matmul", {}, "prob", False),
    "matmul_det_tb": ("matmul", {"transpose_b": 1}, "det", False),
    "matmul_fma": ("matmul", {}, "prob", True),
    "matmul_bcast": ("matmul", {}, "prob", False),
    "linear_prob": ("linear", {}, "prob", False),
    "add": ("add", {}, "prob", False), "sub": ("sub", {}, "prob", False),
    "mul": ("mul", {}, "prob", False), "div": ("div", {}, "prob", False),
    "neg": ("neg", {}, "prob", False),
    "exp": ("exp", {}, "prob", False), "log": ("log", {}, "prob", False),
    "sqrt": ("sqrt", {}, "prob", False), "rsqrt": ("rsqrt", {}, "prob", False),
    "tanh": ("tanh", {}, "prob", False), "gelu": ("gelu", {}, "prob", False),
    "silu": ("silu", {}, "prob", False), "relu": ("relu", {}, "prob", False),
    "max": ("max", {"axis": -1}, "prob", False), "min": ("min", {"axis": 0}, "prob", False),
}
