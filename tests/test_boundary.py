"""CPU: the C-ABI boundary and the product/oracle separation."""

import ast
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_2510_16028_b200"


def header_symbols():
    text = (ROOT / "include" / "nao_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nao_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2510_16028_b200 import _lib
    L = _lib.load(require_cuda=False)
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTED_SYMBOLS)
    assert L.nao_version() == 1


def test_library_is_sm100a():
    import subprocess
    from paper_2510_16028_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.lib_path())],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_text_without_gpu():
    """Invalid arguments are rejected before any CUDA call (-> ValueError in Python)."""
    from paper_2510_16028_b200 import _lib
    L = _lib.load(require_cuda=False)
    rc = L.nao_merkle_root_of(None, 0, 0, None, None, None, 0, None)
    assert rc == _lib.NAO_EINVAL
    assert "at least one leaf" in _lib.last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_product_never_imports_oracle():
    for f in PKG.rglob("*.py"):
        tree = ast.parse(f.read_text())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                names = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                names = [node.module or ""]
            else:
                continue
            assert not any(n == "oracle" or n.startswith("oracle.") for n in names), f


def test_mlp_graph_matches_reference_signatures(ref_mlp):
    """Our lowering of the BASELINE MLP config is the reference's graph:
    same op signatures (commitments.py:68-78) node for node."""
    import hashlib
    import json
    from paper_2510_16028_b200.lowerings import build_mlp
    from paper_2510_16028_b200.tensor import Rng
    c = ref_mlp["config"]
    spec = build_mlp(c["seed"], c["batch"], c["in_dim"], c["hidden"], c["n_classes"])
    sigs = []
    for n in spec.graph.nodes:
        doc = {"name": n.name, "op": "call", "target": n.kind, "args": list(n.inputs),
               "kwargs": {k: v for k, v in n.attrs}}
        sigs.append(hashlib.sha256(json.dumps(doc, sort_keys=True, separators=(",", ":"))
                                   .encode()).hexdigest())
    assert sigs == ref_mlp["signatures"]
    from oracle import commit as OM
    for name, w in spec.graph.weights.items():
        assert hashlib.sha256(OM.canon_tensor(w.array)).hexdigest() == \
            ref_mlp["weights"][name]["digest"], name
    x = spec.make_inputs(Rng(*c["input_rng"]))
    assert hashlib.sha256(OM.canon_tensor(x["x"].array)).hexdigest() == ref_mlp["input_digest"]


def test_partition_and_frontiers():
    from paper_2510_16028_b200.graph import Slice, frontiers, partition
    from paper_2510_16028_b200.lowerings import build_mlp
    assert partition(Slice(0, 10), 4) == [Slice(0, 3), Slice(3, 6), Slice(6, 8), Slice(8, 10)]
    assert partition(Slice(0, 3), 4) == [Slice(0, 1), Slice(1, 2), Slice(2, 3)]
    g = build_mlp(batch=4, in_dim=16, hidden=32).graph
    fr = frontiers(g, Slice(3, 9))
    assert fr.in_nodes == (0, 1, 2) or 2 in fr.in_nodes
    assert all(i < 3 or i >= 9 for i in fr.in_nodes)
