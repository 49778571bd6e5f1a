"""ORACLE -- TEST INFRASTRUCTURE ONLY.  Golden digests of the reference's
on-disk formats: NAOT tensor files
(tensor.py:146-161), trace dumps (engine.py:449-464 save_trace) and bound
dumps (bounds.py:265-282 save_bounds), written by the UNMODIFIED reference
for the MLP 784-256-10 B=64 graph under the sequential profile.  The files
themselves are not committed -- their SHA-256 digests and the manifests are.

    python oracle/gen_golden_traceio.py     # writes tests/golden/ref_traceio.json

Nothing here is imported at test time.
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True  # never write into /root/reference
REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "ref_traceio.json"


def _digests(d: Path) -> dict:
    return {p.name: hashlib.sha256(p.read_bytes()).hexdigest() for p in sorted(d.iterdir())}


def main():
    sys.path.insert(0, REF_SRC)
    from fpverify import bounds as B
    from fpverify.engine import DeviceProfile, save_trace
    from fpverify.models import build_mlp
    from fpverify.tensor import Rng, write_tensor_file

    doc = {}
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        # single NAOT files: edge shapes and both dtypes
        arrs = {"scalar_f32": np.float32(3.5).reshape(()),
                "empty_f32": np.zeros((0, 4), np.float32),
                "ragged_f32": np.arange(7 * 5, dtype=np.float32).reshape(7, 5) * 0.25 - 3,
                "vec_f64": np.linspace(-1, 1, 9, dtype=np.float64)}
        files = {}
        for name, a in arrs.items():
            write_tensor_file(tmp / f"{name}.naot", a)
            files[name] = {"sha256": hashlib.sha256((tmp / f"{name}.naot").read_bytes()).hexdigest(),
                           "shape": list(a.shape), "dtype": str(a.dtype),
                           "values": np.asarray(a, np.float64).reshape(-1).tolist()}
        doc["naot_files"] = files
        # MLP trace + bound dumps (sequential profile, deterministic and probabilistic models)
        spec = build_mlp(seed=0, batch=64, in_dim=784, hidden=256, n_classes=10)
        x = spec.make_inputs(Rng(7))
        seq = DeviceProfile("seq", "sequential")
        for mode in ("probabilistic", "deterministic"):
            model = B.FpModel(mode=mode)
            _, bnds, tr = B.co_execute(spec.graph, x, seq, model, with_trace=True)
            save_trace(tmp / f"trace_{mode}", tr)
            B.save_bounds(tmp / f"bounds_{mode}", bnds, model, seq.id)
            doc[f"trace/{mode}"] = _digests(tmp / f"trace_{mode}")
            doc[f"trace/{mode}/manifest"] = json.loads((tmp / f"trace_{mode}" /
                                                        "manifest.json").read_text())
            doc[f"bounds/{mode}/manifest_text"] = (tmp / f"bounds_{mode}" /
                                                   "manifest.json").read_text()
    json.dump(doc, open(OUT, "w"), indent=1, sort_keys=True)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
