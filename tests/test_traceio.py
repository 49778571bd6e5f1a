"""NAOT files, trace dumps and bound dumps.
CPU: the host NAOT writer is byte-identical to the reference's
(tests/golden/ref_traceio.json, oracle/gen_golden_traceio.py).
GPU: the streaming writers (pinned ring + copy stream + writer thread),
driven from co_execute and from the streaming verifier, produce the
reference's exact trace files and manifests for the MLP graph; bound dumps
have the reference's format with bounds in [ref, ref (1 + 1e-5)]; readers
round-trip."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

GOLD = json.load(open(Path(__file__).resolve().parent / "golden" / "ref_traceio.json"))


def _digests(d: Path) -> dict:
    return {p.name: hashlib.sha256(p.read_bytes()).hexdigest() for p in sorted(d.iterdir())}


def test_naot_files_match_reference(tmp_path):
    from paper_2510_16028_b200.tensor import read_tensor_file, write_tensor_file
    for name, ent in GOLD["naot_files"].items():
        a = np.asarray(ent["values"], dtype=np.dtype(ent["dtype"])).reshape(ent["shape"])
        write_tensor_file(tmp_path / f"{name}.naot", a)
        got = hashlib.sha256((tmp_path / f"{name}.naot").read_bytes()).hexdigest()
        assert got == ent["sha256"], name
        back = read_tensor_file(tmp_path / f"{name}.naot")
        assert back.shape == a.shape and np.array_equal(back, a)


def test_naot_header_matches_host_writer(tmp_path):
    import torch
    from paper_2510_16028_b200.traceio import naot_header
    for shape, dt in (((), torch.float32), ((0, 4), torch.float32), ((7, 5), torch.float64)):
        from paper_2510_16028_b200.tensor import write_tensor_file
        a = np.zeros(shape, np.float32 if dt == torch.float32 else np.float64)
        write_tensor_file(tmp_path / "h.naot", a)
        data = (tmp_path / "h.naot").read_bytes()
        h = naot_header(shape, dt)
        assert data[:len(h)] == h


def _mlp():
    from paper_2510_16028_b200.lowerings import build_mlp
    from paper_2510_16028_b200.tensor import Rng
    spec = build_mlp(seed=0, batch=64, in_dim=784, hidden=256, n_classes=10)
    return spec, spec.make_inputs(Rng(7))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["probabilistic", "deterministic"])
def test_streamed_trace_and_bound_dumps_match_reference(tmp_path, mode):
    from oracle import bounds as OB
    from paper_2510_16028_b200 import bounds as B
    from paper_2510_16028_b200.engine import DeviceProfile
    from paper_2510_16028_b200.tensor import read_tensor_file
    from paper_2510_16028_b200.traceio import BoundWriter, TraceReader, load_trace, save_trace
    spec, x = _mlp()
    seq = DeviceProfile("seq", "sequential")
    model = B.FpModel(mode=mode)
    _, bnds, tr = B.co_execute(spec.graph, x, seq, model, with_trace=True)
    save_trace(tmp_path / "trace", tr)
    assert _digests(tmp_path / "trace") == GOLD[f"trace/{mode}"]
    # bound dump: reference format + manifest, bounds within tolerance of the oracle's
    bw = BoundWriter(tmp_path / "bounds", model, seq.id)
    for i, bt in enumerate(bnds):
        bw.write(i, bt.device_tensor())
    bw.close(len(bnds))
    assert (tmp_path / "bounds" / "manifest.json").read_text() == GOLD[f"bounds/{mode}/manifest_text"]
    _, ref_eps = OB.co_execute(spec.graph, {"x": x["x"].array}, OB.FpModel(mode=mode))
    for i, re in enumerate(ref_eps):
        e = read_tensor_file(tmp_path / "bounds" / f"{i:06d}.naot")
        assert e.dtype == np.float64 and e.shape == re.shape
        assert np.all(e >= re) and np.all(e <= re * (1 + 1e-5))
    # readers
    back = load_trace(tmp_path / "trace")
    r = TraceReader(tmp_path / "trace")
    for i, t in enumerate(tr.tensors):
        assert np.array_equal(back.tensors[i].array, t.array)
        assert np.array_equal(r.node(i).cpu().numpy().reshape(-1), np.asarray(t.array).reshape(-1))


@pytest.mark.gpu
def test_streaming_verifier_dumps_the_claimed_trace(tmp_path):
    """The verifier streams the claimed tensors to disk as it goes (small
    staging slots force multi-chunk files): honest claims under the sequential
    profile reproduce the reference's trace files bit for bit."""
    from paper_2510_16028_b200 import bounds as B
    from paper_2510_16028_b200.commitments import tensor_digest
    from paper_2510_16028_b200.engine import DeviceProfile
    from paper_2510_16028_b200.executor import StreamingVerifier
    from paper_2510_16028_b200.traceio import NaotWriter, TraceWriter
    spec, x = _mlp()
    seq = DeviceProfile("seq", "sequential")
    sv = StreamingVerifier(spec.graph, B.FpModel(), seq, hash_alg="sha256")
    man = GOLD["trace/probabilistic/manifest"]
    tw = TraceWriter(tmp_path / "t", "seq",
                     {k: tensor_digest(v) for k, v in sorted(x.items())},
                     {k: tensor_digest(v) for k, v in sorted(spec.graph.weights.items())},
                     writer=NaotWriter(slots=2, slot_bytes=4096))
    sv.trace_writer = tw
    sv.run(x, lambda node, y: y.clone())
    tw.close(spec.graph.n_nodes)
    assert json.loads((tmp_path / "t" / "manifest.json").read_text()) == man
    assert _digests(tmp_path / "t") == GOLD["trace/probabilistic"]


def test_weight_digests_cached_and_invalidated():
    """co_execute's per-call weight digests (engine.py:362-363) are computed
    once per weight object; a torch weight changed in place is re-hashed."""
    import torch
    from paper_2510_16028_b200 import commitments as CM
    from paper_2510_16028_b200.tensor import Tensor
    w = {"b": Tensor((3,), np.arange(3, dtype=np.float32)),
         "a": torch.ones((2, 2), dtype=torch.float32)}
    d1 = CM.weight_digests(w)
    assert list(d1) == ["a", "b"]
    assert d1 == {k: CM.tensor_digest(v) for k, v in w.items()}
    assert CM.weight_digests(w) == d1
    w["a"].mul_(2.0)
    d2 = CM.weight_digests(w)
    assert d2["a"] == CM.tensor_digest(w["a"]) != d1["a"] and d2["b"] == d1["b"]
