"""Dispute-time records against the reference's own
outputs (tests/golden/ref_subgraph.json, oracle/gen_golden_subgraph.py):
make_subgraph_record / verify_subgraph_record (commitments.py:283-323) and
thresholds_tree (:250-256) on the MLP 784-256-10 B=64 trace; the trace itself
comes from the oracle's sequential restatement and is pinned to the
reference's per-node value digests first (Merkle trees hash on the GPU); and
the challenger's child re-execution (dispute.py:544-559) on the GPU:
FLOPs and worst live-out p_max equal to the reference's."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import bounds as OB

GOLD = Path(__file__).resolve().parent / "golden"
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mlp():
    from paper_2510_16028_b200.commitments import tensor_digest
    from paper_2510_16028_b200.graph import parse_ref
    from paper_2510_16028_b200.lowerings import build_mlp
    from paper_2510_16028_b200.tensor import Rng
    ref = json.load(open(GOLD / "ref_mlp_784_256_10_b64.json"))
    c = ref["config"]
    spec = build_mlp(c["seed"], c["batch"], c["in_dim"], c["hidden"], c["n_classes"])
    g = spec.graph
    x = spec.make_inputs(Rng(*c["input_rng"]))
    vals = []
    for node in g.nodes:
        args = []
        for r in node.inputs:
            cat, key = parse_ref(r)
            args.append(vals[key] if cat == "node" else np.asarray(
                (x[key] if cat == "input" else g.weights[key]).array))
        vals.append(np.asarray(OB.apply_op(node, args), np.float32))
    for v, ent in zip(vals, ref["runs"]["seq/prob"]):
        assert tensor_digest(v) == ent["value_digest"]
    return g, x, vals, ref


def test_subgraph_records_match_reference(mlp):
    from paper_2510_16028_b200 import commitments as CM
    from paper_2510_16028_b200.graph import Slice, frontiers
    g, x, trace, _ = mlp
    gold = json.load(open(GOLD / "ref_subgraph.json"))
    wtree, wnames = CM.weight_tree(g.weights)
    gtree = CM.graph_tree(g)
    assert wtree.root.hex() == gold["weight_root"] and gtree.root.hex() == gold["graph_root"]
    for ent in gold["slices"]:
        s = Slice(ent["start"], ent["end"])
        rec = CM.make_subgraph_record(g, s, trace, x, wtree, wnames, gtree)
        assert rec.h_in.hex() == ent["h_in"] and rec.h_out.hex() == ent["h_out"], s
        assert {n: p.to_wire().hex() for n, p in rec.weight_proofs} == ent["weight_proofs"]
        assert {str(i): p.to_wire().hex() for i, p in rec.sig_proofs} == ent["sig_proofs"]
        fr = frontiers(g, s)
        assert list(fr.out_nodes) == ent["out_nodes"] and list(fr.in_nodes) == ent["in_nodes"]
        ins = ([x[n] for n in fr.in_inputs] + [g.weights[n] for n in fr.in_weights]
               + [trace[i] for i in fr.in_nodes])
        outs = [trace[i] for i in fr.out_nodes]
        assert CM.verify_subgraph_record(rec, g, wtree.root, gtree.root, ins, outs)
        # a tampered live-out, a foreign root, a forged signature index all fail
        bad = [o.copy() for o in outs]
        bad[0].reshape(-1)[0] += 1.0
        assert not CM.verify_subgraph_record(rec, g, wtree.root, gtree.root, ins, bad)
        assert not CM.verify_subgraph_record(rec, g, gtree.root, gtree.root, ins, outs)
        forged = CM.SubgraphRecord(rec.start, rec.end, rec.h_in, rec.h_out, rec.weight_proofs,
                                   ((g.n_nodes, rec.sig_proofs[0][1]),))
        assert not CM.verify_subgraph_record(forged, g, wtree.root, gtree.root, ins, outs)


def test_thresholds_tree_matches_reference(mlp):
    from paper_2510_16028_b200 import commitments as CM
    gold = json.load(open(GOLD / "ref_subgraph.json"))
    assert CM.thresholds_tree(mlp[3]["thresholds"]).root.hex() == gold["thresholds_root"]


def test_child_offense_matches_reference(mlp):
    """run_slice / child_offense on the GPU (sequential profile) against the
    reference's run_subgraph + graph_flops + observed_p_max: the claimed
    live-outs are the trace itself (p_max 0) and the honest pairwise trace,
    which the GPU reproduces bit-exactly (DeviceProfile emulation)."""
    import torch
    from paper_2510_16028_b200.bounds import FpModel, co_execute
    from paper_2510_16028_b200.calibration import ThresholdSet
    from paper_2510_16028_b200.dispute import child_offense
    from paper_2510_16028_b200.engine import DeviceProfile
    from paper_2510_16028_b200.graph import Slice, frontiers
    g, x, trace, ref = mlp
    th = ThresholdSet.from_json(ref["thresholds"])
    _, _, honest = co_execute(g, x, DeviceProfile("pair", "pairwise"), FpModel(), with_trace=True)
    honest = [t._dev.reshape(tuple(t.shape)) if getattr(t, "_dev", None) is not None
              else torch.from_numpy(np.asarray(t.array)) for t in honest.tensors]
    gold = json.load(open(GOLD / "ref_subgraph.json"))
    for ent in gold["slices"]:
        s = Slice(ent["start"], ent["end"])
        fr = frontiers(g, s)
        boundary = {f"input:{n}": x[n] for n in fr.in_inputs}
        boundary.update({f"node:{i}": trace[i] for i in fr.in_nodes})
        seq = DeviceProfile("seq", "sequential")
        w_self, flops = child_offense(g, s, boundary, {i: trace[i] for i in fr.out_nodes}, th, seq)
        assert flops == ent["flops"], s
        assert w_self == ent["worst_p_max"]["self"] == 0.0
        w_h, _ = child_offense(g, s, boundary, {i: honest[i] for i in fr.out_nodes}, th, seq)
        assert w_h == ent["worst_p_max"]["honest"], (s, w_h)
