"""ORACLE -- TEST INFRASTRUCTURE ONLY.  Golden vectors of the dispute-time
records written by the UNMODIFIED reference for the
MLP 784-256-10 B=64 graph (inputs Rng(7, 0), sequential profile):

  * make_subgraph_record (commitments.py:283-304): h_in / h_out and proof
    wires for each child of partition(Slice(0, n), 3) and of partition(child0, 2);
  * the challenger's child re-execution (dispute.py:544-559): run_subgraph
    under the sequential profile, graph_flops, and the worst live-out p_max
    against the honest pairwise trace and a faulted one;
  * thresholds_tree (commitments.py:250-256) root of the golden thresholds.

    python oracle/gen_golden_subgraph.py    # writes tests/golden/ref_subgraph.json

Nothing here is imported at test time.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True  # never write into /root/reference
REF_SRC = "/root/reference/pkg/src"
ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden" / "ref_subgraph.json"


def main():
    sys.path.insert(0, REF_SRC)
    from fpverify import commitments as CM
    from fpverify import dispute as D
    from fpverify.calibration import ThresholdSet
    from fpverify.engine import DeviceProfile, execute, graph_flops, run_subgraph
    from fpverify.graph import Slice, extract_subgraph, frontiers, partition
    from fpverify.models import build_mlp
    from fpverify.tensor import Rng

    mlp = json.load(open(ROOT / "tests" / "golden" / "ref_mlp_784_256_10_b64.json"))
    c = mlp["config"]
    spec = build_mlp(seed=c["seed"], batch=c["batch"], in_dim=c["in_dim"], hidden=c["hidden"],
                     n_classes=c["n_classes"])
    g = spec.graph
    x = spec.make_inputs(Rng(*c["input_rng"]))
    th = ThresholdSet.from_json(mlp["thresholds"])
    seq = DeviceProfile("seq", "sequential")
    _, trace = execute(g, x, seq)
    _, honest = execute(g, x, DeviceProfile("pair", "pairwise"))
    inj_node = mlp["injection"]["node"]
    inj = D.make_injection(th, g.nodes[inj_node].name, trace.tensors[inj_node].shape, 10.0)
    _, faulty = execute(g, x, seq, inject={inj_node: inj})
    wtree, wnames = CM.weight_tree(g.weights)
    gtree = CM.graph_tree(g)

    top = partition(Slice(0, g.n_nodes), 3)
    slices = list(top) + list(partition(top[0], 2))
    out = []
    for s in slices:
        rec = CM.make_subgraph_record(g, s, trace.tensors, x, wtree, wnames, gtree)
        fr = frontiers(g, s)
        ins = ([x[n] for n in fr.in_inputs] + [g.weights[n] for n in fr.in_weights]
               + [trace.tensors[i] for i in fr.in_nodes])
        outs = [trace.tensors[i] for i in fr.out_nodes]
        ok = CM.verify_subgraph_record(rec, g, wtree.root, gtree.root, ins, outs)
        module = extract_subgraph(g, s)
        boundary = {}
        for ref in module.placeholder_refs:
            cat, key = ref.split(":", 1)
            boundary[ref] = x[key] if cat == "input" else trace.tensors[int(key)]
        outputs, sub_trace = run_subgraph(module, boundary, seq)
        flops = graph_flops(module.graph, sub_trace)
        worst = {}
        for tag, claimed in (("self", trace), ("honest", honest), ("fault", faulty)):
            w = 0.0
            for li, pi in enumerate(module.out_nodes):
                w = max(w, D.observed_p_max(outputs[li], claimed.tensors[pi], th,
                                            g.nodes[pi].name))
            worst[tag] = w
        out.append({"start": s.start, "end": s.end, "h_in": rec.h_in.hex(),
                    "h_out": rec.h_out.hex(), "verified": bool(ok),
                    "weight_proofs": {n: p.to_wire().hex() for n, p in rec.weight_proofs},
                    "sig_proofs": {str(i): p.to_wire().hex() for i, p in rec.sig_proofs},
                    "out_nodes": list(module.out_nodes), "in_nodes": list(fr.in_nodes),
                    "flops": int(flops), "worst_p_max": worst})
    doc = {"slices": out, "weight_root": wtree.root.hex(), "graph_root": gtree.root.hex(),
           "thresholds_root": CM.thresholds_tree(mlp["thresholds"]).root.hex(),
           "injection": {"node": inj_node, "value": float(inj.reshape(-1)[0])}}
    json.dump(doc, open(OUT, "w"), indent=1, sort_keys=True)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
