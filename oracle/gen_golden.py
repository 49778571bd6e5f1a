"""ORACLE -- TEST INFRASTRUCTURE ONLY.  Generates tests/golden/* by running the
UNMODIFIED reference (/root/reference/pkg/src/fpverify) in the build
container.  The reference cannot travel to the GPU box, so its outputs are
committed as small fixtures; this script is how they were made:

    python oracle/gen_golden.py        # writes tests/golden/{ref_*.json,ref_ops.npz}

Nothing here is imported at test time.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True  # never write into /root/reference
REF_SRC = "/root/reference/pkg/src"
REF_GOLDEN = "/root/reference/pkg/tests/golden/commitment_vectors.json"
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def main():
    sys.path.insert(0, REF_SRC)
    from fpverify import bounds as B
    from fpverify import calibration as C
    from fpverify import commitments as CM
    from fpverify import dispute as D
    from fpverify.engine import DeviceProfile, apply_op, execute
    from fpverify.graph import build_graph, input_ref, make_node, node_ref
    from fpverify.models import build_mlp
    from fpverify.tensor import Rng, tensor_new

    OUT.mkdir(parents=True, exist_ok=True)

    # ---------------------------------------------------------------- 1. commitment vectors
    ref_vec = json.load(open(REF_GOLDEN))
    t = tensor_new([2, 2], [1.0, -2.0, 0.5, 4.0])
    mine = {
        "canon_2x2": CM.sha256(CM.canon_tensor(t)).hex(),
        "signature_matmul": CM.sha256(CM.op_signature(make_node(
            "mm", "matmul", [input_ref("x"), "weight:w"], {"transpose_b": 1}))).hex(),
        "tree_root_5": CM.build_tree([f"leaf{i}".encode() for i in range(5)]).root.hex(),
        "proof_wire_5_2": CM.prove(CM.build_tree([f"leaf{i}".encode() for i in range(5)]),
                                   2).to_wire().hex(),
    }
    assert mine == ref_vec, (mine, ref_vec)
    vec = dict(ref_vec)
    vec["canon_2x2_bytes"] = CM.canon_tensor(t).hex()
    # build_tree over n byte-leaves for several n (odd-node pairing cases)
    vec["tree_roots"] = {
        str(n): CM.build_tree([bytes([i % 256]) * (i % 7 + 1) for i in range(n)]).root.hex()
        for n in (1, 2, 3, 4, 5, 7, 8, 9, 31, 64, 100, 257, 1000)}
    json.dump(vec, open(OUT / "reference_commitment_vectors.json", "w"), indent=1,
              sort_keys=True)

    # ---------------------------------------------------------------- 2. op-level bounds
    ops = {}
    rng = Rng(2024)
    models = {"prob": B.FpModel(), "det": B.FpModel(mode="deterministic")}
    seq = DeviceProfile("seq", "sequential")
    seqf = DeviceProfile("seqf", "sequential", fma=True)

    def run(tag, node, shapes_inputs, model="prob", prof=seq, transform=None):
        g = build_graph([node], [(f"a{i}", s.shape) for i, s in enumerate(shapes_inputs)], {},
                        [node_ref(0)])
        arrs = [s.array if transform is None else transform(i, s.array)
                for i, s in enumerate(shapes_inputs)]
        y, eps = B.op_bound(g.nodes[0], arrs, models[model], prof)
        for i, a in enumerate(arrs):
            ops[f"{tag}/in{i}"] = np.asarray(a, dtype=np.float32)
        ops[f"{tag}/y"] = np.asarray(y, dtype=np.float32)
        ops[f"{tag}/eps"] = np.asarray(eps, dtype=np.float64)

    def mk(kind, n_in, attrs=None):
        return make_node("op", kind, [input_ref(f"a{i}") for i in range(n_in)], attrs)

    run("softmax_prob", mk("softmax", 1, {"axis": -1}), [rng.uniform((33, 257), -4, 4)])
    run("softmax_det", mk("softmax", 1, {"axis": -1}), [rng.uniform((7, 3, 64), -8, 8)], "det")
    run("softmax_axis0", mk("softmax", 1, {"axis": 0}), [rng.uniform((40, 9), -3, 3)])
    run("softmax_n1", mk("softmax", 1, {"axis": -1}), [rng.uniform((5, 1), -1, 1)], "det")
    run("layernorm_prob", mk("layernorm", 1, {"axis": -1, "eps": 1e-5}),
        [rng.uniform((17, 300), -2, 3)])
    run("layernorm_det", mk("layernorm", 1, {"axis": -1, "eps": 1e-3}),
        [rng.uniform((4, 5, 96), -1, 1)], "det")
    run("sum_prob", mk("sum", 1, {"axis": -1}), [rng.uniform((19, 513), -1, 1)])
    run("sum_axis0", mk("sum", 1, {"axis": 0}), [rng.uniform((50, 6), -1, 1)], "det")
    run("mean_prob", mk("mean", 1, {"axis": 1}), [rng.uniform((8, 77, 5), -3, 1)])
    run("matmul_prob", mk("matmul", 2), [rng.uniform((37, 70), -2, 2), rng.uniform((70, 45), -2, 2)])
    run("matmul_det_tb", mk("matmul", 2, {"transpose_b": 1}),
        [rng.uniform((3, 20, 33), -1, 1), rng.uniform((3, 18, 33), -1, 1)], "det")
    run("matmul_fma", mk("matmul", 2), [rng.uniform((9, 100), -1, 1),
                                        rng.uniform((100, 13), -1, 1)], "prob", seqf)
    run("matmul_bcast", mk("matmul", 2), [rng.uniform((2, 3, 11, 24), -1, 1),
                                          rng.uniform((24, 10), -1, 1)])
    run("linear_prob", mk("linear", 3), [rng.uniform((12, 64), -1, 1),
                                         rng.uniform((64, 40), -0.3, 0.3),
                                         rng.uniform((40,), -0.1, 0.1)])
    for kind, lo, hi in (("add", -2, 2), ("sub", -2, 2), ("mul", -2, 2), ("div", 0.5, 2)):
        run(f"{kind}", mk(kind, 2), [rng.uniform((31, 17), lo, hi), rng.uniform((17,), lo, hi)])
    run("neg", mk("neg", 1), [rng.uniform((300,), -1, 1)])
    for kind, lo, hi in (("exp", -5, 5), ("log", 0.01, 9), ("sqrt", 0, 9), ("rsqrt", 0.01, 9),
                         ("tanh", -4, 4), ("gelu", -6, 6), ("silu", -6, 6), ("relu", -1, 1)):
        run(f"{kind}", mk(kind, 1), [rng.uniform((29, 41), lo, hi)])
    run("max", mk("max", 1, {"axis": -1}), [rng.uniform((6, 50), -1, 1)])
    run("min", mk("min", 1, {"axis": 0}), [rng.uniform((6, 50), -1, 1)])
    np.savez_compressed(OUT / "ref_ops.npz", **ops)

    # ---------------------------------------------------------------- 3. MLP 784-256-10 B=64
    spec = build_mlp(seed=0, batch=64, in_dim=784, hidden=256, n_classes=10)
    g = spec.graph
    x = spec.make_inputs(Rng(7))
    doc = {"config": {"seed": 0, "batch": 64, "in_dim": 784, "hidden": 256, "n_classes": 10,
                      "input_rng": [7, 0], "input_range": [-1.0, 1.0]},
           "graph_root": CM.graph_tree(g).root.hex(),
           "signatures": [hashlib.sha256(CM.op_signature(n)).hexdigest() for n in g.nodes],
           "nodes": [{"name": n.name, "kind": n.kind, "inputs": list(n.inputs),
                      "attrs": {k: v for k, v in n.attrs}} for n in g.nodes],
           "weights": {k: {"shape": list(v.shape), "digest": CM.tensor_digest(v)}
                       for k, v in sorted(g.weights.items())},
           "input_digest": CM.tensor_digest(x["x"])}
    sample_rng = np.random.default_rng(0)
    runs = {}
    traces = {}
    for pname, prof in (("seq", seq), ("seqf", seqf)):
        for mname in ("prob", "det"):
            _, bnds, tr = B.co_execute(g, x, prof, models[mname], with_trace=True)
            traces[(pname, mname)] = tr
            per = []
            for i, (tt, bt) in enumerate(zip(tr.tensors, bnds)):
                n_el = tt.size
                idx = np.unique(sample_rng.integers(0, n_el, size=min(64, n_el)))
                ent = {"value_digest": CM.tensor_digest(tt), "shape": list(tt.shape),
                       "eps_sum": float(bt.eps.sum()), "eps_max": float(bt.eps.max()),
                       "eps_min": float(bt.eps.min()), "idx": idx.tolist(),
                       "eps_sample": [float(v) for v in bt.eps[idx]],
                       "value_sample": [float(v) for v in tt.data[idx]]}
                if mname == "prob":
                    header = CM.canon_tensor(tt)[: 5 + 16 * len(tt.shape)]
                    payload = tt.data.astype("<f4").tobytes()
                    for chunk in (256, 4096):
                        leaves = [header] + [payload[o:o + chunk]
                                             for o in range(0, len(payload), chunk)]
                        ent[f"root_sha256_c{chunk}"] = CM.build_tree(leaves).root.hex()
                per.append(ent)
            runs[f"{pname}/{mname}"] = per
    doc["runs"] = runs
    roots = [bytes.fromhex(e["root_sha256_c4096"]) for e in runs["seq/prob"]]
    doc["trace_root_sha256_c4096"] = CM.build_tree(roots).root.hex()

    # thresholds over the reference default fleet + calibration extras
    fleet = [DeviceProfile.from_spec(s) for s in
             ("sequential", "pairwise", "blocked:32", "permuted:7+fma", "permuted:3", "blocked:4")]
    rng_cal = Rng(101)
    dataset = [spec.make_inputs(rng_cal) for _ in range(12)]
    env = C.calibrate(g, dataset, fleet)
    th = C.build_thresholds(env, alpha=3.0)
    doc["thresholds"] = th.to_json()

    # check goldens: local = sequential trace; claimed = pairwise (honest drift),
    # fault injection (make_injection, dispute.py:369-372), 0.4x / 1.5x eps at the head
    local = traces[("seq", "prob")]
    _, honest = execute(g, x, DeviceProfile("pair", "pairwise"))
    inj_node = [n.index for n in g.nodes if n.name == "mm1"][0]
    inj = D.make_injection(th, "mm1", local.tensors[inj_node].shape, 10.0)
    _, faulty = execute(g, x, seq, inject={inj_node: inj})
    checks = {}
    for cname, claimed in (("honest", honest), ("fault", faulty)):
        per = []
        for i, n in enumerate(g.nodes):
            lt, ct = local.tensors[i], claimed.tensors[i]
            ab, rl = C.elementwise_errors(lt, ct, th.epsilon)
            per.append({"abs_prof": [float(v) for v in C.percentile_profile(ab, th.grid)],
                        "rel_prof": [float(v) for v in C.percentile_profile(rl, th.grid)],
                        "p_max": D.observed_p_max(lt, ct, th, n.name),
                        "claimed_digest": CM.tensor_digest(ct)})
        checks[cname] = per
    doc["checks"] = checks
    doc["injection"] = {"node": inj_node, "scale": 10.0, "value": float(inj.reshape(-1)[0])}
    json.dump(doc, open(OUT / "ref_mlp_784_256_10_b64.json", "w"), indent=0, sort_keys=True)
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
