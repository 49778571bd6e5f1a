"""GPU: the streaming hot path (executor.StreamingVerifier) end to end.

MLP (reference graph, sequential profile): per-node roots equal the oracle's
tensor roots of the reference values, check records equal the oracle's leaf
check / observed_p_max verdicts.  Small Qwen3-shaped decoder (native profile):
node-by-node bounds vs the oracle fed with the same GPU node inputs."""

import numpy as np
import pytest
import torch

from oracle import bounds as OB
from oracle import check as OC
from oracle import commit as OM

pytestmark = pytest.mark.gpu


def test_streaming_mlp_matches_oracle(ref_mlp):
    from paper_2510_16028_b200 import calibration
    from paper_2510_16028_b200.bounds import FpModel
    from paper_2510_16028_b200.engine import DeviceProfile
    from paper_2510_16028_b200.executor import StreamingVerifier, drift_claim
    from paper_2510_16028_b200.lowerings import build_mlp
    from paper_2510_16028_b200.tensor import Rng
    c = ref_mlp["config"]
    spec = build_mlp(c["seed"], c["batch"], c["in_dim"], c["hidden"], c["n_classes"])
    x = spec.make_inputs(Rng(*c["input_rng"]))
    th = calibration.ThresholdSet.from_json(ref_mlp["thresholds"])
    sv = StreamingVerifier(spec.graph, FpModel(), DeviceProfile("seq", "sequential"), th,
                           hash_alg="sha256", chunk_bytes=4096)
    claimed = {}

    def claimed_fn(node, y):
        yc = drift_claim(node, y, seed=1, period=8, fault_node="mm1")
        claimed[node.index] = yc
        return yc

    roots, recs = sv.run(x, claimed_fn)
    troot = sv.trace_root(roots)
    torch.cuda.synchronize()
    from paper_2510_16028_b200.dispute import CheckRecord
    from paper_2510_16028_b200.graph import parse_ref
    host_roots = roots.cpu().numpy()
    cl = {i: t.cpu().numpy() for i, t in claimed.items()}
    model = OB.FpModel()
    tree_roots = []
    for i, node in enumerate(spec.graph.nodes):
        # oracle: the reference leaf adjudication from the claimed inputs
        args = []
        for ref in node.inputs:
            cat, key = parse_ref(ref)
            args.append(cl[key] if cat == "node" else (x[key].array if cat == "input"
                                                        else spec.graph.weights[key].array))
        y_ref, eps = OB.op_bound(node, args, model)
        ref = OC.leaf_check(y_ref, cl[i], eps)
        rec = CheckRecord(recs[i]).host()
        # identical verdicts: the certified band is settled exactly (refine)
        assert rec["n_violations"] == ref["n_violations"], node.name
        assert rec["n_borderline"] == 0, node.name
        if node.name == "mm1":
            assert ref["n_violations"] > 0 and rec["n_violations"] > 0
        op = th.lookup(node.name)
        pm = OC.observed_p_max(y_ref, cl[i], op.tau_abs, op.tau_rel, th.grid, th.epsilon)
        assert bool(rec["threshold_exceeded"]) == (pm > 1.0), node.name
        assert bytes(host_roots[i]) == OM.tensor_root(cl[i], 4096), node.name
        tree_roots.append(bytes(host_roots[i]))
    assert bytes(troot.cpu().numpy()) == OM.trace_root(tree_roots)


def test_streaming_in_band_claims_match_oracle(ref_mlp):
    """Streaming verifier (fused commit+check, FP32 GEMM bounds) with claims
    planted inside the certified band of every linear node: per-node violation
    counts equal the oracle's leaf check exactly, nothing left undecided --
    also when the run is replayed as CUDA graphs."""
    from test_verdict_identity_gpu import plant_in_band
    from paper_2510_16028_b200.bounds import FpModel
    from paper_2510_16028_b200.dispute import CheckRecord
    from paper_2510_16028_b200.engine import DeviceProfile
    from paper_2510_16028_b200.executor import StreamingVerifier
    from paper_2510_16028_b200.graph import parse_ref
    from paper_2510_16028_b200.lowerings import build_mlp
    from paper_2510_16028_b200.tensor import Rng
    c = ref_mlp["config"]
    spec = build_mlp(c["seed"], c["batch"], c["in_dim"], c["hidden"], c["n_classes"])
    g = spec.graph
    x = spec.make_inputs(Rng(*c["input_rng"]))
    sv = StreamingVerifier(g, FpModel(), DeviceProfile("seq", "sequential"), None,
                           hash_alg="keccak256", chunk_bytes=4096)
    claimed, expect = {}, {}
    rng = np.random.default_rng(4)

    def claimed_fn(node, y):
        args = []
        for ref in node.inputs:
            cat, key = parse_ref(ref)
            args.append(claimed[key].cpu().numpy() if cat == "node" else
                        (x[key].array if cat == "input" else g.weights[key].array))
        y_ref, eps = OB.op_bound(node, args, OB.FpModel())
        cl = y_ref
        if node.kind == "linear":
            cl, _, _ = plant_in_band(y_ref, eps, rng, n_max=200, min_each=0)
        expect[node.index] = OC.leaf_check(y_ref, cl, eps)["n_violations"]
        claimed[node.index] = torch.from_numpy(np.ascontiguousarray(cl)).cuda()
        return claimed[node.index].clone()

    roots, recs = sv.run(x, claimed_fn)
    torch.cuda.synchronize()
    n_lin = 0
    for node in g.nodes:
        rec = CheckRecord(recs[node.index]).host()
        assert rec["n_violations"] == expect[node.index], node.name
        assert rec["n_borderline"] == 0, node.name
        n_lin += node.kind == "linear" and expect[node.index] > 0
    assert n_lin >= 1
    # graph replay: same records (the lists are reset by every refine pass)
    run = sv.capture(x, lambda node, y: claimed[node.index].clone())
    for _ in range(2):
        _, recs2 = run.replay()
        torch.cuda.synchronize()
        assert torch.equal(recs2, recs)


def test_streaming_decoder_bounds_vs_oracle():
    from paper_2510_16028_b200.bounds import FpModel, op_bound_device
    from paper_2510_16028_b200.executor import StreamingVerifier, drift_claim, plain_forward
    from paper_2510_16028_b200.graph import parse_ref
    from paper_2510_16028_b200.lowerings import DecoderShape, build_decoder
    from paper_2510_16028_b200.engine import NATIVE, to_device
    from paper_2510_16028_b200.tensor import Rng
    shape = DecoderShape("tiny-qwen", layers=2, hidden=128, heads=4, kv_heads=2, head_dim=32,
                         inter=256, vocab=500, seq=64)
    spec = build_decoder(shape, seed=3)
    g = spec.graph
    ids = spec.make_inputs(Rng(5))
    # node-by-node: GPU bound on the GPU's own node inputs vs oracle op_bound on the same inputs
    model = FpModel()
    values = {}
    for node in g.nodes:
        xs = []
        for ref in node.inputs:
            cat, key = parse_ref(ref)
            xs.append(values[key] if cat == "node" else to_device(
                ids[key] if cat == "input" else g.weights[key]))
        y, eps = op_bound_device(node, xs, model, NATIVE, eps_f64=True)
        values[node.index] = y
        ins = [a.cpu().numpy() for a in xs]
        if node.kind == "embedding":
            continue
        if node.kind in ("matmul", "linear"):
            tb = bool(node.attr("transpose_b", 0))
            K = ins[0].shape[-1]
            ref = OB.matmul_bound(ins[0], ins[1], OB.FpModel(), transpose_b=tb)
            if node.kind == "linear":
                ref = ref + 2.0 ** -24 * np.abs(y.cpu().numpy().astype(np.float64))
        else:
            yr, ref = OB.op_bound(node, ins, OB.FpModel())
            assert np.array_equal(yr.view(np.uint32), y.cpu().numpy().view(np.uint32)) or \
                node.kind in ("exp", "log", "tanh", "gelu", "silu"), node.name
        e = eps.cpu().numpy()
        assert np.all(e >= ref) and np.all(e <= ref * (1 + 1e-5)), node.name
    # and the streaming pipeline runs end to end (native profile) with a planted fault
    sv = StreamingVerifier(g, model, NATIVE, None, "keccak256", 4096)
    roots, recs = sv.run(ids, lambda node, y: drift_claim(node, y, 3, 16, "l1_down", 0.05, 2))
    from paper_2510_16028_b200.dispute import CheckRecord
    viol = {node.name: CheckRecord(recs[i]).host()["n_violations"] for i, node in enumerate(g.nodes)}
    assert viol["l1_down"] > 0
    outs = plain_forward(g, ids)
    assert set(outs) >= {g.n_nodes - 1}


@pytest.mark.parametrize("seg", [7, 1000])
def test_graphed_replay_matches_eager(seg):
    """StreamingVerifier.capture: CUDA-graph replay (segments of `seg` nodes,
    side streams forked/joined inside each graph) gives the eager run's roots,
    check records and outputs bit for bit, replay after replay, and follows
    in-place refills of the input buffer."""
    from paper_2510_16028_b200.bounds import FpModel
    from paper_2510_16028_b200.engine import to_device
    from paper_2510_16028_b200.executor import (GraphedRun, StreamingVerifier, drift_claim,
                                                plain_forward)
    from paper_2510_16028_b200.lowerings import DecoderShape, build_decoder
    from paper_2510_16028_b200.tensor import Rng
    shape = DecoderShape("tiny-qwen", layers=2, hidden=128, heads=4, kv_heads=2, head_dim=32,
                         inter=256, vocab=500, seq=64)
    spec = build_decoder(shape, seed=5)
    g = spec.graph
    ids = spec.make_inputs(Rng(11))
    sv = StreamingVerifier(g, FpModel(), hash_alg="keccak256", chunk_bytes=256)

    def claimed_fn(node, y):
        return drift_claim(node, y, seed=2, period=4, fault_node="l1_down")

    r0, c0 = sv.run(ids, claimed_fn)
    out0 = {k: v.clone() for k, v in sv.outputs.items()}
    r0, c0 = r0.clone(), c0.clone()
    gr = sv.capture(ids, claimed_fn, seg_nodes=seg)
    for _ in range(2):
        r1, c1 = gr.replay()
        torch.cuda.synchronize()
        assert torch.equal(r1, r0)
        assert torch.equal(c1, c0)
        for k, v in out0.items():
            assert torch.equal(gr.outputs[k], v)
    # refill the static input in place: replay follows the new ids
    ids2 = spec.make_inputs(Rng(12))
    ids_dev = to_device(ids["ids"])
    ids_dev.copy_(to_device(ids2["ids"]))
    r2, c2 = gr.replay()
    sv2 = StreamingVerifier(g, FpModel(), hash_alg="keccak256", chunk_bytes=256)
    r3, c3 = sv2.run(ids2, claimed_fn)
    torch.cuda.synchronize()
    assert torch.equal(r2, r3) and torch.equal(c2, c3)
    assert not torch.equal(r2, r0)
    # plain forward graphs: same values as eager
    gp = GraphedRun.record_plain(g, ids, "cuda", 0, None, None, seg_nodes=seg)
    gp.replay()
    ref = plain_forward(g, ids, "cuda")
    torch.cuda.synchronize()
    for k in ref:
        assert torch.equal(gp.outputs[k], ref[k])


@pytest.mark.parametrize("n", [1, 5, 1027, 65536 + 3])
def test_inject_drift_matches_numpy(n):
    """nao_inject_drift (float4 body + scalar tail) against a numpy restatement
    of its per-element hash."""
    from paper_2510_16028_b200.executor import inject_drift
    rng = np.random.default_rng(n)
    y = rng.standard_normal(n).astype(np.float32)
    y[::97] = 0.0
    seed, period, fs, fp = 1234, 5, 1e-3, 7
    out = inject_drift(torch.from_numpy(y).cuda(), seed, period, fs, fp).cpu().numpy()
    i = np.arange(n, dtype=np.uint64)
    m32 = np.uint64(0xFFFFFFFF)
    h = ((i * np.uint64(0x9E3779B1)) & m32) ^ np.uint64(seed)
    h ^= h >> np.uint64(16); h = (h * np.uint64(0x85EBCA6B)) & m32
    h ^= h >> np.uint64(13); h = (h * np.uint64(0xC2B2AE35)) & m32
    h ^= h >> np.uint64(16)
    ref = y.copy()
    flip = ((h % np.uint64(period)) == 0) & (y != 0) & np.isfinite(y)
    bits = ref.view(np.int32)
    step = np.where(((h >> np.uint64(20)) & np.uint64(1)) == 1, 1, -1).astype(np.int32)
    bits[flip] += step[flip]
    fault = ((h >> np.uint64(8)) % np.uint64(fp)) == 0
    ref[fault] = ref[fault] * (np.float32(1.0) + np.float32(fs))
    np.testing.assert_array_equal(out.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("world", [2, 3])
def test_layer_sharded_verification_matches_single_run(world):
    """The multi-GPU path's slices verified one after another on this GPU (real
    kernels): each "rank" runs its layer-aligned slice from the claimed
    residual stream at its frontier (graph.py:244-272); concatenated per-node
    roots / check records and the trace root equal the unsharded run's."""
    from paper_2510_16028_b200 import shard
    from paper_2510_16028_b200.bounds import FpModel
    from paper_2510_16028_b200.executor import StreamingVerifier, drift_claim
    from paper_2510_16028_b200.lowerings import DecoderShape, build_decoder
    from paper_2510_16028_b200.tensor import Rng
    shape = DecoderShape("tiny-qwen", layers=3, hidden=128, heads=4, kv_heads=2, head_dim=32,
                         inter=256, vocab=500, seq=64)
    spec = build_decoder(shape, seed=9)
    g = spec.graph
    ids = spec.make_inputs(Rng(5))
    claimed = {}

    def claimed_fn(node, y):
        yc = drift_claim(node, y, seed=4, period=8, fault_node="l1_up")
        claimed[node.index] = yc
        return yc

    sv = StreamingVerifier(g, FpModel(), hash_alg="keccak256", chunk_bytes=512)
    r_all, c_all = sv.run(ids, claimed_fn)
    t_all = sv.trace_root(r_all)
    roots, recs = [], []
    for rank in range(world):
        start, end = shard.rank_slice(g, shape.layers, rank, world)
        frontier = {k: claimed[k] for k in shard.frontier_refs(g, start, end)}
        svr = StreamingVerifier(g, FpModel(), hash_alg="keccak256", chunk_bytes=512)
        r, c = svr.run(ids, claimed_fn, start, end, frontier)
        roots.append(r)
        recs.append(c)
    r_cat, c_cat = torch.cat(roots), torch.cat(recs)
    torch.cuda.synchronize()
    assert torch.equal(r_cat, r_all)
    assert torch.equal(c_cat, c_all)
    assert torch.equal(sv.trace_root(r_cat), t_all)


@pytest.mark.parametrize("world", [2, 3])
def test_batch_sharded_verification_matches_whole_batch(world):
    """Batch shards (SURVEY 8(e), GPT-2-style B-major graph, sequential profile):
    each "rank" verifies the whole graph on its samples from the claimed trace's
    batch rows, commits its shard of every node (per-shard roots) and emits
    combinable partials; combine_shard_records gives, node by node, the
    unsharded run's violations, max ratio and exact percentile verdicts --
    with thresholds placed at, below and above the true percentiles."""
    from paper_2510_16028_b200 import shard
    from paper_2510_16028_b200.bounds import FpModel
    from paper_2510_16028_b200.calibration import (PERCENTILE_GRID, OpThresholds, ThresholdSet,
                                                   error_profiles_device)
    from paper_2510_16028_b200.commitments import commit_tensors
    from paper_2510_16028_b200.dispute import CheckRecord, partial_from_bytes
    from paper_2510_16028_b200.engine import DeviceProfile
    from paper_2510_16028_b200.executor import StreamingVerifier, drift_claim
    from paper_2510_16028_b200.lowerings import DecoderShape, build_decoder
    from paper_2510_16028_b200.tensor import Rng, Tensor
    B = 6
    base = DecoderShape("tiny-gpt2", layers=2, hidden=64, heads=2, kv_heads=2, head_dim=32,
                        inter=128, vocab=300, seq=32, batch=B, norm="ln", qk_norm=False,
                        rope=False, act="gelu", bias=True, eps=1e-5)
    seq = DeviceProfile("seq", "sequential")
    spec = build_decoder(base, seed=4)
    g = spec.graph
    ids = spec.make_inputs(Rng(8))
    claimed, local = {}, {}

    def claim_full(node, y):
        yc = drift_claim(node, y, seed=6, period=3, fault_node="l1_fc")
        claimed[node.index], local[node.index] = yc, y
        return yc

    StreamingVerifier(g, FpModel(), seq, hash_alg="keccak256", chunk_bytes=256).run(ids, claim_full)
    ops = []
    for k, node in enumerate(g.nodes):  # thresholds: at / below / above the true percentiles
        pa, pr = error_profiles_device(local[node.index], claimed[node.index])
        f = (1.0, 0.5, 3.0)[k % 3]
        ops.append(OpThresholds(node.name, pa.cpu().numpy() * f, pr.cpu().numpy() * f))
    ts = ThresholdSet(alpha=3.0, epsilon=1e-12, grid=PERCENTILE_GRID, ops=ops)
    sv = StreamingVerifier(g, FpModel(), seq, ts, hash_alg="keccak256", chunk_bytes=256)
    _, recs_full = sv.run(ids, lambda node, y: claimed[node.index])
    want = [CheckRecord(recs_full[i]).host() for i in range(g.n_nodes)]

    parts_by_rank, roots_by_rank = [], []
    ids_full = torch.from_numpy(np.array(ids["ids"].array)).reshape(B, -1)
    for r in range(world):
        lo, hi = shard.batch_range(B, r, world)
        shp = DecoderShape(**{**base.__dict__, "batch": hi - lo})
        spec_r = build_decoder(shp, seed=4)
        ids_r = {"ids": Tensor((hi - lo, base.seq), ids_full[lo:hi].float().cuda().reshape(-1))}
        svr = StreamingVerifier(spec_r.graph, FpModel(), seq, ts, hash_alg="keccak256",
                                chunk_bytes=256, partial=True)
        roots, recs = svr.run(ids_r, lambda node, y: shard.batch_rows(
            claimed[node.index], B, r, world).clone().reshape(y.shape))
        torch.cuda.synchronize()
        parts_by_rank.append([partial_from_bytes(recs[i].cpu().numpy().tobytes())
                              for i in range(g.n_nodes)])
        roots_by_rank.append(roots)
        # per-shard roots are the roots of the claimed trace's batch rows
        for i in (0, 5, g.n_nodes - 1):
            sl = shard.batch_rows(claimed[i], B, r, world).contiguous()
            assert torch.equal(roots[i], commit_tensors([sl], 256, "keccak256")[0])
    got = shard.combine_shard_records(
        parts_by_rank, [(ts.lookup(n.name).tau_abs, ts.lookup(n.name).tau_rel) for n in g.nodes])
    exceeded = 0
    for i, node in enumerate(g.nodes):
        for f in ("n", "n_violations", "n_borderline", "n_nonfinite", "threshold_exceeded",
                  "first_exceeded", "max_ratio"):
            assert got[i][f] == want[i][f], (node.name, f, got[i][f], want[i][f])
        exceeded += got[i]["threshold_exceeded"]
    assert exceeded > 0 and got[[n.name for n in g.nodes].index("l1_fc")]["n_violations"] > 0
    assert len(shard.shard_trace_root(roots_by_rank)) == 32


def test_graphed_replay_survives_workspace_growth():
    """Scratch grown between captured segments (small nodes first, a large one
    later; 1 MiB minimum workspace) must not free the buffer earlier segments
    were recorded with (regression: SD-UNet batch 1, illegal address on replay)."""
    from paper_2510_16028_b200 import _lib
    from paper_2510_16028_b200.bounds import FpModel
    from paper_2510_16028_b200.executor import StreamingVerifier, drift_claim
    from paper_2510_16028_b200.graph import build_graph, input_ref
    from paper_2510_16028_b200.lowerings import _Builder
    b = _Builder()
    h = b.add("a0", "exp", [input_ref("x")])
    for i in range(1, 6):
        h = b.add(f"a{i}", "tanh", [h])
    big = b.add("wide", "concat", [h] * 4096, {"axis": 1})
    out = b.add("out", "relu", [big])
    g = build_graph(b.nodes, [("x", (64, 64))], b.weights, [out])
    x = {"x": torch.randn((64, 64), device="cuda") * 0.1}
    sv = StreamingVerifier(g, FpModel(), hash_alg="keccak256", chunk_bytes=64)
    claimed = lambda node, y: drift_claim(node, y, seed=1, period=4)  # noqa: E731
    r0, c0 = sv.run(x, claimed)
    r0, c0 = r0.clone(), c0.clone()
    _lib._ws.clear()  # force growth inside the capture
    kept = len(_lib._ws_captured)
    gr = sv.capture(x, claimed, seg_nodes=2)
    assert len(_lib._ws_captured) > kept  # the outgrown buffer stays alive with the graph
    torch.cuda.empty_cache()
    for _ in range(3):
        r1, c1 = gr.replay()
        torch.cuda.synchronize()
        assert torch.equal(r1, r0) and torch.equal(c1, c0)


def test_streaming_conv_in_band_claims_match_oracle():
    """A small ResNet (conv -> BN -> relu, maxpool, residual blocks) through the
    streaming verifier with claims planted inside the certified band of every
    conv node (FP32 tensor-core bounds, conv refine by implicit-im2col
    double-double dots): per-node violation counts equal the oracle's exactly,
    nothing undecided."""
    from test_verdict_identity_gpu import plant_in_band
    from paper_2510_16028_b200.bounds import FpModel
    from paper_2510_16028_b200.dispute import CheckRecord
    from paper_2510_16028_b200.engine import DeviceProfile
    from paper_2510_16028_b200.executor import StreamingVerifier
    from paper_2510_16028_b200.graph import parse_ref
    from paper_2510_16028_b200.lowerings import build_resnet18
    from paper_2510_16028_b200.tensor import Rng
    spec = build_resnet18(batch=2, side=32, n_classes=10, width=16)
    g = spec.graph
    x = spec.make_inputs(Rng(3))
    sv = StreamingVerifier(g, FpModel(), DeviceProfile("seq", "sequential"), None,
                           hash_alg="keccak256", chunk_bytes=1024)
    claimed, expect = {}, {}
    rng = np.random.default_rng(6)

    def claimed_fn(node, y):
        args = []
        for ref in node.inputs:
            cat, key = parse_ref(ref)
            args.append(claimed[key].cpu().numpy() if cat == "node" else
                        (x[key].array if cat == "input" else g.weights[key].array))
        if node.kind == "conv2d":
            y_ref, eps = OB.op_bound(node, args, OB.FpModel())
            assert np.array_equal(y_ref.view(np.uint32), y.cpu().numpy().view(np.uint32))
            cl, _, _ = plant_in_band(y_ref, eps, rng, n_max=100, min_each=0)
            expect[node.index] = OC.leaf_check(y_ref, cl, eps)["n_violations"]
        else:
            cl = y.cpu().numpy()
        claimed[node.index] = torch.from_numpy(np.ascontiguousarray(cl)).cuda()
        return claimed[node.index].clone()

    roots, recs = sv.run(x, claimed_fn)
    torch.cuda.synchronize()
    planted = 0
    for node in g.nodes:
        rec = CheckRecord(recs[node.index]).host()
        assert rec["n_borderline"] == 0, node.name
        if node.index in expect:
            assert rec["n_violations"] == expect[node.index], node.name
            planted += expect[node.index]
        else:
            assert rec["n_violations"] == 0, node.name
    assert planted > 0


@pytest.mark.parametrize("seg", [7, 1000])
def test_stream_options_keep_roots_and_records(seg):
    """The verifier's stream options -- abs-GEMM bounds on their own stream,
    claims made on a claim stream, the commit stream at another priority --
    give the serial run's roots and check records, eagerly and replayed as
    CUDA graphs (segments of `seg` nodes)."""
    import os
    from paper_2510_16028_b200.bounds import FpModel
    from paper_2510_16028_b200.executor import StreamingVerifier, drift_claim
    from paper_2510_16028_b200.lowerings import DecoderShape, build_decoder
    from paper_2510_16028_b200.tensor import Rng
    shape = DecoderShape("tiny-qwen", layers=2, hidden=128, heads=4, kv_heads=2, head_dim=32,
                         inter=256, vocab=500, seq=64)
    spec = build_decoder(shape, seed=7)
    g = spec.graph
    ids = spec.make_inputs(Rng(13))

    def claimed_fn(node, y):
        return drift_claim(node, y, seed=3, period=4, fault_node="l1_up")

    ref = StreamingVerifier(g, FpModel(), hash_alg="keccak256", chunk_bytes=256, overlap=False)
    r0, c0 = ref.run(ids, claimed_fn)
    r0, c0 = r0.clone(), c0.clone()
    sv = StreamingVerifier(g, FpModel(), hash_alg="keccak256", chunk_bytes=256,
                           claim_stream=True, commit_priority=-1, bound_stream=True)
    assert sv._s_bnd is not None and sv._s_clm is not None
    r1, c1 = sv.run(ids, claimed_fn)
    torch.cuda.synchronize()
    assert torch.equal(r1, r0) and torch.equal(c1, c0)
    sv.release()  # the eager run's deferred frees
    assert sv._deferred == []
    gr = sv.capture(ids, claimed_fn, seg_nodes=seg)
    for _ in range(2):
        r2, c2 = gr.replay()
        torch.cuda.synchronize()
        assert torch.equal(r2, r0) and torch.equal(c2, c0)


def test_reference_digest_cache_follows_in_place_updates():
    """The broadcast-reference digests (causal-mask shortcut) are recommitted
    after an in-place update of the reference tensor."""
    from paper_2510_16028_b200.bounds import FpModel
    from paper_2510_16028_b200.commitments import commit_tensors
    from paper_2510_16028_b200.executor import StreamingVerifier
    from paper_2510_16028_b200.lowerings import DecoderShape, build_decoder
    shape = DecoderShape("tiny-qwen", layers=1, hidden=128, heads=4, kv_heads=2, head_dim=32,
                         inter=256, vocab=500, seq=64)
    sv = StreamingVerifier(build_decoder(shape, seed=1).graph, FpModel(), hash_alg="keccak256",
                           chunk_bytes=4096)
    w = torch.randn(64, 256, device="cuda")
    p1 = sv._ref_chunk_digests(w)
    assert sv._ref_chunk_digests(w) == p1  # cached
    w.add_(1.0)
    p2 = sv._ref_chunk_digests(w)
    assert p2[0] == p1[0] and p2[1] != p1[1]
    ref = torch.empty((1 + w.numel() * 4 // 4096, 32), dtype=torch.uint8, device="cuda")
    commit_tensors([w], 4096, "keccak256", leaf_digests=ref)
    got = [v for v in sv._ref_cache.values() if v[1].data_ptr() + 32 == p2[1]][0][1]
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
