"""CPU, world_size 2 over gloo: the multi-GPU path's host logic.

Each rank takes its contiguous slice of a small decoder graph (shard.rank_slice),
computes its nodes' chunked tensor roots (oracle hashing stands in for the
kernels, which need a GPU), exchanges (root, record) rows with ONE all_gather
(shard.gather_node_records) and rank 0 builds the trace root: it must equal
the single-process trace root bit for bit, for any rank count."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _values():
    """Deterministic stand-in trace: one array per node (shape from the graph)."""
    from paper_2510_16028_b200.lowerings import DecoderShape, build_decoder
    shape = DecoderShape("tiny", layers=4, hidden=32, heads=2, kv_heads=1, head_dim=16,
                         inter=64, vocab=50, seq=8)
    spec = build_decoder(shape, device="cpu", seed=1)
    g = spec.graph
    rng = np.random.default_rng(0)
    vals = [rng.standard_normal(8 + (i % 5)).astype(np.float32) for i in range(g.n_nodes)]
    return g, vals


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import commit as OM
        from paper_2510_16028_b200 import shard
        g, vals = _values()
        start, end = shard.rank_slice(g, 4, rank, world)
        roots = torch.tensor(np.stack([np.frombuffer(OM.tensor_root(v, 64, OM.KECCAK256),
                                                     np.uint8) for v in vals[start:end]]))
        recs = torch.full((end - start, 56), rank, dtype=torch.uint8)
        full_roots, full_recs = shard.gather_node_records(roots, recs)
        if rank == 0:
            q.put((bytes(OM.trace_root([bytes(r) for r in full_roots.numpy()], OM.KECCAK256)),
                   full_recs[:, 0].tolist(), (start, end)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_trace_root_is_rank_count_invariant(world):
    from oracle import commit as OM
    from paper_2510_16028_b200 import shard
    g, vals = _values()
    ref = OM.trace_root([OM.tensor_root(v, 64, OM.KECCAK256) for v in vals], OM.KECCAK256)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, owners, _ = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got == ref
    # records arrive in canonical node order, each from the rank owning the node
    slices = [shard.rank_slice(g, 4, r, world) for r in range(world)]
    expect = [r for r, (s, e) in enumerate(slices) for _ in range(s, e)]
    assert owners == expect


def test_rank_slices_cover_graph_contiguously():
    from paper_2510_16028_b200 import shard
    g, _ = _values()
    for world in (1, 2, 3, 4):
        sl = [shard.rank_slice(g, 4, r, world) for r in range(world)]
        assert sl[0][0] == 0 and sl[-1][1] == g.n_nodes
        assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
        starts = shard.layer_starts(g)
        for s, _ in sl[1:]:
            assert s in starts
            # frontier of a layer-aligned slice is only the residual stream
            fr = shard.frontier_refs(g, s, g.n_nodes)
            assert len(fr) == 1
    with pytest.raises(ValueError):
        shard.rank_slice(g, 4, 0, 5)


def _bs_worker(rank, world, port, q):
    """Batch shards over gloo: each rank builds its shard's partial (oracle
    restatement stands in for the GPU kernel), packs it as a nao_check_partial
    row, one all_gather, rank 0 combines -> the whole tensor's verdicts."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import check as OC
        from paper_2510_16028_b200 import _lib, shard
        from paper_2510_16028_b200.dispute import partial_from_bytes
        y, yc, eps, ta, tr = _bs_data()
        B = 12
        lo, hi = shard.batch_range(B, rank, world)
        per = y.size // B
        part = OC.shard_partial(y[lo * per:hi * per], yc[lo * per:hi * per],
                                eps[lo * per:hi * per], ta, tr)
        row = _lib.CheckPartial()
        for f in ("n", "n_violations", "n_borderline", "n_nonfinite", "max_ratio"):
            setattr(row, f, part[f])
        for f in ("hist_abs", "hist_rel", "min_abs", "max_abs", "min_rel", "max_rel"):
            getattr(row, f)[:] = list(part[f])
        t = torch.frombuffer(bytearray(bytes(row)), dtype=torch.uint8)
        rows = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(rows, t)
        if rank == 0:
            parts = [[partial_from_bytes(x.numpy().tobytes())] for x in rows]
            rec = shard.combine_shard_records(parts, [(ta, tr)])[0]
            q.put(rec)
    finally:
        dist.destroy_process_group()


def _bs_data():
    from oracle import check as OC
    rng = np.random.default_rng(77)
    n = 12 * 500
    y = (rng.standard_normal(n) * 10.0 ** rng.integers(-2, 2, size=n)).astype(np.float32)
    yc = y.copy()
    idx = rng.random(n) < 0.3
    bits = yc.view(np.int32)
    bits[idx] += rng.integers(-4, 5, size=int(idx.sum())).astype(np.int32)
    eps = 3.0 * 2.0 ** -24 * np.abs(y.astype(np.float64))
    a, r = OC.elementwise_errors(y, yc)
    pa, pr = OC.percentile_profile(a), OC.percentile_profile(r)
    ta = pa * np.where(np.arange(pa.size) % 2 == 0, 1.0, 0.9)  # at / just below the truth
    tr = pr * np.where(np.arange(pr.size) % 3 == 0, 1.0, 1.2)
    return y, yc, eps, ta, tr


@pytest.mark.parametrize("world", [2, 3])
def test_batch_shard_partials_combine_over_gloo(world):
    from oracle import check as OC
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bs_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    rec = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    y, yc, eps, ta, tr = _bs_data()
    lc = OC.leaf_check(y, yc, eps)
    pm = OC.observed_p_max(y, yc, ta, tr)
    assert rec["n"] == y.size
    assert rec["n_violations"] == lc["n_violations"]
    assert rec["max_ratio"] == lc["max_ratio"]
    assert bool(rec["threshold_exceeded"]) == (pm > 1.0)
