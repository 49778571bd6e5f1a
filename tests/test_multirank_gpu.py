"""GPU, world_size 2 and 3 over gloo, every rank a separate process on cuda:0:
the multi-GPU path end to end with the real kernels (the one-GPU gpurun box
stands in for the 8-GPU node; NCCL and gloo run the same shard code).

Each rank regenerates the deterministic claimed trace of a small Qwen3-shaped
decoder (proposer harness with a planted fault), verifies only its
layer-aligned slice from the claimed residual stream at its frontier
(shard.rank_slice / frontier_refs; graph.py:244-272), exchanges (root,
record) rows with ONE all_gather (shard.gather_node_records), and rank 0
builds the trace root.  Roots, check records and the trace root must equal
the single-process run's, and the fault must be reported at its own node."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SHAPE = dict(name="tiny-qwen", layers=4, hidden=128, heads=4, kv_heads=2, head_dim=32,
             inter=256, vocab=500, seq=64)
FAULT = "l2_up"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    from paper_2510_16028_b200.lowerings import DecoderShape, build_decoder
    from paper_2510_16028_b200.tensor import Rng
    shape = DecoderShape(**SHAPE)
    spec = build_decoder(shape, seed=9)
    return shape, spec.graph, spec.make_inputs(Rng(5))


def _claimed_fn(store):
    from paper_2510_16028_b200.executor import drift_claim

    def fn(node, y):
        yc = drift_claim(node, y, seed=4, period=8, fault_node=FAULT)
        store[node.index] = yc
        return yc
    return fn


def _verifier(g):
    from paper_2510_16028_b200.bounds import FpModel
    from paper_2510_16028_b200.executor import StreamingVerifier
    return StreamingVerifier(g, FpModel(), hash_alg="keccak256", chunk_bytes=512)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2510_16028_b200 import shard
        shape, g, ids = _setup()
        start, end = shard.rank_slice(g, shape.layers, rank, world)
        # the claimed trace up to this slice (the committed frontier tensors)
        claimed = {}
        if start > 0:
            _verifier(g).run(ids, _claimed_fn(claimed), 0, start)
        frontier = {k: claimed[k] for k in shard.frontier_refs(g, start, end)}
        roots, recs = _verifier(g).run(ids, _claimed_fn({}), start, end, frontier)
        torch.cuda.synchronize()
        all_roots, all_recs = shard.gather_node_records(roots.cpu(), recs.cpu())
        if rank == 0:
            troot = _verifier(g).trace_root(all_roots.cuda()).cpu()
            q.put((all_roots.numpy().tobytes(), all_recs.numpy().tobytes(),
                   troot.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_shards_match_single_run(world):
    from paper_2510_16028_b200.dispute import CheckRecord
    shape, g, ids = _setup()
    sv = _verifier(g)
    r_all, c_all = sv.run(ids, _claimed_fn({}))
    t_all = sv.trace_root(r_all)
    torch.cuda.synchronize()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    roots_b, recs_b, troot_b = q.get(timeout=600)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert roots_b == r_all.cpu().numpy().tobytes()
    assert recs_b == c_all.cpu().numpy().tobytes()
    assert troot_b == t_all.cpu().numpy().tobytes()
    flagged = [g.nodes[i].name for i in range(g.n_nodes)
               if CheckRecord(c_all[i]).host()["n_violations"]]
    assert flagged == [FAULT]
