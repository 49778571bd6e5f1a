"""Multi-GPU sharding of the verified forward.

Two unit kinds, both without a data-path collective:
  * layer slices (below) for single-sequence models (Qwen3-8B, S=2048);
  * batch shards (batch_rows, combine_shard_records) for the batched configs
    (GPT-2 B=8, SD-UNet B=8): samples are independent, every rank verifies the
    whole graph on its samples, commits each node's shard as its own tensor
    (per-shard roots, north_star (5)) and emits combinable check partials, from
    which rank 0 decides every node's verdict exactly as on the whole tensor.

Units are contiguous canonical-order op slices -- the reference's partition
unit (graph.py:275-293) -- aligned to layer boundaries so that each rank's
frontier is the residual stream (the reference re-executes a child slice from
its committed frontier tensors, graph.py:244-272, dispute.py:544-559).
There is no data-path collective: ranks verify independently, then ONE
all_gather of fixed-size per-node records (32 B root + check record) lets
rank 0 build the trace root over all node roots in canonical order, which is
bit-exact for any number of ranks.  Works over NCCL (CUDA tensors) or gloo
(CPU tensors, tests/test_multirank.py).
"""

from __future__ import annotations

import torch

from .graph import parse_ref


def layer_starts(graph) -> list:
    """Index of the first node of every decoder layer (names 'l{k}_*')."""
    starts = []
    for i, n in enumerate(graph.nodes):
        head = n.name.split("_")[0]
        if head.startswith("l") and head[1:].isdigit() and int(head[1:]) == len(starts):
            starts.append(i)
    return starts


def rank_slice(graph, n_layers: int, rank: int, world: int):
    """[start, end) of rank's slice: layers split into contiguous groups whose
    sizes differ by <= 1 (larger first, like partition); rank 0 also owns the
    prologue, the last rank the epilogue."""
    if world <= 1:
        return 0, graph.n_nodes
    starts = layer_starts(graph)
    if len(starts) < world:
        raise ValueError(f"{len(starts)} layers cannot be split over {world} ranks")
    base, extra = divmod(n_layers, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    start = 0 if rank == 0 else starts[lo]
    end = graph.n_nodes if rank == world - 1 else starts[hi]
    return start, end


def frontier_refs(graph, start: int, end: int) -> list:
    """External producer nodes consumed inside [start, end) (frontiers, graph.py:193-225)."""
    need = set()
    for node in graph.nodes[start:end]:
        for ref in node.inputs:
            cat, key = parse_ref(ref)
            if cat == "node" and key < start:
                need.add(key)
    return sorted(need)


def gather_node_records(roots: torch.Tensor, records: torch.Tensor, group=None, dst: int = 0):
    """All-gather per-node (root, record) rows from every rank's slice; returns
    the concatenation in rank order (== canonical node order) on every rank.
    Rows are padded to the largest slice so one fixed-size collective suffices."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if world == 1:
        return roots, records
    dev = roots.device
    n_local = torch.tensor([roots.shape[0]], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    row = torch.zeros((mx, 32 + records.shape[1]), dtype=torch.uint8, device=dev)
    row[:roots.shape[0], :32] = roots
    row[:roots.shape[0], 32:] = records
    out = [torch.empty_like(row) for _ in range(world)]
    dist.all_gather(out, row, group=group)
    full = torch.cat([o[:s] for o, s in zip(out, sizes)])
    return full[:, :32].contiguous(), full[:, 32:].contiguous()


# ------------------------------------------------------------ batch shards

def batch_range(batch: int, rank: int, world: int):
    """[lo, hi) samples of rank (contiguous, sizes differ by <= 1, larger first)."""
    base, extra = divmod(int(batch), int(world))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def batch_rows(t: torch.Tensor, batch: int, rank: int, world: int) -> torch.Tensor:
    """The rank's samples of a batch-major tensor (leading extent = batch x k)."""
    lo, hi = batch_range(batch, rank, world)
    per = t.shape[0] // batch
    return t[lo * per:hi * per]


def combine_shard_records(partials_by_rank, thresholds_by_node, grid=None) -> list:
    """Rank 0 after the gather: per node, combine the shards' nao_check_partial
    rows (dispute.combine_partials) into the whole tensor's record.
    partials_by_rank[r][i] = decoded partial dict of node i on rank r;
    thresholds_by_node[i] = (tau_abs, tau_rel)."""
    from .calibration import PERCENTILE_GRID
    from .dispute import combine_partials
    grid = PERCENTILE_GRID if grid is None else grid
    n_nodes = len(partials_by_rank[0])
    out = []
    for i in range(n_nodes):
        parts = [partials_by_rank[r][i] for r in range(len(partials_by_rank))
                 if partials_by_rank[r][i]["n"] > 0]
        ta, tr = thresholds_by_node[i]
        out.append(combine_partials(parts, ta, tr, grid) if parts else
                   {"n": 0, "n_violations": 0, "n_borderline": 0, "n_nonfinite": 0,
                    "max_ratio": 0.0, "threshold_exceeded": 0, "first_exceeded": -1})
    return out


def shard_trace_root(roots_by_rank, alg="keccak256") -> bytes:
    """Trace root of a batch-sharded run: Merkle tree over the per-(node, shard)
    roots in node-major, rank-minor order (leaf = H(0x00 || root))."""
    from .commitments import build_tree
    leaves = []
    n_nodes = roots_by_rank[0].shape[0]
    host = [r.cpu().numpy() for r in roots_by_rank]
    for i in range(n_nodes):
        for h in host:
            leaves.append(bytes(h[i]))
    return build_tree(leaves, alg).root
