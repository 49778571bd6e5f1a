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


def _weight_numel(graph, ref) -> int:
    cat, key = parse_ref(ref)
    if cat != "weight":
        return 0
    w = graph.weights
    shp = w.shape_of(key) if hasattr(w, "shape_of") else tuple(w[key].shape)
    n = 1
    for d in shp:
        n *= int(d)
    return n


def epilogue_cost(graph, starts) -> float:
    """Verified-time weight of the nodes after the last layer (final norm +
    lm_head), in layer units: the GEMM weight elements behind them relative to
    one layer's, times the GEMM share of a verified layer's time (~0.5 on the
    B200: the commit and the row kernels scale with activations, not weights).
    Qwen3-8B: lm_head 622 M vs 193 M per layer -> ~1.6 layers."""
    if len(starts) < 2:
        return 0.0
    mm = ("matmul", "linear", "conv2d")
    layer = sum(_weight_numel(graph, r) for n in graph.nodes[starts[0]:starts[1]]
                if n.kind in mm for r in n.inputs[1:2])
    tail = sum(_weight_numel(graph, r) for n in graph.nodes[starts[-1]:]
               if n.kind in mm for r in n.inputs[1:2]) - layer
    return 0.5 * max(tail, 0) / layer if layer else 0.0


def rank_slice(graph, n_layers: int, rank: int, world: int):
    """[start, end) of rank's slice: contiguous groups of whole layers; rank 0
    also owns the prologue, the last rank the epilogue.  Groups balance the
    estimated verified time, with the epilogue (lm_head) weighted by
    epilogue_cost, so the last rank takes fewer layers when the head is
    heavy (Qwen3-8B on 8 ranks: 5,5,5,5,4,4,4,3 + head instead of 5,5,5,5,4,4,4,4 + head)."""
    if world <= 1:
        return 0, graph.n_nodes
    starts = layer_starts(graph)
    if len(starts) < world:
        raise ValueError(f"{len(starts)} layers cannot be split over {world} ranks")
    n = len(starts)
    cost = [1.0] * n
    cost[-1] += epilogue_cost(graph, starts)
    total = sum(cost)
    # layer j goes to the rank whose share holds the midpoint of its cost
    owner, acc = [], 0.0
    for j in range(n):
        mid = acc + cost[j] / 2.0
        owner.append(min(world - 1, int(mid * world / total)))
        acc += cost[j]
    # every rank keeps at least one layer (contiguous, monotone owners)
    for r in range(world):
        if r not in owner:
            return _even_slice(graph, starts, n, rank, world)
    lo = owner.index(rank)
    hi = len(owner) - owner[::-1].index(rank)
    start = 0 if rank == 0 else starts[lo]
    end = graph.n_nodes if rank == world - 1 else starts[hi]
    return start, end


def _even_slice(graph, starts, n, rank, world):
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return (0 if rank == 0 else starts[lo]), (graph.n_nodes if rank == world - 1 else starts[hi])


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
