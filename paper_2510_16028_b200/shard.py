"""Multi-GPU sharding of the verified forward.

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
