"""Streaming co-execution on one B200: the NAO hot path at model scale.

Trace-driven verification, the challenger's per-operator adjudication
(dispute.py:605-657) applied to every node in canonical order (optionally a
contiguous op slice, the reference's partition unit, graph.py:275-293):

    y      = op(claimed inputs)            (re-execution from the committed trace)
    eps    = bound template of that op     (fused where it needs FP32 parts)
    check  = one pass over (y, claimed y', eps): bound violations |y'-y| > eps,
             max violation ratio, exact p_max > 1 verdict (dispute.py:114-158)
    commit = chunked Merkle root of the claimed tensor y' (batched per flush)

Downstream nodes consume the claimed values, so an injected fault is flagged
at its own node and nowhere else (the localisation property of the game).

Only per-node roots (32 B) and check records (56 B) survive a node; the trace
is never resident.  No host synchronisation happens
until `finish()`.  Elementwise bounds are never materialised: the check
kernel recomputes c|y| on the fly.

`plain_forward` runs the same lowered graph with values only (cuBLAS FP32,
TF32 off, torch eager ops) -- the baseline the overhead is measured against.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F

from . import _lib
from .bounds import (INTRINSIC_KINDS, ROW_KINDS, FpModel, apply_value, certified_overestimate,
                     op_bound_device, release_activation_split, apply_value,
                     gemm_bound_device, GEMM_BOUND_KINDS)
from .calibration import DEFAULT_EPSILON, PERCENTILE_GRID
from .commitments import DEFAULT_CHUNK_BYTES, alg_id, commit_tensors, root_of_digests
from .dispute import new_result_buffer
from .engine import NATIVE, ExecutionError, _batch_view, fma_of, to_device
from .graph import parse_ref

_EXP_SKIP_COMMIT = os.environ.get("NAO_EXP_SKIP_COMMIT") == "1"
INF_TAU = np.full(len(PERCENTILE_GRID), np.inf)


def last_uses(graph, start: int = 0, end: int | None = None) -> dict:
    """node index -> last consumer index within [start, end) (outputs live to the end)."""
    end = graph.n_nodes if end is None else end
    last = {}
    for node in graph.nodes[start:end]:
        for ref in node.inputs:
            cat, key = parse_ref(ref)
            if cat == "node":
                last[key] = node.index
    for ref in graph.outputs:
        last[parse_ref(ref)[1]] = end
    return last


REDUCTION_KINDS = frozenset({"matmul", "linear", "softmax", "layernorm", "sum", "mean"})


def drift_claim(node, y: torch.Tensor, seed: int = 0, period: int = 16, fault_node=None,
                fault_scale: float = 1e-3, fault_period: int = 64) -> torch.Tensor:
    """Harness proposer: reduction ops drift by +-1 ulp on ~1/period elements
    (a different device's summation order); deterministic ops are reproduced
    exactly; `fault_node` additionally carries a relative fault."""
    faulty = fault_node is not None and node.name == fault_node
    if node.kind in REDUCTION_KINDS or faulty:
        return inject_drift(y, seed * 7919 + node.index, period if node.kind in REDUCTION_KINDS
                            else 0, fault_scale if faulty else 0.0, fault_period if faulty else 0)
    # a separate claimed buffer holding the same bytes (nao_inject_drift's copy
    # path: ~2x the bandwidth of torch's clone on the B200)
    return inject_drift(y, 0, 0, 0.0, 0)


def inject_drift(y: torch.Tensor, seed: int, period: int = 16, fault_scale: float = 0.0,
                 fault_period: int = 0) -> torch.Tensor:
    """Claimed tensor = y with honest +-1-ulp drift (+ optional fault); see nao_inject_drift."""
    y = y.contiguous()
    if y.data_ptr() % 16:
        y = y.clone()
    out = torch.empty_like(y)
    _lib.call("nao_inject_drift", y.data_ptr(), out.data_ptr(), y.numel(), seed & 0xFFFFFFFF,
              period, float(fault_scale), fault_period, _lib.stream_ptr(y.device))
    return out


def _materialise_eps(eps, y: torch.Tensor) -> torch.Tensor:
    """FP64 bound tensor of a node for a bound dump (lazy templates expanded)."""
    if isinstance(eps, tuple):
        if eps[0] == "scaled":
            return torch.abs(y.double()) * float(eps[1])
        return torch.zeros(y.shape, dtype=torch.float64, device=y.device)
    return eps.double().reshape(y.shape)


class _RunState:
    """Carry-over between the stream segments of one run."""

    def __init__(self):
        self.pending, self.pend_idx, self.pend_bytes = [], [], 0
        self.pend_checks, self.pend_keep = [], []  # fused check descriptors / their operands
        self.pend_refine = []  # nao_refine_desc of the flush's GEMM / conv / intrinsic nodes
        self.pend_reuse = []   # (src position, block_chunks, repeats) or None per pending tensor
        self.pend_pos = {}     # node index -> position in `pending`


GEMM_KINDS = frozenset({"matmul", "linear", "conv2d"})


def check_band(node, xs, eps):
    """(eps kind, eps pointer, scale, lo_factor, uses the borderline list) of a
    node's check.  lo_factor = 1/R with R the certified over-estimate of the
    node's bound path (bounds.certified_overestimate): diff in (eps/R, eps] is
    borderline -- recorded for GEMM / conv nodes (settled exactly by
    nao_refine_borderline), only counted for row kernels (FP64 bounds, band
    ~1e-12: numpy's own summation order)."""
    if isinstance(eps, tuple):
        if eps[0] == "scaled":  # u|y|, 2u|y|: the reference's FP64 product, exactly
            return _lib.EPS_SCALED_LOCAL, None, float(eps[1]), 1.0, False
        return _lib.EPS_ZERO, None, 0.0, 1.0, False
    f32 = eps.dtype == torch.float32
    kind = _lib.EPS_TENSOR_F32 if f32 else _lib.EPS_TENSOR_F64
    if node.kind in GEMM_KINDS:
        K = xs[1][0].numel() if node.kind == "conv2d" else xs[0].shape[-1]
        R = certified_overestimate(node.kind, K=K, eps_f32=f32)
        return kind, eps.data_ptr(), 0.0, 1.0 / R, True
    if node.kind in ROW_KINDS:
        ax = int(node.attr("axis", -1)) % xs[0].dim()
        R = certified_overestimate(node.kind, n=xs[0].shape[ax], eps_f32=f32)
        return kind, eps.data_ptr(), 0.0, 1.0 / R, False
    return kind, eps.data_ptr(), 0.0, (1.0 / (1.0 + 2.0 ** -22) if f32 else 1.0), False


def refine_desc(node, xs, y, yc, record_ptr, border, model, profile=None, eps_scale=0.0):
    """nao_refine_desc of one node (None when its check needs no settling) and
    the operand tensors it reads (keep them alive until the refine ran)."""
    k = node.kind
    d = _lib.RefineDesc()
    d.list, d.cap, d.result = border.data_ptr(), border.numel() - 1, record_ptr
    d.local, d.claimed = y.data_ptr(), yc.data_ptr()
    if k in INTRINSIC_KINDS:
        x = xs[0].contiguous()
        d.kind, d.unary_kind, d.a, d.u = _lib.REFINE_UNARY, _lib.UNARY[k], x.data_ptr(), eps_scale
        return d, [x]
    if k in ("matmul", "linear"):
        tb = bool(node.attr("transpose_b", 0)) if k == "matmul" else False
        a3, b3, sa, sb, nb, M, N, K, _ = _batch_view(xs[0], xs[1], tb)
        d.kind, d.a, d.b = _lib.REFINE_GEMM, a3.data_ptr(), b3.data_ptr()
        d.batch, d.M, d.N, d.K, d.stride_a, d.stride_b = nb, M, N, K, sa, sb
        d.transpose_b, d.has_y = int(tb), int(k == "linear")
        d.gamma_const = model.reduction_const(K if fma_of(profile) else 2 * K - 1)
        d.u = model.u
        return d, [a3, b3]
    if k == "conv2d":
        x, w = xs[0].contiguous(), xs[1].contiguous()
        B, C, H, W = x.shape
        kk, st, pd = w.shape[-1], int(node.attr("stride", 1)), int(node.attr("pad", 0))
        OH, OW = (H + 2 * pd - kk) // st + 1, (W + 2 * pd - kk) // st + 1
        K = C * kk * kk
        d.kind, d.a, d.b = _lib.REFINE_CONV, w.data_ptr(), x.data_ptr()
        d.batch, d.M, d.N, d.K = B, OH * OW, w.shape[0], K
        d.C, d.H, d.W, d.k, d.stride, d.pad, d.OW = C, H, W, kk, st, pd, OW
        d.gamma_const = model.reduction_const(K if fma_of(profile) else 2 * K - 1)
        return d, [x, w]
    return None, []


def chunk_reuse(node, xs, pos_of, chunk: int):
    """nao_chunk_reuse of a data-movement node whose local output is a copy of
    a claimed tensor pending in the same commit (positions via pos_of): reshape
    (same bytes) or concat of one tensor with itself (GQA expansion: whole
    blocks repeated).  None when the chunks do not line up."""
    srcs = {parse_ref(r) for r in node.inputs}
    if len(srcs) != 1:
        return None
    cat, key = next(iter(srcs))
    if cat != "node" or key not in pos_of:
        return None
    x = xs[0]
    nbytes = x.numel() * 4
    if nbytes == 0:
        return None
    if node.kind == "reshape":
        return (pos_of[key], -(-nbytes // chunk), 1)
    if node.kind == "concat":
        ax = int(node.attr("axis", 0)) % x.dim()
        inner = 4
        for d in x.shape[ax:]:
            inner *= int(d)
        if inner % chunk == 0:
            return (pos_of[key], inner // chunk, len(node.inputs))
    return None


# x + c / x - c with c a weight: where c is 0 the claimed output can equal the
# operand chunk for chunk (a causal-mask add keeps the scores' lower triangle)
SAME_OFFSET_KINDS = frozenset({"add", "sub"})


def row_chunks(y: torch.Tensor, chunk: int) -> int:
    """Chunks per row of y's last axis when rows are whole chunks and their
    count divides the commit CTA's 128 chunks, else 0 (nao_chunk_reuse.row_chunks)."""
    if y.dim() < 2 or y.numel() == 0:
        return 0
    rb = int(y.shape[-1]) * 4
    if rb % chunk:
        return 0
    rc = rb // chunk
    return rc if 1 < rc <= 128 and 128 % rc == 0 else 0


def broadcast_ref(w: torch.Tensor, y: torch.Tensor, chunk: int) -> bool:
    """w broadcasts to y over leading dims only, in whole chunks (a reference
    tensor for the digest shortcut)."""
    return (w.dim() >= 1 and w.dtype == torch.float32 and w.is_contiguous() and w.numel() > 0
            and (w.numel() * 4) % chunk == 0 and y.numel() % w.numel() == 0
            and tuple(y.shape[y.dim() - w.dim():]) == tuple(w.shape) and w.data_ptr() % 16 == 0)


def chunk_plan(node, xs, y, pos_of, chunk: int, ref_digests=None):
    """nao_chunk_reuse entry of a checked node's claimed tensor, or None:
    data-movement reuse (chunk_reuse); for x + w / x - w (w a weight) the
    same-offset reuse of x's equal chunks and w as a broadcast reference
    (ref_digests(w) -> (payload ptr, chunk-digest ptr, bytes), cached by the
    caller); and the row-chunk mapping."""
    rc = row_chunks(y, chunk)
    r = chunk_reuse(node, xs, pos_of, chunk) if node.kind in ("reshape", "concat") else None
    if r is not None:
        return (r[0], r[1], r[2], _lib.REUSE_LOCAL_COPY, rc)
    # (only tensors of at least one commit CTA of chunks: the source-first launch
    # phase a reuse entry adds costs more than it saves on small graphs)
    if node.kind in SAME_OFFSET_KINDS and len(node.inputs) == 2 and y.numel() * 4 >= 128 * chunk:
        (c0, k0), (c1, _) = parse_ref(node.inputs[0]), parse_ref(node.inputs[1])
        if c0 == "node" and c1 == "weight" and tuple(xs[0].shape) == tuple(y.shape):
            src = (pos_of[k0], -(-y.numel() * 4 // chunk), 1, _lib.REUSE_SAME_OFFSET) \
                if k0 in pos_of else (-1, 0, 0, _lib.REUSE_LOCAL_COPY)
            ref = (None, None, 0)
            if ref_digests is not None and broadcast_ref(xs[1], y, chunk):
                ref = ref_digests(xs[1])
            if src[0] >= 0 or ref[0] is not None:
                return src + (rc,) + ref
    return (-1, 0, 0, _lib.REUSE_LOCAL_COPY, rc) if rc else None


def run_refine(descs) -> None:
    """One nao_refine_borderline launch on the current stream."""
    if descs:
        arr = (_lib.RefineDesc * len(descs))(*descs)
        _lib.call("nao_refine_borderline", arr, len(descs), _lib.stream_ptr())


def _segments(lo: int, hi: int, size: int):
    return [(a, min(a + size, hi)) for a in range(lo, hi, size)]


class GraphedRun:
    """A verification (or plain forward) recorded as CUDA graphs: replay() is
    one cudaGraphLaunch per segment; outputs land in the same buffers."""

    def __init__(self):
        self.graphs, self.pool, self.stream = [], None, None
        self.roots = self.records = None
        self.outputs = {}

    @classmethod
    def record(cls, sv, inputs, claimed_fn, start, end, frontier, seg_nodes):
        self = cls()
        self.pool = torch.cuda.graph_pool_handle()
        self.stream = torch.cuda.Stream(sv.dev)
        torch.cuda.synchronize(sv.dev)
        sv._deferred.clear()  # every eager use has completed (no event queries in a capture)
        st = sv._begin(inputs, start, end, frontier)
        for lo, hi in _segments(start, st.end, seg_nodes):
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph, pool=self.pool, stream=self.stream):
                sv._nodes(st, lo, hi, claimed_fn)
            self.graphs.append(gph)
        self.roots, self.records = sv._finish(st)
        self.outputs = sv.outputs
        torch.cuda.synchronize(sv.dev)
        return self

    @classmethod
    def record_plain(cls, graph, inputs, device, start, end, frontier, seg_nodes=96):
        self = cls()
        dev = torch.device(device)
        self.pool = torch.cuda.graph_pool_handle()
        self.stream = torch.cuda.Stream(dev)
        torch.cuda.synchronize(dev)
        end = graph.n_nodes if end is None else end
        values = dict(frontier or {})
        last = last_uses(graph, start, end)
        for lo, hi in _segments(start, end, seg_nodes):
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph, pool=self.pool, stream=self.stream):
                _plain_nodes(graph, inputs, dev, values, last, lo, hi)
            self.graphs.append(gph)
        self.outputs = values
        torch.cuda.synchronize(dev)
        return self

    def replay(self):
        """Enqueue every segment on the caller's current stream."""
        cur = torch.cuda.current_stream()
        self.stream.wait_stream(cur)
        with torch.cuda.stream(self.stream):
            for gph in self.graphs:
                gph.replay()
        cur.wait_stream(self.stream)
        return self.roots, self.records


@dataclass
class NodeStats:
    bytes_committed: int = 0
    elements_checked: int = 0
    gemm_flops: int = 0


class StreamingVerifier:
    def __init__(self, graph, model: FpModel | None = None, profile=NATIVE, thresholds=None,
                 hash_alg: str = "keccak256", chunk_bytes: int = DEFAULT_CHUNK_BYTES,
                 flush_bytes: int = 2 << 30, device="cuda", epsilon: float = DEFAULT_EPSILON,
                 grid=PERCENTILE_GRID, overlap: bool = True, fuse_check: bool = True,
                 max_lag: int = 0, partial: bool = False, missing_thresholds: str = "raise",
                 commit_priority: int | None = None, claim_stream: bool = False,
                 bound_stream: bool | None = None):
        self.g = graph
        self.model = model or FpModel()
        self.profile = profile
        self.thresholds = thresholds
        if missing_thresholds not in ("raise", "inf"):
            raise ValueError("missing_thresholds must be 'raise' or 'inf'")
        self.missing_thresholds = missing_thresholds
        self.alg = alg_id(hash_alg)
        self.chunk = int(chunk_bytes)
        self.flush_bytes = int(flush_bytes)
        self.dev = torch.device(device)
        self.epsilon = float(epsilon)
        self.grid = tuple(grid)
        self._tau_cache = {}
        # fuse_check: the acceptance check runs inside the Merkle commit pass
        # (nao_commit_check_tensors: the ALU-bound Keccak hides its HBM read);
        # False: a separate nao_check launch per node on its own side stream
        self.fuse_check = bool(fuse_check)
        # optional streaming dumps (traceio.TraceWriter / BoundWriter): the claimed
        # trace and the bounds leave the device on a copy stream as nodes finish
        self.trace_writer = None
        self.bound_writer = None
        # max_lag > 0: the main stream waits for commit flush k - max_lag before
        # issuing more work (bounds the claimed / local tensors pinned by a
        # side stream that runs behind, e.g. under a high-priority main stream)
        self.max_lag = int(max_lag)
        self._com_events = []
        self._host_events = []  # commit-flush events the host has not waited for
        # eager runs: tensors a side stream reads stay referenced here until an
        # event recorded on that stream after the use has completed (a deferred
        # free instead of Tensor.record_stream: with the expandable-segments
        # allocator, record_stream'ed blocks of the eager warm-up faulted later
        # runs of the GPT-2 config -- DESIGN.md §6)
        self._deferred = []  # [(event, [tensors])]
        self.host_lag_bytes = int(float(os.environ.get("NAO_HOST_LAG_GB", "32")) * (1 << 30))
        self._ref_cache = {}  # (ptr, numel, version, chunk, alg) -> (weight, its chunk digests)
        # partial: records are combinable nao_check_partial rows (a batch shard of
        # every node; shard.combine_shard_records decides the whole-tensor verdicts)
        self.partial = bool(partial)
        if self.partial and not self.fuse_check:
            raise ValueError("partial (batch-shard) records need the fused check")
        # device verdict specs: {node index: device address}; every uploaded blob
        # stays alive with the verifier (in-flight commits may still read it)
        self._spec_addr: dict = {}
        self._spec_blobs: list = []
        # side streams: the memory-bound check and the ALU-bound hashing run
        # concurrently with the next nodes' GEMMs / bound kernels
        # (equal priorities: a low-priority side stream starves and the memory its
        # pending work pins via record_stream balloons -- measured 2x slower)
        self.overlap = bool(overlap)
        self._s_chk = torch.cuda.Stream(self.dev) if overlap else None
        # commit_priority: the commit stream's CUDA priority (lower = higher);
        # at the caller's main-stream priority the commit takes SMs as soon as
        # the value path frees them (bench: -1, 66.7-67.1 vs 67.5-67.6 % at 0)
        if commit_priority is None:
            commit_priority = int(os.environ.get("NAO_COMMIT_PRIO", "0"))
        self._s_com = (torch.cuda.Stream(self.dev, priority=int(commit_priority))
                       if overlap else None)
        # abs-GEMM bounds of matmul / linear / conv nodes on their own stream:
        # the value path (main) runs on while the tensor-core bound fills the
        # SMs the SIMT GEMMs' last waves leave idle; commits wait for it
        # (NAO_BOUND_STREAM=0 turns it off.  With Tensor.record_stream for the
        # eager side-stream reads it faulted intermittently on the GPT-2 config
        # under expandable segments; the deferred free below fixed that.)
        if bound_stream is None:
            bound_stream = os.environ.get("NAO_BOUND_STREAM", "1") != "0"
        self.bound_stream = overlap and bool(bound_stream)
        # claim_stream: call claimed_fn on its own stream (a proposer harness
        # that derives claims from the local values: a node's claim is then
        # made while independent nodes' values run; consumers wait per node)
        self._s_clm = torch.cuda.Stream(self.dev) if (overlap and claim_stream) else None
        self._s_bnd = (torch.cuda.Stream(self.dev, priority=int(os.environ.get("NAO_BOUND_PRIO", "0")))
                       if self.bound_stream else None)
        self._s_main = None

    # ---------------------------------------------------------- thresholds
    def _ref_chunk_digests(self, w: torch.Tensor):
        """(payload ptr, chunk-digest ptr, bytes) of a static broadcast reference
        tensor (a weight), its chunk digests committed once and cached."""
        # the version counter keys in-place updates (a stale digest would be
        # copied for chunks that equal the tensor's new bytes)
        key = (w.data_ptr(), w.numel(), w._version, self.chunk, self.alg)
        hit = self._ref_cache.get(key)
        if hit is None:
            if len(self._ref_cache) >= 64:  # weights are static: a handful of masks
                return (None, None, 0)
            n = w.numel() * 4 // self.chunk
            dig = torch.empty((1 + n, 32), dtype=torch.uint8, device=w.device)
            commit_tensors([w], self.chunk, self.alg, leaf_digests=dig)
            hit = self._ref_cache[key] = (w, dig)
        w, dig = hit
        return (w.data_ptr(), dig.data_ptr() + 32, w.numel() * 4)

    def release(self) -> None:
        """Wait for the side streams and drop every tensor an eager run kept
        alive for them (the deferred frees of the last flushes)."""
        for s in (self._s_chk, self._s_com, self._s_bnd, self._s_clm):
            if s is not None:
                s.synchronize()
        self._deferred.clear()

    def _sync_thresholds(self):
        """Drop the cached taus / device specs when `thresholds` was replaced."""
        if getattr(self, "_spec_for", None) is not self.thresholds:
            self._spec_addr, self._tau_cache = {}, {}
            self._spec_for = self.thresholds

    def _taus(self, name):
        """(tau_abs, tau_rel) of a node.  Without a ThresholdSet the threshold
        verdict is off (tau = +inf); with one, a node it does not cover raises
        KeyError like the reference's ThresholdSet.lookup (calibration.py:189-191),
        unless the verifier was built with missing_thresholds="inf"."""
        if self.thresholds is None:
            return INF_TAU, INF_TAU
        self._sync_thresholds()
        t = self._tau_cache.get(name)
        if t is None:
            try:
                op = self.thresholds.lookup(name)
                t = (op.tau_abs, op.tau_rel)
            except KeyError:
                if self.missing_thresholds != "inf":
                    raise
                t = (INF_TAU, INF_TAU)
            self._tau_cache[name] = t
        return t

    def _spec_table(self, start, end):
        """Device address of every node's nao_verdict_spec in [start, end); the
        missing ones are uploaded in one copy."""
        self._sync_thresholds()
        missing = [n for n in self.g.nodes[start:end] if n.index not in self._spec_addr]
        if missing:
            size = int(_lib.load().nao_verdict_spec_bytes())
            blob = b"".join(_lib.verdict_spec(self.grid, *self._taus(n.name), self.epsilon)
                            for n in missing)
            dev_blob = torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(self.dev)
            self._spec_blobs.append(dev_blob)
            for k, n in enumerate(missing):
                self._spec_addr[n.index] = dev_blob.data_ptr() + k * size
        return self._spec_addr

    # ----------------------------------------------------------------- run
    def run(self, inputs: dict, claimed_fn, start: int = 0, end: int | None = None,
            frontier: dict | None = None, stats: NodeStats | None = None):
        """Verify nodes [start, end).  claimed_fn(node, y) -> the claimed CUDA tensor
        of node (the proposer's trace; given the locally recomputed y for harnesses).
        frontier maps external producer node index -> tensor (slice execution,
        graph.py:244-272).  Returns (roots [n,32] uint8, records [n, R] uint8)."""
        st = self._begin(inputs, start, end, frontier)
        self._nodes(st, start, st.end, claimed_fn, stats)
        return self._finish(st)

    def _begin(self, inputs, start, end, frontier, roots=None, records=None):
        g = self.g
        end = g.n_nodes if end is None else end
        n = end - start
        _lib.load()
        st = _RunState()
        st.inputs, st.start, st.end = inputs, start, end
        st.roots = roots if roots is not None else torch.empty((n, 32), dtype=torch.uint8,
                                                                device=self.dev)
        if records is None:
            records = (torch.zeros((n, _lib.CHECK_PARTIAL_BYTES), dtype=torch.uint8,
                                   device=self.dev) if self.partial
                       else new_result_buffer(self.dev, n))
        st.records = records
        st.last = last_uses(g, start, end)
        st.values = dict(frontier or {})
        st.all_idx = torch.arange(n, device=self.dev)
        # per-node borderline / value-ambiguity lists (word 0 = count, reset by
        # the refine pass that consumes them)
        st.border = torch.zeros((n, 1 + _lib.BORDER_CAP), dtype=torch.int64, device=self.dev)
        st.grid_arr = _lib.dbl_array(self.grid)
        if self.fuse_check:
            st.specs = self._spec_table(start, end)
        return st

    def _finish(self, st):
        self.outputs = {k: v for k, v in st.values.items()}
        return st.roots, st.records

    def _nodes(self, st, lo, hi, claimed_fn, stats=None):
        """Process nodes [lo, hi) of the run, then flush pending commits and
        join the side streams (a self-contained stream segment: it can be
        captured as one CUDA graph)."""
        g = self.g
        main = torch.cuda.current_stream(self.dev)
        s_chk = self._s_chk or main
        s_com = self._s_com or main
        capturing = torch.cuda.is_current_stream_capturing()
        if not capturing:  # references whose side-stream reads have completed
            while self._deferred and self._deferred[0][0].query():
                self._deferred.pop(0)
        s_bnd = self._s_bnd if (self.overlap and self._s_bnd is not None) else None
        s_clm = self._s_clm if (self.overlap and self._s_clm is not None) else None
        clm_ev = {}  # node index -> event after its claim (claim stream)
        if self.overlap:  # side streams start after everything already queued on main
            s_chk.wait_stream(main)
            s_com.wait_stream(main)
        if s_bnd is not None:
            s_bnd.wait_stream(main)
        if s_clm is not None:
            s_clm.wait_stream(main)
        with torch.cuda.stream(s_chk):
            ws_chk = _lib.check_accumulator(self.dev)
        chk_ptr = s_chk.cuda_stream
        start = st.start
        # tensors read on a side stream: deferred-freed when eager; held until
        # the segment's join when capturing (a capture cannot record events)
        keep = []

        uses = {}  # eager: side stream -> tensors it read since the last release point

        def side_use(t, s):
            if not self.overlap:
                return
            if capturing:
                keep.append(t)
            else:
                uses.setdefault(s, []).append(t)

        def defer_uses():
            """Eager: one event per side stream after its queued uses; drop the
            references whose events have completed (in order)."""
            for s, ts in uses.items():
                ev = torch.cuda.Event()
                ev.record(s)
                self._deferred.append((ev, ts))
            uses.clear()
            while not capturing and self._deferred and self._deferred[0][0].query():
                self._deferred.pop(0)

        def flush():
            if not st.pending:
                return
            if self.overlap:
                s_com.wait_stream(main)
            if s_bnd is not None:  # the flush's GEMM bounds
                s_com.wait_stream(s_bnd)
            if s_clm is not None:  # the flush's claims
                s_com.wait_stream(s_clm)
            with torch.cuda.stream(s_com):
                if _EXP_SKIP_COMMIT:  # timing experiment only: main-stream work alone
                    st.pending, st.pend_idx, st.pend_bytes = [], [], 0
                    st.pend_checks, st.pend_keep, st.pend_refine = [], [], []
                    st.pend_reuse, st.pend_pos = [], {}
                    return
                r = commit_tensors(st.pending, self.chunk, self.alg,
                                   checks=st.pend_checks if self.fuse_check else None,
                                   reuse=st.pend_reuse if self.fuse_check else None)
                if self.fuse_check:
                    run_refine(st.pend_refine)  # settle the flush's borderline elements
                lo_i, hi_i = st.pend_idx[0], st.pend_idx[-1] + 1
                if hi_i - lo_i == len(st.pend_idx):
                    st.roots[lo_i:hi_i].copy_(r)
                else:
                    st.roots.index_copy_(0, st.all_idx[torch.as_tensor(st.pend_idx)], r)
            for t in st.pending + st.pend_keep:
                side_use(t, s_com)
            defer_uses()
            if self.overlap and capturing:
                keep.append(r)
            if self.overlap and self.max_lag > 0 and not capturing:
                ev = torch.cuda.Event()
                ev.record(s_com)
                self._com_events.append(ev)
                if len(self._com_events) > self.max_lag:
                    old_ev = self._com_events.pop(0)
                    main.wait_event(old_ev)
                    # the host may run at most ~host_lag_bytes of claimed tensors
                    # (in flushes) further ahead: blocks freed while a side stream
                    # still uses them stay reserved until it passes (claimed + local
                    # + eps per node), so unbounded run-ahead fills HBM and turns
                    # into allocator OOM retries (device syncs).  The bound must stay
                    # loose: the host enqueues only ~8 % faster than the GPU runs,
                    # and a tight one (6 flushes) left the main stream starved
                    # (77 -> 90-130 % on the bench)
                    self._host_events.append(old_ev)
                    n_host = max(self.max_lag, int(self.host_lag_bytes // max(1, self.flush_bytes)))
                    while len(self._host_events) > n_host:
                        self._host_events.pop(0).synchronize()
            st.pending, st.pend_idx, st.pend_bytes = [], [], 0
            st.pend_checks, st.pend_keep, st.pend_refine = [], [], []
            st.pend_reuse, st.pend_pos = [], {}

        values, last = st.values, st.last
        for node in g.nodes[lo:hi]:
            xs = []
            for ref in node.inputs:
                cat, key = parse_ref(ref)
                if cat == "node":
                    xs.append(values[key])
                    ev = clm_ev.pop(key, None) if s_clm is not None else None
                    if ev is not None:  # this input's claim is made on the claim stream
                        main.wait_event(ev)
                elif cat == "input":
                    xs.append(to_device(st.inputs[key], self.dev))
                else:
                    xs.append(to_device(g.weights[key], self.dev))
            i = node.index - start
            border = st.border[i]
            try:
                if s_bnd is not None and node.kind in GEMM_BOUND_KINDS:
                    # value on main, abs-GEMM bound on the bound stream (matmul /
                    # conv: from the inputs alone, concurrently with the value
                    # GEMM; linear: after it, for the u|y| term)
                    early = node.kind != "linear"
                    if early:
                        s_bnd.wait_stream(main)
                    y = apply_value(node, xs, self.profile)
                    if not early:
                        s_bnd.wait_stream(main)
                    with torch.cuda.stream(s_bnd):
                        eps = gemm_bound_device(node, xs, y, self.model, self.profile, False)
                    for t in xs:
                        side_use(t, s_bnd)
                    side_use(y, s_bnd)
                else:
                    y, eps = op_bound_device(node, xs, self.model, self.profile, eps_f64=None,
                                             amb=border if node.kind in INTRINSIC_KINDS else None)
            except (ExecutionError, NotImplementedError):
                raise
            except Exception as exc:
                raise ExecutionError(f"node {node.index} ({node.name!r}, {node.kind}): {exc}",
                                     node_index=node.index, node_name=node.name) from exc
            y = y.contiguous()
            if s_clm is not None:
                s_clm.wait_stream(main)
                with torch.cuda.stream(s_clm):
                    yc = claimed_fn(node, y)
                ev = torch.cuda.Event()
                ev.record(s_clm)
                clm_ev[node.index] = ev
                side_use(y, s_clm)
            else:
                yc = claimed_fn(node, y)
            if not (isinstance(yc, torch.Tensor) and yc.dtype == torch.float32
                    and tuple(yc.shape) == tuple(y.shape) and yc.device == y.device):
                # the reference raises on a claimed tensor of another shape
                # (elementwise_errors / leaf_payload broadcasting); the kernels
                # would read the local tensor out of bounds
                raise ExecutionError(
                    f"node {node.index} ({node.name!r}): claimed tensor "
                    f"{getattr(yc, 'dtype', type(yc))} {tuple(getattr(yc, 'shape', ()))} does not "
                    f"match the recomputed float32 {tuple(y.shape)} on {y.device}",
                    node_index=node.index, node_name=node.name)
            yc = yc.contiguous()
            if s_clm is not None:
                side_use(yc, main)  # made on the claim stream, read on main / commit
            if self.trace_writer is not None:
                if s_clm is not None:
                    main.wait_stream(s_clm)
                self.trace_writer.write(node.index, yc)
            if self.bound_writer is not None:
                if s_bnd is not None:
                    main.wait_stream(s_bnd)
                self.bound_writer.write(node.index, _materialise_eps(eps, y))
            tau_a, tau_r = self._taus(node.name)
            kind, eps_ptr, scale, lo_f, listed = check_band(node, xs, eps)
            blist = border.data_ptr() if listed else None
            rdesc, rkeep = (None, [])
            if y.numel() and (listed or node.kind in INTRINSIC_KINDS):
                rdesc, rkeep = refine_desc(node, xs, y, yc, st.records[i].data_ptr(), border,
                                           self.model, self.profile, eps_scale=scale)
            desc = None
            if y.numel() and self.fuse_check:
                desc = _lib.CheckDesc(y.data_ptr(), eps_ptr, st.specs[node.index],
                                      st.records[i].data_ptr(), scale, lo_f, kind,
                                      _lib.CHECK_PARTIAL if self.partial else 0,
                                      blist, _lib.BORDER_CAP)
                st.pend_keep.append(y)
                if not isinstance(eps, tuple):
                    st.pend_keep.append(eps)
                if rdesc is not None:
                    st.pend_refine.append(rdesc)
                    st.pend_keep.extend(rkeep)
            elif y.numel():
                if self.overlap:
                    s_chk.wait_stream(main)
                    if s_bnd is not None:
                        s_chk.wait_stream(s_bnd)
                    side_use(y, s_chk)
                    side_use(yc, s_chk)
                    if not isinstance(eps, tuple):
                        side_use(eps, s_chk)
                    for t in rkeep:
                        side_use(t, s_chk)
                with torch.cuda.stream(s_chk):
                    _lib.call("nao_check", y.data_ptr(), yc.data_ptr(), y.numel(), kind, eps_ptr,
                              scale, lo_f, st.grid_arr, _lib.dbl_array(tau_a),
                              _lib.dbl_array(tau_r), len(self.grid), self.epsilon,
                              st.records[i].data_ptr(), ws_chk.data_ptr(), ws_chk.numel(),
                              blist, _lib.BORDER_CAP, chk_ptr)
                    if rdesc is not None:
                        run_refine([rdesc])
            if stats is not None:
                stats.elements_checked += y.numel()
                stats.bytes_committed += y.numel() * 4
                if node.kind in ("matmul", "linear"):
                    stats.gemm_flops += 2 * y.numel() * xs[0].shape[-1]
                elif node.kind == "conv2d":  # implicit GEMM, K = C k k
                    stats.gemm_flops += 2 * y.numel() * xs[1][0].numel()
            del eps, y
            values[node.index] = yc
            st.pend_reuse.append(chunk_plan(node, xs, yc, st.pend_pos, self.chunk,
                                            self._ref_chunk_digests)
                                 if desc is not None else None)
            st.pend_pos[node.index] = len(st.pending)
            st.pending.append(yc)
            st.pend_checks.append(desc)
            st.pend_idx.append(i)
            st.pend_bytes += yc.numel() * 4
            if st.pend_bytes >= self.flush_bytes or len(st.pending) >= 120:
                flush()
            for ref in node.inputs:
                cat, key = parse_ref(ref)
                if cat == "node" and last.get(key, -1) == node.index and key in values:
                    del values[key]
            if last.get(node.index, -1) <= node.index and node.index in values:
                del values[node.index]
        flush()
        if self.overlap:
            main.wait_stream(s_chk)
            main.wait_stream(s_com)
        if s_bnd is not None:
            main.wait_stream(s_bnd)
        if s_clm is not None:
            main.wait_stream(s_clm)
        defer_uses()
        keep.clear()
        release_activation_split()  # the memo must not pin a split past the segment

    # ------------------------------------------------------------ graphs
    def capture(self, inputs: dict, claimed_fn, start: int = 0, end: int | None = None,
                frontier: dict | None = None, seg_nodes: int = 96):
        """Record the verification of nodes [start, end) as a chain of CUDA
        graphs (segments of ~seg_nodes nodes, one shared memory pool) and
        return a GraphedRun whose replay() re-runs it with no host work per
        node.  `inputs` / `frontier` / weights must stay at the same device
        addresses (refill them in place between replays).  Call run() once
        first (warm-up: weight split caches, workspaces)."""
        return GraphedRun.record(self, inputs, claimed_fn, start, end, frontier, seg_nodes)

    def trace_root(self, roots: torch.Tensor) -> torch.Tensor:
        """Merkle root over per-node roots (leaf = H(0x00||root)), on device."""
        n = roots.shape[0]
        offs = torch.arange(0, 32 * (n + 1), 32, dtype=torch.int64, device=roots.device)
        leaves = torch.empty((n, 32), dtype=torch.uint8, device=roots.device)
        _lib.call("nao_merkle_hash_leaves", roots.contiguous().data_ptr(), offs.data_ptr(), n,
                  self.alg, leaves.data_ptr(), _lib.stream_ptr(roots.device))
        return root_of_digests(leaves, self.alg)


# ------------------------------------------------------------ plain forward

def plain_value(node, xs, profile=NATIVE) -> torch.Tensor:
    """Values only, torch eager FP32 (the baseline forward of the same graph)."""
    k = node.kind
    if k == "softmax":
        return torch.softmax(xs[0], dim=int(node.attr("axis", -1)))
    if k == "layernorm":
        ax = int(node.attr("axis", -1)) % xs[0].dim()
        x = xs[0].movedim(ax, -1)
        y = F.layer_norm(x, (x.shape[-1],), eps=float(node.attr("eps", 1e-5)))
        return y.movedim(-1, ax)
    if k in ("sum", "mean", "max", "min"):
        ax = int(node.attr("axis", -1))
        return {"sum": torch.sum, "mean": torch.mean, "max": torch.amax,
                "min": torch.amin}[k](xs[0], dim=ax)
    if k in ("exp", "log", "sqrt", "rsqrt", "tanh"):
        return getattr(torch, k)(xs[0])
    if k == "gelu":
        return F.gelu(xs[0], approximate="tanh")
    if k == "silu":
        return F.silu(xs[0])
    return apply_value(node, xs, profile)


def _plain_nodes(g, inputs, dev, values, last, lo, hi):
    for node in g.nodes[lo:hi]:
        xs = []
        for ref in node.inputs:
            cat, key = parse_ref(ref)
            if cat == "node":
                xs.append(values[key])
            elif cat == "input":
                xs.append(to_device(inputs[key], dev))
            else:
                xs.append(to_device(g.weights[key], dev))
        values[node.index] = plain_value(node, xs)
        for ref in node.inputs:
            cat, key = parse_ref(ref)
            if cat == "node" and last.get(key, -1) == node.index and key in values:
                del values[key]


def plain_forward(graph, inputs: dict, device="cuda", start: int = 0, end: int | None = None,
                  frontier: dict | None = None):
    g = graph
    end = g.n_nodes if end is None else end
    last = last_uses(g, start, end)
    values = dict(frontier or {})
    _plain_nodes(g, inputs, torch.device(device), values, last, start, end)
    return values
