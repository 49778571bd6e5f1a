"""Threshold check and leaf bound check on the GPU -- drop-in for the hot-path
part of /root/reference/pkg/src/fpverify/dispute.py (p_max :114-127,
observed_p_max :130-141, screen :144-150, select_offending :153-158, the leaf
route of Challenger.leaf_payload :639-657).  The ledger / protocol state
machine is the reference's control plane and out of scope.

Two GPU entry points:
  * observed_p_max: exact percentiles (sort) -> exact p_max value, as the
    reference returns it.
  * check_node (nao_check): ONE pass deciding the same verdict p_max > 1 plus
    bound violations / max violation ratio -- the streaming hot-path check.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .calibration import DEFAULT_EPSILON, PERCENTILE_GRID, error_profiles_device
from .engine import to_device


def p_max(abs_profile, rel_profile, tau_abs, tau_rel) -> float:
    """dispute.py:114-127 (0/0 -> 0, x/0 -> inf)."""
    if len(abs_profile) != len(tau_abs) or len(rel_profile) != len(tau_rel):
        raise ValueError("percentile grid mismatch between observation and thresholds")
    worst = 0.0
    for obs, tau in ((abs_profile, tau_abs), (rel_profile, tau_rel)):
        obs = np.asarray(obs, dtype=np.float64)
        tau = np.asarray(tau, dtype=np.float64)
        with np.errstate(divide="ignore", invalid="ignore"):
            ratio = np.where(tau > 0.0, obs / np.where(tau > 0.0, tau, 1.0),
                             np.where(obs > 0.0, np.inf, 0.0))
        worst = max(worst, float(np.max(ratio)) if ratio.size else 0.0)
    return worst


def _payload(t):
    if isinstance(t, (torch.Tensor, np.ndarray)):
        return t
    if getattr(t, "_dev", None) is not None:
        return t._dev
    return np.asarray(t.data)


def observed_p_max(local, claimed, thresholds, name: str) -> float:
    """dispute.py:130-141: exact p_max (relative denominator = local magnitudes)."""
    pa, pr = error_profiles_device(_payload(local), _payload(claimed), thresholds.grid,
                                   thresholds.epsilon)
    op = thresholds.lookup(name)
    return p_max(pa.cpu().numpy(), pr.cpu().numpy(), op.tau_abs, op.tau_rel)


def screen(local_outputs, claimed_outputs, output_names, thresholds):
    """dispute.py:144-150."""
    details = {}
    for local, claimed, name in zip(local_outputs, claimed_outputs, output_names):
        details[name] = observed_p_max(local, claimed, thresholds, name)
    return any(v > 1.0 for v in details.values()), details


def select_offending(offense_ratios):
    """dispute.py:153-158."""
    for j, ratio in enumerate(offense_ratios):
        if ratio is not None and ratio > 1.0:
            return j
    return None


# ----------------------------------------------------- streaming node check

class CheckRecord:
    """Device-side nao_check_result; `.host()` reads it (one small D2H)."""

    def __init__(self, buf: torch.Tensor):
        self.buf = buf

    def host(self) -> dict:
        raw = self.buf.cpu().numpy().tobytes()
        r = _lib.CheckResult.from_buffer_copy(raw[:_lib.CHECK_RESULT_BYTES])
        return {f: getattr(r, f) for f, _ in _lib.CheckResult._fields_ if f != "reserved"}


def new_result_buffer(device, n: int = 1) -> torch.Tensor:
    return torch.zeros((n, _lib.CHECK_RESULT_BYTES), dtype=torch.uint8, device=device)


def check_node(local: torch.Tensor, claimed: torch.Tensor, eps, tau_abs, tau_rel,
               grid=PERCENTILE_GRID, epsilon: float = DEFAULT_EPSILON, lo_factor: float = 1.0,
               out: torch.Tensor | None = None, border: torch.Tensor | None = None) -> CheckRecord:
    """One-pass check of a node.  eps: FP32/FP64 CUDA tensor, ("scaled", c)
    for c|local| templates, or ("zero",).  border: int64 [1 + cap] list that
    receives the borderline elements (for nao_refine_borderline).  No host sync."""
    from .engine import require_f32
    require_f32(local, claimed)
    a = to_device(local).reshape(-1).contiguous()
    b = to_device(claimed).reshape(-1).contiguous()
    if a.numel() != b.numel():
        raise ValueError("shape mismatch between local and claimed")
    n = a.numel()
    if n == 0:
        raise ValueError("percentile profile of empty input")
    if len(tau_abs) != len(grid) or len(tau_rel) != len(grid):
        raise ValueError("percentile grid mismatch between observation and thresholds")
    eps_ptr, kind, scale = None, _lib.EPS_ZERO, 0.0
    if isinstance(eps, tuple):
        if eps[0] == "scaled":
            kind, scale = _lib.EPS_SCALED_LOCAL, float(eps[1])
    else:
        e = eps.reshape(-1).contiguous()
        if e.numel() != n:
            raise ValueError("bound shape mismatch")
        kind = _lib.EPS_TENSOR_F64 if e.dtype == torch.float64 else _lib.EPS_TENSOR_F32
        if e.dtype == torch.float32 and lo_factor == 1.0:
            lo_factor = 1.0 / (1.0 + 2.0 ** -22)
        eps_ptr = e.data_ptr()
    res = out if out is not None else new_result_buffer(a.device)
    L = _lib.load()
    ws = _lib.check_accumulator(a.device)
    _lib.call("nao_check", a.data_ptr(), b.data_ptr(), n, kind, eps_ptr, scale, float(lo_factor),
              _lib.dbl_array(grid), _lib.dbl_array(tau_abs), _lib.dbl_array(tau_rel), len(grid),
              float(epsilon), res.data_ptr(), ws.data_ptr(), ws.numel(), _lib.ptr(border),
              (border.numel() - 1) if border is not None else 0, _lib.stream_ptr(a.device))
    return CheckRecord(res)


def commit_check_nodes(claimed, local, eps, taus, chunk_bytes: int = 4096, alg="keccak256",
                       grid=PERCENTILE_GRID, epsilon: float = DEFAULT_EPSILON,
                       partial: bool = False):
    """Merkle-commit every claimed tensor and check it against its local
    recomputation in the same pass (nao_commit_check_tensors).  eps[i] as in
    check_node; taus[i] = (tau_abs, tau_rel).  Returns (roots [n,32],
    records [n, R]) on the device (records of empty tensors stay zero)."""
    from .commitments import commit_tensors
    n = len(claimed)
    if not (len(local) == len(eps) == len(taus) == n):
        raise ValueError("claimed/local/eps/taus lengths differ")
    dev = to_device(claimed[0]).device
    recs = (torch.zeros((n, _lib.CHECK_PARTIAL_BYTES), dtype=torch.uint8, device=dev) if partial
            else new_result_buffer(dev, n))
    blobs, descs, keep = [], [], []
    for i in range(n):
        a = to_device(local[i]).contiguous()
        b = to_device(claimed[i]).contiguous()
        if a.numel() != b.numel():
            raise ValueError("shape mismatch between local and claimed")
        ta, tr = taus[i]
        if len(ta) != len(grid) or len(tr) != len(grid):
            raise ValueError("percentile grid mismatch between observation and thresholds")
        blobs.append(_lib.verdict_spec(grid, ta, tr, epsilon))
        kind, eps_ptr, scale, lo = _lib.EPS_ZERO, None, 0.0, 1.0
        e = eps[i]
        if isinstance(e, tuple):
            if e[0] == "scaled":
                kind, scale = _lib.EPS_SCALED_LOCAL, float(e[1])
        else:
            e = e.reshape(-1).contiguous()
            if e.numel() != a.numel():
                raise ValueError("bound shape mismatch")
            kind = _lib.EPS_TENSOR_F64 if e.dtype == torch.float64 else _lib.EPS_TENSOR_F32
            lo = 1.0 if e.dtype == torch.float64 else 1.0 / (1.0 + 2.0 ** -22)
            eps_ptr = e.data_ptr()
            keep.append(e)
        keep += [a, b]
        descs.append((a, b, kind, eps_ptr, scale, lo))
    size = len(blobs[0])
    spec = torch.frombuffer(bytearray(b"".join(blobs)), dtype=torch.uint8).to(dev)
    checks = []
    for i, (a, b, kind, eps_ptr, scale, lo) in enumerate(descs):
        checks.append(_lib.CheckDesc(a.data_ptr(), eps_ptr, spec.data_ptr() + i * size,
                                     recs[i].data_ptr(), scale, lo, kind,
                                     _lib.CHECK_PARTIAL if partial else 0, None, 0)
                      if a.numel() else None)
    roots = commit_tensors([d[1] for d in descs], chunk_bytes, alg, checks=checks)
    for t in keep + [spec]:
        t.record_stream(torch.cuda.current_stream(dev))
    return roots, recs


def partial_from_bytes(raw: bytes) -> dict:
    """Decode one nao_check_partial row."""
    r = _lib.CheckPartial.from_buffer_copy(bytes(raw)[:_lib.CHECK_PARTIAL_BYTES])
    out = {f: getattr(r, f) for f in ("n", "n_violations", "n_borderline", "n_nonfinite",
                                      "max_ratio")}
    for f in ("hist_abs", "hist_rel", "min_abs", "max_abs", "min_rel", "max_rel"):
        out[f] = np.array(getattr(r, f)[:])
    return out


def _np_lerp(a, b, t):
    """numpy _lerp (_function_base_impl.py:4657-4679)."""
    d = b - a
    r = a + d * t
    if t >= 0.5:
        r = b - d * (1.0 - t)
    return r


def combine_partials(partials, tau_abs, tau_rel, grid=PERCENTILE_GRID) -> dict:
    """Merge shard partials of one tensor (nao_check_partial: interval counts +
    per-interval key ranges) into the whole tensor's record: violation counts
    add, max ratios max, and the threshold verdict observed_p_max > 1
    (dispute.py:114-141) is decided exactly -- including numpy's interpolation
    between order statistics, from the interval key ranges."""
    G = len(grid)
    n = int(sum(p["n"] for p in partials))
    rec = {"n": n, "n_violations": int(sum(p["n_violations"] for p in partials)),
           "n_borderline": int(sum(p["n_borderline"] for p in partials)),
           "n_nonfinite": int(sum(p["n_nonfinite"] for p in partials)),
           "max_ratio": float(max(p["max_ratio"] for p in partials)) if partials else 0.0}
    exceeded, first = False, -1
    for arr, (taus, key) in enumerate(((tau_abs, "abs"), (tau_rel, "rel"))):
        eff = np.array([t if t > 0.0 else 0.0 for t in np.asarray(taus, dtype=np.float64)])
        srt = np.sort(eff)
        hist = np.sum([p[f"hist_{key}"][:G + 1] for p in partials], axis=0).astype(np.int64)
        cnt = np.sum([(p[f"hist_{key}"][:G + 1] > 0) for p in partials], axis=0)
        with np.errstate(invalid="ignore"):
            mx = np.max([np.where(p[f"hist_{key}"][:G + 1] > 0, p[f"max_{key}"][:G + 1], -np.inf)
                         for p in partials], axis=0)
            mn = np.min([np.where(p[f"hist_{key}"][:G + 1] > 0, p[f"min_{key}"][:G + 1], np.inf)
                         for p in partials], axis=0)
        del cnt
        for i in range(G):
            tau = float(eff[i])
            L = int(np.searchsorted(srt, tau, side="left"))  # #{sorted t < tau}
            cle = int(hist[:L + 1].sum())
            q = np.float64(grid[i]) / 100.0
            vi = (n - 1) * q
            if vi >= n - 1:
                ex = cle < n
            else:
                prev = int(np.floor(vi))
                g = vi - np.floor(vi)
                if cle <= prev:
                    ex = True
                elif cle >= prev + 2:
                    ex = False
                else:  # exactly prev+1 keys <= tau: the prev-th / next order statistics
                    a = float(np.max(mx[:L + 1]))
                    b = float(np.min(mn[L + 1:])) if L + 1 <= G else np.inf
                    ex = _np_lerp(a, b, g) > tau
            if ex and not exceeded:
                exceeded, first = True, arr * G + i
    rec["threshold_exceeded"] = int(exceeded)
    rec["first_exceeded"] = first
    return rec


def leaf_check(claimed, y_ref, eps) -> dict:
    """dispute.py:641-648 on the GPU for a given bound: any(|claimed - y_ref| > eps)
    and its count (thresholds are irrelevant: grid of one point, tau = +inf).
    With a bound computed by this package prefer leaf_bound_check, which also
    settles the elements inside the bound's certified over-estimate."""
    e = eps if isinstance(eps, tuple) else to_device_eps(eps)
    rec = check_node(y_ref, claimed, e, [np.inf], [np.inf], grid=(100.0,)).host()
    return {"n_violations": int(rec["n_violations"]), "n_borderline": int(rec["n_borderline"]),
            "max_ratio": float(rec["max_ratio"]), "any_violation": rec["n_violations"] > 0}


def _node_args(args):
    from .engine import to_device
    xs = []
    for a in args:
        if isinstance(a, torch.Tensor) and a.is_cuda:
            xs.append(a)
        elif isinstance(a, np.ndarray) and a.dtype.kind in "iu":
            xs.append(torch.from_numpy(np.ascontiguousarray(a)).cuda())
        else:
            xs.append(to_device(a))
    return xs


def leaf_bound_check(node, args, claimed, model=None, profile=None) -> dict:
    """The leaf's bound check exactly as the reference decides it
    (Challenger.leaf_payload, dispute.py:639-648: y_ref, eps = op_bound(...);
    any(|claimed - y_ref| > eps)).  The GPU bound over-estimates eps_ref by at
    most its certified factor R; elements in (eps/R, eps] are recorded by the
    check and settled by nao_refine_borderline (GEMM / conv: the reference's
    eps recomputed for that element; intrinsics: every FP32 value numpy's libm
    could give).  Returns counts of certain violations, the undecided rest
    (n_borderline; the reference's own FP64 summation order is the only
    source left), y and eps (device)."""
    from .bounds import FpModel, INTRINSIC_KINDS, SINGLE_ROUNDING_KINDS, op_bound_device
    from .executor import check_band, refine_desc, run_refine
    model = model or FpModel()
    xs = _node_args(args)
    c = claimed._dev if getattr(claimed, "_dev", None) is not None else claimed
    c = _node_args([c])[0]
    border = torch.zeros(1 + _lib.BORDER_CAP, dtype=torch.int64, device=xs[0].device)
    intrinsic = node.kind in INTRINSIC_KINDS
    y, eps = op_bound_device(node, xs, model, profile, eps_f64=True,
                             amb=border if intrinsic else None)
    y = y.contiguous()
    if tuple(c.shape) != tuple(y.shape):
        raise ValueError(f"claimed shape {tuple(c.shape)} differs from the output {tuple(y.shape)}")
    c = c.contiguous()
    if intrinsic or node.kind in ("matmul", "linear", "conv2d"):
        # the API path sizes the list to the node (every listed element is settled)
        cap = max(_lib.BORDER_CAP, min(int(y.numel()), 1 << 24))
        if cap > _lib.BORDER_CAP:
            big = torch.zeros(1 + cap, dtype=torch.int64, device=y.device)
            if intrinsic:  # the ambiguity list was filled by the value kernel
                n_amb = int(border[0])
                if n_amb > _lib.BORDER_CAP:  # re-run the value pass into the big list
                    _ = op_bound_device(node, xs, model, profile, eps_f64=True, amb=big)
                else:
                    big[:1 + _lib.BORDER_CAP].copy_(border)
            border = big
    eps_chk = eps
    if intrinsic:
        eps_chk = ("scaled", 2.0 * model.u)
    elif node.kind in SINGLE_ROUNDING_KINDS:
        eps_chk = ("scaled", model.u)
    rec = new_result_buffer(y.device)
    if y.numel() == 0:
        return {"n_violations": 0, "n_borderline": 0, "max_ratio": 0.0, "any_violation": False,
                "certain": True, "y": y, "eps": eps}
    kind, _, scale, lo, listed = check_band(node, xs, eps_chk)
    check_node(y, c, eps_chk, [np.inf], [np.inf], grid=(100.0,), lo_factor=lo, out=rec,
               border=border if listed else None)
    if listed or intrinsic:
        d, keep = refine_desc(node, xs, y, c, rec.data_ptr(), border, model, profile,
                              eps_scale=scale)
        run_refine([d])
        del keep
    h = CheckRecord(rec).host()
    return {"n_violations": int(h["n_violations"]), "n_borderline": int(h["n_borderline"]),
            "max_ratio": float(h["max_ratio"]), "any_violation": h["n_violations"] > 0,
            "certain": h["n_borderline"] == 0, "y": y, "eps": eps}


def oracle_recheck(node, args, claimed, eps, model=None, profile=None) -> dict:
    """The theoretical path (dispute.py:649-656): y_oracle = apply_op(node,
    args64, None, fp64=True) on the GPU (engine.apply_op_fp64: sequential FP64
    folds, bit-identical to numpy's except transcendental last ulps), then
    all(|claimed - y_oracle| <= eps).  Against the GPU's eps (>= eps_ref) the
    elements inside its certified band are re-adjudicated for GEMM / conv
    nodes with the reference's eps recomputed (nao_refine_borderline on the
    FP64 oracle values)."""
    from .bounds import FpModel
    from .engine import apply_op_fp64
    from .executor import GEMM_KINDS, check_band, refine_desc, run_refine
    model = model or FpModel()
    xs = _node_args(args)
    c = claimed._dev if getattr(claimed, "_dev", None) is not None else claimed
    c = _node_args([c])[0].contiguous()
    y_or = apply_op_fp64(node, xs).contiguous()
    e = eps.double().reshape(y_or.shape) if isinstance(eps, torch.Tensor) else \
        to_device_eps(eps).reshape(y_or.shape)
    diff = (c.double() - y_or).abs()
    excess = diff - e
    fail = diff > e
    n_fail = int(fail.sum())
    n_border = 0
    if node.kind in GEMM_KINDS and diff.numel():
        _, _, _, lo, _ = check_band(node, xs, eps if isinstance(eps, torch.Tensor) else e)
        band = (~fail) & (diff > e * lo)
        idx = torch.nonzero(band.reshape(-1)).reshape(-1)
        n_border = int(idx.numel())
        if n_border:
            y32 = None
            if node.kind == "linear":  # the u|y| term takes the FP32 value
                from .bounds import op_bound_device
                y32, _ = op_bound_device(node, xs, model, profile, eps_f64=None)
                y32 = y32.contiguous()
            cap = max(_lib.BORDER_CAP, n_border)  # the API path settles every band element
            border = torch.zeros(1 + cap, dtype=torch.int64, device=y_or.device)
            border[0] = n_border
            border[1:1 + n_border] = idx
            rec = new_result_buffer(y_or.device)
            r = torch.zeros(2, dtype=torch.int64, device=y_or.device)
            r[0], r[1] = n_fail, n_border
            rec.view(torch.int64)[0, 1:3].copy_(r)
            d, keep = refine_desc(node, xs, y32 if y32 is not None else c, c, rec.data_ptr(),
                                  border, model, profile)
            d.local64 = y_or.data_ptr()
            if y32 is None:
                d.local = None
            run_refine([d])
            h = CheckRecord(rec).host()
            n_fail, n_border = int(h["n_violations"]), int(h["n_borderline"])
            del keep
    return {"ok": n_fail == 0, "n_fail": n_fail, "n_borderline": n_border,
            "max_excess": float(excess.max()) if excess.numel() else float("-inf"),
            "y_oracle": y_or}


def sample_committee(pool, size: int, seed: int):
    """dispute.py:675-682: committee members without replacement (Rng(seed))."""
    from .tensor import Rng
    if size % 2 == 0:
        raise ValueError("committee size must be odd")
    if size > len(pool):
        raise ValueError(f"committee size {size} exceeds profile pool {len(pool)}")
    order = Rng(seed).permutation(len(pool))
    return [pool[i] for i in order[:size]]


def member_value(node, xs, member) -> torch.Tensor:
    """apply_op(node, args, member, fp64=False) on the GPU (the member's
    DeviceProfile emulated bit-exactly, csrc/profile_fold.cuh)."""
    from .bounds import FpModel, ROW_KINDS, apply_value, op_bound_device
    if node.kind in ROW_KINDS:
        y, _ = op_bound_device(node, xs, FpModel(), member, eps_f64=False)
        return y
    return apply_value(node, xs, member)


def leaf_route(node, args, claimed, thresholds=None, committee_pool=None, committee_size=3,
               committee_seed=0, model=None, profile=None, leaf=None) -> dict:
    """Challenger.leaf_payload's verdict (dispute.py:639-671) on the GPU, from
    the leaf's arguments on: the bound check (leaf_bound_check, exact), then
    either the theoretical FP64-oracle recheck or the committee vote -- each
    member re-executes the node under its DeviceProfile and votes
    observed_p_max <= 1 against the claimed tensor; majority wins.  Returns
    {"path", "winner", "evidence", "flops"} like the reference (evidence adds
    the undecided-element counts)."""
    from .bounds import FpModel
    from .commitments import tensor_digest
    from .tensor import Tensor
    model = model or FpModel()
    xs = _node_args(args)
    res = leaf_bound_check(node, xs, claimed, model, profile)
    y = res["y"]
    flops = node_flops(node, tuple(y.shape), [tuple(a.shape) for a in xs])
    c = claimed._dev if getattr(claimed, "_dev", None) is not None else claimed
    c = _node_args([c])[0]
    evidence = {"leaf": leaf if leaf is not None else getattr(node, "index", None),
                "leaf_name": node.name,
                "claimed_digest": tensor_digest(Tensor(tuple(c.shape), c.cpu().numpy().reshape(-1))),
                "undecided_bound_elements": res["n_borderline"]}
    if res["any_violation"]:
        orc = oracle_recheck(node, xs, c, res["eps"], model, profile)
        evidence["max_excess"] = orc["max_excess"]
        evidence["undecided_oracle_elements"] = orc["n_borderline"]
        return {"path": "theoretical", "winner": "proposer" if orc["ok"] else "challenger",
                "evidence": evidence, "flops": flops}
    if thresholds is None or committee_pool is None:
        raise ValueError("committee path needs thresholds and a profile pool")
    members = sample_committee(committee_pool, committee_size, committee_seed)
    votes = []
    for member in members:
        ym = member_value(node, xs, member)
        votes.append(observed_p_max(ym, c, thresholds, node.name) <= 1.0)
    within = sum(votes)
    evidence["votes_within"] = within
    evidence["committee"] = ",".join(m.id for m in members)
    return {"path": "committee", "winner": "proposer" if within * 2 > len(votes) else "challenger",
            "evidence": evidence, "flops": flops}


def to_device_eps(eps) -> torch.Tensor:
    if isinstance(eps, torch.Tensor):
        return eps if eps.is_cuda else eps.cuda()
    if hasattr(eps, "device_tensor"):
        return eps.device_tensor()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(eps, dtype=np.float64))).cuda()


__all__ = ["p_max", "observed_p_max", "screen", "select_offending", "check_node", "leaf_check",
           "leaf_bound_check", "oracle_recheck", "leaf_route", "sample_committee",
           "CheckRecord", "new_result_buffer", "commit_check_nodes", "combine_partials",
           "partial_from_bytes"]
_ = ctypes


# ------------------------------------------- challenger child re-execution
# Challenger._child_offense (dispute.py:544-559) on the
# GPU.  The child slice runs straight from the parent graph (no extracted
# sub-graph object): boundary tensors keyed by the parent refs the reference's
# SubgraphModule.placeholder_refs use ("input:<name>", "node:<i>"), weights
# from the graph, values under the challenger's DeviceProfile.

_FLOP_WEIGHTS = {"add": 1, "sub": 1, "mul": 1, "div": 1, "neg": 1, "relu": 1,
                 "exp": 4, "log": 4, "sqrt": 2, "rsqrt": 3, "tanh": 4, "gelu": 8, "silu": 6}


def node_flops(node, out_shape, in_shapes) -> int:
    """engine.py:409-429 analytic FLOP model (+ the extension kinds: conv2d as
    its implicit GEMM, the other extensions as data movement)."""
    from .graph import DATA_MOVEMENT_KINDS
    kind = node.kind
    out_size = int(np.prod(out_shape, dtype=np.int64)) if out_shape else 1
    if kind in DATA_MOVEMENT_KINDS or kind in ("transpose", "maxpool2d", "upsample2x"):
        return 0
    if kind in _FLOP_WEIGHTS:
        return _FLOP_WEIGHTS[kind] * out_size
    if kind in ("sum", "mean", "max", "min"):
        return int(np.prod(in_shapes[0], dtype=np.int64))
    if kind == "softmax":
        return 4 * int(np.prod(in_shapes[0], dtype=np.int64))
    if kind == "layernorm":
        return 8 * int(np.prod(in_shapes[0], dtype=np.int64))
    if kind == "matmul":
        return 2 * in_shapes[0][-1] * out_size
    if kind == "linear":
        return 2 * in_shapes[0][-1] * out_size + out_size
    if kind == "conv2d":
        return 2 * int(np.prod(in_shapes[1][1:], dtype=np.int64)) * out_size
    raise ValueError(f"no flop model for kind {kind!r}")


def run_slice(g, s, boundary: dict, profile=None, device=None):
    """engine.py:393-400 run_subgraph for nodes [s.start, s.end) of g on the
    GPU.  Returns ({node index: value}, flops) -- flops as graph_flops
    (engine.py:432-446) over the slice."""
    from .bounds import FpModel, apply_value, op_bound_device
    from .engine import DeviceProfile, ExecutionError
    from .graph import parse_ref
    profile = profile or DeviceProfile("seq", "sequential")
    dev = torch.device(device) if device is not None else torch.device("cuda")
    values, flops, model = {}, 0, FpModel()
    for i in range(s.start, s.end):
        node = g.nodes[i]
        xs, from_boundary = [], []
        for ref in node.inputs:
            cat, key = parse_ref(ref)
            if cat == "node" and s.contains(key):
                xs.append(values[key])
            elif cat == "weight":
                xs.append(to_device(g.weights[key], dev))
            else:
                if ref not in boundary:
                    raise ExecutionError(f"missing boundary tensor for {ref}")
                xs.append(to_device(boundary[ref], dev))
            from_boundary.append(cat != "weight" and not (cat == "node" and s.contains(key)))
        if node.kind in ("softmax", "layernorm", "sum", "mean", "max", "min"):
            y, _ = op_bound_device(node, xs, model, profile, eps_f64=None)
        else:
            y = apply_value(node, xs, profile)
        values[i] = y.contiguous()
        # graph_flops sees boundary tensors as the sub-graph's inputs, whose
        # shape it takes from the node's own output (engine.py:435-444)
        flops += node_flops(node, tuple(y.shape), [tuple(y.shape) if fb else tuple(x.shape)
                                                   for x, fb in zip(xs, from_boundary)])
    return values, flops


def child_offense(g, child, boundary: dict, claimed_outputs: dict, thresholds, profile=None,
                  device=None):
    """dispute.py:544-559: re-execute one child from its committed inputs and
    return (worst live-out p_max against the claimed tensors, FLOPs spent).
    claimed_outputs: {parent node index: claimed tensor} for the live-outs."""
    from .graph import frontiers
    values, flops = run_slice(g, child, boundary, profile, device)
    worst = 0.0
    for i in frontiers(g, child).out_nodes:
        worst = max(worst, observed_p_max(values[i], claimed_outputs[i], thresholds,
                                          g.nodes[i].name))
    return worst, flops
