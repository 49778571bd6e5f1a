"""Percentile thresholds on the GPU -- drop-in for the hot-path part of
/root/reference/pkg/src/fpverify/calibration.py (PERCENTILE_GRID :16,
percentile :23-30, percentile_profile :33-37, elementwise_errors :40-49,
error_profiles :52-55, OpThresholds/ThresholdSet :117-191,
build_thresholds :194-203).

Percentiles are numpy's method="linear" computed exactly (full radix sort of
the FP64 keys, numpy _lerp arithmetic) in nao_percentile_profile /
nao_error_profiles.  Offline calibration (`calibrate`, stability reports)
is SURVEY.md 8(f) row 1 ("next").
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .engine import to_device

PERCENTILE_GRID = (0.0, 1.0) + tuple(float(p) for p in range(5, 100, 5)) + (99.0, 100.0)
THRESHOLD_FILE_VERSION = 1
DEFAULT_EPSILON = 1e-12
DEFAULT_ALPHA = 3.0


def _flat_f64(values) -> torch.Tensor:
    if isinstance(values, torch.Tensor):
        t = values.reshape(-1)
        return (t if t.is_cuda else t.cuda()).double().contiguous()
    arr = np.ascontiguousarray(np.asarray(values, dtype=np.float64).reshape(-1))
    return torch.from_numpy(arr).cuda()


def percentile_profile_device(values: torch.Tensor, grid=PERCENTILE_GRID) -> torch.Tensor:
    v = _flat_f64(values)
    n = v.numel()
    if n == 0:
        raise ValueError("percentile profile of empty input")
    out = torch.empty(len(grid), dtype=torch.float64, device=v.device)
    ws = _lib.workspace(_lib.load().nao_percentile_workspace(n), v.device)
    _lib.call("nao_percentile_profile", v.data_ptr(), n, _lib.dbl_array(grid), len(grid),
              out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr(v.device))
    return out


def percentile_profile(values, grid=PERCENTILE_GRID) -> np.ndarray:
    """calibration.py:33-37 (exact numpy "linear")."""
    return percentile_profile_device(values, grid).cpu().numpy()


def percentile(values, p: float) -> float:
    """calibration.py:23-30."""
    return float(percentile_profile(values, (float(p),))[0])


def error_profiles_device(local: torch.Tensor, claimed: torch.Tensor, grid=PERCENTILE_GRID,
                          epsilon: float = DEFAULT_EPSILON):
    """Exact percentile profiles of |a-b| and |a-b|/(|a|+eps) (calibration.py:40-55)."""
    a = to_device(local).reshape(-1).contiguous()
    b = to_device(claimed).reshape(-1).contiguous()
    if a.numel() != b.numel():
        raise ValueError(f"shape mismatch: {a.numel()} vs {b.numel()}")
    n = a.numel()
    if n == 0:
        raise ValueError("percentile profile of empty input")
    pa = torch.empty(len(grid), dtype=torch.float64, device=a.device)
    pr = torch.empty(len(grid), dtype=torch.float64, device=a.device)
    ws = _lib.workspace(_lib.load().nao_percentile_workspace(n), a.device)
    _lib.call("nao_error_profiles", a.data_ptr(), b.data_ptr(), n, float(epsilon),
              _lib.dbl_array(grid), len(grid), pa.data_ptr(), pr.data_ptr(), ws.data_ptr(),
              ws.numel(), _lib.stream_ptr(a.device))
    return pa, pr


def elementwise_errors(y_a, y_b, epsilon: float = DEFAULT_EPSILON):
    """calibration.py:40-49 (host arrays, exact FP64 like the reference)."""
    if tuple(y_a.shape) != tuple(y_b.shape):
        raise ValueError(f"shape mismatch: {y_a.shape} vs {y_b.shape}")
    a = to_device(y_a.data if hasattr(y_a, "data") and not isinstance(y_a, torch.Tensor) else y_a)
    b = to_device(y_b.data if hasattr(y_b, "data") and not isinstance(y_b, torch.Tensor) else y_b)
    a64, b64 = a.reshape(-1).double(), b.reshape(-1).double()
    abs_err = (a64 - b64).abs()
    rel_err = abs_err / (a64.abs() + epsilon)
    return abs_err.cpu().numpy(), rel_err.cpu().numpy()


def error_profiles(y_a, y_b, grid=PERCENTILE_GRID, epsilon: float = DEFAULT_EPSILON):
    if tuple(y_a.shape) != tuple(y_b.shape):
        raise ValueError(f"shape mismatch: {y_a.shape} vs {y_b.shape}")
    pa, pr = error_profiles_device(_payload(y_a), _payload(y_b), grid, epsilon)
    return pa.cpu().numpy(), pr.cpu().numpy()


def _payload(t):
    if isinstance(t, torch.Tensor) or isinstance(t, np.ndarray):
        return t
    if hasattr(t, "_dev") and t._dev is not None:
        return t._dev
    return np.asarray(t.data)


@dataclass(frozen=True)
class OpThresholds:
    name: str
    tau_abs: np.ndarray
    tau_rel: np.ndarray


@dataclass
class ThresholdSet:
    """calibration.py:124-191."""
    alpha: float
    epsilon: float
    grid: tuple
    ops: list

    def __post_init__(self):
        self._by_name = {op.name: op for op in self.ops}

    def lookup(self, name: str) -> OpThresholds:
        if name not in self._by_name:
            raise KeyError(f"no thresholds for operator {name!r}")
        return self._by_name[name]

    def scaled(self, alpha: float) -> "ThresholdSet":
        if alpha <= 0:
            raise ValueError("alpha must be positive")
        f = alpha / self.alpha
        return ThresholdSet(alpha=alpha, epsilon=self.epsilon, grid=self.grid,
                            ops=[OpThresholds(o.name, o.tau_abs * f, o.tau_rel * f)
                                 for o in self.ops])

    def to_json(self) -> dict:
        return {"version": THRESHOLD_FILE_VERSION, "alpha": self.alpha, "epsilon": self.epsilon,
                "grid": list(self.grid),
                "ops": [{"name": o.name, "tau_abs": [float(v) for v in o.tau_abs],
                         "tau_rel": [float(v) for v in o.tau_rel]} for o in self.ops]}

    @classmethod
    def from_json(cls, doc: dict) -> "ThresholdSet":
        if doc.get("version") != THRESHOLD_FILE_VERSION:
            raise ValueError(f"unsupported threshold file version {doc.get('version')}")
        ops = [OpThresholds(e["name"], np.asarray(e["tau_abs"], dtype=np.float64),
                            np.asarray(e["tau_rel"], dtype=np.float64)) for e in doc["ops"]]
        return cls(alpha=doc["alpha"], epsilon=doc["epsilon"], grid=tuple(doc["grid"]), ops=ops)

    def save(self, path) -> None:
        with open(path, "w") as fh:
            json.dump(self.to_json(), fh, sort_keys=True, indent=1)

    @classmethod
    def load(cls, path) -> "ThresholdSet":
        with open(path) as fh:
            return cls.from_json(json.load(fh))


def build_thresholds(names, abs_env, rel_env, grid=PERCENTILE_GRID, alpha: float = DEFAULT_ALPHA,
                     epsilon: float = DEFAULT_EPSILON) -> ThresholdSet:
    """calibration.py:194-203 from per-node envelopes."""
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    ops = [OpThresholds(n, alpha * np.asarray(a, np.float64), alpha * np.asarray(r, np.float64))
           for n, a, r in zip(names, abs_env, rel_env)]
    return ThresholdSet(alpha=alpha, epsilon=epsilon, grid=tuple(grid), ops=ops)


# ------------------------------------------------------------ calibration
# calibrate / build_thresholds on the GPU.

@dataclass
class EnvelopeSet:
    """calibration.py:58-67."""
    grid: tuple
    abs_env: list
    rel_env: list
    node_names: list
    per_sample_abs: list


def calibrate(g, dataset, profiles, grid=PERCENTILE_GRID, epsilon: float = DEFAULT_EPSILON,
              device="cuda") -> EnvelopeSet:
    """calibration.py:70-114: every input under every profile; per node the
    pointwise max over (input, profile pair) of the exact abs percentile
    profile and of the rel profile in BOTH orientations.  The profiles run in
    lockstep node by node, so only one node's values per profile are live
    beyond their last use (no full traces)."""
    from .bounds import apply_value, reduce_device, softmax_device, layernorm_device, FpModel
    from .engine import require_supported
    from .executor import last_uses
    from .graph import parse_ref
    if len(profiles) < 2:
        raise ValueError("calibration requires at least 2 device profiles")
    if not dataset:
        raise ValueError("calibration requires at least 1 input")
    for p in profiles:
        require_supported(p)
    n_nodes, G = g.n_nodes, len(grid)
    dev = torch.device(device)
    abs_env = [torch.zeros(G, dtype=torch.float64, device=dev) for _ in range(n_nodes)]
    rel_env = [torch.zeros(G, dtype=torch.float64, device=dev) for _ in range(n_nodes)]
    per_sample_abs = [[] for _ in range(n_nodes)]
    last = last_uses(g)
    model = FpModel()

    def value(node, xs, prof):
        k = node.kind
        if k == "softmax":
            return softmax_device(xs[0], int(node.attr("axis", -1)), model, False, prof)[0]
        if k == "layernorm":
            return layernorm_device(xs[0], int(node.attr("axis", -1)),
                                    float(node.attr("eps", 1e-5)), model, False, prof)[0]
        if k in ("sum", "mean", "max", "min"):
            return reduce_device(k, xs[0], int(node.attr("axis", -1)), model, False, prof)[0]
        return apply_value(node, xs, prof)

    for sample in dataset:
        vals = [dict() for _ in profiles]
        for node in g.nodes:
            outs = []
            for pi, prof in enumerate(profiles):
                xs = []
                for ref in node.inputs:
                    cat, key = parse_ref(ref)
                    xs.append(vals[pi][key] if cat == "node" else to_device(
                        sample[key] if cat == "input" else g.weights[key], dev))
                y = value(node, xs, prof).contiguous()
                vals[pi][node.index] = y
                outs.append(y.reshape(-1))
            i = node.index
            sample_abs = torch.zeros(G, dtype=torch.float64, device=dev)
            for j in range(len(profiles)):
                for k in range(j + 1, len(profiles)):
                    pa, pr_j = error_profiles_device(outs[j], outs[k], grid, epsilon)
                    _, pr_k = error_profiles_device(outs[k], outs[j], grid, epsilon)
                    torch.maximum(abs_env[i], pa, out=abs_env[i])
                    torch.maximum(rel_env[i], pr_j, out=rel_env[i])
                    torch.maximum(rel_env[i], pr_k, out=rel_env[i])
                    torch.maximum(sample_abs, pa, out=sample_abs)
            per_sample_abs[i].append(sample_abs)
            for pi in range(len(profiles)):
                for ref in node.inputs:
                    cat, key = parse_ref(ref)
                    if cat == "node" and last.get(key, -1) == node.index:
                        vals[pi].pop(key, None)
    return EnvelopeSet(grid=tuple(grid), abs_env=[e.cpu().numpy() for e in abs_env],
                       rel_env=[e.cpu().numpy() for e in rel_env],
                       node_names=[n.name for n in g.nodes],
                       per_sample_abs=[[s.cpu().numpy() for s in row] for row in per_sample_abs])


def build_thresholds_from_envelopes(env: EnvelopeSet, alpha: float = DEFAULT_ALPHA,
                                    epsilon: float = DEFAULT_EPSILON) -> ThresholdSet:
    """calibration.py:194-203."""
    return build_thresholds(env.node_names, env.abs_env, env.rel_env, env.grid, alpha, epsilon)
