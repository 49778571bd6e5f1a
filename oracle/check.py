"""ORACLE -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the threshold check
and the leaf bound check:
  /root/reference/pkg/src/fpverify/calibration.py:16-49  (grid, percentile, errors)
  /root/reference/pkg/src/fpverify/dispute.py:114-158    (p_max, observed_p_max, screen)
  /root/reference/pkg/src/fpverify/dispute.py:639-657    (leaf: any(|y'-y| > eps))
The percentile arithmetic is numpy 2.3's method="linear" (third-party,
pinned in the container: numpy 2.3.5, numpy/lib/_function_base_impl.py:126-129
(n-1)*q, :4277 q = p/100, :4753-4786 _get_indexes, :4657-4679 _lerp).
`percentile_profile_sorted` restates that arithmetic from a full sort so the
GPU radix-select path has an independent, explicit oracle.
"""

from __future__ import annotations

import math

import numpy as np

PERCENTILE_GRID = (0.0, 1.0) + tuple(float(p) for p in range(5, 100, 5)) + (99.0, 100.0)  # calibration.py:16
DEFAULT_EPSILON = 1e-12  # calibration.py:19


def percentile_profile(values, grid=PERCENTILE_GRID) -> np.ndarray:
    """calibration.py:33-37."""
    arr = np.asarray(values, dtype=np.float64).reshape(-1)
    if arr.size == 0:
        raise ValueError("percentile profile of empty input")
    return np.percentile(arr, list(grid), method="linear")


def lerp(a: float, b: float, t: float) -> float:
    """numpy _lerp (_function_base_impl.py:4657-4679), scalar FP64, no FMA."""
    d = b - a
    r = a + d * t
    if t >= 0.5:
        r = b - d * (1.0 - t)
    return r


def percentile_from_sorted(xs: np.ndarray, p: float) -> float:
    n = xs.shape[0]
    q = float(p) / 100.0
    vi = (n - 1) * q
    if vi >= n - 1:
        prev = nxt = n - 1
        g = vi - (-1.0)
    else:
        prev = int(math.floor(vi))
        nxt = prev + 1
        g = vi - prev
    return lerp(float(xs[prev]), float(xs[nxt]), g)


def percentile_profile_sorted(values, grid=PERCENTILE_GRID) -> np.ndarray:
    xs = np.sort(np.asarray(values, dtype=np.float64).reshape(-1))
    if xs.size == 0:
        raise ValueError("percentile profile of empty input")
    return np.array([percentile_from_sorted(xs, p) for p in grid])


def elementwise_errors(local, claimed, epsilon=DEFAULT_EPSILON):
    """calibration.py:40-49 / dispute.py:134-138: denominator = |local| + eps."""
    a = np.asarray(local, dtype=np.float32).reshape(-1).astype(np.float64)
    b = np.asarray(claimed, dtype=np.float32).reshape(-1).astype(np.float64)
    abs_err = np.abs(a - b)
    rel_err = abs_err / (np.abs(a) + epsilon)
    return abs_err, rel_err


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


def observed_p_max(local, claimed, tau_abs, tau_rel, grid=PERCENTILE_GRID,
                   epsilon=DEFAULT_EPSILON) -> float:
    """dispute.py:130-141."""
    abs_e, rel_e = elementwise_errors(local, claimed, epsilon)
    return p_max(percentile_profile(abs_e, grid), percentile_profile(rel_e, grid),
                 tau_abs, tau_rel)


def leaf_check(local, claimed, eps) -> dict:
    """dispute.py:641-648: violation iff |claimed - y_ref| > eps (strict)."""
    diff = np.abs(np.asarray(claimed, np.float32).astype(np.float64)
                  - np.asarray(local, np.float32).astype(np.float64)).reshape(-1)
    eps = np.asarray(eps, dtype=np.float64).reshape(-1)
    viol = diff > eps
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(eps > 0, diff / np.where(eps > 0, eps, 1.0),
                         np.where(diff > 0, np.inf, 0.0))
    return {"n_violations": int(np.count_nonzero(viol)),
            "max_ratio": float(ratio.max()) if ratio.size else 0.0,
            "any_violation": bool(viol.any())}


def calibrate(graph, dataset, fmas, grid=PERCENTILE_GRID, epsilon=DEFAULT_EPSILON):
    """calibration.py:70-114 restated for the sequential profile family
    (fmas: list of bool, one simulated device each): max envelope over
    (input, pair) of abs profiles and of rel profiles in both orientations."""
    from . import bounds as OB
    n_nodes = len(graph.nodes)
    G = len(grid)
    abs_env = [np.zeros(G) for _ in range(n_nodes)]
    rel_env = [np.zeros(G) for _ in range(n_nodes)]
    for sample in dataset:
        traces = [OB.co_execute(graph, sample, OB.FpModel(), fma=f)[0] for f in fmas]
        for i in range(n_nodes):
            flats = [t[i].reshape(-1).astype(np.float64) for t in traces]
            for j in range(len(fmas)):
                for k in range(j + 1, len(fmas)):
                    diff = np.abs(flats[j] - flats[k])
                    stacked = np.stack([diff, diff / (np.abs(flats[j]) + epsilon),
                                        diff / (np.abs(flats[k]) + epsilon)])
                    profs = np.percentile(stacked, list(grid), axis=1, method="linear")
                    np.maximum(abs_env[i], profs[:, 0], out=abs_env[i])
                    np.maximum(rel_env[i], profs[:, 1], out=rel_env[i])
                    np.maximum(rel_env[i], profs[:, 2], out=rel_env[i])
    return abs_env, rel_env


def shard_partial(local, claimed, eps, tau_abs, tau_rel, grid=PERCENTILE_GRID,
                  epsilon=DEFAULT_EPSILON) -> dict:
    """A shard's combinable check state (the nao_check_partial the GPU emits for
    batch-sharded verification; not a reference function -- it restates the
    pieces of dispute.py:130-141 / :641-648 that add up across shards): exact
    FP64 keys bucketed by the number of sorted effective thresholds strictly
    below them, bucket counts and key ranges, violation counts, max ratio."""
    G = len(grid)
    a, r = elementwise_errors(local, claimed, epsilon)
    out = {"n": int(a.size)}
    lc = leaf_check(local, claimed, eps)
    out["n_violations"], out["max_ratio"] = lc["n_violations"], lc["max_ratio"]
    out["n_borderline"], out["n_nonfinite"] = 0, 0
    for key, vals, taus in (("abs", a, tau_abs), ("rel", r, tau_rel)):
        srt = np.sort(np.maximum(np.asarray(taus, dtype=np.float64), 0.0))
        b = np.searchsorted(srt, vals, side="left")  # #{t < key}
        hist = np.bincount(b, minlength=33)[:33].astype(np.uint64)
        mn = np.full(33, np.inf)
        mx = np.zeros(33)
        for k in range(G + 1):
            sel = vals[b == k]
            if sel.size:
                mn[k], mx[k] = sel.min(), sel.max()
        out[f"hist_{key}"], out[f"min_{key}"], out[f"max_{key}"] = hist, mn, mx
    return out
