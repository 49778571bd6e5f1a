"""ORACLE -- TEST INFRASTRUCTURE ONLY.  numpy restatement of the reference
bound templates and the FP32 value path they are co-computed with:
  /root/reference/pkg/src/fpverify/bounds.py   (FpModel, gamma, templates)
  /root/reference/pkg/src/fpverify/engine.py   (reduction orders, parts, apply_op)
Reduction orders (engine.py:75-113): "sequential" (default proposer profile,
config.py:14), "pairwise", "blocked" and "permuted" (Philox permutation), each
with and without fma; `profile` arguments are duck-typed DeviceProfiles
(.reduction, .block_size, .perm_seed, .fma), None = sequential.
Extension kinds (not in the reference) are marked as such;
their parity is unpinned by reference tests.
"""

from __future__ import annotations

import math

import numpy as np

FP32_UNIT_ROUNDOFF = 2.0 ** -24  # bounds.py:23
_SQRT_2_OVER_PI = math.sqrt(2.0 / math.pi)  # engine.py:23
_GELU_COEFF = 0.044715  # engine.py:24

DATA_MOVEMENT_KINDS = frozenset({"concat", "slice", "reshape", "embedding"})  # graph.py:27
EXT_DATA_MOVEMENT_KINDS = frozenset({"transpose", "maxpool2d", "upsample2x"})  # extensions
SINGLE_ROUNDING_KINDS = frozenset({"add", "sub", "mul", "div", "neg"})  # bounds.py:172
INTRINSIC_KINDS = frozenset({"exp", "log", "sqrt", "rsqrt", "tanh", "gelu", "silu"})  # :173


def gamma(k: int, u: float = FP32_UNIT_ROUNDOFF) -> float:
    """bounds.py:52-59."""
    if k < 0:
        raise ValueError("k must be nonnegative")
    ku = k * u
    if ku >= 1.0:
        raise ValueError(f"gamma undefined: k*u = {ku} >= 1")
    return ku / (1.0 - ku)


def gamma_tilde(k: int, lam: float = 4.0, u: float = FP32_UNIT_ROUNDOFF) -> float:
    """bounds.py:62-66."""
    if k < 0:
        raise ValueError("k must be nonnegative")
    return math.expm1(lam * math.sqrt(k) * u + k * u * u / (1.0 - u))


class FpModel:
    """bounds.py:26-49."""

    def __init__(self, u=FP32_UNIT_ROUNDOFF, lam=4.0, mode="probabilistic"):
        self.u, self.lam, self.mode = u, lam, mode

    def reduction_const(self, k: int) -> float:
        if self.mode == "deterministic":
            return gamma(k, self.u)
        return gamma_tilde(k, self.lam, self.u)


# ------------------------------------------------------------- value path


def fold_last(arr: np.ndarray) -> np.ndarray:
    """Sequential left fold over the last axis (engine.py:80-84)."""
    acc = arr[..., 0]
    for k in range(1, arr.shape[-1]):
        acc = acc + arr[..., k]
    return acc


def permutation(seed: int, n: int) -> np.ndarray:
    """engine.py:75-77 (numpy Philox: the permuted profile's fixed order)."""
    gen = np.random.Generator(np.random.Philox(key=seed, counter=n << 128))
    return gen.permutation(n)


def pairwise_last(arr: np.ndarray) -> np.ndarray:
    """engine.py:87-92: recursive halving, left half = ceil(n/2)."""
    n = arr.shape[-1]
    if n == 1:
        return arr[..., 0]
    mid = (n + 1) // 2
    return pairwise_last(arr[..., :mid]) + pairwise_last(arr[..., mid:])


def reduce_last_axis(arr: np.ndarray, profile=None) -> np.ndarray:
    """engine.py:95-113: the trailing-axis reduction in the profile's order."""
    n = arr.shape[-1]
    if n == 0:
        raise ValueError("cannot reduce an empty axis")
    red = "sequential" if profile is None else profile.reduction
    if red == "sequential":
        return fold_last(arr)
    if red == "pairwise":
        return pairwise_last(arr)
    if red == "blocked":
        b = max(1, int(profile.block_size))
        parts = [fold_last(arr[..., i:min(i + b, n)]) for i in range(0, n, b)]
        acc = parts[0]
        for q in parts[1:]:
            acc = acc + q
        return acc
    if red == "permuted":
        return fold_last(arr[..., permutation(int(profile.perm_seed), n)])
    raise ValueError(f"unknown reduction strategy {red!r}")


def _fma(profile, fma):
    return bool(fma) or bool(getattr(profile, "fma", False))


def unary_intrinsic(kind: str, x: np.ndarray) -> np.ndarray:
    """FP64 evaluation rounded once to FP32 (engine.py:133-154)."""
    with np.errstate(all="ignore"):
        x64 = x.astype(np.float64)
        if kind == "exp":
            out = np.exp(x64)
        elif kind == "log":
            out = np.log(x64)
        elif kind == "sqrt":
            out = np.sqrt(x64)
        elif kind == "rsqrt":
            out = 1.0 / np.sqrt(x64)
        elif kind == "tanh":
            out = np.tanh(x64)
        elif kind == "gelu":
            inner = _SQRT_2_OVER_PI * (x64 + _GELU_COEFF * x64 ** 3)
            out = 0.5 * x64 * (1.0 + np.tanh(inner))
        elif kind == "silu":
            out = x64 / (1.0 + np.exp(-x64))
        else:
            raise ValueError(kind)
    return out.astype(np.float32)


def matmul_value(a, b, transpose_b=False, fma=False, profile=None) -> np.ndarray:
    """matmul_op (engine.py:157-182): FP32 products reduced over K in the
    profile's order (sequential: column by column, no (..., M, K, N) product);
    fma: the sequential FP64-step loop whatever the order."""
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    if transpose_b:
        b = np.swapaxes(b, -1, -2)
    if a.shape[-1] != b.shape[-2]:
        raise ValueError(f"matmul inner dims disagree: {a.shape} @ {b.shape}")
    k_dim = a.shape[-1]
    fma = _fma(profile, fma)
    if not fma and profile is not None and profile.reduction != "sequential":
        prods = a[..., :, :, None] * b[..., None, :, :]  # (..., M, K, N) fp32
        return reduce_last_axis(np.moveaxis(prods, -2, -1), profile)
    if fma:
        a64 = a.astype(np.float64)
        b64 = b.astype(np.float64)
        acc = None
        for k in range(k_dim):
            step = a64[..., :, k, None] * b64[..., None, k, :]
            acc = step if acc is None else step + acc.astype(np.float64)
            acc = acc.astype(np.float32)
        return acc
    acc = None
    for k in range(k_dim):
        prod = a[..., :, k, None] * b[..., None, k, :]  # fp32 product rounding
        acc = prod if acc is None else acc + prod
    return acc


def softmax_parts(x, axis, profile=None):
    """engine.py:185-194."""
    xm = np.moveaxis(x, axis % x.ndim, -1)
    m = np.max(xm, axis=-1, keepdims=True)
    z = xm - m
    e = unary_intrinsic("exp", z)
    s = reduce_last_axis(e, profile)[..., None]
    y = e / s
    return {"m": m, "z": z, "e": e, "s": s, "y": np.moveaxis(y, -1, axis % x.ndim)}


def layernorm_parts(x, axis, eps, profile=None):
    """engine.py:197-213."""
    xm = np.moveaxis(x, axis % x.ndim, -1)
    n = xm.shape[-1]
    inv_n = np.float32(n)
    mu = (reduce_last_axis(xm, profile) / inv_n)[..., None]
    xc = xm - mu
    sq = xc * xc
    var = (reduce_last_axis(sq, profile) / inv_n)[..., None]
    sp = var + np.float32(eps)
    sigma = np.sqrt(sp)
    y = xc / sigma
    return {"mu": mu, "xc": xc, "sq": sq, "var": var, "sp": sp, "sigma": sigma,
            "y": np.moveaxis(y, -1, axis % x.ndim)}


def _parse_shape(spec) -> tuple:
    return tuple(int(t) for t in str(spec).split(",") if t != "")


def apply_op(node, arrays, fma=False, profile=None) -> np.ndarray:
    """engine.py:220-285 (FP32) under `profile` (None: sequential)."""
    kind = node.kind
    if kind in ("add", "sub", "mul", "div"):
        a, b = arrays
        return {"add": np.add, "sub": np.subtract, "mul": np.multiply,
                "div": np.divide}[kind](a, b)
    if kind == "neg":
        return -arrays[0]
    if kind == "relu":
        return np.maximum(arrays[0], np.zeros_like(arrays[0]))
    if kind in INTRINSIC_KINDS:
        return unary_intrinsic(kind, arrays[0])
    if kind in ("sum", "mean"):
        axis = int(node.attr("axis", -1))
        xm = np.moveaxis(arrays[0], axis % arrays[0].ndim, -1)
        red = reduce_last_axis(xm, profile)
        return red if kind == "sum" else red / np.float32(xm.shape[-1])
    if kind in ("max", "min"):
        axis = int(node.attr("axis", -1))
        fn = np.max if kind == "max" else np.min
        return fn(arrays[0], axis=axis % arrays[0].ndim)
    if kind == "matmul":
        return matmul_value(arrays[0], arrays[1], bool(node.attr("transpose_b", 0)), fma,
                            profile)
    if kind == "linear":
        x, w, b = arrays
        return matmul_value(x, w, False, fma, profile) + b
    if kind == "softmax":
        return softmax_parts(arrays[0], int(node.attr("axis", -1)), profile)["y"]
    if kind == "layernorm":
        return layernorm_parts(arrays[0], int(node.attr("axis", -1)),
                               float(node.attr("eps", 1e-5)), profile)["y"]
    if kind == "concat":
        return np.concatenate(arrays, axis=int(node.attr("axis", 0)))
    if kind == "slice":
        x = arrays[0]
        axis = int(node.attr("axis", 0))
        idx = [slice(None)] * x.ndim
        idx[axis % x.ndim] = slice(int(node.attr("start", 0)), int(node.attr("stop", 0)))
        return x[tuple(idx)]
    if kind == "reshape":
        return arrays[0].reshape(_parse_shape(node.attr("shape")))
    if kind == "embedding":
        ids, table = arrays
        idx = ids.astype(np.int64)
        if idx.size and (idx.min() < 0 or idx.max() >= table.shape[0]):
            raise ValueError("embedding index out of range")
        return table[idx]
    if kind == "transpose":  # extension: permutation of axes, pure data movement
        return np.transpose(arrays[0], _parse_shape(node.attr("perm")))
    if kind == "conv2d":  # extension: sequential matmul over im2col, K order (c, kh, kw)
        x, w = arrays
        col, (B, OH, OW) = im2col(x, w.shape[-1], int(node.attr("stride", 1)),
                                  int(node.attr("pad", 0)))
        out = matmul_value(col, w.reshape(w.shape[0], -1), True, fma)
        return np.ascontiguousarray(out.reshape(B, OH, OW, w.shape[0]).transpose(0, 3, 1, 2))
    if kind == "upsample2x":  # extension: nearest-neighbour 2x
        return np.repeat(np.repeat(arrays[0], 2, axis=-2), 2, axis=-1)
    if kind == "maxpool2d":  # extension: exact max over windows (padding = -inf)
        x = arrays[0]
        k, st, pd = int(node.attr("k", 2)), int(node.attr("stride", 2)), int(node.attr("pad", 0))
        xp = np.pad(x, ((0, 0), (0, 0), (pd, pd), (pd, pd)), constant_values=-np.inf)
        B, C, H, W = xp.shape
        OH, OW = (H - k) // st + 1, (W - k) // st + 1
        out = np.full((B, C, OH, OW), -np.inf, dtype=np.float32)
        for i in range(k):
            for j in range(k):
                out = np.maximum(out, xp[:, :, i:i + st * OH:st, j:j + st * OW:st])
        return out
    raise ValueError(f"unsupported op kind {kind!r}")


def im2col(x, k: int, stride: int, pad: int):
    """[B, C, H, W] -> ([B, OH*OW, C*k*k], (B, OH, OW)); K ordered (c, kh, kw)."""
    x = np.asarray(x, dtype=np.float32)
    B, C, H, W = x.shape
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    OH, OW = (H + 2 * pad - k) // stride + 1, (W + 2 * pad - k) // stride + 1
    cols = np.empty((B, C, k, k, OH, OW), dtype=np.float32)
    for i in range(k):
        for j in range(k):
            cols[:, :, i, j] = xp[:, :, i:i + stride * OH:stride, j:j + stride * OW:stride]
    return cols.reshape(B, C * k * k, OH * OW).transpose(0, 2, 1), (B, OH, OW)


# --------------------------------------------------------------- templates


def _abs64(a) -> np.ndarray:
    return np.abs(np.asarray(a).astype(np.float64))


def matmul_bound(a, b, model: FpModel, fma=False, transpose_b=False) -> np.ndarray:
    """bounds.py:100-111: const(count) * (|A|64 @ |B|64), count = 2K-1 or K."""
    a64 = _abs64(a)
    b64 = _abs64(b)
    if transpose_b:
        b64 = np.swapaxes(b64, -1, -2)
    k_dim = a64.shape[-1]
    if k_dim != b64.shape[-2]:
        raise ValueError(f"matmul inner dims disagree: {a64.shape} @ {b64.shape}")
    count = k_dim if fma else 2 * k_dim - 1
    return model.reduction_const(count) * (a64 @ b64)


def softmax_bound_parts(x, axis, model: FpModel, profile=None):
    """bounds.py:114-135."""
    x = np.asarray(x)
    parts = softmax_parts(x, axis, profile)
    u = model.u
    n = parts["e"].shape[-1]
    rc = model.reduction_const(n - 1)
    xm = np.moveaxis(x, axis % x.ndim, -1).astype(np.float64)
    m64 = parts["m"].astype(np.float64)
    e64 = _abs64(parts["e"])
    s64 = _abs64(parts["s"])
    y_last = np.moveaxis(parts["y"], axis % x.ndim, -1)
    eps_z = u * (np.abs(xm) + np.abs(m64))
    eps_e = e64 * eps_z + 2.0 * u * e64
    eps_s = rc * np.sum(e64, axis=-1, keepdims=True) + (rc + 1.0) * np.sum(
        eps_e, axis=-1, keepdims=True)
    eps_y = eps_e / s64 + e64 * eps_s / s64 ** 2 + u * _abs64(y_last)
    return parts["y"], np.moveaxis(eps_y, -1, axis % x.ndim)


def layernorm_bound_parts(x, axis, eps_attr, model: FpModel, profile=None):
    """bounds.py:143-169."""
    x = np.asarray(x)
    parts = layernorm_parts(x, axis, eps_attr, profile)
    u = model.u
    n = parts["xc"].shape[-1]
    rc = model.reduction_const(n - 1)
    xm64 = np.moveaxis(x, axis % x.ndim, -1).astype(np.float64)
    mu = _abs64(parts["mu"])
    xc = _abs64(parts["xc"])
    sq = _abs64(parts["sq"])
    var = _abs64(parts["var"])
    sp = _abs64(parts["sp"])
    sigma = _abs64(parts["sigma"])
    y_last = np.moveaxis(parts["y"], axis % x.ndim, -1)
    eps_mu = rc * np.sum(np.abs(xm64), axis=-1, keepdims=True) / n + u * mu
    eps_xc = eps_mu + u * xc
    eps_sq = 2.0 * xc * eps_xc + u * sq
    eps_ssq = rc * np.sum(sq, axis=-1, keepdims=True) + (rc + 1.0) * np.sum(
        eps_sq, axis=-1, keepdims=True)
    eps_var = eps_ssq / n + u * var
    eps_sp = eps_var + u * sp
    eps_sigma = eps_sp / (2.0 * sigma) + u * sigma
    eps_y = eps_xc / sigma + xc * eps_sigma / sigma ** 2 + u * _abs64(y_last)
    return parts["y"], np.moveaxis(eps_y, -1, axis % x.ndim)


def op_bound(node, arrays, model: FpModel, fma=False, profile=None):
    """bounds.py:176-218 -> (y float32, eps float64)."""
    kind = node.kind
    fma = _fma(profile, fma)
    if kind == "softmax":
        return softmax_bound_parts(arrays[0], int(node.attr("axis", -1)), model, profile)
    if kind == "layernorm":
        return layernorm_bound_parts(arrays[0], int(node.attr("axis", -1)),
                                     float(node.attr("eps", 1e-5)), model, profile)
    out = apply_op(node, arrays, fma, profile)
    u = model.u
    if kind in DATA_MOVEMENT_KINDS or kind in EXT_DATA_MOVEMENT_KINDS or kind in (
            "relu", "max", "min"):
        return out, np.zeros(out.shape, dtype=np.float64)
    if kind in SINGLE_ROUNDING_KINDS:
        return out, u * _abs64(out)
    if kind in INTRINSIC_KINDS:
        return out, 2.0 * u * _abs64(out)
    if kind in ("sum", "mean"):
        axis = int(node.attr("axis", -1)) % arrays[0].ndim
        x64 = np.abs(arrays[0].astype(np.float64))
        n = x64.shape[axis]
        rc = model.reduction_const(n - 1)
        eps = rc * np.sum(x64, axis=axis)
        if kind == "mean":
            eps = eps / n + u * _abs64(out)
        return out, eps
    if kind == "matmul":
        return out, matmul_bound(arrays[0], arrays[1], model, fma,
                                 bool(node.attr("transpose_b", 0)))
    if kind == "linear":
        return out, matmul_bound(arrays[0], arrays[1], model, fma) + u * _abs64(out)
    if kind == "conv2d":  # extension: matmul_bound over the implicit im2col
        x, w = arrays
        col, (B, OH, OW) = im2col(x, w.shape[-1], int(node.attr("stride", 1)),
                                  int(node.attr("pad", 0)))
        eps = matmul_bound(col, w.reshape(w.shape[0], -1), model, fma, transpose_b=True)
        return out, np.ascontiguousarray(eps.reshape(B, OH, OW, w.shape[0]).transpose(0, 3, 1, 2))
    raise ValueError(f"no bound template for kind {kind!r}")


def co_execute(graph, inputs: dict, model: FpModel, fma=False, inject=None):
    """bounds.py:221-262 over numpy arrays: returns (values, bounds) lists in
    canonical node order.  `inject` mirrors engine.py:348-351."""
    values, bounds = [], []
    for node in graph.nodes:
        args = []
        for ref in node.inputs:
            cat, _, key = ref.partition(":")
            if cat == "node":
                args.append(values[int(key)])
            elif cat == "input":
                args.append(np.asarray(inputs[key], dtype=np.float32))
            else:
                args.append(np.asarray(graph.weight_array(key), dtype=np.float32))
        out, eps = op_bound(node, args, model, fma)
        out = np.ascontiguousarray(out, dtype=np.float32)
        if inject and node.index in inject:
            out = np.ascontiguousarray(out + np.asarray(inject[node.index], np.float32),
                                       dtype=np.float32)
        if out.size and not np.all(np.isfinite(out)):
            raise FloatingPointError(f"non-finite intermediate at node {node.index}")
        values.append(out)
        bounds.append(np.asarray(eps, dtype=np.float64))
    return values, bounds


# ------------------------------------------- FP64 oracle (theoretical path)

def matmul_fp64(a, b, transpose_b=False) -> np.ndarray:
    """engine.py:173-177 (fp64=True): FP64 products, sequential fold over K
    (reduce_last_axis(profile=None), engine.py:95-103).  Folded k-slice by
    k-slice instead of materialising the (M, K, N) product array -- the same
    additions in the same order."""
    a = np.asarray(a, np.float32).astype(np.float64)
    b = np.asarray(b, np.float32).astype(np.float64)
    if transpose_b:
        b = np.swapaxes(b, -1, -2)
    acc = a[..., :, 0:1] * b[..., 0:1, :]
    for k in range(1, a.shape[-1]):
        acc = acc + a[..., :, k:k + 1] * b[..., k:k + 1, :]
    return acc


def apply_op_fp64(node, arrays) -> np.ndarray:
    """apply_op(node, args64, None, fp64=True) (engine.py:220-285) for the
    reduction kinds and matmul (the leaf route's FP64 oracle recheck,
    dispute.py:648-656): sequential FP64 folds."""
    kind = node.kind
    x = np.asarray(arrays[0], np.float32).astype(np.float64)
    if kind == "matmul":
        return matmul_fp64(arrays[0], arrays[1], bool(node.attr("transpose_b", 0)))
    if kind == "linear":
        return matmul_fp64(arrays[0], arrays[1]) + np.asarray(arrays[2], np.float32).astype(np.float64)
    axis = int(node.attr("axis", -1)) % x.ndim
    xm = np.moveaxis(x, axis, -1)
    n = xm.shape[-1]
    if kind in ("sum", "mean"):
        red = fold_last(xm)
        return red if kind == "sum" else red / np.float64(n)
    if kind == "softmax":  # engine.py:185-194
        m = np.max(xm, axis=-1, keepdims=True)
        e = np.exp(xm - m)
        y = e / fold_last(e)[..., None]
        return np.moveaxis(y, -1, axis)
    if kind == "layernorm":  # engine.py:197-213 (eps as the attribute's double)
        mu = (fold_last(xm) / np.float64(n))[..., None]
        xc = xm - mu
        var = (fold_last(xc * xc) / np.float64(n))[..., None]
        y = xc / np.sqrt(var + np.float64(float(node.attr("eps", 1e-5))))
        return np.moveaxis(y, -1, axis)
    raise ValueError(f"oracle apply_op_fp64: kind {kind!r} not restated")
