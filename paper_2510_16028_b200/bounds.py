"""Per-operator IEEE-754 bounds co-computed with FP32 execution on the B200 --
drop-in for /root/reference/pkg/src/fpverify/bounds.py.

Same API and semantics (FpModel, gamma, gamma_tilde, BoundTensor,
matmul_bound, softmax_bound(_parts), layernorm_bound_parts, op_bound,
co_execute, save_bounds); the arithmetic runs in libnao_b200.so:
  * matmul / linear  -> nao_abs_gemm_bound   (bounds.py:100-111, :209-217)
  * softmax          -> nao_softmax_bound    (bounds.py:114-135)
  * layernorm        -> nao_layernorm_bound  (bounds.py:143-169)
  * sum/mean/max/min -> nao_reduce_bound     (bounds.py:194-208)
  * u|y|, 2u|y|      -> nao_scaled_abs_bound (bounds.py:196-199)
Guarantee vs the reference (tests/test_bounds_gpu.py):
  eps_ref <= eps_gpu <= eps_ref * (1 + 1e-5).
numpy arrays in -> numpy arrays out (host sync, like the reference);
CUDA tensors in -> CUDA tensors out (asynchronous).
"""

from __future__ import annotations

import math
import os
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .engine import (ExecutionError, fma_of, matmul_value, parse_shape_attr, relu,
                     profile_arg, require_f32, require_supported, to_device, unary,
                     _batch_view)
from .graph import DATA_MOVEMENT_KINDS, parse_ref
from .tensor import Tensor

FP32_UNIT_ROUNDOFF = 2.0 ** -24
SINGLE_ROUNDING_KINDS = frozenset({"add", "sub", "mul", "div", "neg"})
INTRINSIC_KINDS = frozenset({"exp", "log", "sqrt", "rsqrt", "tanh", "gelu", "silu"})
ZERO_BOUND_KINDS = DATA_MOVEMENT_KINDS | {"transpose", "relu", "max", "min", "maxpool2d",
                                          "upsample2x"}


@dataclass(frozen=True)
class FpModel:
    """bounds.py:26-49."""
    u: float = FP32_UNIT_ROUNDOFF
    lam: float = 4.0
    mode: str = "probabilistic"

    def __post_init__(self):
        if self.u <= 0:
            raise ValueError("unit roundoff must be positive")
        if self.lam <= 0:
            raise ValueError("lambda must be positive")
        if self.mode not in ("deterministic", "probabilistic"):
            raise ValueError(f"unknown bound mode {self.mode!r}")

    def reduction_const(self, k: int) -> float:
        if self.mode == "deterministic":
            return gamma(k, self.u)
        return gamma_tilde(k, self.lam, self.u)

    def confidence(self) -> float:
        return 1.0 - 2.0 * math.exp(-self.lam ** 2 * (1.0 - self.u) ** 2 / 2.0)


def gamma(k: int, u: float = FP32_UNIT_ROUNDOFF) -> float:
    """Deterministic k u / (1 - k u)  (bounds.py:52-59)."""
    if k < 0:
        raise ValueError("k must be nonnegative")
    ku = k * u
    if ku >= 1.0:
        raise ValueError(f"gamma undefined: k*u = {ku} >= 1")
    return ku / (1.0 - ku)


def gamma_tilde(k: int, lam: float = 4.0, u: float = FP32_UNIT_ROUNDOFF) -> float:
    """Probabilistic expm1(lam sqrt(k) u + k u^2/(1-u))  (bounds.py:62-66)."""
    if k < 0:
        raise ValueError("k must be nonnegative")
    return math.expm1(lam * math.sqrt(k) * u + k * u * u / (1.0 - u))


# Slack factors: eps_gpu = template * (1 + slack).  They cover only FP64
# summation-order differences vs numpy (pairwise np.sum / BLAS), so they sit
# ~1e-12 -- far inside rtol 1e-5 -- while keeping eps_gpu >= eps_ref.
def sum_slack(n: int) -> float:
    return 4.0 * max(int(n), 1) * 2.0 ** -53 + 2.0 ** -50


def gemm_slack(k: int) -> float:
    return (int(k) + int(k) // 32 + 16) * 2.0 ** -52


# Certified over-estimates R: eps_ref <= eps_gpu <= R * eps_ref for every
# element, per bound path.  A check counts eps_gpu/R < diff <=
# eps_gpu as borderline (its lo_factor is 1/R); those elements are settled
# exactly by nao_refine_borderline.
def _tc_overestimate(K: int, f16: bool) -> float:
    """tcgen05 3-split: split excess (hi+lo < |x|(1+2^-20), per operand),
    the dropped-lo compensation, the acc0 chunk compensation (the MMA
    accumulation is modelled as losing <= 3*2^-23 per instruction, never
    gaining), the acc1 compensation on its <= 2^-8 share, FP16 tiny parts
    (<= 2^-20) and the epilogue's slack."""
    kchunk = int(_lib.load(require_cuda=False).nao_abs_gemm_tc_kchunk())
    bk = 32 if f16 else 16
    kp = (K + 7) // 8 * 8 if f16 else (K + 3) // 4 * 4
    nkb = -(-kp // bk)
    mma = 3.0 * 2.0 ** -23
    comp0 = 1.0 / (1.0 - (kchunk // 16) * 2 * mma)  # KCHUNK_KB k-blocks of 64 B, 2 MMAs each
    comp1 = 1.0 / (1.0 - 2.0 * nkb * 2 * mma)
    comp_split = 1.0 / (1.0 - 1.002 * 2.0 ** -20)
    r = comp_split * comp0 * (1.0 + (comp1 - 1.0) * 2.0 ** -8) * (1.0 + 2.0 ** -20) ** 2
    if f16:
        r *= 1.0 + 2.0 ** -20
    return r * (1.0 + gemm_slack(K)) * (1.0 + 2.0 ** -50) * (1.0 + 2.0 ** -48)


def certified_overestimate(kind: str, K: int = 0, n: int = 0, path: int | None = None,
                           eps_f32: bool = True) -> float:
    # path None: the path abs_gemm_bound picks for this eps dtype
    """R of one node's bound.  kind: matmul/linear/conv2d (K = reduced length,
    path = the abs-GEMM path), softmax/layernorm/sum/mean (n = row length),
    anything else 1.0 (templates evaluated exactly as the reference does)."""
    store = 1.0 + 2.0 ** -23 if eps_f32 else 1.0  # FP32 rounded up
    if kind in ("matmul", "linear", "conv2d"):
        path = default_gemm_path(K, api=not eps_f32) if path is None else path
        if path == _lib.GEMM_FFMA_RU:  # every partial rounds up, chains of 32
            r = (1.0 + 2.0 ** -23) ** 34 * (1.0 + gemm_slack(K)) * (1.0 + 2.0 ** -48)
        elif path == _lib.GEMM_FP64:  # both FP64 sums within gamma_K of the exact one
            g = (K + 2) * 2.0 ** -53
            r = (1.0 + g) / (1.0 - g) * (1.0 + gemm_slack(K)) * (1.0 + 2.0 ** -48)
        else:
            r = _tc_overestimate(K, path == _lib.GEMM_TC_F16X3)
        return r * store
    if kind in ("softmax", "layernorm", "sum", "mean"):
        return (1.0 + sum_slack(n)) ** 2 * (1.0 + 2.0 ** -48) * store
    return 1.0


class BoundTensor:
    """Same-shape non-negative cap (bounds.py:69-93); eps is FP64, flat,
    held on the GPU or the host."""

    __slots__ = ("shape", "_eps_np", "_eps_dev")

    def __init__(self, shape, eps):
        self.shape = tuple(int(d) for d in shape)
        if isinstance(eps, torch.Tensor):
            self._eps_dev, self._eps_np = eps.reshape(-1), None
        else:
            arr = np.ascontiguousarray(np.asarray(eps, dtype=np.float64)).reshape(-1)
            if arr.size and float(arr.min()) < 0.0:
                raise ValueError("bound must be nonnegative")
            self._eps_dev, self._eps_np = None, arr

    @property
    def eps(self) -> np.ndarray:
        if self._eps_np is None:
            self._eps_np = self._eps_dev.double().cpu().numpy()
        return self._eps_np

    @property
    def array(self) -> np.ndarray:
        return self.eps.reshape(self.shape)

    def device_tensor(self) -> torch.Tensor:
        if self._eps_dev is None:
            self._eps_dev = torch.from_numpy(self._eps_np).cuda()
        return self._eps_dev.reshape(self.shape)

    @classmethod
    def from_array(cls, arr) -> "BoundTensor":
        if isinstance(arr, torch.Tensor):
            return cls(tuple(arr.shape), arr.double())
        arr = np.asarray(arr, dtype=np.float64)
        return cls(arr.shape, arr)

    @classmethod
    def zeros(cls, shape) -> "BoundTensor":
        n = int(np.prod(tuple(shape), dtype=np.int64)) if tuple(shape) else 1
        return cls(tuple(shape), np.zeros(n, dtype=np.float64))


def _eps_buffer(shape, device, f64: bool) -> torch.Tensor:
    return torch.empty(shape, dtype=torch.float64 if f64 else torch.float32, device=device)


# ---------------------------------------------------------------- kernels

F16_MIN_K = 256  # short K is epilogue bound: the TF32 split wins there (kbench)


def default_gemm_path(K: int | None = None, api: bool = False) -> int:
    """NAO_GEMM_PATH = auto (default), tc / tf32, f16, ffma or fp64.  auto:
    the streaming verifier's FP32 bounds run on tcgen05 (FP16 3-split for
    K > 256, 3xTF32 below); API calls returning the reference's FP64 bound
    (api=True: matmul_bound, op_bound, co_execute) use the FP64 path, the
    reference's own arithmetic.  All are sound."""
    env = os.environ.get("NAO_GEMM_PATH", "auto").lower()
    if env in ("ffma", "simt", "0"):
        return _lib.GEMM_FFMA_RU
    if env in ("f16", "tc16", "2"):
        return _lib.GEMM_TC_F16X3
    if env in ("tc", "tf32", "1"):
        return _lib.GEMM_TC_TF32X3
    if env in ("fp64", "3") or api:
        return _lib.GEMM_FP64
    return _lib.GEMM_TC_F16X3 if (K is not None and K > F16_MIN_K) else _lib.GEMM_TC_TF32X3


# hi/lo TF32 splits of operands that outlive a call (weights), keyed by the
# identity of the torch tensor object; dropped when that object dies.
_SPLITS: dict = {}


def tf32_split(x3: torch.Tensor, rows: int, K: int, transpose: bool, cache: bool):
    """|x| -> (hi, lo) K-major [batch, rows, Kp] TF32 parts (nao_tf32_split)."""
    key = id(x3)
    if cache:
        hit = _SPLITS.get(key)
        if hit is not None and hit[0]() is x3 and hit[1] == x3._version:
            return hit[2], hit[3]
    batch = x3.numel() // (rows * K) if rows * K else 1
    Kp = (K + 3) // 4 * 4
    hi = torch.empty((batch, rows, Kp), dtype=torch.float32, device=x3.device)
    lo = torch.empty_like(hi)
    ld = rows if transpose else K
    _lib.call("nao_tf32_split", x3.data_ptr(), hi.data_ptr(), lo.data_ptr(), batch, rows, K, ld,
              rows * K, int(transpose), _lib.stream_ptr(x3.device))
    if cache:
        _SPLITS[key] = (weakref.ref(x3, lambda _r, k=key: _SPLITS.pop(k, None)), x3._version,
                        hi, lo)
    return hi, lo


def f16_split(x3: torch.Tensor, rows: int, K: int, transpose: bool, cache: bool, owner=None):
    """|x| -> (hi, lo, row_exp): K-major [batch, rows, Kp] FP16 parts with
    |x| <= 2^e (hi + 2^-10 lo) per row (nao_f16_split).  `owner` (default x3)
    is the tensor the cache entry is keyed on (a weight whose view x3 is)."""
    owner = x3 if owner is None else owner
    key = ("f16", id(owner))
    if cache:
        hit = _SPLITS.get(key)
        if hit is not None and hit[0]() is owner and hit[1] == owner._version:
            return hit[2], hit[3], hit[4]
    batch = x3.numel() // (rows * K) if rows * K else 1
    if transpose and not cache:
        # per-call operand stored [K, rows] (e.g. V of p @ v): one transposing
        # copy, then the row kernel (the column kernel is meant for one-time
        # weight splits)
        x3 = x3.reshape(batch, K, rows).transpose(1, 2).contiguous()
        transpose = False
    Kp = (K + 7) // 8 * 8
    hi = torch.empty((batch, rows, Kp), dtype=torch.float16, device=x3.device)
    lo = torch.empty_like(hi)
    ex = torch.empty((2, batch, rows), dtype=torch.int32, device=x3.device)  # exps, tiny counts
    ld = rows if transpose else K
    _lib.call("nao_f16_split", x3.data_ptr(), hi.data_ptr(), lo.data_ptr(), ex.data_ptr(), batch,
              rows, K, ld, rows * K, int(transpose), _lib.stream_ptr(x3.device))
    if cache:
        _SPLITS[key] = (weakref.ref(owner, lambda _r, k=key: _SPLITS.pop(k, None)),
                        owner._version, hi, lo, ex)
    return hi, lo, ex


_ACT_MEMO: list = []  # [(weakref(x3), version, M, K, hi, lo, ex)]: the last activation split


def _act_split(x3: torch.Tensor, M: int, K: int):
    """f16_split of a per-call A operand, memoised for the most recent tensor:
    consecutive GEMMs reading the same activation (q/k/v, gate/up) split it once."""
    if _ACT_MEMO:
        ref, ver, m, k, hi, lo, ex = _ACT_MEMO[0]
        if ref() is x3 and ver == x3._version and (m, k) == (M, K):
            return hi, lo, ex
    hi, lo, ex = f16_split(x3, M, K, False, False)
    _ACT_MEMO[:] = [(weakref.ref(x3), x3._version, M, K, hi, lo, ex)]
    return hi, lo, ex


def release_activation_split() -> None:
    _ACT_MEMO.clear()


def abs_gemm_bound(a: torch.Tensor, b: torch.Tensor, const: float, transpose_b=False,
                   y: torch.Tensor | None = None, u: float = 0.0, eps_f64=True,
                   path: int | None = None, cache_b: bool = False,
                   a_owner: torch.Tensor | None = None) -> torch.Tensor:
    """const * (|A| @ |B|) (* (1+slack)) [+ u|y|] on the GPU (device tensors).
    a_owner: A is a (2-D view of a) static weight -- cache its split on it."""
    require_f32(a, b, y)
    a3, b3, sa, sb, nb, M, N, K, out_shape = _batch_view(a, b, transpose_b)
    path = default_gemm_path(K, api=bool(eps_f64)) if path is None else path
    eps = _eps_buffer(out_shape, a.device, eps_f64)
    yc = None
    if y is not None:
        yc = y.contiguous()
        if tuple(yc.shape) != tuple(out_shape):
            raise ValueError("linear bound: output shape mismatch")
    if path == _lib.GEMM_TC_F16X3:
        cb = cache_b and b3.data_ptr() == b.data_ptr()
        ca = a_owner is not None and a3.data_ptr() == a.data_ptr()
        if ca:
            ahi, alo, aex = f16_split(a3, M, K, False, True, a_owner)
        else:
            ahi, alo, aex = _act_split(a3, M, K)
        bhi, blo, bex = f16_split(b if cb else b3, N, K, not transpose_b, cb)
        fix = _lib.gemm_fix_workspace(a.device)
        bsrc = b if cb else b3
        _lib.call("nao_abs_gemm_tc16", ahi.data_ptr(), alo.data_ptr(), aex.data_ptr(),
                  bhi.data_ptr(), blo.data_ptr(), bex.data_ptr(), a3.data_ptr(), bsrc.data_ptr(),
                  int(transpose_b), eps.data_ptr(), int(eps_f64), nb, nb if sa else 1,
                  nb if sb else 1, M, N, K, N, M * N, float(const), _lib.ptr(yc), float(u),
                  gemm_slack(K), fix.data_ptr(), fix.numel(), _lib.stream_ptr(a.device))
        return eps
    if path == _lib.GEMM_TC_TF32X3:
        ahi, alo = tf32_split(a3, M, K, False, False)
        bhi, blo = tf32_split(b if (cache_b and b3.data_ptr() == b.data_ptr()) else b3,
                              N, K, not transpose_b, cache_b and b3.data_ptr() == b.data_ptr())
        _lib.call("nao_abs_gemm_tc", ahi.data_ptr(), alo.data_ptr(), bhi.data_ptr(),
                  blo.data_ptr(), eps.data_ptr(), int(eps_f64), nb, nb if sa else 1,
                  nb if sb else 1, M, N, K, N, M * N, float(const), _lib.ptr(yc), float(u),
                  gemm_slack(K), _lib.stream_ptr(a.device))
        return eps
    ldb = K if transpose_b else N
    _lib.call("nao_abs_gemm_bound", a3.data_ptr(), b3.data_ptr(), eps.data_ptr(), int(eps_f64), nb,
              M, N, K, K, ldb, N, sa, sb, M * N, int(transpose_b), float(const), _lib.ptr(yc),
              float(u), gemm_slack(K), int(path), _lib.stream_ptr(a.device))
    return eps


def _rows_last(x: torch.Tensor, axis: int):
    require_f32(x)
    ax = axis % x.dim()
    xm = x.movedim(ax, -1).contiguous()
    n = xm.shape[-1]
    rows = xm.numel() // n if n else 0
    return xm, ax, rows, n


def softmax_device(x: torch.Tensor, axis: int, model: FpModel, eps_f64=True, profile=None):
    xm, ax, rows, n = _rows_last(x, axis)
    if n == 0:
        raise ValueError("cannot reduce an empty axis")
    y = torch.empty_like(xm)
    eps = _eps_buffer(xm.shape, x.device, eps_f64)
    _lib.call("nao_softmax_bound", xm.data_ptr(), y.data_ptr(), eps.data_ptr(), int(eps_f64), rows,
              n, model.u, model.reduction_const(n - 1), sum_slack(n),
              profile_arg(profile, n, x.device), _lib.stream_ptr(x.device))
    return y.movedim(-1, ax), eps.movedim(-1, ax)


def layernorm_device(x: torch.Tensor, axis: int, ln_eps: float, model: FpModel, eps_f64=True,
                     profile=None):
    xm, ax, rows, n = _rows_last(x, axis)
    if n == 0:
        raise ValueError("cannot reduce an empty axis")
    y = torch.empty_like(xm)
    eps = _eps_buffer(xm.shape, x.device, eps_f64)
    _lib.call("nao_layernorm_bound", xm.data_ptr(), y.data_ptr(), eps.data_ptr(), int(eps_f64),
              rows, n, float(np.float32(ln_eps)), model.u, model.reduction_const(n - 1),
              sum_slack(n), profile_arg(profile, n, x.device), _lib.stream_ptr(x.device))
    return y.movedim(-1, ax), eps.movedim(-1, ax)


_RED = {"sum": _lib.RED_SUM, "mean": _lib.RED_MEAN, "max": _lib.RED_MAX, "min": _lib.RED_MIN}


def reduce_device(kind: str, x: torch.Tensor, axis: int, model: FpModel, eps_f64=True,
                  profile=None):
    xm, ax, rows, n = _rows_last(x, axis)
    if n == 0:
        raise ValueError("cannot reduce an empty axis")
    y = torch.empty(xm.shape[:-1], dtype=torch.float32, device=x.device)
    eps = _eps_buffer(xm.shape[:-1], x.device, eps_f64)
    _lib.call("nao_reduce_bound", xm.data_ptr(), y.data_ptr(), eps.data_ptr(), int(eps_f64), rows,
              n, _RED[kind], model.u, model.reduction_const(n - 1), sum_slack(n),
              profile_arg(profile, n, x.device), _lib.stream_ptr(x.device))
    return y, eps


def scaled_abs(y: torch.Tensor, scale: float, eps_f64=True) -> torch.Tensor:
    yc = y.contiguous()
    eps = _eps_buffer(yc.shape, y.device, eps_f64)
    _lib.call("nao_scaled_abs_bound", yc.data_ptr(), eps.data_ptr(), int(eps_f64), yc.numel(),
              float(scale), _lib.stream_ptr(y.device))
    return eps


# ------------------------------------------------------------ public API

def _to_host_pair(y, eps):
    return y.cpu().numpy(), eps.double().cpu().numpy()


def matmul_bound(a, b, model: FpModel, fma: bool = False, transpose_b: bool = False) -> BoundTensor:
    """bounds.py:100-111."""
    host = not isinstance(a, torch.Tensor)
    A, B = to_device(a), to_device(b)
    k_dim = A.shape[-1]
    kb = B.shape[-1] if transpose_b else B.shape[-2]
    if k_dim != kb:
        raise ValueError(f"matmul inner dims disagree: {tuple(A.shape)} @ {tuple(B.shape)}")
    count = k_dim if fma else 2 * k_dim - 1
    eps = abs_gemm_bound(A, B, model.reduction_const(count), transpose_b)
    return BoundTensor.from_array(eps.cpu().numpy() if host else eps)


def softmax_bound_parts(x, axis, model: FpModel, profile=None):
    """bounds.py:114-135 -> (y float32, eps float64) on the original axis layout."""
    require_supported(profile)
    host = not isinstance(x, torch.Tensor)
    y, eps = softmax_device(to_device(x), int(axis), model, profile=profile)
    return _to_host_pair(y, eps) if host else (y, eps)


def softmax_bound(x, axis, model: FpModel, profile=None) -> BoundTensor:
    _, eps = softmax_bound_parts(x, axis, model, profile)
    return BoundTensor.from_array(eps)


def layernorm_bound_parts(x, axis, eps_attr, model: FpModel, profile=None):
    """bounds.py:143-169."""
    require_supported(profile)
    host = not isinstance(x, torch.Tensor)
    y, eps = layernorm_device(to_device(x), int(axis), float(eps_attr), model, profile=profile)
    return _to_host_pair(y, eps) if host else (y, eps)


def apply_value(node, xs, profile) -> torch.Tensor:
    """FP32 value of one non-fused node on the GPU (engine.py:220-285)."""
    kind = node.kind
    if kind in ("add", "sub", "mul", "div"):
        a, b = xs
        return {"add": torch.add, "sub": torch.sub, "mul": torch.mul, "div": torch.div}[kind](a, b)
    if kind == "neg":
        return torch.neg(xs[0])
    if kind == "relu":
        return relu(xs[0])
    if kind in INTRINSIC_KINDS:
        return unary(kind, xs[0])
    if kind == "matmul":
        return matmul_value(xs[0], xs[1], profile, bool(node.attr("transpose_b", 0)))
    if kind == "linear":
        return torch.add(matmul_value(xs[0], xs[1], profile), xs[2])
    if kind == "concat":
        return torch.cat(list(xs), dim=int(node.attr("axis", 0)))
    if kind == "slice":
        x = xs[0]
        ax = int(node.attr("axis", 0)) % x.dim()
        start, stop = int(node.attr("start", 0)), int(node.attr("stop", 0))
        idx = [slice(None)] * x.dim()
        idx[ax] = slice(start, stop)
        return x[tuple(idx)].contiguous()
    if kind == "reshape":
        return xs[0].reshape(parse_shape_attr(node.attr("shape")))
    if kind == "transpose":  # extension: axis permutation
        return xs[0].permute(parse_shape_attr(node.attr("perm"))).contiguous()
    if kind == "conv2d":  # extension: value = cuDNN (native) or im2col + profile matmul
        x, w = xs
        st, pd = int(node.attr("stride", 1)), int(node.attr("pad", 0))
        if (profile is None or profile.reduction != "native"):
            col, (B, OH, OW) = im2col(x, w.shape[-1], st, pd)
            out = matmul_value(col, w.reshape(w.shape[0], -1), profile, transpose_b=True)
            return out.reshape(B, OH, OW, w.shape[0]).permute(0, 3, 1, 2).contiguous()
        return torch.nn.functional.conv2d(x, w, stride=st, padding=pd)
    if kind == "upsample2x":  # extension: nearest-neighbour, pure data movement
        return xs[0].repeat_interleave(2, dim=-2).repeat_interleave(2, dim=-1).contiguous()
    if kind == "maxpool2d":
        return torch.nn.functional.max_pool2d(xs[0], int(node.attr("k", 2)),
                                              int(node.attr("stride", 2)),
                                              int(node.attr("pad", 0)))
    if kind == "embedding":
        ids, table = xs
        idx = ids.to(torch.int64)
        # the range check reads back to the host; a CUDA-graph capture validates
        # its ids before recording (executor.GraphedRun) and skips it here
        if idx.numel() and not torch.cuda.is_current_stream_capturing() and (
                int(idx.min()) < 0 or int(idx.max()) >= table.shape[0]):
            raise ValueError("embedding index out of range")
        return table[idx]
    raise ExecutionError(f"unsupported op kind {kind!r}")


ROW_KINDS = frozenset({"softmax", "layernorm", "sum", "mean"})


def op_bound_device(node, xs, model: FpModel, profile, eps_f64=True, amb=None):
    """(y, eps) for one node on device tensors.  eps is a tensor, or a
    ("scaled", c) / ("zero",) tag when eps_f64 is None (lazy: the check
    kernel recomputes c|y| on the fly and nothing is materialised; row
    kernels then write FP64 bounds, GEMMs FP32 rounded up).  amb: the
    value-ambiguity list of an intrinsic node (csrc/unary.cuh)."""
    kind = node.kind
    lazy = eps_f64 is None
    f64 = bool(eps_f64) if not lazy else kind in ROW_KINDS
    u = model.u
    if kind == "softmax":
        require_supported(profile)
        return softmax_device(xs[0], int(node.attr("axis", -1)), model, f64, profile)
    if kind == "layernorm":
        require_supported(profile)
        return layernorm_device(xs[0], int(node.attr("axis", -1)), float(node.attr("eps", 1e-5)),
                                model, f64, profile)
    if kind in ("sum", "mean", "max", "min"):
        require_supported(profile)
        y, eps = reduce_device(kind, xs[0], int(node.attr("axis", -1)), model, f64, profile)
        if lazy and kind in ("max", "min"):
            return y, ("zero",)
        return y, eps
    if kind in INTRINSIC_KINDS:
        if lazy:
            return unary(kind, xs[0], amb=amb), ("scaled", 2.0 * u)
        return unary(kind, xs[0], amb=amb, eps_scale=2.0 * u, eps_f64=f64)
    y = apply_value(node, xs, profile)
    if kind in ZERO_BOUND_KINDS:
        return y, (("zero",) if lazy else torch.zeros(y.shape, dtype=torch.float64 if f64 else
                                                      torch.float32, device=y.device))
    if kind in SINGLE_ROUNDING_KINDS:
        return y, (("scaled", u) if lazy else scaled_abs(y, u, f64))
    if kind in GEMM_BOUND_KINDS:
        return y, gemm_bound_device(node, xs, y, model, profile, f64)
    raise ValueError(f"no bound template for kind {kind!r}")


GEMM_BOUND_KINDS = frozenset({"matmul", "linear", "conv2d"})


def gemm_bound_device(node, xs, y, model: FpModel, profile, f64: bool) -> torch.Tensor:
    """The abs-GEMM bound of a matmul / linear / conv2d node (bounds.py:100-111,
    209-217) on the current stream, given its inputs and (linear: u|y|) its
    value -- separable from the value so a caller can run it on another stream."""
    kind, u = node.kind, model.u
    if kind in ("matmul", "linear"):
        tb = bool(node.attr("transpose_b", 0)) if kind == "matmul" else False
        k_dim = xs[0].shape[-1]
        count = k_dim if fma_of(profile) else 2 * k_dim - 1
        const = model.reduction_const(count)
        static_b = xs[1].dim() == 2  # 2-D right operands are weights in every lowering
        if kind == "matmul":
            return abs_gemm_bound(xs[0], xs[1], const, tb, eps_f64=f64, cache_b=static_b)
        return abs_gemm_bound(xs[0], xs[1], const, False, y=y, u=u, eps_f64=f64,
                              cache_b=static_b)
    # conv2d: eps[b] = const |W| @ |col_b|^T: the weight is the (cached) A operand
    # and the patch rows are K-major B rows, so the GEMM writes NCHW directly
    x, w = xs
    col, (B, OH, OW) = im2col(x, w.shape[-1], int(node.attr("stride", 1)),
                              int(node.attr("pad", 0)))
    K = col.shape[-1]
    count = K if fma_of(profile) else 2 * K - 1
    eps = abs_gemm_bound(w.reshape(w.shape[0], -1), col, model.reduction_const(count), True,
                         eps_f64=f64, a_owner=w)
    return eps.reshape(B, w.shape[0], OH, OW)


def im2col(x: torch.Tensor, k: int, stride: int, pad: int):
    """[B, C, H, W] -> [B, OH*OW, C*k*k] patches (zero padding included in K,
    SURVEY.md 2.3), K ordered (c, kh, kw) as torch.nn.functional.unfold."""
    B, C, H, W = x.shape
    OH = (H + 2 * pad - k) // stride + 1
    OW = (W + 2 * pad - k) // stride + 1
    xc = x.contiguous()
    col = torch.empty((B, OH * OW, C * k * k), dtype=torch.float32, device=x.device)
    _lib.call("nao_im2col_rows", xc.data_ptr(), col.data_ptr(), B, C, H, W, k, stride, pad,
              _lib.stream_ptr(x.device))
    return col, (B, OH, OW)


def op_bound(node, arrays, model: FpModel, profile=None):
    """bounds.py:176-218: co-compute (FP32 value, FP64 bound) for one operator."""
    host = any(not isinstance(a, torch.Tensor) for a in arrays)
    xs = [to_device(a) for a in arrays]
    if node.kind == "embedding":
        xs[0] = to_device(arrays[0])
    y, eps = op_bound_device(node, xs, model, profile, eps_f64=True)
    if host:
        return _to_host_pair(y, eps)
    return y, eps


def _resolve(ref, g, inputs, values):
    cat, key = parse_ref(ref)
    if cat == "node":
        return values[key]
    if cat == "input":
        return to_device(inputs[key])
    return to_device(g.weights[key])


def _check_declared_inputs(g, inputs):
    """engine.py:312-321."""
    declared = dict(g.inputs)
    missing = set(declared) - set(inputs)
    if missing:
        raise ExecutionError(f"missing graph inputs: {sorted(missing)}")
    for name, shape in declared.items():
        if shape is not None and tuple(inputs[name].shape) != tuple(shape):
            raise ExecutionError(f"input {name!r} has shape {inputs[name].shape}, declared {shape}")


def co_execute(g, inputs, profile, model: FpModel, with_trace: bool = False):
    """bounds.py:221-262 on the GPU: returns (outputs, bounds[, trace]) with
    device-resident Tensors / BoundTensors (numpy views materialise lazily)."""
    from .commitments import tensor_digest, weight_digests
    from .engine_trace import Trace

    _check_declared_inputs(g, inputs)
    values, bounds = [], []
    for node in g.nodes:
        xs = [_resolve(r, g, inputs, values) for r in node.inputs]
        try:
            y, eps = op_bound_device(node, xs, model, profile, eps_f64=True)
        except ExecutionError:
            raise
        except NotImplementedError:
            raise
        except Exception as exc:
            raise ExecutionError(f"node {node.index} ({node.name!r}, {node.kind}): {exc}",
                                 node_index=node.index, node_name=node.name) from exc
        y = y.contiguous()
        if y.numel() and not bool(torch.isfinite(y).all()):
            raise ExecutionError(f"non-finite intermediate at node {node.index} ({node.name!r})",
                                 node_index=node.index, node_name=node.name)
        values.append(y)
        bounds.append(BoundTensor(tuple(y.shape), eps))
    release_activation_split()
    outputs = [Tensor(values[parse_ref(r)[1]].shape, values[parse_ref(r)[1]]) for r in g.outputs]
    if not with_trace:
        return outputs, bounds
    trace = Trace(tensors=[Tensor(v.shape, v) for v in values],
                  profile_id=getattr(profile, "id", "seq"),
                  input_digests={k: tensor_digest(v) for k, v in sorted(inputs.items())},
                  weight_digests=weight_digests(g.weights))
    return outputs, bounds, trace


def save_bounds(dirpath, bounds, model: FpModel, profile_id: str) -> None:
    """bounds.py:265-282: FP64 NAOT files + manifest."""
    import json
    from pathlib import Path

    from .tensor import write_tensor_file

    dirpath = Path(dirpath)
    dirpath.mkdir(parents=True, exist_ok=True)
    for i, bt in enumerate(bounds):
        write_tensor_file(dirpath / f"{i:06d}.naot", bt.array)
    manifest = {"n_nodes": len(bounds), "profile_id": profile_id,
                "fp_model": {"u": model.u, "lambda": model.lam, "mode": model.mode}}
    with open(dirpath / "manifest.json", "w") as fh:
        json.dump(manifest, fh, sort_keys=True, indent=1)
