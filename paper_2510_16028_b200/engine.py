"""FP32 operator values on the GPU, mirroring the reference executor
(/root/reference/pkg/src/fpverify/engine.py).

Profiles: the reference simulates devices by reduction order (engine.py:29-65).
This B200 build executes
  * "sequential" (with/without "+fma") bit-exactly -- the reference's default
    proposer profile (config.py:14) -- for every reduction (matmul via
    nao_matmul_profile, softmax/layernorm/sum/mean via the fused bound kernels);
  * "native": GEMMs on cuBLAS FP32 (TF32 off), the production forward whose
    values are *not* any simulated profile (the B200 is its own device).
  * "pairwise" / "blocked" / "permuted": the same
    kernels fold in that profile's order (csrc/profile_fold.cuh), bit-exact
    with the reference (tests/golden/ref_profiles.npz); the permuted order's
    Philox permutation is computed on the host exactly as engine.py:75-77.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

REDUCTIONS = ("sequential", "pairwise", "blocked", "permuted", "native")


@dataclass(frozen=True)
class DeviceProfile:
    """engine.py:29-55 (plus the B200 "native" profile)."""
    id: str
    reduction: str = "sequential"
    block_size: int = 32
    perm_seed: int = 0
    fma: bool = False

    def __post_init__(self):
        if self.reduction not in REDUCTIONS:
            raise ValueError(f"unknown reduction strategy {self.reduction!r}")

    @classmethod
    def from_spec(cls, spec: str, id: str | None = None) -> "DeviceProfile":
        fma = spec.endswith("+fma")
        if fma:
            spec = spec[: -len("+fma")]
        head, _, arg = spec.partition(":")
        kw = {}
        if head == "blocked" and arg:
            kw["block_size"] = int(arg)
        elif head == "permuted" and arg:
            kw["perm_seed"] = int(arg)
        return cls(id=id or spec + ("+fma" if fma else ""), reduction=head, fma=fma, **kw)


def default_profiles():
    """engine.py:58-65."""
    return [DeviceProfile("seq", "sequential"), DeviceProfile("pair", "pairwise"),
            DeviceProfile("blk32", "blocked", block_size=32),
            DeviceProfile("perm7+fma", "permuted", perm_seed=7, fma=True)]


NATIVE = DeviceProfile("b200", "native")


class ExecutionError(RuntimeError):
    """engine.py:68-72."""

    def __init__(self, message, node_index=None, node_name=None):
        super().__init__(message)
        self.node_index = node_index
        self.node_name = node_name


def require_supported(profile) -> str:
    red = "sequential" if profile is None else profile.reduction
    if red not in REDUCTIONS:
        raise ValueError(f"unknown reduction strategy {red!r}")
    return red


_PERMS: dict = {}


def permutation_device(seed: int, n: int, device) -> torch.Tensor:
    """engine.py:75-77: the permuted profile's order (numpy Philox, computed
    once per (seed, n) on the host -- it is data independent -- and kept on the
    device as int64)."""
    dev = torch.device(device)
    key = (int(seed), int(n), dev.index)
    t = _PERMS.get(key)
    if t is None:
        gen = np.random.Generator(np.random.Philox(key=int(seed), counter=int(n) << 128))
        t = torch.from_numpy(gen.permutation(int(n)).astype(np.int64)).to(dev)
        _PERMS[key] = t
    return t


def profile_arg(profile, n: int, device):
    """ctypes nao_profile* for a DeviceProfile reducing length n (None for
    sequential without fma and for the native profile)."""
    if profile is None or profile.reduction == "native":
        return None
    if profile.reduction == "sequential" and not profile.fma:
        return None
    p = _lib.Profile(_lib.ORDER[profile.reduction], int(profile.block_size), None, 0,
                     int(bool(profile.fma)), 0)
    if profile.reduction == "permuted":
        perm = permutation_device(profile.perm_seed, n, device)
        p.perm, p.perm_n = perm.data_ptr(), int(n)
    return ctypes.pointer(p)


def fma_of(profile) -> bool:
    return bool(profile.fma) if profile is not None else False


# ------------------------------------------------------------------ values

def to_device(a, device=None) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        t = a if a.is_cuda else a.to(device or "cuda")
        return t if t.dtype == torch.float32 else t.float()
    if hasattr(a, "device_view"):
        return a.device_view(device)
    if hasattr(a, "cuda") and hasattr(a, "shape") and not isinstance(a, np.ndarray):
        return a.cuda(device).reshape(a.shape)
    if not isinstance(a, np.ndarray) and hasattr(a, "array"):  # the reference's Tensor
        a = a.array
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    if not arr.flags.writeable:  # the reference freezes its arrays (tensor.py:36-37)
        arr = arr.copy()
    return torch.from_numpy(arr).to(device or "cuda")


def require_f32(*ts) -> None:
    """The kernels read FP32 words: any other dtype is rejected at the boundary
    (ValueError, the reference's error type for bad inputs) instead of being
    reinterpreted -- e.g. a float64 array from float32 / np.float64 promotion."""
    for t in ts:
        if isinstance(t, torch.Tensor) and t.dtype != torch.float32:
            raise ValueError(f"expected a float32 tensor, got {t.dtype}")


def unary(kind: str, x: torch.Tensor, amb: torch.Tensor | None = None, eps_scale: float = 0.0,
          eps_f64: bool | None = None):
    """engine.py:133-154 (FP64 evaluation rounded once).  amb: the node's
    value-ambiguity list (int64 [1 + cap], csrc/unary.cuh); eps_f64 not None:
    also return the intrinsic bound eps_scale*|y| at the largest candidate."""
    require_f32(x)
    x = x.contiguous()
    y = torch.empty_like(x)
    eps = None
    if eps_f64 is not None:
        eps = torch.empty(x.shape, dtype=torch.float64 if eps_f64 else torch.float32,
                          device=x.device)
    _lib.call("nao_unary_fp64", x.data_ptr(), y.data_ptr(), x.numel(), _lib.UNARY[kind],
              _lib.ptr(eps), int(bool(eps_f64)), float(eps_scale), _lib.ptr(amb),
              (amb.numel() - 1) if amb is not None else 0, _lib.stream_ptr(x.device))
    return y if eps_f64 is None else (y, eps)


def _batch_view(a: torch.Tensor, b: torch.Tensor, transpose_b: bool):
    """numpy-@ broadcasting over leading dims.  Returns contiguous operands
    A [nb,M,K], B [nb,K,N] (or [nb,N,K] with transpose_b), their batch strides
    (0 = broadcast 2-D operand), nb, M, N, K and the output shape."""
    if a.dim() < 2 or b.dim() < 2:
        raise ValueError("matmul operands must be at least 2-D")
    kb, nn = (b.shape[-1], b.shape[-2]) if transpose_b else (b.shape[-2], b.shape[-1])
    M, K = a.shape[-2], a.shape[-1]
    if K != kb:
        raise ValueError(f"matmul inner dims disagree: {tuple(a.shape)} @ {tuple(b.shape)}"
                         f"{' (transpose_b)' if transpose_b else ''}")
    batch = tuple(torch.broadcast_shapes(a.shape[:-2], b.shape[:-2]))
    nb = int(np.prod(batch, dtype=np.int64)) if batch else 1

    def prep(t, inner):
        if t.dim() == 2 or nb == 1:
            return t.contiguous(), 0
        if tuple(t.shape[:-2]) == batch:
            return t.contiguous(), inner
        return t.expand(*batch, *t.shape[-2:]).contiguous(), inner

    a3, sa = prep(a, M * K)
    b3, sb = prep(b, b.shape[-2] * b.shape[-1])
    return a3, b3, sa, sb, nb, M, nn, K, batch + (M, nn)


def matmul_value(a: torch.Tensor, b: torch.Tensor, profile, transpose_b=False) -> torch.Tensor:
    """engine.py:157-182 under the sequential profile, or cuBLAS FP32 (native)."""
    red = require_supported(profile)
    if red == "native":
        bb = b.transpose(-1, -2) if transpose_b else b
        return torch.matmul(a, bb)
    a3, b3, sa, sb, nb, M, N, K, out_shape = _batch_view(a, b, transpose_b)
    out = torch.empty(out_shape, dtype=torch.float32, device=a.device)
    ldb = K if transpose_b else N
    _lib.call("nao_matmul_profile", a3.data_ptr(), b3.data_ptr(), out.data_ptr(), nb, M, N, K, K,
              ldb, sa, sb, M * N, int(transpose_b), profile_arg(profile, K, a.device),
              _lib.stream_ptr(a.device))
    return out


def relu(x: torch.Tensor) -> torch.Tensor:
    # np.maximum(x, 0): keeps -0.0 (a >= b ? a : b)
    return torch.where(x >= 0, x, torch.zeros((), dtype=x.dtype, device=x.device))


def parse_shape_attr(spec) -> tuple:
    return tuple(int(tok) for tok in str(spec).split(",") if tok != "")


# ------------------------------------------------ FP64 oracle (theoretical path)

def _rows_fp64(kind: int, x: torch.Tensor, axis: int, ln_eps: float = 0.0) -> torch.Tensor:
    """nao_rows_fp64 over `axis` (moved last and back)."""
    require_f32(x)
    ax = axis % x.dim()
    xm = x.movedim(ax, -1).contiguous()
    n = xm.shape[-1]
    if n == 0:
        raise ValueError("cannot reduce an empty axis")
    rows = xm.numel() // n
    out_shape = xm.shape[:-1] if kind >= 2 else xm.shape
    y = torch.empty(out_shape, dtype=torch.float64, device=x.device)
    _lib.call("nao_rows_fp64", kind, xm.data_ptr(), y.data_ptr(), rows, n, float(ln_eps),
              _lib.stream_ptr(x.device))
    return y if kind >= 2 else y.movedim(-1, ax)


def matmul_fp64(a: torch.Tensor, b: torch.Tensor, transpose_b: bool = False) -> torch.Tensor:
    """matmul_op(fp64=True) (engine.py:173-177): exact FP64 products folded
    sequentially -- bit-identical to the reference."""
    require_f32(a, b)
    a3, b3, sa, sb, nb, M, N, K, out_shape = _batch_view(a, b, transpose_b)
    out = torch.empty(out_shape, dtype=torch.float64, device=a.device)
    _lib.call("nao_matmul_fp64", a3.data_ptr(), b3.data_ptr(), out.data_ptr(), nb, M, N, K, sa, sb,
              int(transpose_b), _lib.stream_ptr(a.device))
    return out


def apply_op_fp64(node, xs) -> torch.Tensor:
    """apply_op(node, args64, None, fp64=True) (engine.py:220-285) on the GPU:
    the reference's FP64 oracle of one operator (execute_fp64 :369-390; the
    leaf route's theoretical recheck, dispute.py:648-656).  xs: FP32 CUDA
    tensors (the node's arguments, promoted to FP64 as args64 is)."""
    k = node.kind
    if k in ("add", "sub", "mul", "div"):
        a, b = xs[0].double(), xs[1].double()
        return {"add": torch.add, "sub": torch.sub, "mul": torch.mul, "div": torch.div}[k](a, b)
    if k == "neg":
        return torch.neg(xs[0].double())
    if k == "relu":
        return relu(xs[0].double())
    if k in UNARY_F64:
        x = xs[0].contiguous()
        require_f32(x)
        y = torch.empty(x.shape, dtype=torch.float64, device=x.device)
        _lib.call("nao_unary_f64out", x.data_ptr(), y.data_ptr(), x.numel(), _lib.UNARY[k],
                  _lib.stream_ptr(x.device))
        return y
    if k in ("sum", "mean"):
        return _rows_fp64(2 if k == "sum" else 3, xs[0], int(node.attr("axis", -1)))
    if k in ("max", "min"):
        ax = int(node.attr("axis", -1)) % xs[0].dim()
        return (torch.amax if k == "max" else torch.amin)(xs[0].double(), dim=ax)
    if k == "matmul":
        return matmul_fp64(xs[0], xs[1], bool(node.attr("transpose_b", 0)))
    if k == "linear":
        return torch.add(matmul_fp64(xs[0], xs[1]), xs[2].double())
    if k == "softmax":
        return _rows_fp64(0, xs[0], int(node.attr("axis", -1)))
    if k == "layernorm":
        return _rows_fp64(1, xs[0], int(node.attr("axis", -1)), float(node.attr("eps", 1e-5)))
    if k == "conv2d":  # extension: the implicit-im2col GEMM in FP64
        from .bounds import im2col
        x, w = xs
        col, (B, OH, OW) = im2col(x, w.shape[-1], int(node.attr("stride", 1)),
                                  int(node.attr("pad", 0)))
        out = matmul_fp64(w.reshape(w.shape[0], -1).contiguous(), col, transpose_b=True)
        return out.reshape(B, w.shape[0], OH, OW)
    # data movement: exact in any precision
    from .bounds import apply_value
    return apply_value(node, list(xs), DeviceProfile("seq", "sequential")).double()


UNARY_F64 = frozenset({"exp", "log", "sqrt", "rsqrt", "tanh", "gelu", "silu"})
