"""ctypes binding of the in-tree C-ABI library libnao_b200.so (include/nao_b200.h).

There is no CPU fallback: if the library or a CUDA device is missing every
entry point raises.  Device pointers come from torch tensors; the stream is
torch's current stream on the tensors' device.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import torch

import os

# NAO_LIB_PATH: an alternative in-tree build of the same library (A/B kernel experiments)
_LIB_PATH = Path(os.environ.get("NAO_LIB_PATH") or
                 Path(__file__).resolve().parent / "libnao_b200.so")
_lib = None
_lock = threading.Lock()

c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_sz = ctypes.c_size_t
c_vp = ctypes.c_void_p

NAO_OK, NAO_EINVAL, NAO_ECUDA, NAO_ENONFINITE = 0, 1, 2, 3
HASH_SHA256, HASH_KECCAK256 = 0, 1
EPS_TENSOR_F32, EPS_TENSOR_F64, EPS_SCALED_LOCAL, EPS_ZERO = 0, 1, 2, 3
RED_SUM, RED_MEAN, RED_MAX, RED_MIN = 0, 1, 2, 3
UNARY = {"exp": 0, "log": 1, "sqrt": 2, "rsqrt": 3, "tanh": 4, "gelu": 5, "silu": 6}
GEMM_FFMA_RU, GEMM_TC_TF32X3, GEMM_TC_F16X3, GEMM_FP64 = 0, 1, 2, 3
BORDER_CAP = 1023  # borderline / ambiguity list entries per node (word 0 = count)


class CheckResult(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("n_violations", ctypes.c_uint64),
                ("n_borderline", ctypes.c_uint64), ("n_nonfinite", ctypes.c_uint64),
                ("max_ratio", ctypes.c_double), ("threshold_exceeded", ctypes.c_int32),
                ("first_exceeded", ctypes.c_int32), ("n_ambiguous", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


CHECK_RESULT_BYTES = ctypes.sizeof(CheckResult)

ORDER = {"sequential": 0, "pairwise": 1, "blocked": 2, "permuted": 3}


class Profile(ctypes.Structure):
    """nao_profile: a DeviceProfile's reduction order for the value kernels."""
    _fields_ = [("order", ctypes.c_int32), ("block_size", ctypes.c_int32),
                ("perm", ctypes.c_void_p), ("perm_n", ctypes.c_int64),
                ("fma", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class CheckDesc(ctypes.Structure):
    """nao_check_desc: the check fused into nao_commit_check_tensors."""
    _fields_ = [("local", c_vp), ("eps", c_vp), ("spec", c_vp), ("result", c_vp),
                ("eps_scale", ctypes.c_double), ("lo_factor", ctypes.c_double),
                ("eps_kind", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("border_list", c_vp), ("border_cap", ctypes.c_int64)]


class ChunkReuse(ctypes.Structure):
    """nao_chunk_reuse: a data-movement node's chunk digests copied from its source."""
    _fields_ = [("src", ctypes.c_int64), ("block_chunks", ctypes.c_uint64),
                ("repeats", ctypes.c_uint64), ("mode", ctypes.c_int32),
                ("row_chunks", ctypes.c_uint32), ("ref_payload", ctypes.c_void_p),
                ("ref_digests", ctypes.c_void_p), ("ref_bytes", ctypes.c_uint64)]


REUSE_LOCAL_COPY, REUSE_SAME_OFFSET = 0, 1


REFINE_GEMM, REFINE_CONV, REFINE_UNARY = 0, 1, 2


class RefineDesc(ctypes.Structure):
    """nao_refine_desc: one node's borderline list and what recomputes its bound."""
    _fields_ = [("kind", ctypes.c_int32), ("unary_kind", ctypes.c_int32),
                ("list", c_vp), ("cap", ctypes.c_int64), ("result", c_vp),
                ("local", c_vp), ("local64", c_vp), ("claimed", c_vp), ("a", c_vp), ("b", c_vp),
                ("batch", ctypes.c_int64), ("M", ctypes.c_int64), ("N", ctypes.c_int64),
                ("K", ctypes.c_int64), ("stride_a", ctypes.c_int64), ("stride_b", ctypes.c_int64),
                ("transpose_b", ctypes.c_int32), ("has_y", ctypes.c_int32),
                ("C", ctypes.c_int64), ("H", ctypes.c_int64), ("W", ctypes.c_int64),
                ("k", ctypes.c_int64), ("stride", ctypes.c_int64), ("pad", ctypes.c_int64),
                ("OW", ctypes.c_int64), ("gamma_const", ctypes.c_double), ("u", ctypes.c_double)]


CHECK_PARTIAL = 1  # NAO_CHECK_PARTIAL


class CheckPartial(ctypes.Structure):
    """nao_check_partial: a shard's combinable check state."""
    _fields_ = [("n", ctypes.c_uint64), ("n_violations", ctypes.c_uint64),
                ("n_borderline", ctypes.c_uint64), ("n_nonfinite", ctypes.c_uint64),
                ("max_ratio", ctypes.c_double),
                ("hist_abs", ctypes.c_uint64 * 33), ("hist_rel", ctypes.c_uint64 * 33),
                ("min_abs", ctypes.c_double * 33), ("max_abs", ctypes.c_double * 33),
                ("min_rel", ctypes.c_double * 33), ("max_rel", ctypes.c_double * 33)]


CHECK_PARTIAL_BYTES = ctypes.sizeof(CheckPartial)

# name -> (restype, argtypes)
_SIGS = {
    "nao_version": (c_int, []),
    "nao_last_error": (c_int, [ctypes.c_char_p, c_sz]),
    "nao_device_info": (c_int, [ctypes.POINTER(c_int)] * 3),
    "nao_merkle_commit_workspace": (c_sz, [c_i64, ctypes.POINTER(c_u64), c_u64]),
    "nao_merkle_commit_tensors": (c_int, [c_i64, ctypes.POINTER(c_vp), ctypes.POINTER(c_u64),
                                          ctypes.POINTER(c_vp), ctypes.POINTER(ctypes.c_uint32),
                                          c_u64, c_int, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "nao_merkle_hash_leaves": (c_int, [c_vp, c_vp, c_i64, c_int, c_vp, c_vp]),
    "nao_merkle_root_workspace": (c_sz, [c_i64]),
    "nao_merkle_root_of": (c_int, [c_vp, c_i64, c_int, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "nao_check_workspace": (c_sz, []),
    "nao_verdict_spec_bytes": (c_sz, []),
    "nao_verdict_spec_fill": (c_int, [c_vp, ctypes.POINTER(c_dbl), ctypes.POINTER(c_dbl),
                                      ctypes.POINTER(c_dbl), c_int, c_dbl]),
    "nao_commit_check_accum_bytes": (c_sz, []),
    "nao_commit_stats": (c_int, [ctypes.POINTER(c_u64), c_int]),
    "nao_commit_check_tensors": (c_int, [c_i64, ctypes.POINTER(c_vp), ctypes.POINTER(c_u64),
                                         ctypes.POINTER(c_vp), ctypes.POINTER(ctypes.c_uint32),
                                         c_u64, c_int, ctypes.POINTER(CheckDesc),
                                         ctypes.POINTER(ChunkReuse), c_vp, c_vp, c_vp, c_sz,
                                         c_vp]),
    "nao_check": (c_int, [c_vp, c_vp, c_i64, c_int, c_vp, c_dbl, c_dbl,
                          ctypes.POINTER(c_dbl), ctypes.POINTER(c_dbl), ctypes.POINTER(c_dbl),
                          c_int, c_dbl, c_vp, c_vp, c_sz, c_vp, c_i64, c_vp]),
    "nao_percentile_workspace": (c_sz, [c_i64]),
    "nao_error_profiles": (c_int, [c_vp, c_vp, c_i64, c_dbl, ctypes.POINTER(c_dbl), c_int,
                                   c_vp, c_vp, c_vp, c_sz, c_vp]),
    "nao_percentile_profile": (c_int, [c_vp, c_i64, ctypes.POINTER(c_dbl), c_int, c_vp, c_vp,
                                       c_sz, c_vp]),
    "nao_softmax_bound": (c_int, [c_vp, c_vp, c_vp, c_int, c_i64, c_i64, c_dbl, c_dbl, c_dbl,
                                  ctypes.POINTER(Profile), c_vp]),
    "nao_layernorm_bound": (c_int, [c_vp, c_vp, c_vp, c_int, c_i64, c_i64, ctypes.c_float,
                                    c_dbl, c_dbl, c_dbl, ctypes.POINTER(Profile), c_vp]),
    "nao_reduce_bound": (c_int, [c_vp, c_vp, c_vp, c_int, c_i64, c_i64, c_int, c_dbl, c_dbl,
                                 c_dbl, ctypes.POINTER(Profile), c_vp]),
    "nao_unary_fp64": (c_int, [c_vp, c_vp, c_i64, c_int, c_vp, c_int, c_dbl, c_vp, c_i64, c_vp]),
    "nao_refine_borderline": (c_int, [ctypes.POINTER(RefineDesc), c_int, c_vp]),
    "nao_matmul_fp64": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_int,
                                c_vp]),
    "nao_rows_fp64": (c_int, [c_int, c_vp, c_vp, c_i64, c_i64, c_dbl, c_vp]),
    "nao_unary_f64out": (c_int, [c_vp, c_vp, c_i64, c_int, c_vp]),
    "nao_im2col_rows": (c_int, [c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64,
                                c_vp]),
    "nao_scaled_abs_bound": (c_int, [c_vp, c_vp, c_int, c_i64, c_dbl, c_vp]),
    "nao_abs_gemm_bound": (c_int, [c_vp, c_vp, c_vp, c_int, c_i64, c_i64, c_i64, c_i64, c_i64,
                                   c_i64, c_i64, c_i64, c_i64, c_i64, c_int, c_dbl, c_vp, c_dbl,
                                   c_dbl, c_int, c_vp]),
    "nao_matmul_profile": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64,
                                   c_i64, c_i64, c_i64, c_int, ctypes.POINTER(Profile), c_vp]),
    "nao_tf32_split_cols": (c_i64, [c_i64]),
    "nao_abs_gemm_tc_kchunk": (c_int, []),
    "nao_tf32_split": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_int, c_vp]),
    "nao_abs_gemm_tc": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_i64, c_i64, c_i64, c_i64,
                                c_i64, c_i64, c_i64, c_i64, c_dbl, c_vp, c_dbl, c_dbl, c_vp]),
    "nao_f16_split_cols": (c_i64, [c_i64]),
    "nao_f16_split": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_int,
                              c_vp]),
    "nao_abs_gemm_tc16_fix_workspace": (c_sz, []),
    "nao_abs_gemm_tc16": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_vp,
                                  c_int, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64,
                                  c_dbl, c_vp, c_dbl, c_dbl, c_vp, c_sz, c_vp]),
    "nao_inject_drift": (c_int, [c_vp, c_vp, c_i64, ctypes.c_uint32, ctypes.c_uint32,
                                 ctypes.c_float, ctypes.c_uint32, c_vp]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)


class NaoError(RuntimeError):
    pass


def lib_path() -> Path:
    return _LIB_PATH


def load(require_cuda: bool = True):
    """Load the library (building it first if it is missing and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not _LIB_PATH.exists():
            from . import _build
            _build.build()
        L = ctypes.CDLL(str(_LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    if require_cuda and not torch.cuda.is_available():
        raise NaoError("paper_2510_16028_b200 needs a CUDA device (no CPU fallback)")
    return _lib


def last_error() -> str:
    L = load(require_cuda=False)
    buf = ctypes.create_string_buffer(2048)
    L.nao_last_error(buf, 2048)
    return buf.value.decode(errors="replace")


def check(rc: int, what: str = ""):
    if rc == NAO_OK:
        return
    msg = last_error()
    if rc == NAO_EINVAL:
        raise ValueError(msg or what)
    raise NaoError(f"{what}: {msg} (status {rc})")


# optional per-entry-point CUDA-event timing (bench.py roofline): name -> events/units
_timer = None


def set_timer(store, units_fn, stream):
    """Start (store=dict) or stop (None) event timing of every `call`.  On stop,
    store[name] = {"ms": [...], "units": [...]} per launch (needs a prior sync)."""
    global _timer
    if store is None and _timer is not None:
        d = _timer[0]
        for name, ent in d.items():
            ent["ms"] = [a.elapsed_time(b) for a, b in ent.pop("ev")]
        _timer = None
        return
    _timer = (store, units_fn, stream) if store is not None else None


def call(name: str, *args):
    fn = getattr(load(), name)
    if _timer is None:
        check(fn(*args), name)
        return
    store, units_fn, _ = _timer
    stream = torch.cuda.current_stream()  # the stream this entry point launches on
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    rc = fn(*args)
    e1.record(stream)
    check(rc, name)
    ent = store.setdefault(name, {"ev": [], "units": []})
    ent["ev"].append((e0, e1))
    ent["units"].append(units_fn(name, args) if units_fn else 0.0)


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def dbl_array(values):
    vals = [float(v) for v in values]
    return (c_dbl * len(vals))(*vals)


# ------------------------------------------------------------------ workspace
_ws: dict = {}


_ws_captured: list = []  # scratch buffers baked into captured CUDA graphs


def workspace(nbytes: int, device) -> torch.Tensor:
    """Per (device, stream) growable scratch buffer.  A buffer outgrown while
    a CUDA graph is being captured stays alive: the graph's earlier kernels
    keep its address (replaying them after it was freed faults)."""
    dev = torch.device(device)
    key = (dev.index, torch.cuda.current_stream(dev).cuda_stream)
    buf = _ws.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 1 << 20), dtype=torch.uint8, device=dev)
        _ws[key] = buf
    if torch.cuda.is_current_stream_capturing() and not any(b is buf for b in _ws_captured):
        # every buffer a graph records stays alive, also one handed out before
        # the capture and outgrown by a later eager call
        _ws_captured.append(buf)
    return buf


def commit_check_accumulator(device) -> torch.Tensor:
    """Zero-initialised accumulator of nao_commit_check_tensors per (device, stream)."""
    dev = torch.device(device)
    key = ("commit_check", dev.index, torch.cuda.current_stream(dev).cuda_stream)
    buf = _ws.get(key)
    if buf is None:
        buf = torch.zeros(int(load().nao_commit_check_accum_bytes()), dtype=torch.uint8,
                          device=dev)
        _ws[key] = buf
    return buf


def verdict_spec(grid, tau_abs, tau_rel, epsilon) -> bytes:
    """Host bytes of one nao_verdict_spec (upload them to the device)."""
    L = load(require_cuda=False)
    buf = ctypes.create_string_buffer(int(L.nao_verdict_spec_bytes()))
    check(L.nao_verdict_spec_fill(buf, dbl_array(grid), dbl_array(tau_abs), dbl_array(tau_rel),
                                  len(grid), float(epsilon)), "nao_verdict_spec_fill")
    return buf.raw


def gemm_fix_workspace(device) -> torch.Tensor:
    """Zeroed fix-up list of nao_abs_gemm_tc16 per (device, stream)."""
    dev = torch.device(device)
    key = ("tc16fix", dev.index, torch.cuda.current_stream(dev).cuda_stream)
    buf = _ws.get(key)
    if buf is None:
        buf = torch.zeros(int(load().nao_abs_gemm_tc16_fix_workspace()), dtype=torch.uint8,
                          device=dev)
        _ws[key] = buf
    return buf


def check_accumulator(device) -> torch.Tensor:
    """Dedicated zero-initialised nao_check accumulator per (device, stream);
    every nao_check call leaves it zeroed (include/nao_b200.h)."""
    dev = torch.device(device)
    key = ("check", dev.index, torch.cuda.current_stream(dev).cuda_stream)
    buf = _ws.get(key)
    if buf is None:
        buf = torch.zeros(int(load().nao_check_workspace()), dtype=torch.uint8, device=dev)
        _ws[key] = buf
    return buf
