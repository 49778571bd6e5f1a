"""ORACLE -- TEST INFRASTRUCTURE ONLY.  Builds/loads oracle/hashes.c (plain C,
gcc) into oracle/_build/liboracle.so and exposes it through ctypes."""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "hashes.c"
_OUT = _HERE / "_build" / "liboracle.so"
_lib = None


def build(force: bool = False) -> Path:
    if _OUT.exists() and not force and _OUT.stat().st_mtime >= _SRC.stat().st_mtime:
        return _OUT
    _OUT.parent.mkdir(parents=True, exist_ok=True)
    tmp = _OUT.with_suffix(f".{os.getpid()}.tmp")
    subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC",
                           str(_SRC), "-o", str(tmp)])
    os.replace(tmp, _OUT)
    return _OUT


def lib():
    global _lib
    if _lib is None:
        path = build()
        L = ctypes.CDLL(str(path))
        u8p = ctypes.c_void_p
        L.oracle_hash.argtypes = [ctypes.c_int, u8p, ctypes.c_size_t, u8p, ctypes.c_size_t, u8p]
        L.oracle_hash.restype = None
        L.oracle_chunk_leaves.argtypes = [ctypes.c_int, u8p, ctypes.c_uint64, ctypes.c_uint64,
                                          u8p, ctypes.c_int]
        L.oracle_chunk_leaves.restype = None
        L.oracle_tree_level.argtypes = [ctypes.c_int, u8p, ctypes.c_int64, u8p, ctypes.c_int]
        L.oracle_tree_level.restype = None
        _lib = L
    return _lib
