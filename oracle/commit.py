"""ORACLE -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference
commitment primitives (/root/reference/pkg/src/fpverify/commitments.py) with
a hash parameter, plus the chunked per-tensor tree and the trace tree that
the B200 path commits (north_star (4)).

Tensor commitment format (shared with the product):
    leaves(t)      = [canon_header(t)] + [payload[i*C:(i+1)*C] for i in ...]
    tensor_root(t) = MerkleTree([leaf_digest(x) for x in leaves(t)]).root
    trace_root     = MerkleTree([leaf_digest(r) for r in tensor_roots]).root
In SHA-256 mode tensor_root(t) == reference build_tree(leaves(t)).root
(commitments.py:141-142) bit for bit.
"""

from __future__ import annotations

import ctypes
import hashlib
import struct

import numpy as np

from ._clib import lib

SHA256 = 0
KECCAK256 = 1
_ALG_NAMES = {"sha256": SHA256, "keccak256": KECCAK256}

LEAF_TAG = b"\x00"  # commitments.py:27
NODE_TAG = b"\x01"  # commitments.py:28


def alg_id(alg) -> int:
    if isinstance(alg, str):
        return _ALG_NAMES[alg]
    return int(alg)


def _ptr(b) -> ctypes.c_void_p:
    return ctypes.cast(ctypes.c_char_p(b), ctypes.c_void_p)


def hash_bytes(data: bytes, alg=SHA256) -> bytes:
    """H(data).  SHA-256 goes through hashlib exactly like commitments.py:31-32;
    Keccak-256 through the C restatement (oracle/hashes.c)."""
    a = alg_id(alg)
    if a == SHA256:
        return hashlib.sha256(data).digest()
    out = ctypes.create_string_buffer(32)
    lib().oracle_hash(a, None, 0, _ptr(data), len(data), out)
    return out.raw


def sha3_256_via_keccak_sponge(data: bytes) -> bytes:
    """Same sponge with FIPS-202 pad byte 0x06 -- must equal hashlib.sha3_256
    (the free cross-check of the Keccak restatement)."""
    out = ctypes.create_string_buffer(32)
    lib().oracle_hash(2, None, 0, _ptr(data), len(data), out)
    return out.raw


def leaf_digest(data: bytes, alg=SHA256) -> bytes:
    """H(0x00 || x)  (commitments.py:137-138)."""
    return hash_bytes(LEAF_TAG + data, alg)


def node_digest(left: bytes, right: bytes, alg=SHA256) -> bytes:
    """H(0x01 || L || R)  (commitments.py:125)."""
    return hash_bytes(NODE_TAG + left + right, alg)


class MerkleTree:
    """Level list with odd-node self-pairing (commitments.py:112-134)."""

    def __init__(self, leaf_digests, alg=SHA256):
        if len(leaf_digests) == 0:
            raise ValueError("merkle tree requires at least one leaf")
        self.alg = alg_id(alg)
        self.levels = [list(leaf_digests)]
        while len(self.levels[-1]) > 1:
            prev = self.levels[-1]
            nxt = []
            for i in range(0, len(prev), 2):
                left = prev[i]
                right = prev[i + 1] if i + 1 < len(prev) else prev[i]
                nxt.append(node_digest(left, right, self.alg))
            self.levels.append(nxt)

    @property
    def root(self) -> bytes:
        return self.levels[-1][0]

    @property
    def n_leaves(self) -> int:
        return len(self.levels[0])


def build_tree(leaves, alg=SHA256) -> MerkleTree:
    """commitments.py:141-142."""
    return MerkleTree([leaf_digest(x, alg) for x in leaves], alg)


def fast_root_of_digests(digests: np.ndarray, alg=SHA256, n_threads: int = 1) -> bytes:
    """Root over an (n, 32) uint8 array of leaf digests via the C level loop
    (same construction as MerkleTree, used for big trees)."""
    d = np.ascontiguousarray(digests, dtype=np.uint8).reshape(-1, 32)
    if d.shape[0] == 0:
        raise ValueError("merkle tree requires at least one leaf")
    a = alg_id(alg)
    while d.shape[0] > 1:
        out = np.empty(((d.shape[0] + 1) // 2, 32), dtype=np.uint8)
        lib().oracle_tree_level(a, d.ctypes.data, d.shape[0], out.ctypes.data, n_threads)
        d = out
    return bytes(d[0])


# --------------------------------------------------------------- canon bytes


def canon_header(shape, dtype=np.float32) -> bytes:
    """u8 dtype code || u32 rank || rank x u64 dims || rank x u64 contiguous
    element strides  (commitments.py:39-61)."""
    dt = np.dtype(dtype)
    if dt == np.float32:
        code = 0
    elif dt == np.float64:
        code = 1
    else:
        raise ValueError(f"unsupported dtype {dt}")
    shape = tuple(int(d) for d in shape)
    strides = []
    acc = 1
    for d in reversed(shape):
        strides.append(acc)
        acc *= d
    strides.reverse()
    head = struct.pack("<BI", code, len(shape))
    dims = b"".join(struct.pack("<Q", d) for d in shape)
    strd = b"".join(struct.pack("<Q", s) for s in strides)
    return head + dims + strd


def canon_tensor(arr) -> bytes:
    arr = np.asarray(arr)
    if arr.dtype not in (np.float32, np.float64):
        raise ValueError(f"unsupported dtype {arr.dtype}")
    dt = np.dtype("<f4") if arr.dtype == np.float32 else np.dtype("<f8")
    return canon_header(arr.shape, arr.dtype) + np.ascontiguousarray(arr, dtype=dt).tobytes()


def tensor_leaves(arr, chunk_bytes: int) -> list[bytes]:
    arr = np.asarray(arr)
    payload = np.ascontiguousarray(arr).tobytes()
    leaves = [canon_header(arr.shape, arr.dtype)]
    leaves += [payload[i:i + chunk_bytes] for i in range(0, len(payload), chunk_bytes)]
    return leaves


def tensor_leaf_digests(arr, chunk_bytes: int, alg=SHA256, n_threads: int = 1) -> np.ndarray:
    """(1 + ceil(nbytes/C), 32) leaf digests: header leaf then payload chunks."""
    arr = np.asarray(arr)
    shape = arr.shape  # np.ascontiguousarray would turn a 0-d array into shape (1,)
    arr = np.ascontiguousarray(arr)
    a = alg_id(alg)
    nbytes = arr.nbytes
    n_chunks = (nbytes + chunk_bytes - 1) // chunk_bytes
    out = np.empty((1 + n_chunks, 32), dtype=np.uint8)
    out[0] = np.frombuffer(leaf_digest(canon_header(shape, arr.dtype), a), dtype=np.uint8)
    if n_chunks:
        lib().oracle_chunk_leaves(a, arr.ctypes.data, nbytes, chunk_bytes,
                                  out[1:].ctypes.data, n_threads)
    return out


def tensor_root(arr, chunk_bytes: int = 4096, alg=SHA256, n_threads: int = 1) -> bytes:
    return fast_root_of_digests(tensor_leaf_digests(arr, chunk_bytes, alg, n_threads), alg,
                                n_threads)


def trace_root(tensor_roots, alg=SHA256) -> bytes:
    """Root over per-node tensor roots in canonical node order."""
    return build_tree(list(tensor_roots), alg).root
