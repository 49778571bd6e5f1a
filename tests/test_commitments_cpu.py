"""CPU: dispute-time commitments -- interface hashes,
c0 commitments, weight / graph trees' leaf encoding -- against the reference's
golden vectors and hashlib compositions (commitments.py:68-78, :172-247)."""

import hashlib

import numpy as np
import pytest

from paper_2510_16028_b200 import commitments as C
from paper_2510_16028_b200.graph import input_ref, make_node, weight_ref
from paper_2510_16028_b200.tensor import tensor_new


def test_signature_golden(ref_vectors):
    n = make_node("mm", "matmul", [input_ref("x"), weight_ref("w")], {"transpose_b": 1})
    assert hashlib.sha256(C.op_signature(n)).hexdigest() == ref_vectors["signature_matmul"]


def test_interface_hash_composition():
    assert C.interface_hash([]) == hashlib.sha256(b"").digest()
    ts = [tensor_new([2], [1, 2]), tensor_new([3], [1, 2, 3]), tensor_new([1], [5])]
    inner = b"".join(hashlib.sha256(C.canon_tensor(t)).digest() for t in ts)
    assert C.interface_hash(ts) == hashlib.sha256(inner).digest()
    assert C.interface_hash(ts[::-1]) != C.interface_hash(ts)


def test_commitment_round_trip_and_tamper():
    meta = {"device": "b200", "kernel": "v1", "dtype": "fp32", "window": 10}
    x, y = [tensor_new([2], [1, 2])], [tensor_new([2], [3, 4])]
    roots = (C.sha256(b"w"), C.sha256(b"g"), C.sha256(b"e"))
    c = C.make_commitment(*roots, x, y, meta)
    assert C.verify_commitment(c, x, y)
    assert not C.verify_commitment(c, x, [tensor_new([2], [3, 5])])
    with pytest.raises(ValueError):
        C.make_commitment(*roots, x, y, {"bad": [1, 2]})
