"""GPU parity: Merkle commitment kernels vs the oracle / reference goldens.
Bit-exact roots and leaf digests (north_star: "Merkle roots and leaf hashes
must be bit-exact given the same committed tensor bytes")."""

import hashlib

import numpy as np
import pytest
import torch

from oracle import commit as OM

pytestmark = pytest.mark.gpu

ALGS = ["sha256", "keccak256"]


@pytest.fixture(scope="module")
def C():
    from paper_2510_16028_b200 import commitments
    return commitments


@pytest.mark.parametrize("alg", ALGS)
def test_leaf_digests_generic_lengths(C, alg):
    leaves = [bytes((i * 31 + j) % 256 for j in range(n))
              for i, n in enumerate([0, 1, 3, 4, 54, 55, 56, 63, 64, 65, 119, 134, 135, 136, 137,
                                     200, 271, 272, 1000, 4096, 4097])]
    got = C.hash_leaves(leaves, alg).cpu().numpy()
    for row, leaf in zip(got, leaves):
        assert bytes(row) == OM.leaf_digest(leaf, alg)


def test_reference_golden_vectors(C, ref_vectors):
    leaves = [f"leaf{i}".encode() for i in range(5)]
    tree = C.build_tree(leaves)
    assert tree.root.hex() == ref_vectors["tree_root_5"]
    assert C.prove(tree, 2).to_wire().hex() == ref_vectors["proof_wire_5_2"]
    for n, root in ref_vectors["tree_roots"].items():
        n = int(n)
        lv = [bytes([i % 256]) * (i % 7 + 1) for i in range(n)]
        assert C.build_tree(lv).root.hex() == root
    canon = C.canon_tensor(np.array([[1.0, -2.0], [0.5, 4.0]], dtype=np.float32))
    assert hashlib.sha256(canon).hexdigest() == ref_vectors["canon_2x2"]


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("n", [1, 2, 3, 5, 511, 512, 513, 1023, 1024, 1025, 262145])
def test_tree_levels_and_root(C, alg, n):
    rng = np.random.default_rng(n)
    digs = rng.integers(0, 256, size=(n, 32), dtype=np.uint8)
    d = torch.from_numpy(digs).cuda()
    root = bytes(C.root_of_digests(d, alg).cpu().numpy())
    assert root == OM.fast_root_of_digests(digs, alg)
    if n <= 1025:
        tree = C.MerkleTree(d, alg)
        ref = OM.MerkleTree([bytes(r) for r in digs], alg)
        assert tree.levels == ref.levels


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("chunk", [64, 256, 4096, 16384])
def test_tensor_roots_batched(C, alg, chunk):
    g = torch.Generator(device="cuda").manual_seed(chunk)
    shapes = [(1,), (3,), (16,), (17,), (2, 33), (64, 256), (1000, 37), (4096 * 3 + 4,),
              (8, 16, 17), ()]
    ts = [torch.randn(s, generator=g, device="cuda") for s in shapes]
    roots = C.commit_tensors(ts, chunk, alg).cpu().numpy()
    for t, r in zip(ts, roots):
        assert bytes(r) == OM.tensor_root(t.cpu().numpy(), chunk, alg), (t.shape, chunk, alg)


def test_empty_tensor_and_errors(C):
    e = torch.empty((0, 5), device="cuda")
    r = C.commit_tensors([e], 4096).cpu().numpy()[0]
    assert bytes(r) == OM.tensor_root(np.empty((0, 5), np.float32), 4096)
    with pytest.raises(ValueError):
        C.build_tree([])
    with pytest.raises(ValueError):
        C.commit_tensors([torch.ones(4, device="cuda")], 100)  # not a multiple of 64


def test_sha256_tensor_root_matches_reference_build_tree(C, ref_mlp):
    """Roots of the reference MLP trace values (regenerated bit-exactly by the oracle)."""
    from oracle import bounds as OB
    from paper_2510_16028_b200.lowerings import build_mlp
    from paper_2510_16028_b200.tensor import Rng
    c = ref_mlp["config"]
    spec = build_mlp(c["seed"], c["batch"], c["in_dim"], c["hidden"], c["n_classes"])
    x = spec.make_inputs(Rng(*c["input_rng"]))
    vals, _ = OB.co_execute(spec.graph, {"x": x["x"].array}, OB.FpModel())
    ts = [torch.from_numpy(v).cuda() for v in vals]
    for chunk in (256, 4096):
        roots = C.commit_tensors(ts, chunk).cpu().numpy()
        for r, ent in zip(roots, ref_mlp["runs"]["seq/prob"]):
            assert bytes(r).hex() == ent[f"root_sha256_c{chunk}"]
    roots = C.commit_tensors(ts, 4096)
    assert C.trace_root(roots).hex() == ref_mlp["trace_root_sha256_c4096"]


@pytest.mark.parametrize("alg", ALGS)
def test_large_tensor_root(C, alg):
    t = torch.randn(2048 * 4096 + 12, device="cuda")
    r = bytes(C.commit_tensors([t], 4096, alg).cpu().numpy()[0])
    assert r == OM.tensor_root(t.cpu().numpy(), 4096, alg, n_threads=8)


def test_proofs_roundtrip(C):
    for n in (1, 2, 3, 5, 8, 13):
        leaves = [f"L{i}".encode() for i in range(n)]
        tree = C.build_tree(leaves)
        for i in range(n):
            assert C.verify(tree.root, leaves[i], C.prove(tree, i))
        if n > 1:
            assert not C.verify(tree.root, b"tampered", C.prove(tree, 0))
