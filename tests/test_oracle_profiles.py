"""CPU: the oracle's restatement of the reference's non-sequential device
profiles (pairwise / blocked / permuted, +fma; engine.py:75-113, :157-213)
reproduces the reference's own outputs (tests/golden/ref_profiles.npz, made by
oracle/gen_golden_profiles.py from the unmodified reference): values
bit-exact, bounds to 1e-12."""

from pathlib import Path

import numpy as np
import pytest

from oracle import bounds as OB

GOLD = Path(__file__).resolve().parent / "golden" / "ref_profiles.npz"
PROFILES = {"pair": ("pairwise", 32, 0, False), "blk32": ("blocked", 32, 0, False),
            "blk7": ("blocked", 7, 0, False), "perm7": ("permuted", 32, 7, False),
            "perm3fma": ("permuted", 32, 3, True), "pairfma": ("pairwise", 32, 0, True)}


class Prof:
    def __init__(self, red, blk, seed, fma):
        self.reduction, self.block_size, self.perm_seed, self.fma = red, blk, seed, fma


class _Node:
    def __init__(self, kind, attrs):
        self.kind, self.attrs = kind, attrs

    def attr(self, k, d=None):
        return self.attrs.get(k, d)


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def _cases(gold, tag, what):
    keys = sorted({k.rsplit("/", 1)[0] for k in gold if k.startswith(f"{tag}/{what}/")})
    return keys


@pytest.mark.parametrize("tag", sorted(PROFILES))
def test_reduce_orders_bit_exact(gold, tag):
    p = Prof(*PROFILES[tag])
    for key in _cases(gold, tag, "reduce"):
        y = OB.reduce_last_axis(gold[key + "/x"], p)
        assert np.array_equal(y.view(np.uint32), gold[key + "/y"].view(np.uint32)), key


@pytest.mark.parametrize("tag", sorted(PROFILES))
def test_profile_matmul_and_bounds(gold, tag):
    p = Prof(*PROFILES[tag])
    for key in _cases(gold, tag, "matmul"):
        tb = key.endswith("x1")
        a, b = gold[key + "/a"], gold[key + "/b"]
        y, eps = OB.op_bound(_Node("matmul", {"transpose_b": int(tb)}), [a, b], OB.FpModel(),
                             profile=p)
        assert np.array_equal(y.view(np.uint32), gold[key + "/y"].view(np.uint32)), key
        np.testing.assert_allclose(eps, gold[key + "/eps"], rtol=1e-12, err_msg=key)


@pytest.mark.parametrize("tag", sorted(PROFILES))
@pytest.mark.parametrize("kind", ["softmax", "layernorm", "sum", "mean"])
def test_profile_row_ops(gold, tag, kind):
    p = Prof(*PROFILES[tag])
    attrs = {"axis": -1}
    for key in _cases(gold, tag, kind):
        if kind == "layernorm":
            attrs["eps"] = 1e-5 if key.endswith("x96") else 1e-6
        y, eps = OB.op_bound(_Node(kind, attrs), [gold[key + "/x"]], OB.FpModel(), profile=p)
        assert np.array_equal(np.asarray(y, np.float32).view(np.uint32),
                              np.asarray(gold[key + "/y"], np.float32).view(np.uint32)), key
        np.testing.assert_allclose(eps, gold[key + "/eps"], rtol=1e-12, err_msg=key)
