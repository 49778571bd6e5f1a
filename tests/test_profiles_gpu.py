"""GPU parity for the reference's non-sequential device profiles (SURVEY.md
8(f) row 3): pairwise / blocked / permuted reduction orders, with and without
fma, through the drop-in API (op_bound / matmul value kernels / softmax /
layernorm / sum / mean) against the UNMODIFIED reference's outputs
(tests/golden/ref_profiles.npz, oracle/gen_golden_profiles.py): values
bit-exact, bounds within [ref, ref (1 + 1e-5)].  Larger shapes compare with
the oracle restatement (pinned to those goldens by test_oracle_profiles.py)."""

from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import bounds as OB

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden" / "ref_profiles.npz"
PROFILES = {"pair": ("pairwise", 32, 0, False), "blk32": ("blocked", 32, 0, False),
            "blk7": ("blocked", 7, 0, False), "perm7": ("permuted", 32, 7, False),
            "perm3fma": ("permuted", 32, 3, True), "pairfma": ("pairwise", 32, 0, True)}
RTOL = 1e-5


class _Node:
    def __init__(self, kind, attrs):
        self.kind, self.attrs, self.index, self.name, self.inputs = kind, attrs, 0, "op", ()

    def attr(self, k, d=None):
        return self.attrs.get(k, d)


def _prof(tag):
    from paper_2510_16028_b200.engine import DeviceProfile
    red, blk, seed, fma = PROFILES[tag]
    return DeviceProfile(tag, red, block_size=blk, perm_seed=seed, fma=fma)


def _bits_equal(a, b):
    return np.array_equal(np.asarray(a, np.float32).view(np.uint32),
                          np.asarray(b, np.float32).view(np.uint32))


def _assert_bound(got, ref, what):
    got = np.asarray(got, np.float64).reshape(-1)
    ref = np.asarray(ref, np.float64).reshape(-1)
    assert np.all(got >= ref), what
    assert np.all(got <= ref * (1 + RTOL)), (what, float(np.max(got / ref - 1)))


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def _keys(gold, tag, what):
    return sorted({k.rsplit("/", 1)[0] for k in gold if k.startswith(f"{tag}/{what}/")})


@pytest.mark.parametrize("tag", sorted(PROFILES))
def test_profile_reductions_match_reference(gold, tag):
    """sum over the trailing axis (reduce_last_axis) for n = 1 .. 1000."""
    from paper_2510_16028_b200.bounds import FpModel, op_bound
    for key in _keys(gold, tag, "reduce"):
        x = gold[key + "/x"]
        y, eps = op_bound(_Node("sum", {"axis": -1}), [x], FpModel(), _prof(tag))
        assert _bits_equal(y, gold[key + "/y"]), key


@pytest.mark.parametrize("tag", sorted(PROFILES))
def test_profile_matmul_matches_reference(gold, tag):
    from paper_2510_16028_b200.bounds import FpModel, op_bound
    for key in _keys(gold, tag, "matmul"):
        tb = key.endswith("x1")
        y, eps = op_bound(_Node("matmul", {"transpose_b": int(tb)}),
                          [gold[key + "/a"], gold[key + "/b"]], FpModel(), _prof(tag))
        assert _bits_equal(y, gold[key + "/y"]), key
        _assert_bound(eps, gold[key + "/eps"], key)


@pytest.mark.parametrize("tag", sorted(PROFILES))
@pytest.mark.parametrize("kind", ["softmax", "layernorm", "sum", "mean"])
def test_profile_row_ops_match_reference(gold, tag, kind):
    from paper_2510_16028_b200.bounds import FpModel, op_bound
    attrs = {"axis": -1}
    for key in _keys(gold, tag, kind):
        if kind == "layernorm":
            attrs["eps"] = 1e-5 if key.endswith("x96") else 1e-6
        y, eps = op_bound(_Node(kind, attrs), [gold[key + "/x"]], FpModel(), _prof(tag))
        assert _bits_equal(y, gold[key + "/y"]), key
        _assert_bound(eps, gold[key + "/eps"], key)


@pytest.mark.parametrize("tag", ["pair", "blk7", "perm7"])
def test_profile_larger_shapes_vs_oracle(tag):
    """Many rows (several CTAs, R rows per CTA), ragged n, batched matmul."""
    from paper_2510_16028_b200.bounds import FpModel, op_bound
    rng = np.random.default_rng(len(tag))
    p = _prof(tag)
    x = (rng.standard_normal((700, 513)) * 2).astype(np.float32)
    for kind, attrs in (("softmax", {"axis": -1}), ("layernorm", {"axis": -1, "eps": 1e-5}),
                        ("mean", {"axis": -1})):
        y, eps = op_bound(_Node(kind, attrs), [x], FpModel(), p)
        y_ref, e_ref = OB.op_bound(_Node(kind, attrs), [x], OB.FpModel(), profile=p)
        assert _bits_equal(y, y_ref), kind
        _assert_bound(eps, e_ref, kind)
    a = rng.standard_normal((3, 40, 77)).astype(np.float32)
    b = rng.standard_normal((3, 77, 21)).astype(np.float32)
    y, eps = op_bound(_Node("matmul", {}), [a, b], FpModel(), p)
    y_ref, e_ref = OB.op_bound(_Node("matmul", {}), [a, b], OB.FpModel(), profile=p)
    assert _bits_equal(y, y_ref)
    _assert_bound(eps, e_ref, "matmul")


def test_profile_default_fleet_co_execute(ref_mlp):
    """The reference's default fleet (engine.py:58-65) co-executes the MLP
    graph on the GPU with values bit-exact against the oracle under every
    profile (the committee's cross-profile traces)."""
    from paper_2510_16028_b200 import bounds as B
    from paper_2510_16028_b200.engine import default_profiles
    from paper_2510_16028_b200.lowerings import build_mlp
    from paper_2510_16028_b200.tensor import Rng
    c = ref_mlp["config"]
    spec = build_mlp(c["seed"], c["batch"], c["in_dim"], c["hidden"], c["n_classes"])
    x = spec.make_inputs(Rng(*c["input_rng"]))
    for prof in default_profiles():
        outs, bnds, trace = B.co_execute(spec.graph, x, prof, B.FpModel(), with_trace=True)
        vals = [np.asarray(x["x"].array, np.float32)]
        ref_vals = []
        cur = {}
        for node in spec.graph.nodes:
            args = []
            for ref in node.inputs:
                cat, _, key = ref.partition(":")
                args.append(cur[int(key)] if cat == "node" else
                            (np.asarray(x[key].array, np.float32) if cat == "input"
                             else np.asarray(spec.graph.weights[key].array, np.float32)))
            y, _ = OB.op_bound(node, args, OB.FpModel(), profile=prof)
            cur[node.index] = np.asarray(y, np.float32)
            ref_vals.append(cur[node.index])
        for t, rv in zip(trace.tensors, ref_vals):
            assert _bits_equal(t.array, rv), prof.id
