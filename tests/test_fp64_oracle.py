"""The FP64 oracle path (apply_op(fp64=True), engine.py:220-285; the leaf
route's theoretical recheck, dispute.py:648-656) against golden vectors of
the unmodified reference (oracle/gen_golden_fp64.py -> tests/golden/ref_fp64.npz):
the oracle restatement on the CPU, engine.apply_op_fp64 on the GPU.  Matmul /
linear / sum / mean / layernorm are bit-exact (exact products, sequential
FP64 folds); softmax and the intrinsics differ only in the libm's last FP64
ulps (numpy's SIMD exp / tanh vs CUDA's)."""

import ast

import numpy as np
import pytest

from _helpers import GOLDEN

EXACT = {"matmul", "linear", "sum", "mean", "layernorm"}


class _Node:
    def __init__(self, kind, attrs):
        self.kind, self.attrs = kind, attrs

    def attr(self, k, d=None):
        return self.attrs.get(k, d)


def _cases():
    z = np.load(GOLDEN / "ref_fp64.npz")
    tags = sorted({k.split("/")[0] for k in z.files})
    out = []
    for t in tags:
        ins, i = [], 0
        while f"{t}/in{i}" in z.files:
            ins.append(z[f"{t}/in{i}"])
            i += 1
        out.append((t, str(z[f"{t}/kind"]), ast.literal_eval(str(z[f"{t}/attrs"])), ins,
                    z[f"{t}/y"]))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c[0])
def test_oracle_fp64_matches_reference(case):
    from oracle import bounds as OB
    tag, kind, attrs, ins, y = case
    if kind not in EXACT | {"softmax"}:
        pytest.skip("intrinsics: the oracle restates only the reduction kinds")
    got = OB.apply_op_fp64(_Node(kind, attrs), ins)
    assert np.array_equal(got, y), tag


@pytest.mark.gpu
@pytest.mark.parametrize("case", _cases(), ids=lambda c: c[0])
def test_gpu_fp64_matches_reference(case):
    import torch
    from paper_2510_16028_b200.engine import apply_op_fp64
    tag, kind, attrs, ins, y = case
    got = apply_op_fp64(_Node(kind, attrs), [torch.from_numpy(a).cuda() for a in ins])
    got = got.cpu().numpy()
    assert got.shape == y.shape and got.dtype == np.float64
    if kind in EXACT:
        assert np.array_equal(got, y), tag
    elif kind == "gelu":  # 0.5 x (1 + tanh(.)) cancels for x << 0: |x| times tanh's ulps
        x = ins[0].astype(np.float64)
        assert np.all(np.abs(got - y) <= 8 * np.spacing(np.abs(y)) + np.abs(x) * 2.0 ** -49), tag
    else:
        np.testing.assert_allclose(got, y, rtol=8 * 2.0 ** -52, atol=0, err_msg=tag)
