"""GPU parity: per-operator values and bounds vs the reference goldens
(tests/golden/ref_ops.npz, ref_mlp_784_256_10_b64.json; made by
oracle/gen_golden.py from the unmodified reference).

Tolerance (north_star): bounds within rtol 1e-5 of the reference and never
below it:  eps_ref <= eps_gpu <= eps_ref * (1 + 1e-5).  Values under the
sequential profile: bit-exact."""

import hashlib

import numpy as np
import pytest
import torch

from _helpers import OP_SPECS, op_cases
from oracle import bounds as OB
from oracle import commit as OM

pytestmark = pytest.mark.gpu
RTOL = 1e-5
INTRINSIC_TRANSCENDENTAL = {"exp", "log", "tanh", "gelu", "silu"}


def _sub32(e_ref):
    """Slack of an FP32 bound rounded up from the FP64 one: two FP32 spacings,
    only where e_ref is below FP32's normal range (elsewhere rounding up costs
    at most 2^-23 relative, inside rtol)."""
    return np.where(e_ref < np.finfo(np.float32).tiny, 2 * np.spacing(e_ref.astype(np.float32)),
                    0.0)


def assert_bound(eps_gpu, eps_ref, what=""):
    eps_gpu = np.asarray(eps_gpu, dtype=np.float64).reshape(-1)
    eps_ref = np.asarray(eps_ref, dtype=np.float64).reshape(-1)
    assert eps_gpu.shape == eps_ref.shape, what
    below = eps_gpu < eps_ref
    assert not below.any(), (what, int(below.sum()), float((eps_ref - eps_gpu)[below].max()))
    over = eps_gpu > eps_ref * (1.0 + RTOL)
    assert not over.any(), (what, int(over.sum()),
                            float(np.max(eps_gpu[over] / eps_ref[over] - 1.0)))


class _Node:
    def __init__(self, kind, attrs):
        self.kind, self.attrs, self.index, self.name, self.inputs = kind, attrs, 0, "op", ()

    def attr(self, k, d=None):
        return self.attrs.get(k, d)


@pytest.fixture(scope="module")
def B():
    from paper_2510_16028_b200 import bounds
    return bounds


@pytest.mark.parametrize("tag", sorted(OP_SPECS))
def test_op_bound_matches_reference(B, ref_ops, tag):
    from paper_2510_16028_b200.engine import DeviceProfile
    ins, y_ref, eps_ref = op_cases(ref_ops)[tag]
    kind, attrs, mode, fma = OP_SPECS[tag]
    model = B.FpModel(mode="deterministic" if mode == "det" else "probabilistic")
    prof = DeviceProfile("seqf" if fma else "seq", "sequential", fma=fma)
    y, eps = B.op_bound(_Node(kind, attrs), ins, model, prof)
    assert y.dtype == np.float32 and eps.dtype == np.float64
    assert y.shape == y_ref.shape and eps.shape == eps_ref.shape
    yu, ru = y.view(np.int32).astype(np.int64), y_ref.astype(np.float32).view(np.int32)
    same = yu == ru
    if kind in INTRINSIC_TRANSCENDENTAL:
        # numpy's FP64 libm is not correctly rounded: the GPU value equals the
        # reference's on every element except the flagged value-ambiguous ones
        # (csrc/unary.cuh), and the bound (taken at the largest candidate) is
        # never below the reference's anywhere
        import torch
        from paper_2510_16028_b200 import _lib
        from paper_2510_16028_b200.engine import unary
        amb = torch.zeros(1 + _lib.BORDER_CAP, dtype=torch.int64, device="cuda")
        unary(kind, torch.from_numpy(np.ascontiguousarray(ins[0])).cuda(), amb=amb)
        a = amb.cpu().numpy()
        flagged = np.zeros(y.size, bool)
        flagged[a[1:1 + min(int(a[0]), _lib.BORDER_CAP)]] = True
        assert np.all(flagged[~same.reshape(-1)]), (tag, int((~same).sum()))
        # gelu on U(-6, 6): 1 + tanh cancels for x < ~-3 (its FP32 value there
        # depends on the libm's last FP64 ulps); the others: ~never
        assert flagged.mean() <= (0.15 if kind == "gelu" else 1e-3), (tag, flagged.mean())
        e, er = eps.reshape(-1), eps_ref.reshape(-1)
        assert np.all(e >= er), tag
        assert_bound(e[~flagged], er[~flagged], tag)
    else:
        assert same.all(), tag
        assert_bound(eps, eps_ref, tag)


def test_matmul_bound_api(B):
    a = np.array([[2.0]], dtype=np.float32)
    b = np.array([[3.0]], dtype=np.float32)
    bt = B.matmul_bound(a, b, B.FpModel(mode="deterministic"))
    ref = B.gamma(1) * 6.0
    assert ref <= bt.array[0, 0] <= ref * (1 + RTOL)
    with pytest.raises(ValueError):
        B.matmul_bound(np.ones((2, 3), np.float32), np.ones((4, 2), np.float32), B.FpModel())


PATHS = [0, 1, 2]  # NAO_GEMM_FFMA_RU, NAO_GEMM_TC_TF32X3, NAO_GEMM_TC_F16X3
TC_PATHS = [1, 2]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("shape", [(1, 1, 1), (7, 33, 5), (128, 128, 128), (129, 300, 131),
                                   (64, 4096, 96), (300, 17, 1000), (256, 12288, 256),
                                   (2048, 128, 640)])
@pytest.mark.parametrize("tb", [False, True])
def test_abs_gemm_vs_fp64_blas(B, shape, tb, path):
    M, K, N = shape
    rng = np.random.default_rng(M * 7 + K)
    a = rng.standard_normal((M, K)).astype(np.float32)
    b = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    model = B.FpModel()
    ref = OB.matmul_bound(a, b, OB.FpModel(), transpose_b=tb)
    got = B.abs_gemm_bound(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
                           model.reduction_const(2 * K - 1), tb, path=path).cpu().numpy()
    assert_bound(got, ref, str(shape))
    got32 = B.abs_gemm_bound(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
                             model.reduction_const(2 * K - 1), tb, eps_f64=False,
                             path=path).cpu().numpy()
    assert_bound(got32, ref, str(shape) + " f32")


@pytest.mark.parametrize("path", PATHS)
def test_abs_gemm_heterogeneous_rows(B, path):
    """Softmax-like rows (one dominant entry, tiny rest) and wide dynamic range."""
    rng = np.random.default_rng(5)
    M, K, N = 64, 2048, 128
    p = np.exp(rng.standard_normal((M, K)) * 8).astype(np.float32)
    p /= p.sum(axis=1, keepdims=True)
    v = (rng.standard_normal((K, N)) * 10.0 ** rng.integers(-20, 20, size=(K, N))).astype(
        np.float32)
    ref = OB.matmul_bound(p, v, OB.FpModel())
    got = B.abs_gemm_bound(torch.from_numpy(p).cuda(), torch.from_numpy(v).cuda(),
                           OB.FpModel().reduction_const(2 * K - 1), path=path).cpu().numpy()
    assert_bound(got, ref, "hetero")


@pytest.mark.parametrize("path", TC_PATHS)
@pytest.mark.parametrize("case", ["equal", "ramp", "sparse", "tf32_edge", "subnormal",
                                  "wide_range", "one_hot_rows"])
def test_abs_gemm_tc_adversarial(B, case, path):
    """Data that stresses the tensor-core accumulation / split error model:
    long runs of equal terms (truncation bias), values on TF32 boundaries,
    sparse rows and subnormals.  Must stay inside [ref, ref (1 + 1e-5)]."""
    rng = np.random.default_rng(17)
    M, K, N = 256, 8192, 256
    if case == "equal":
        a = np.full((M, K), 1.0 + 2.0 ** -12, np.float32)
        b = np.full((K, N), 3.0 - 2.0 ** -11, np.float32)
    elif case == "ramp":
        a = np.tile(np.linspace(1e-3, 1e3, K, dtype=np.float32), (M, 1))
        b = rng.random((K, N)).astype(np.float32) + 1
    elif case == "sparse":
        a = (rng.random((M, K)) < 0.01).astype(np.float32) * rng.standard_normal((M, K)).astype(np.float32)
        b = rng.standard_normal((K, N)).astype(np.float32)
    elif case == "tf32_edge":
        base = (rng.random((M, K)) + 1).astype(np.float32)
        a = (base.view(np.uint32) | 0x1FFF).view(np.float32)  # all 13 dropped bits set
        b = ((rng.random((K, N)) + 1).astype(np.float32).view(np.uint32) | 0x1000).view(np.float32)
    elif case == "subnormal":
        a = (rng.random((M, K)) * 1e-39).astype(np.float32)
        b = (rng.random((K, N)) * 1e-3).astype(np.float32)
    elif case == "wide_range":  # 2^-40 .. 2^40 inside every row and column
        a = (2.0 ** rng.integers(-40, 40, size=(M, K)) * (rng.random((M, K)) + 1)).astype(np.float32)
        b = (2.0 ** rng.integers(-40, 40, size=(K, N)) * (rng.random((K, N)) + 1)).astype(np.float32)
    else:  # one huge entry per row paired with a zero of B; the rest tiny (FP16 tiny parts)
        a = np.full((M, K), 1e-12, np.float32)
        a[:, 0] = 1e3
        b = (rng.random((K, N)) + 0.5).astype(np.float32)
        b[0, :] = 0.0
    ref = OB.matmul_bound(a, b, OB.FpModel())
    got = B.abs_gemm_bound(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
                           OB.FpModel().reduction_const(2 * K - 1), path=path).cpu().numpy()
    if case == "subnormal":  # absolute floor K*2^-120 dominates tiny products: sound, not tight
        assert np.all(got >= ref)
    else:
        assert_bound(got, ref, case)


@pytest.mark.parametrize("path", TC_PATHS)
def test_abs_gemm_tc_batched_and_cached_weight(B, path):
    rng = np.random.default_rng(2)
    q = torch.from_numpy(rng.standard_normal((8, 200, 64)).astype(np.float32)).cuda()
    k = torch.from_numpy(rng.standard_normal((8, 300, 64)).astype(np.float32)).cuda()
    ref = OB.matmul_bound(q.cpu().numpy(), k.cpu().numpy(), OB.FpModel(), transpose_b=True)
    c = OB.FpModel().reduction_const(127)
    got = B.abs_gemm_bound(q, k, c, True, path=path).cpu().numpy()
    assert_bound(got, ref, "batched tb")
    w = torch.from_numpy(rng.standard_normal((64, 96)).astype(np.float32)).cuda()
    ref = OB.matmul_bound(q.cpu().numpy(), w.cpu().numpy(), OB.FpModel())
    for _ in range(2):  # second call hits the cached weight split
        got = B.abs_gemm_bound(q, w, c, False, path=path, cache_b=True).cpu().numpy()
        assert_bound(got, ref, "bcast weight")
    w.mul_(2.0)  # in-place change bumps _version -> cache must not be used
    ref = OB.matmul_bound(q.cpu().numpy(), w.cpu().numpy(), OB.FpModel())
    got = B.abs_gemm_bound(q, w, c, False, path=path, cache_b=True).cpu().numpy()
    assert_bound(got, ref, "weight changed")


def test_batched_broadcast_matmul(B):
    rng = np.random.default_rng(9)
    a = rng.standard_normal((4, 3, 20, 33)).astype(np.float32)
    b = rng.standard_normal((3, 18, 33)).astype(np.float32)
    ref = OB.matmul_bound(a, b, OB.FpModel(), transpose_b=True)
    got = B.matmul_bound(a, b, B.FpModel(), transpose_b=True).array
    assert_bound(got, ref, "bcast")


def test_softmax_layernorm_large_rows(B):
    """Qwen-shaped rows: softmax over n=2048, layernorm over n=4096."""
    rng = np.random.default_rng(1)
    x = (rng.standard_normal((96, 2048)) * 3).astype(np.float32)
    y_ref, e_ref = OB.softmax_bound_parts(x, -1, OB.FpModel())
    y, e = B.softmax_bound_parts(x, -1, B.FpModel())
    assert np.array_equal(y.view(np.uint32), y_ref.view(np.uint32))
    assert_bound(e, e_ref, "softmax")
    x = (rng.standard_normal((40, 4096)) + 0.5).astype(np.float32)
    y_ref, e_ref = OB.layernorm_bound_parts(x, -1, 1e-6, OB.FpModel())
    y, e = B.layernorm_bound_parts(x, -1, 1e-6, B.FpModel())
    assert np.array_equal(y.view(np.uint32), y_ref.view(np.uint32))
    assert_bound(e, e_ref, "layernorm")


@pytest.mark.parametrize("shape", [(3, 81920), (2, 100003), (5, 24577)])
@pytest.mark.parametrize("kind", ["layernorm", "sum", "mean", "max", "min"])
def test_rows_beyond_shared_memory(B, kind, shape):
    """GroupNorm-length rows (C/G*H*W up to 122880 in the SD UNet) stream
    through the double-buffered one-CTA-per-row kernel: values bit-exact to the
    sequential fold, bounds within [ref, ref(1+1e-5)]; odd n exercises the
    unaligned (scalar) loader."""
    from paper_2510_16028_b200.engine import DeviceProfile
    rng = np.random.default_rng(shape[1] + len(kind))
    x = (rng.standard_normal(shape) * 2 + 0.75).astype(np.float32)
    attrs = {"axis": -1, "eps": 1e-5}
    y_ref, e_ref = OB.op_bound(_Node(kind, attrs), [x], OB.FpModel())
    y, e = B.op_bound(_Node(kind, attrs), [x], B.FpModel(), DeviceProfile("seq", "sequential"))
    assert np.array_equal(np.asarray(y, np.float32).view(np.uint32),
                          np.asarray(y_ref, np.float32).view(np.uint32)), kind
    if kind in ("max", "min"):
        assert not np.any(e)
    else:
        assert_bound(e, e_ref, kind)


def test_mlp_co_execute_matches_reference(B, ref_mlp):
    """Full reference MLP (784-256-10, B=64) under the sequential profile:
    every node value bit-exact (digest), bounds within [ref, ref(1+1e-5)]."""
    from paper_2510_16028_b200 import commitments
    from paper_2510_16028_b200.engine import DeviceProfile
    from paper_2510_16028_b200.lowerings import build_mlp
    from paper_2510_16028_b200.tensor import Rng
    c = ref_mlp["config"]
    spec = build_mlp(c["seed"], c["batch"], c["in_dim"], c["hidden"], c["n_classes"])
    x = spec.make_inputs(Rng(*c["input_rng"]))
    for run, fma in (("seq", False), ("seqf", True)):
        for mode, mname in (("prob", "probabilistic"), ("det", "deterministic")):
            prof = DeviceProfile(run, "sequential", fma=fma)
            outs, bnds, trace = B.co_execute(spec.graph, x, prof, B.FpModel(mode=mname),
                                             with_trace=True)
            for i, (t, bt, ent) in enumerate(zip(trace.tensors, bnds, ref_mlp["runs"][f"{run}/{mode}"])):
                node = spec.graph.nodes[i].name
                assert commitments.tensor_digest(t) == ent["value_digest"], (run, mode, node)
                flat = bt.eps
                ref_s = np.asarray(ent["eps_sample"])
                assert_bound(flat[ent["idx"]], ref_s, f"{run}/{mode}/{node}")
                assert ent["eps_sum"] <= flat.sum() * (1 + 1e-12)
                assert flat.sum() <= ent["eps_sum"] * (1 + RTOL)


@pytest.mark.parametrize("shape,f64", [((4096, 384), True), ((4096, 384), False),
                                       ((1536, 131), True), ((1030, 2048), False),
                                       ((1030, 2048), True), ((777, 1024), False),
                                       ((6, 2048), True), ((3000, 1024), True)])
def test_softmax_many_long_rows(B, shape, f64):
    """Design C (max/exp warp per row, lane-per-row sequential fold, epilogue)
    at GPT-2 (n=1024) and Qwen (n=2048) row lengths: values bit-exact, bound
    within [ref, ref(1+1e-5)] (FP32 eps rounded up)."""
    rng = np.random.default_rng(shape[0] + shape[1])
    x = (rng.standard_normal(shape) * 4).astype(np.float32)
    x[3, :7] = -np.inf  # exp(-inf - m) = 0 participates in the fold
    x[5, 11] = 80.0
    y_ref, e_ref = OB.softmax_bound_parts(x, -1, OB.FpModel())
    y, e = B.softmax_device(torch.from_numpy(x).cuda(), -1, B.FpModel(), eps_f64=f64)
    y, e = y.cpu().numpy(), e.cpu().numpy().astype(np.float64)
    assert np.array_equal(y.view(np.uint32), y_ref.view(np.uint32))
    nan = np.isnan(e_ref)  # x = -inf: eps_z = inf, 0 * inf in the reference formula
    assert np.array_equal(np.isnan(e), nan)
    e, e_ref = e[~nan], e_ref[~nan]
    if f64:
        assert_bound(e, e_ref, "softmax C f64")
    else:
        assert np.all(e >= e_ref)
        # FP32 storage rounds up: beyond rtol only below FP32's normal range
        assert np.all(e <= e_ref * (1 + RTOL) + _sub32(e_ref))


@pytest.mark.parametrize("shape", [(4096, 2048), (2048, 4096), (300, 100), (8, 30000)])
def test_softmax_exp_wide_range(B, shape):
    """z = x - max spread uniformly over [-90, 0] (FP32-normal and FP32-subnormal
    e values, exp(-inf) = 0): probabilities bit-exact against the oracle
    (numpy's FP64 exp rounded to FP32) on every row kernel (design G rows,
    long rows, short-row batches), bound within [ref, ref(1+1e-5)]."""
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    x = -rng.uniform(0.0, 90.0, shape).astype(np.float32)
    x[:, 0] = 0.0
    x[1, 1:9] = -np.inf
    y_ref, e_ref = OB.softmax_bound_parts(x, -1, OB.FpModel())
    y, e = B.softmax_device(torch.from_numpy(x).cuda(), -1, B.FpModel(), eps_f64=True)
    assert np.array_equal(y.cpu().numpy().view(np.uint32), y_ref.view(np.uint32))
    e, ok = e.cpu().numpy(), ~np.isnan(e_ref)
    assert_bound(e[ok], e_ref[ok], "softmax wide z")


@pytest.mark.parametrize("path", TC_PATHS)
@pytest.mark.parametrize("K", [1, 64, 128, 256])
def test_abs_gemm_tc_short_k_persistent(B, K, path):
    """K <= one TMEM chunk -> the persistent k_absgemm_tc_short (FP32 eps): many
    more tiles than SMs (slot reuse), ragged M/N, batched q k^T, linear u|y|."""
    rng = np.random.default_rng(K)
    q = rng.standard_normal((40, 300, K)).astype(np.float32)
    k = rng.standard_normal((40, 333, K)).astype(np.float32)
    c = OB.FpModel().reduction_const(2 * K - 1)
    ref = OB.matmul_bound(q, k, OB.FpModel(), transpose_b=True)
    got = B.abs_gemm_bound(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(), c, True,
                           eps_f64=False, path=path).cpu().numpy()
    assert_bound(got, ref, "scores")
    x = rng.standard_normal((1000, K)).astype(np.float32)
    w = rng.standard_normal((K, 700)).astype(np.float32)
    y = (x @ w).astype(np.float32)
    u = 2.0 ** -24
    ref = OB.matmul_bound(x, w, OB.FpModel()) + u * np.abs(y.astype(np.float64))
    got = B.abs_gemm_bound(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), c, False,
                           y=torch.from_numpy(y).cuda(), u=u, eps_f64=False, path=path,
                           cache_b=True).cpu().numpy()
    assert_bound(got, ref, "linear")


@pytest.mark.parametrize("geom", [(2, 3, 17, 13, 7, 2, 3), (3, 5, 8, 8, 3, 1, 1),
                                  (1, 4, 9, 6, 1, 1, 0), (2, 2, 5, 7, 3, 2, 0)])
def test_im2col_rows_matches_unfold(B, geom):
    """nao_im2col_rows == torch unfold (K order c, kh, kw; zero padding) transposed
    to [B, OH*OW, K]: the patch-row operand of the conv2d abs-GEMM bound."""
    b, c, h, w, k, st, pd = geom
    x = torch.randn((b, c, h, w), device="cuda")
    col, (nb, oh, ow) = B.im2col(x, k, st, pd)
    ref = torch.nn.functional.unfold(x, k, padding=pd, stride=st).transpose(1, 2)
    assert (nb, oh * ow) == (b, ref.shape[1])
    assert torch.equal(col, ref)


def test_softmax_design_c_parity():
    """The opt-in three-kernel softmax (NAO_SOFTMAX_DESIGN=C, read once per
    process; the default is the shared-memory design G) against the oracle,
    in a subprocess."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, torch\n"
        "from oracle import bounds as OB\n"
        "from paper_2510_16028_b200 import bounds as B\n"
        "for shape in ((1030, 2048), (2048, 1024), (1500, 516)):\n"
        "    rng = np.random.default_rng(shape[1])\n"
        "    x = (rng.standard_normal(shape) * 4).astype(np.float32)\n"
        "    x[3, :7] = -np.inf\n"
        "    y_ref, e_ref = OB.softmax_bound_parts(x, -1, OB.FpModel())\n"
        "    for f64 in (True, False):\n"
        "        y, e = B.softmax_device(torch.from_numpy(x).cuda(), -1, B.FpModel(), eps_f64=f64)\n"
        "        y, e = y.cpu().numpy(), e.cpu().numpy().astype(np.float64)\n"
        "        assert np.array_equal(y.view(np.uint32), y_ref.view(np.uint32))\n"
        "        ok = ~np.isnan(e_ref)\n"
        "        assert np.array_equal(np.isnan(e), ~ok)\n"
        "        assert np.all(e[ok] >= e_ref[ok])\n"
        "        er = e_ref[ok]\n"
        "        sp = 0 if f64 else np.where(er < np.finfo(np.float32).tiny,\n"
        "                                    2 * np.spacing(er.astype(np.float32)), 0.0)\n"
        "        assert np.all(e[ok] <= e_ref[ok] * (1 + 1e-5) + sp)\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, NAO_SOFTMAX_DESIGN="C", PYTHONPATH=root)
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("MKN", [(2048, 4096, 4096), (2048, 4096, 12288), (2048, 12288, 4096),
                                 (2048, 4096, 1024)])
def test_abs_gemm_full_qwen_shapes(B, MKN):
    """Qwen3-8B projection shapes at full size on the default (FP16 3-split)
    path: 24 sampled output rows against the FP64 reference template, and two
    size-independent properties over the whole output -- exact power-of-two
    homogeneity eps(8A) == 8 eps(A) (the split, the MMAs, the FP64 drains and
    the round-up all commute with 2^3) and eps(A) == eps(A) over a row
    permutation of A (rows are independent)."""
    M, K, N = MKN
    rng = np.random.default_rng(K + N)
    a = torch.from_numpy((rng.standard_normal((M, K)) * 0.5).astype(np.float32)).cuda()
    w = torch.from_numpy((rng.uniform(-1, 1, (K, N)) / np.sqrt(K)).astype(np.float32)).cuda()
    c = B.FpModel().reduction_const(2 * K - 1)
    eps = B.abs_gemm_bound(a, w, c, False, eps_f64=False)
    rows = np.r_[0, M - 1, rng.choice(M, 22, replace=False)]
    ref = OB.matmul_bound(a[rows].cpu().numpy(), w.cpu().numpy(), OB.FpModel())
    assert_bound(eps[rows].cpu().numpy().astype(np.float64), ref, str(MKN))
    eps8 = B.abs_gemm_bound(a * 8.0, w, c, False, eps_f64=False)
    assert torch.equal(eps8, eps * 8.0)
    perm = torch.from_numpy(rng.permutation(M)).cuda()
    epsp = B.abs_gemm_bound(a[perm].contiguous(), w, c, False, eps_f64=False)
    assert torch.equal(epsp, eps[perm])


def test_non_fp32_inputs_rejected(B):
    """A float64 operand (e.g. float32 / np.float64 promotion) is a ValueError at
    the boundary, never reinterpreted as FP32 words by the kernels."""
    from paper_2510_16028_b200.dispute import check_node
    a32 = torch.ones((4, 8), device="cuda")
    a64 = torch.ones((4, 8), device="cuda", dtype=torch.float64)
    c = B.FpModel().reduction_const(15)
    with pytest.raises(ValueError):
        B.abs_gemm_bound(a32, a64.T.contiguous(), c)
    with pytest.raises(ValueError):
        B.softmax_device(a64, -1, B.FpModel())
    with pytest.raises(ValueError):
        B.reduce_device("sum", a64, -1, B.FpModel())
    with pytest.raises(ValueError):
        check_node(a32, a64, ("zero",), np.full(23, np.inf), np.full(23, np.inf))


def test_softmax_full_qwen_scores(B):
    """Qwen3-8B attention probabilities at full size (32 x 2048 x 2048, causal
    -1e9 mask as in the lowering): 16 sampled rows bit-exact / within tolerance
    against the oracle, and the whole output equivariant under a permutation of
    the 65536 rows (rows are independent in every design)."""
    S, H = 2048, 32
    rng = np.random.default_rng(S)
    x = torch.randn((H, S, S), device="cuda") * 4.0
    mask = torch.triu(torch.full((S, S), -1e9, device="cuda"), diagonal=1)
    x = (x + mask).contiguous()
    y, e = B.softmax_device(x, -1, B.FpModel(), eps_f64=False)
    flat_x, flat_y, flat_e = x.reshape(-1, S), y.reshape(-1, S), e.reshape(-1, S)
    rows = np.r_[0, S - 1, rng.choice(H * S, 14, replace=False)]
    xr = flat_x[rows].cpu().numpy()
    y_ref, e_ref = OB.softmax_bound_parts(xr, -1, OB.FpModel())
    got_y, got_e = flat_y[rows].cpu().numpy(), flat_e[rows].cpu().numpy().astype(np.float64)
    assert np.array_equal(got_y.view(np.uint32), y_ref.view(np.uint32))
    assert np.all(got_e >= e_ref)
    assert np.all(got_e <= e_ref * (1 + RTOL) + _sub32(e_ref))
    perm = torch.from_numpy(rng.permutation(H * S)).cuda()
    yp, ep = B.softmax_device(flat_x[perm].contiguous(), -1, B.FpModel(), eps_f64=False)
    assert torch.equal(yp, flat_y[perm]) and torch.equal(ep, flat_e[perm])
