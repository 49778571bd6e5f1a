"""GPU: empirical check of the tcgen05 accumulation error model behind
nao_abs_gemm_tc (csrc/absgemm_tc.cu header): with TF32-exact operands the lo
parts vanish, every product is exact, and the output is
    eps = scale0 * sum_chunks acc0_chunk   (scale0 known)
so the accumulator's relative loss per k-chunk (nao_abs_gemm_tc_kchunk()/8 MMAs)
can be measured exactly against an FP64 sum and compared with the modelled
bound J0 * 3 * 2^-23.
The runs are built to maximise truncation loss: long runs of equal terms
(every addition aligns the same low bits away) and growing partial sums.
Both tcgen05 paths: kind::tf32 (path 1) and the default kind::f16 (path 2,
every Qwen projection): operands with 11 significant bits are exact in TF32
and, after the split's exact power-of-two row scaling, in FP16 (lo = 0, no
tiny parts), so the same identity isolates the FP16 MMA accumulation."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

MMA_REL = 3.0 * 2.0 ** -23


def _j0():
    from paper_2510_16028_b200 import _lib
    return _lib.load().nao_abs_gemm_tc_kchunk() // 8


def _scale0(c, K):
    from paper_2510_16028_b200.bounds import gemm_slack
    comp_split = 1.0 / (1.0 - 1.002 * 2.0 ** -20)
    comp0 = 1.0 / (1.0 - _j0() * MMA_REL)
    return c * comp_split * (1.0 + gemm_slack(K)) * (1.0 + 2.0 ** -50) * comp0, comp0


def _tf32_exact(x):
    return (x.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


@pytest.mark.parametrize("path", [1, 2])
@pytest.mark.parametrize("case", ["equal", "equal_big", "random_tf32", "ramp"])
def test_tc_accumulation_loss_within_model(case, path):
    from paper_2510_16028_b200.bounds import abs_gemm_bound
    rng = np.random.default_rng(3)
    M, K, N = 128, 8192, 128
    if case == "equal":
        a = np.full((M, K), 1.0 + 2.0 ** -10, np.float32)
        b = np.full((K, N), 1.0 + 2.0 ** -9, np.float32)
    elif case == "equal_big":
        a = np.full((M, K), 1.9990234375, np.float32)  # 11 significant bits
        b = np.full((K, N), 1.9990234375, np.float32)
    elif case == "random_tf32":
        a = _tf32_exact((rng.random((M, K)) + 0.5).astype(np.float32))
        b = _tf32_exact((rng.random((K, N)) + 0.5).astype(np.float32))
    else:
        a = _tf32_exact(np.tile(np.linspace(1.0, 2.0, K, dtype=np.float32), (M, 1)))
        b = _tf32_exact((rng.random((K, N)) + 1.0).astype(np.float32))
    exact = np.abs(a.astype(np.float64)) @ np.abs(b.astype(np.float64))
    c = 1.0
    got = abs_gemm_bound(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), c, path=path)
    got = got.cpu().numpy()
    scale0, comp0 = _scale0(c, K)
    raw = got / scale0  # = sum of the per-chunk TMEM sums (lo parts are exactly zero)
    loss = 1.0 - raw / exact  # relative loss of the tensor-core accumulation
    worst = float(loss.max())
    j0 = _j0()
    print(f"{case} path {path}: worst relative accumulation loss {worst:.3e} "
          f"(model per chunk {j0 * MMA_REL:.3e})")
    assert worst <= j0 * MMA_REL
    assert np.all(got >= exact)  # the compensated bound stays sound
