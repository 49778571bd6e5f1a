"""CPU: the drop-in binding's host logic (no kernels run here).

* refbind.install() rebinds the unmodified reference's hot-path names
   -- including the by-name imports in dispute.py -- keeps
  the reference's own types at the boundary and is idempotent;
* the certified over-estimates used for the borderline band are >= 1,
  grow with K, and the tensor-core ones stay near the 1e-5 contract;
* chunk-digest reuse is only proposed where chunks line up."""

import sys
from pathlib import Path

import pytest
import torch

REF_SRC = Path("/root/reference/pkg/src")


@pytest.fixture(scope="module")
def fpverify():
    if not REF_SRC.is_dir():
        pytest.skip("reference not present")
    sys.path.insert(0, str(REF_SRC))
    import fpverify
    from fpverify import bounds, calibration, commitments, dispute  # noqa: F401
    return fpverify


def test_refbind_rebinds_reference_names(fpverify):
    from fpverify import bounds as rb, calibration as rc, commitments as rcm, dispute as rd
    orig = (rb.op_bound, rc.percentile_profile, rcm.build_tree, rd.Challenger.leaf_payload)
    names = {rb: ("op_bound", "matmul_bound", "softmax_bound_parts", "softmax_bound",
                  "layernorm_bound_parts"),
             rc: ("percentile_profile", "percentile", "calibrate"),
             rcm: ("build_tree",), rd: ("op_bound", "percentile_profile", "sample_committee")}
    saved = {(m, n): getattr(m, n) for m, ns in names.items() for n in ns}
    from paper_2510_16028_b200 import refbind
    try:
        refbind.install()
        refbind.install()  # idempotent
        assert rb.op_bound is not orig[0] and rd.op_bound is rb.op_bound
        assert rd.percentile_profile is rc.percentile_profile is not orig[1]
        assert rcm.build_tree is not orig[2]
        assert rd.Challenger.leaf_payload is not orig[3]
        assert rb.op_bound.__wrapped__.__module__ == "paper_2510_16028_b200.refbind"
    finally:  # leave the reference modules as they were for the other CPU tests
        for (m, n), v in saved.items():
            setattr(m, n, v)
        rd.Challenger.leaf_payload = orig[3]
        refbind._INSTALLED = False


def test_certified_overestimates():
    from paper_2510_16028_b200 import _lib
    from paper_2510_16028_b200.bounds import certified_overestimate as R
    for K in (16, 128, 4096, 12288):
        for path in (_lib.GEMM_FFMA_RU, _lib.GEMM_TC_TF32X3, _lib.GEMM_TC_F16X3, _lib.GEMM_FP64):
            r32, r64 = R("matmul", K=K, path=path), R("matmul", K=K, path=path, eps_f32=False)
            assert r32 >= r64 > 1.0
    assert R("matmul", K=4096, path=_lib.GEMM_TC_F16X3) - 1 < 1.1e-5
    assert R("matmul", K=4096, path=_lib.GEMM_FP64, eps_f32=False) - 1 < 1e-11
    assert R("softmax", n=2048, eps_f32=False) - 1 < 1e-11
    assert R("add") == R("exp") == 1.0
    assert R("matmul", K=12288, path=_lib.GEMM_TC_F16X3) > R("matmul", K=64, path=_lib.GEMM_TC_F16X3)


class _N:
    def __init__(self, kind, inputs, attrs=None):
        self.kind, self.inputs, self.attrs = kind, inputs, attrs or {}

    def attr(self, k, d=None):
        return self.attrs.get(k, d)


def test_chunk_reuse_proposals():
    from paper_2510_16028_b200.executor import chunk_reuse
    x = torch.zeros(8, 1, 2048, 128)
    pos = {5: 3}
    assert chunk_reuse(_N("reshape", ["node:5"]), [x], pos, 4096) == (3, 2048 * 128 * 4 * 8 // 4096, 1)
    # GQA: 4 copies of each 1 MB block along axis 1
    assert chunk_reuse(_N("concat", ["node:5"] * 4, {"axis": 1}), [x] * 4, pos, 4096) == \
        (3, 2048 * 128 * 4 // 4096, 4)
    # blocks that do not fill whole chunks, other inputs, or a source not pending: none
    y = torch.zeros(8, 1, 3, 5)
    assert chunk_reuse(_N("concat", ["node:5"] * 2, {"axis": 1}), [y] * 2, pos, 4096) is None
    assert chunk_reuse(_N("concat", ["node:5", "node:6"], {"axis": 1}), [x, x], pos, 4096) is None
    assert chunk_reuse(_N("reshape", ["node:7"]), [x], pos, 4096) is None


def test_chunk_plan_proposals():
    """row_chunks only for rows of whole chunks dividing the CTA's 128; same-offset
    reuse only for node +/- weight of the output's shape, pending in the commit."""
    import torch
    from paper_2510_16028_b200 import _lib
    from paper_2510_16028_b200.executor import chunk_plan, row_chunks
    assert row_chunks(torch.empty(4, 2048), 4096) == 2
    assert row_chunks(torch.empty(4, 1000), 4096) == 0
    assert row_chunks(torch.empty(4, 3 * 1024), 4096) == 0   # 3 does not divide 128
    assert row_chunks(torch.empty(2048), 4096) == 0
    y = torch.empty(2, 64, 2048)
    pos = {5: 3}
    m = torch.empty(64, 2048)
    assert chunk_plan(_N("add", ["node:5", "weight:mask"]), [y, m], y, pos,
                      4096) == (3, 2 * 64 * 2, 1, _lib.REUSE_SAME_OFFSET, 2, None, None, 0)
    # the weight as a broadcast reference (digests from the caller's cache)
    fake = lambda w: (111, 222, w.numel() * 4)  # noqa: E731
    assert chunk_plan(_N("add", ["node:5", "weight:mask"]), [y, m], y, {}, 4096, fake) == \
        (-1, 0, 0, _lib.REUSE_LOCAL_COPY, 2, 111, 222, 64 * 2048 * 4)
    assert chunk_plan(_N("add", ["node:5", "weight:b"]), [y, torch.empty(2048)], y, {}, 4096,
                      fake) == (-1, 0, 0, _lib.REUSE_LOCAL_COPY, 2, 111, 222, 2048 * 4)
    assert chunk_plan(_N("add", ["node:5", "weight:b"]), [y, torch.empty(1000)], y, {}, 4096,
                      fake) == (-1, 0, 0, _lib.REUSE_LOCAL_COPY, 2)  # not whole chunks
    assert chunk_plan(_N("add", ["node:5", "node:6"]), [y, y], y, {5: 3, 6: 4}, 4096) == \
        (-1, 0, 0, _lib.REUSE_LOCAL_COPY, 2)
    assert chunk_plan(_N("mul", ["node:5", "weight:w"]), [y, y], y, pos, 4096) == \
        (-1, 0, 0, _lib.REUSE_LOCAL_COPY, 2)
    small = torch.empty(4, 2048)  # below one commit CTA of chunks: no same-offset entry
    assert chunk_plan(_N("add", ["node:5", "weight:mask"]), [small, torch.empty(2048)], small,
                      pos, 4096) == (-1, 0, 0, _lib.REUSE_LOCAL_COPY, 2)
    z = torch.empty(2, 64, 1000)
    assert chunk_plan(_N("add", ["node:7", "weight:w"]), [z, z], z, pos, 4096) is None
