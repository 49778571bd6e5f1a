"""Probe: fused commit+check time of one Qwen3-8B attention block's committed
tensors (scores -> scaled -> masked -> probs, 32 x 2048 x 2048 each) with and
without the digest shortcuts (all-zero chunks, same-offset reuse of the mask
add, row_chunks thread mapping).  CUDA events, best of --reps.

    python tools/shortcut_probe.py [--reps 5]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--seq", type=int, default=2048)
    args = ap.parse_args()
    from paper_2510_16028_b200 import _lib
    from paper_2510_16028_b200.commitments import commit_tensors
    from paper_2510_16028_b200.executor import inject_drift, row_chunks
    H, S = args.heads, args.seq
    g = torch.Generator(device="cuda").manual_seed(0)
    scores = torch.randn((H, S, S), generator=g, device="cuda") * 4
    scaled = scores * 0.08838834764831845
    mask = torch.triu(torch.full((S, S), -1e9, device="cuda"), diagonal=1)
    masked = scaled + mask
    probs = torch.softmax(masked, dim=-1)
    locals_ = [scores, scaled, masked, probs]
    claims = [inject_drift(scores, 1, 16), scaled.clone(), masked.clone(), inject_drift(probs, 2, 16)]
    spec = torch.frombuffer(bytearray(_lib.verdict_spec([50.0], [float("inf")], [float("inf")],
                                                         1e-12)), dtype=torch.uint8).cuda()
    recs = torch.zeros((4, _lib.CHECK_RESULT_BYTES), dtype=torch.uint8, device="cuda")
    checks = [_lib.CheckDesc(l.data_ptr(), None, spec.data_ptr(), recs[i].data_ptr(),
                             2.0 ** -22, 1.0, _lib.EPS_SCALED_LOCAL, 0, None, 0)
              for i, l in enumerate(locals_)]
    rc = row_chunks(probs, 4096)
    nch = probs.numel() * 4 // 4096
    mdig = torch.empty((1 + mask.numel() * 4 // 4096, 32), dtype=torch.uint8, device="cuda")
    commit_tensors([mask], 4096, "keccak256", leaf_digests=mdig)
    ref = (mask.data_ptr(), mdig.data_ptr() + 32, mask.numel() * 4)
    plans = {
        "none": None,
        "rows_only": [(-1, 0, 0, 0, rc)] * 4,
        "shortcuts_identity_map": [None, None, (1, nch, 1, _lib.REUSE_SAME_OFFSET, 0), (-1, 0, 0, 0, 0)],
        "shortcuts_no_mask_ref": [(-1, 0, 0, 0, rc), (-1, 0, 0, 0, rc),
                                  (1, nch, 1, _lib.REUSE_SAME_OFFSET, rc), (-1, 0, 0, 0, rc)],
        "shortcuts": [(-1, 0, 0, 0, rc), (-1, 0, 0, 0, rc),
                      (1, nch, 1, _lib.REUSE_SAME_OFFSET, rc) + ref, (-1, 0, 0, 0, rc)],
    }

    def timed(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    res = {"mask_fill_chunk_frac_masked": float(
        (masked.view(-1, 1024) == -1e9).all(dim=1).float().mean()),
        "zero_chunk_frac_probs": float(
        (probs.view(-1, 1024) == 0).all(dim=1).float().mean()),
        "masked_eq_scaled_chunk_frac": float(
        (masked.view(-1, 1024) == scaled.view(-1, 1024)).all(dim=1).float().mean())}
    roots = {}
    for name, plan in plans.items():
        fn = lambda: commit_tensors(claims, 4096, "keccak256", checks=checks, reuse=plan)  # noqa
        fn()
        roots[name] = fn().cpu()
        res[name + "_ms"] = round(min(timed(fn) for _ in range(args.reps)), 3)
    res["roots_equal"] = all(torch.equal(roots["none"], r) for r in roots.values())
    # all-zero tensor: every chunk takes the zero digest (memory-bound pass)
    z, zl = torch.zeros_like(probs), torch.zeros_like(probs)
    zc = [_lib.CheckDesc(zl.data_ptr(), None, spec.data_ptr(), recs[0].data_ptr(),
                         2.0 ** -22, 1.0, _lib.EPS_SCALED_LOCAL, 0, None, 0)]
    fz = lambda: commit_tensors([z], 4096, "keccak256", checks=zc, reuse=[(-1, 0, 0, 0, rc)])  # noqa
    fz()
    res["all_zero_ms"] = round(min(timed(fz) for _ in range(args.reps)), 3)
    fr = lambda: commit_tensors([probs], 4096, "keccak256", checks=zc[:0] + [  # noqa
        _lib.CheckDesc(probs.data_ptr(), None, spec.data_ptr(), recs[0].data_ptr(),
                       2.0 ** -22, 1.0, _lib.EPS_SCALED_LOCAL, 0, None, 0)], reuse=[(-1, 0, 0, 0, rc)])
    fr()
    res["probs_alone_ms"] = round(min(timed(fr) for _ in range(args.reps)), 3)
    fs = lambda: commit_tensors([scores], 4096, "keccak256", checks=[  # noqa
        _lib.CheckDesc(scores.data_ptr(), None, spec.data_ptr(), recs[0].data_ptr(),
                       2.0 ** -22, 1.0, _lib.EPS_SCALED_LOCAL, 0, None, 0)], reuse=[(-1, 0, 0, 0, rc)])
    fs()
    res["scores_alone_ms"] = round(min(timed(fs) for _ in range(args.reps)), 3)
    res["gb"] = round(4 * sum(t.numel() for t in claims) * 4 / 4 / 1e9, 3)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
