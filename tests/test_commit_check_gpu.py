"""GPU parity: the acceptance check fused into the Merkle commit pass
(nao_commit_check_tensors) gives, per tensor, the same record as the
standalone one-pass check (nao_check) and the oracle's verdicts, and the same
roots as the plain commit -- across eps kinds, drift/fault/non-finite claims,
thresholds that force the exact second pass, ragged sizes and >128-tensor
batches (several launches)."""

import numpy as np
import pytest
import torch

from oracle import check as OC
from oracle import commit as OM

pytestmark = pytest.mark.gpu
GRID = OC.PERCENTILE_GRID
INF = np.full(len(GRID), np.inf)
FIELDS = ("n", "n_violations", "n_borderline", "n_nonfinite", "max_ratio",
          "threshold_exceeded", "first_exceeded", "n_ambiguous")


def _drift(y, frac, ulps, rng):
    yc = y.copy()
    idx = rng.random(y.size) < frac
    bits = yc.view(np.int32).reshape(-1)
    bits[idx] += rng.integers(-ulps, ulps + 1, size=int(idx.sum())).astype(np.int32)
    return yc


def _case(rng, n, mode, eps_kind, tau_mode):
    y = (rng.standard_normal(n) * 10.0 ** rng.integers(-2, 2, size=n)).astype(np.float32)
    if mode == "equal":
        yc = y.copy()
    elif mode == "drift":
        yc = _drift(y, 1 / 16, 1, rng)
    elif mode == "heavy":
        yc = _drift(y, 1.0, 6, rng)
        k = rng.integers(0, n, size=max(1, n // 100))
        yc[k] = yc[k] * np.float32(37.0) + np.float32(1e3)
        k = rng.integers(0, n, size=max(1, n // 100))
        yc[k] = -yc[k]
    else:  # nonfinite
        yc = _drift(y, 0.1, 2, rng)
        yc[rng.integers(0, n, size=max(1, n // 500))] = np.inf
        yc[rng.integers(0, n, size=max(1, n // 700))] = np.nan
        y[rng.integers(0, n, size=max(1, n // 900))] = np.nan
    c = 3.3 * 2.0 ** -24
    eps64 = c * np.abs(y.astype(np.float64))
    if eps_kind == "scaled":
        eps, ref_eps = ("scaled", c), eps64
    elif eps_kind == "f64":
        eps, ref_eps = torch.from_numpy(eps64).cuda(), eps64
    elif eps_kind == "f32":
        e32 = eps64.astype(np.float32)
        eps, ref_eps = torch.from_numpy(e32).cuda(), e32.astype(np.float64)
    else:
        eps, ref_eps = ("zero",), np.zeros(n)
    if tau_mode == "inf":
        taus = (INF, INF)
    else:
        with np.errstate(invalid="ignore"):
            a, r = OC.elementwise_errors(y, yc)
        pa, pr = OC.percentile_profile(a), OC.percentile_profile(r)
        taus = (pa, pr) if tau_mode == "exact" else (pa * 0.5, pr * 3.0)
    return y, yc, eps, ref_eps, taus


def _records(recs):
    from paper_2510_16028_b200.dispute import CheckRecord
    return [CheckRecord(recs[i]).host() for i in range(recs.shape[0])]


@pytest.mark.parametrize("alg,chunk", [("keccak256", 4096), ("keccak256", 256),
                                       ("sha256", 1024)])
def test_fused_matches_standalone_check(alg, chunk):
    from paper_2510_16028_b200 import dispute
    from paper_2510_16028_b200.commitments import commit_tensors
    rng = np.random.default_rng(hash((alg, chunk)) & 0xFFFF)
    sizes = [1, 3, 64, 1025, 4097, 70001, 262147]
    modes = ["equal", "drift", "heavy", "nonfinite"]
    kinds = ["scaled", "f32", "f64", "zero"]
    taus_m = ["inf", "exact", "scaled"]
    cases = []
    for k in range(24):
        n = sizes[k % len(sizes)]
        mode = modes[k % len(modes)]
        if mode == "nonfinite" and n < 8:
            mode = "drift"
        tm = taus_m[(k // 4) % 3] if mode != "nonfinite" else "inf"
        cases.append(_case(rng, n, mode, kinds[(k // 2) % 4], tm))
    claimed = [torch.from_numpy(c[1]).cuda() for c in cases]
    local = [torch.from_numpy(c[0]).cuda() for c in cases]
    roots, recs = dispute.commit_check_nodes(claimed, local, [c[2] for c in cases],
                                             [c[4] for c in cases], chunk, alg)
    plain = commit_tensors(claimed, chunk, alg)
    torch.cuda.synchronize()
    assert torch.equal(roots, plain)
    got = _records(recs)
    for i, (y, yc, eps, ref_eps, taus) in enumerate(cases):
        want = dispute.check_node(local[i], claimed[i], eps, taus[0], taus[1]).host()
        for f in FIELDS:
            if f == "max_ratio" and np.isnan(want[f]):
                continue
            assert got[i][f] == want[f], (i, f, got[i][f], want[f])
        # and the oracle's verdicts directly
        with np.errstate(invalid="ignore"):
            ref = OC.leaf_check(y, yc, ref_eps)
        if np.all(np.isfinite(y)):
            assert got[i]["n_violations"] == ref["n_violations"], i
            pm = OC.observed_p_max(y, yc, taus[0], taus[1])
            assert bool(got[i]["threshold_exceeded"]) == (pm > 1.0), i
        assert bytes(roots[i].cpu().numpy()) == OM.tensor_root(
            yc, chunk, OM.KECCAK256 if alg == "keccak256" else OM.SHA256), i


def test_fused_many_tensors_and_empty():
    """>128 tensors (several launches), an empty tensor in the batch (root
    only, no record), and the accumulator left clean for the next call."""
    from paper_2510_16028_b200 import dispute
    from paper_2510_16028_b200.commitments import commit_tensors
    rng = np.random.default_rng(3)
    ys, ycs = [], []
    for i in range(300):
        n = int(rng.integers(0, 3000)) if i != 5 else 0
        y = rng.standard_normal(n).astype(np.float32)
        ys.append(y)
        ycs.append(_drift(y, 0.3, 2, rng))
    claimed = [torch.from_numpy(c).cuda() for c in ycs]
    local = [torch.from_numpy(c).cuda() for c in ys]
    eps = [("scaled", 2.0 ** -23)] * len(ys)
    taus = [(INF, INF)] * len(ys)
    for rep in range(2):
        roots, recs = dispute.commit_check_nodes(claimed, local, eps, taus, 256, "keccak256")
        plain = commit_tensors(claimed, 256, "keccak256")
        torch.cuda.synchronize()
        assert torch.equal(roots, plain)
        got = _records(recs)
        for i, (y, yc) in enumerate(zip(ys, ycs)):
            if y.size == 0:
                assert got[i]["n"] == 0
                continue
            ref = OC.leaf_check(y, yc, 2.0 ** -23 * np.abs(y.astype(np.float64)))
            assert got[i]["n"] == y.size
            assert got[i]["n_violations"] == ref["n_violations"], (rep, i)


@pytest.mark.parametrize("pieces", [1, 2, 3, 5])
def test_partial_records_combine_to_whole_tensor_verdict(pieces):
    """Batch-sharded checks: each shard emits a combinable
    nao_check_partial; combine_partials reproduces the whole tensor's record
    from the pieces -- violations, borderline, max ratio and the exact
    percentile verdict incl. thresholds AT the true percentiles (numpy's
    interpolation between order statistics, decided from the key ranges)."""
    from paper_2510_16028_b200 import dispute
    rng = np.random.default_rng(pieces)
    for mode, kind, tm in (("drift", "scaled", "exact"), ("heavy", "f32", "exact"),
                           ("heavy", "f64", "scaled"), ("drift", "zero", "inf"),
                           ("equal", "scaled", "exact"), ("heavy", "scaled", "exact")):
        y, yc, eps, ref_eps, taus = _case(rng, 12000 + 7 * pieces, mode, kind, tm)
        want = dispute.check_node(torch.from_numpy(y).cuda(), torch.from_numpy(yc).cuda(), eps,
                                  taus[0], taus[1]).host()
        cuts = np.linspace(0, y.size, pieces + 1).astype(int)
        claimed = [torch.from_numpy(yc[a:b]).cuda() for a, b in zip(cuts[:-1], cuts[1:])]
        local = [torch.from_numpy(y[a:b]).cuda() for a, b in zip(cuts[:-1], cuts[1:])]
        if isinstance(eps, tuple):
            epss = [eps] * pieces
        else:
            epss = [eps[a:b] for a, b in zip(cuts[:-1], cuts[1:])]
        _, recs = dispute.commit_check_nodes(claimed, local, epss, [taus] * pieces, 256,
                                             "keccak256", partial=True)
        torch.cuda.synchronize()
        parts = [dispute.partial_from_bytes(recs[i].cpu().numpy().tobytes())
                 for i in range(pieces)]
        got = dispute.combine_partials(parts, taus[0], taus[1])
        for f in ("n", "n_violations", "n_borderline", "n_nonfinite", "threshold_exceeded",
                  "first_exceeded"):
            assert got[f] == want[f], (mode, kind, tm, f, got[f], want[f])
        assert got["max_ratio"] == want["max_ratio"], (mode, kind, tm)
        with np.errstate(invalid="ignore"):
            pm = OC.observed_p_max(y, yc, taus[0], taus[1])
        assert bool(got["threshold_exceeded"]) == (pm > 1.0)


def test_fused_full_qwen_scores_tensor():
    """One Qwen3-8B attention-scores-sized tensor (32 x 2048 x 2048 FP32, 537 MB)
    with 1/16 of the elements drifted by one ulp, an FP32 bound tensor and
    thresholds at the exact percentile profile of its own errors (every grid
    point on the boundary: the exact second pass runs): the fused record equals
    the standalone check's, the verdicts equal the oracle's numpy ones, and the
    Keccak root equals the C restatement's."""
    from paper_2510_16028_b200 import dispute
    from paper_2510_16028_b200.commitments import commit_tensors
    rng = np.random.default_rng(2048)
    n = 32 * 2048 * 2048
    y = (rng.standard_normal(n, dtype=np.float32) * 3.0).astype(np.float32)
    yc = _drift(y, 1 / 16, 1, rng)
    c = 3.3 * 2.0 ** -24
    e32 = (c * np.abs(y.astype(np.float64))).astype(np.float32)
    e32[rng.integers(0, n, size=64)] = 0.0  # a few zero bounds: violations where drifted
    with np.errstate(invalid="ignore"):
        a, r = OC.elementwise_errors(y, yc)
    pa, pr = OC.percentile_profile(a), OC.percentile_profile(r)
    del a, r
    local, claimed = torch.from_numpy(y).cuda(), torch.from_numpy(yc).cuda()
    eps = torch.from_numpy(e32).cuda()
    roots, recs = dispute.commit_check_nodes([claimed], [local], [eps], [(pa, pr)], 4096,
                                             "keccak256")
    plain = commit_tensors([claimed], 4096, "keccak256")
    want = dispute.check_node(local, claimed, eps, pa, pr).host()
    got = _records(recs)[0]
    torch.cuda.synchronize()
    assert torch.equal(roots, plain)
    for f in FIELDS:
        assert got[f] == want[f], (f, got[f], want[f])
    ref = OC.leaf_check(y, yc, e32.astype(np.float64))
    assert got["n_violations"] == ref["n_violations"] > 0
    assert bool(got["threshold_exceeded"]) == (OC.observed_p_max(y, yc, pa, pr) > 1.0)
    import os
    assert bytes(roots[0].cpu().numpy()) == OM.tensor_root(yc, 4096, OM.KECCAK256,
                                                           n_threads=os.cpu_count() or 1)


@pytest.mark.parametrize("chunk", [512, 4096])
def test_chunk_digest_reuse_keeps_roots(chunk):
    """nao_chunk_reuse (data-movement nodes copy their source's chunk digests):
    a reshape chain and a GQA-style concat of one tensor with itself, with
    claims equal to the local copy, with one differing word, and with an inf,
    give the same roots as hashing every chunk and the same check records."""
    from paper_2510_16028_b200 import _lib
    from paper_2510_16028_b200.commitments import commit_tensors
    from paper_2510_16028_b200.dispute import CheckRecord
    rng = np.random.default_rng(3)
    S, hd = 64, 32  # block = S*hd*4 = 8 KiB = whole chunks
    src = torch.from_numpy(rng.standard_normal((2, 1, S, hd)).astype(np.float32)).cuda()
    spec = torch.frombuffer(bytearray(_lib.verdict_spec(GRID, INF, INF, 1e-12)),
                            dtype=torch.uint8).cuda()
    for mode in ("equal", "word", "inf"):
        # every local is the data movement of the CLAIMED inputs (as in the executor)
        c0 = src.clone()
        l1 = c0.reshape(2, S, hd)             # reshape node (a view of claim 0)
        c1 = l1.clone()
        l2 = torch.cat([c0] * 4, dim=1)       # GQA concat of claim 0 with itself
        c2 = l2.clone()
        if mode == "word":
            c2.view(-1)[1000] += 1.0
        elif mode == "inf":
            c1.view(-1)[5] = float("inf")
        l3 = c2.reshape(8, S, hd)             # reshape of the concat's claim (chain)
        c3 = l3.clone()
        if mode == "word":
            c3.view(-1)[3000] -= 1.0
        claims = [c0, c1, c2, c3]
        locals_ = [None, l1, l2, l3]
        recs = torch.zeros((4, _lib.CHECK_RESULT_BYTES), dtype=torch.uint8, device="cuda")
        checks = [None] + [_lib.CheckDesc(l.data_ptr(), None, spec.data_ptr(), recs[i + 1].data_ptr(),
                                          0.0, 1.0, _lib.EPS_ZERO, 0, None, 0)
                           for i, l in enumerate(locals_[1:])]
        nch = -(-src.numel() * 4 // chunk)
        blk = S * hd * 4 // chunk
        reuse = [None, (0, nch, 1), (0, blk, 4), (2, 4 * nch, 1)]
        got = commit_tensors(claims, chunk, "keccak256", checks=checks, reuse=reuse)
        plain = commit_tensors(claims, chunk, "keccak256")
        torch.cuda.synchronize()
        assert torch.equal(got, plain), mode
        for i, t in enumerate(claims):
            assert bytes(got[i].cpu().numpy()) == OM.tensor_root(t.cpu().numpy(), chunk,
                                                                 OM.KECCAK256), (mode, i)
        r = [CheckRecord(recs[i]).host() for i in range(1, 4)]
        if mode == "equal":
            assert all(x["n_violations"] == 0 for x in r)
        elif mode == "word":
            assert [x["n_violations"] for x in r] == [0, 1, 1]
        else:
            assert r[0]["n_violations"] == 1 and r[0]["n_nonfinite"] == 1


@pytest.mark.parametrize("chunk,width", [(4096, 2048), (512, 512), (4096, 1024)])
def test_digest_shortcuts_keep_roots_and_records(chunk, width):
    """Digest shortcuts of the fused commit+check: all-zero claimed chunks take
    the zero-chunk digest, a causal-mask add (x + mask) copies the digest of
    the operand's equal chunks (REUSE_SAME_OFFSET), rows of several chunks
    map one chunk position per warp (row_chunks) -- with claims equal to the
    local tensors, with a drifted word inside a zero / reused chunk and with a
    local word that is not zero under a zero claim: roots equal the plain
    commit and the oracle's, records equal the unshortcut fused check."""
    from paper_2510_16028_b200 import _lib
    from paper_2510_16028_b200.commitments import commit_tensors
    from paper_2510_16028_b200.dispute import CheckRecord
    from paper_2510_16028_b200.executor import row_chunks
    rng = np.random.default_rng(11)
    H, S = 3, 192
    spec = torch.frombuffer(bytearray(_lib.verdict_spec(GRID, INF, INF, 1e-12)),
                            dtype=torch.uint8).cuda()
    scaled = torch.from_numpy((rng.standard_normal((H, S, width)) * 3).astype(np.float32)).cuda()
    cols = torch.arange(width, device="cuda")
    rows = torch.arange(S, device="cuda") * (width // S + 1)
    mask = torch.where(cols[None, :] > rows[:, None], -1e9, 0.0).float()  # causal-style
    masked = scaled + mask
    probs = torch.softmax(masked, dim=-1)
    assert (probs == 0).any() and (masked == scaled).any()
    rc = row_chunks(masked, chunk)
    if width * 4 > chunk:  # rows of several chunks: whole fill chunks exist
        assert ((masked.view(-1, chunk // 4) == -1e9).all(dim=1)).any()
    for mode in ("equal", "drift", "local"):
        c_scaled, c_masked, c_probs = scaled.clone(), masked.clone(), probs.clone()
        l_masked, l_probs = masked.clone(), probs.clone()
        if mode == "drift":  # claimed words moved inside shortcut chunks
            c_masked[0, S - 1, 3] += 1.0          # lower triangle: equals scaled elsewhere
            c_masked[2, 0, width - 1] = -1e9 * (1 + 2 ** -20)  # a fill chunk (rc > 1)
            c_probs[0, 0, width - 5] = 1e-3       # the zero upper triangle of row 0
        elif mode == "local":  # local non-zero where the claim is zero
            l_probs[1, 0, width - 9] = 2.0 ** -40
        claims = [c_scaled, c_masked, c_probs]
        locals_ = [scaled, l_masked, l_probs]

        def run(reuse):
            recs = torch.zeros((3, _lib.CHECK_RESULT_BYTES), dtype=torch.uint8, device="cuda")
            checks = [_lib.CheckDesc(l.data_ptr(), None, spec.data_ptr(), recs[i].data_ptr(),
                                     0.0, 1.0, _lib.EPS_ZERO, 0, None, 0)
                      for i, l in enumerate(locals_)]
            roots = commit_tensors(claims, chunk, "keccak256", checks=checks, reuse=reuse)
            torch.cuda.synchronize()
            return roots, [CheckRecord(recs[i]).host() for i in range(3)]

        nch = -(-masked.numel() * 4 // chunk)
        # the mask as a broadcast reference (its fill chunks: x + -1e9 == -1e9)
        mdig = torch.empty((1 + mask.numel() * 4 // chunk, 32), dtype=torch.uint8, device="cuda")
        commit_tensors([mask], chunk, "keccak256", leaf_digests=mdig)
        ref = (mask.data_ptr(), mdig.data_ptr() + 32, mask.numel() * 4)
        got, r_got = run([(-1, 0, 0, 0, rc), (0, nch, 1, _lib.REUSE_SAME_OFFSET, rc) + ref,
                          (-1, 0, 0, 0, rc)])
        got2, r_got2 = run([None, (-1, 0, 0, 0, 0) + ref, None])
        assert torch.equal(got2, got) and r_got2 == r_got, mode
        ref, r_ref = run(None)
        plain = commit_tensors(claims, chunk, "keccak256")
        torch.cuda.synchronize()
        assert torch.equal(got, plain) and torch.equal(ref, plain), mode
        for i, t in enumerate(claims):
            assert bytes(got[i].cpu().numpy()) == OM.tensor_root(t.cpu().numpy(), chunk,
                                                                 OM.KECCAK256), (mode, i)
        assert r_got == r_ref, mode
        nv = [x["n_violations"] for x in r_got]
        assert nv == {"equal": [0, 0, 0], "drift": [0, 2, 1], "local": [0, 0, 1]}[mode], (mode, nv)
