"""GPU parity: the one-pass check (nao_check) and exact percentiles vs the
oracle.  Verdicts must be identical; percentiles are bit-exact."""

import numpy as np
import pytest
import torch

from oracle import check as OC

pytestmark = pytest.mark.gpu
GRID = OC.PERCENTILE_GRID


@pytest.fixture(scope="module")
def D():
    from paper_2510_16028_b200 import calibration, dispute
    return dispute, calibration


def _drift(y, frac, ulps, rng):
    yc = y.copy()
    idx = rng.random(y.size) < frac
    bits = yc.view(np.int32).reshape(-1)
    bits[idx] += rng.integers(-ulps, ulps + 1, size=int(idx.sum())).astype(np.int32)
    return yc


@pytest.mark.parametrize("n", [1, 2, 3, 7, 100, 4097, 100003])
def test_percentile_profile_exact(D, n):
    _, cal = D
    rng = np.random.default_rng(n)
    v = rng.standard_normal(n) * 10.0 ** rng.integers(-3, 3, size=n)
    np.testing.assert_array_equal(cal.percentile_profile(v), OC.percentile_profile(v))
    v2 = np.abs(v)
    np.testing.assert_array_equal(cal.percentile_profile(v2), OC.percentile_profile(v2))


@pytest.mark.parametrize("n", [1, 5, 1000, 65537, 1 << 20])
def test_error_profiles_exact(D, n):
    _, cal = D
    rng = np.random.default_rng(n + 1)
    y = rng.standard_normal(n).astype(np.float32)
    yc = _drift(y, 0.3, 3, rng)
    pa, pr = cal.error_profiles_device(torch.from_numpy(y).cuda(), torch.from_numpy(yc).cuda())
    a, r = OC.elementwise_errors(y, yc)
    np.testing.assert_array_equal(pa.cpu().numpy(), OC.percentile_profile(a))
    np.testing.assert_array_equal(pr.cpu().numpy(), OC.percentile_profile(r))


def _random_taus(a, r, rng, scale):
    ta = OC.percentile_profile(a) * scale
    tr = OC.percentile_profile(r) * scale
    return ta, tr


@pytest.mark.parametrize("n", [1, 2, 9, 1000, 4099, 262147])
@pytest.mark.parametrize("scale", [0.5, 0.999, 1.0, 1.001, 3.0])
def test_threshold_verdict_matches_oracle(D, n, scale):
    dsp, _ = D
    rng = np.random.default_rng(7 * n)
    y = (rng.standard_normal(n) * 10.0 ** rng.integers(-2, 2, size=n)).astype(np.float32)
    yc = _drift(y, 0.2, 4, rng)
    a, r = OC.elementwise_errors(y, yc)
    ta, tr = _random_taus(a, r, rng, scale)
    ref = OC.observed_p_max(y, yc, ta, tr)
    rec = dsp.check_node(torch.from_numpy(y).cuda(), torch.from_numpy(yc).cuda(), ("zero",),
                         ta, tr).host()
    assert bool(rec["threshold_exceeded"]) == (ref > 1.0), (ref, rec)
    # exact threshold = profile itself (ratio exactly 1 -> not exceeded): exercises pass 2
    rec2 = dsp.check_node(torch.from_numpy(y).cuda(), torch.from_numpy(yc).cuda(), ("zero",),
                          OC.percentile_profile(a), OC.percentile_profile(r)).host()
    assert rec2["threshold_exceeded"] == 0


def test_threshold_zero_tau_guard(D):
    dsp, _ = D
    y = np.ones(1000, np.float32)
    yc = y.copy()
    z = np.zeros(len(GRID))
    rec = dsp.check_node(torch.from_numpy(y).cuda(), torch.from_numpy(yc).cuda(), ("zero",), z,
                         z).host()
    assert rec["threshold_exceeded"] == 0  # 0/0 -> 0
    yc[3] = np.nextafter(np.float32(1), np.float32(2))
    rec = dsp.check_node(torch.from_numpy(y).cuda(), torch.from_numpy(yc).cuda(), ("zero",), z,
                         z).host()
    assert rec["threshold_exceeded"] == 1  # x/0 -> inf at p100


@pytest.mark.parametrize("kind", ["scaled", "f32", "f64", "zero"])
def test_bound_violations_exact(D, kind):
    dsp, _ = D
    rng = np.random.default_rng(11)
    n = 300007
    y = rng.standard_normal(n).astype(np.float32)
    u = 2.0 ** -24
    eps64 = u * np.abs(y.astype(np.float64))
    yc = y.copy()
    # put claims just inside / outside the bound
    k = rng.integers(0, n, size=2000)
    fac = rng.choice([0.5, 0.99, 1.5, 3.0], size=k.size)
    yc[k] = (y[k].astype(np.float64) + fac * eps64[k] * 1.0000001 * 2).astype(np.float32)
    if kind == "scaled":
        eps, ref_eps = ("scaled", u), eps64
    elif kind == "f64":
        eps, ref_eps = torch.from_numpy(eps64).cuda(), eps64
    elif kind == "f32":
        e32 = eps64.astype(np.float32)
        eps, ref_eps = torch.from_numpy(e32).cuda(), e32.astype(np.float64)
    else:
        eps, ref_eps = ("zero",), np.zeros(n)
    ref = OC.leaf_check(y, yc, ref_eps)
    rec = dsp.check_node(torch.from_numpy(y).cuda(), torch.from_numpy(yc).cuda(), eps,
                         np.full(len(GRID), np.inf), np.full(len(GRID), np.inf)).host()
    assert rec["n_violations"] == ref["n_violations"]
    if np.isfinite(ref["max_ratio"]):
        assert rec["max_ratio"] == pytest.approx(ref["max_ratio"], rel=1e-12)
    else:
        assert rec["max_ratio"] == np.inf


def test_mlp_golden_checks(D, ref_mlp):
    """The reference's observed_p_max on the MLP fault injection (golden) vs GPU."""
    dsp, cal = D
    from oracle import bounds as OB
    from paper_2510_16028_b200.lowerings import build_mlp
    from paper_2510_16028_b200.tensor import Rng
    c = ref_mlp["config"]
    spec = build_mlp(c["seed"], c["batch"], c["in_dim"], c["hidden"], c["n_classes"])
    x = spec.make_inputs(Rng(*c["input_rng"]))
    vals, _ = OB.co_execute(spec.graph, {"x": x["x"].array}, OB.FpModel())
    inj = ref_mlp["injection"]
    faulty, _ = OB.co_execute(spec.graph, {"x": x["x"].array}, OB.FpModel(),
                              inject={inj["node"]: np.full(vals[inj["node"]].shape, inj["value"])})
    th = cal.ThresholdSet.from_json(ref_mlp["thresholds"])
    for i, node in enumerate(spec.graph.nodes):
        ent = ref_mlp["checks"]["fault"][i]
        a, b = torch.from_numpy(vals[i]).cuda(), torch.from_numpy(faulty[i]).cuda()
        pa, pr = cal.error_profiles_device(a, b, th.grid, th.epsilon)
        np.testing.assert_array_equal(pa.cpu().numpy(), ent["abs_prof"])
        np.testing.assert_array_equal(pr.cpu().numpy(), ent["rel_prof"])
        pm = dsp.observed_p_max(a, b, th, node.name)
        assert pm == ent["p_max"]
        op = th.lookup(node.name)
        rec = dsp.check_node(a, b, ("zero",), op.tau_abs, op.tau_rel, th.grid, th.epsilon).host()
        assert bool(rec["threshold_exceeded"]) == (ent["p_max"] > 1.0), node.name


def _heavy_claims(y, rng):
    """Every element drifts: ulp noise, some sign flips, some large faults,
    some tiny values (FP32 fast path must hand these to the FP64 keys)."""
    yc = _drift(y, 1.0, 6, rng)
    n = y.size
    k = rng.integers(0, n, size=max(1, n // 50))
    yc[k] = -yc[k]
    k = rng.integers(0, n, size=max(1, n // 100))
    yc[k] = yc[k] * np.float32(37.0) + np.float32(1e3)
    k = rng.integers(0, n, size=max(1, n // 100))
    yc[k] = np.float32(1e-38) * rng.standard_normal(k.size).astype(np.float32)
    return yc


@pytest.mark.parametrize("n", [4, 1001, 262147])
def test_threshold_verdict_heavy_drift_edges(D, n):
    """Thresholds exactly at the true percentiles (not exceeded) and one FP64
    ulp below them, per grid point (exceeded) -- the FP32 interval search
    must fall back to the exact keys inside its guard band."""
    dsp, _ = D
    rng = np.random.default_rng(n + 99)
    y = (rng.standard_normal(n) * 10.0 ** rng.integers(-3, 3, size=n)).astype(np.float32)
    y[rng.integers(0, n, size=max(1, n // 100))] = 1e-39
    yc = _heavy_claims(y, rng)
    a, r = OC.elementwise_errors(y, yc)
    pa, pr = OC.percentile_profile(a), OC.percentile_profile(r)
    gy, gc = torch.from_numpy(y).cuda(), torch.from_numpy(yc).cuda()
    rec = dsp.check_node(gy, gc, ("zero",), pa, pr).host()
    assert rec["threshold_exceeded"] == 0
    for arr in (0, 1):
        for i in range(0, len(GRID), 3):
            ta, tr = pa.copy(), pr.copy()
            t = ta if arr == 0 else tr
            if t[i] == 0.0:
                continue
            t[i] = np.nextafter(t[i], -np.inf)
            ref = OC.observed_p_max(y, yc, ta, tr)
            assert ref > 1.0
            rec = dsp.check_node(gy, gc, ("zero",), ta, tr).host()
            assert rec["threshold_exceeded"] == 1, (arr, i)
            assert rec["first_exceeded"] == arr * len(GRID) + i


@pytest.mark.parametrize("kind", ["scaled", "f32", "f64"])
def test_bound_violations_heavy_drift(D, kind):
    dsp, _ = D
    rng = np.random.default_rng(5)
    n = 200003
    y = (rng.standard_normal(n) * 10.0 ** rng.integers(-3, 3, size=n)).astype(np.float32)
    yc = _heavy_claims(y, rng)
    c = 3.3 * 2.0 ** -24  # not a power of two: FP32 and FP64 products differ
    eps64 = c * np.abs(y.astype(np.float64))
    if kind == "scaled":
        eps, ref_eps = ("scaled", c), eps64
    elif kind == "f64":
        eps, ref_eps = torch.from_numpy(eps64).cuda(), eps64
    else:
        e32 = eps64.astype(np.float32)
        eps, ref_eps = torch.from_numpy(e32).cuda(), e32.astype(np.float64)
    ref = OC.leaf_check(y, yc, ref_eps)
    rec = dsp.check_node(torch.from_numpy(y).cuda(), torch.from_numpy(yc).cuda(), eps,
                         np.full(len(GRID), np.inf), np.full(len(GRID), np.inf)).host()
    assert rec["n_violations"] == ref["n_violations"]
    assert rec["max_ratio"] == pytest.approx(ref["max_ratio"], rel=1e-12)
