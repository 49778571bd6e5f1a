"""GPU: SURVEY.md 8(f) "next" rows built so far.
Row 1 -- calibrate / build_thresholds on the GPU vs the oracle restatement of
calibration.py:70-114 (profiles the B200 emulates bit-exactly: sequential,
sequential+fma), envelopes bit-identical."""

import numpy as np
import pytest

from oracle import check as OC

pytestmark = pytest.mark.gpu


def test_gpu_calibrate_matches_oracle():
    from paper_2510_16028_b200 import calibration
    from paper_2510_16028_b200.engine import DeviceProfile
    from paper_2510_16028_b200.lowerings import build_mlp
    from paper_2510_16028_b200.tensor import Rng
    spec = build_mlp(seed=0, batch=4, in_dim=16, hidden=32)
    rng = Rng(101)
    data = [spec.make_inputs(rng) for _ in range(3)]
    profs = [DeviceProfile("seq", "sequential"), DeviceProfile("seqf", "sequential", fma=True)]
    env = calibration.calibrate(spec.graph, data, profs)
    ref_abs, ref_rel = OC.calibrate(spec.graph, [{"x": d["x"].array} for d in data],
                                    [False, True])
    for i in range(spec.graph.n_nodes):
        np.testing.assert_array_equal(env.abs_env[i], ref_abs[i])
        np.testing.assert_array_equal(env.rel_env[i], ref_rel[i])
    th = calibration.build_thresholds_from_envelopes(env, alpha=3.0)
    assert th.lookup("mm1").tau_abs.shape == (len(calibration.PERCENTILE_GRID),)
    assert np.all(th.lookup("mm1").tau_abs == 3.0 * env.abs_env[6])
    with pytest.raises(ValueError):
        calibration.calibrate(spec.graph, data, profs[:1])


def test_gpu_calibrate_reproduces_reference_thresholds(ref_mlp):
    """Row f1 pinned to the reference itself: calibrate + build_thresholds on the
    GPU over the reference's own 6-profile fleet (default_profiles + the
    calibration extras, conftest.py:9-13; every order emulated bit-exactly,
    csrc/profile_fold.cuh) on Rng(101)'s first 12 MLP inputs, alpha = 3
    (oracle/gen_golden.py), reproduces the reference-generated ThresholdSet in
    tests/golden/ref_mlp_784_256_10_b64.json bit for bit."""
    from paper_2510_16028_b200 import calibration
    from paper_2510_16028_b200.engine import DeviceProfile
    from paper_2510_16028_b200.lowerings import build_mlp
    from paper_2510_16028_b200.tensor import Rng
    c = ref_mlp["config"]
    spec = build_mlp(c["seed"], c["batch"], c["in_dim"], c["hidden"], c["n_classes"])
    fleet = [DeviceProfile.from_spec(s) for s in
             ("sequential", "pairwise", "blocked:32", "permuted:7+fma", "permuted:3", "blocked:4")]
    rng = Rng(101)
    data = [spec.make_inputs(rng) for _ in range(12)]
    env = calibration.calibrate(spec.graph, data, fleet)
    th = calibration.build_thresholds_from_envelopes(env, alpha=3.0)
    ref = calibration.ThresholdSet.from_json(ref_mlp["thresholds"])
    assert th.grid == ref.grid and th.alpha == ref.alpha and th.epsilon == ref.epsilon
    for node in spec.graph.nodes:
        a, b = th.lookup(node.name), ref.lookup(node.name)
        assert np.array_equal(a.tau_abs, b.tau_abs), node.name
        assert np.array_equal(a.tau_rel, b.tau_rel), node.name
