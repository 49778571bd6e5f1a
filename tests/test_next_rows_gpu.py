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
