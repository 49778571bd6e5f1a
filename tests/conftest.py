import json
import sys
from pathlib import Path

import numpy as np
import pytest

from _helpers import GOLDEN, ROOT  # noqa: F401


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ref_vectors():
    return json.load(open(GOLDEN / "reference_commitment_vectors.json"))


@pytest.fixture(scope="session")
def ref_mlp():
    return json.load(open(GOLDEN / "ref_mlp_784_256_10_b64.json"))


@pytest.fixture(scope="session")
def ref_ops():
    z = np.load(GOLDEN / "ref_ops.npz")
    return {k: z[k] for k in z.files}


