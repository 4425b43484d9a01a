"""The CPU oracle still reproduces the frozen golden logits (tests/golden/logits_*.npz,
oracle/make_golden_logits.py): the GPU parity tests compare the device against these
frozen values, so a drift of the oracle itself (torch / torchvision / the parameter
generator) must show up here, on the CPU."""

import os

import numpy as np
import pytest

from oracle import make_golden_logits

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ARCHS = sorted(f[len("logits_"):-4] for f in os.listdir(GOLDEN) if f.startswith("logits_"))


@pytest.mark.parametrize("name", ARCHS)
def test_oracle_reproduces_frozen_logits(name):
    frozen = np.load(os.path.join(GOLDEN, f"logits_{name}.npz"))["logits"]
    assert frozen.shape[0] == 16
    got = make_golden_logits.golden(name)
    np.testing.assert_allclose(got, frozen, rtol=1e-4, atol=1e-4 * np.abs(frozen).max())
