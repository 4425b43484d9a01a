"""Freeze golden logits of the CPU fp32 oracle — TEST INFRASTRUCTURE ONLY.

    python oracle/make_golden_logits.py [arch ...]

For each arch: the torchvision-definition network with the repo's deterministic
random-init parameters (arch.make_params(spec, seed=0)), evaluated in fp32 on the CPU
(oracle/resnet_oracle.py) on the first 16 synthetic request inputs
(arch.make_inputs(16, spec): image i = N(0,1) from numpy default_rng(i)). Writes
tests/golden/logits_<arch>.npz with `logits` [16][classes] float32 and `request_ids`.
The GPU tests compare the device logits of every batch size against these frozen values
(tolerance in resnet_oracle.compare); tests/test_golden_logits.py checks the oracle still
reproduces them (a drift in torch / torchvision would show there first).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from oracle import resnet_oracle  # noqa: E402
from paper_2006_02464_b200 import arch  # noqa: E402

N = 16


def golden(name: str) -> np.ndarray:
    spec = arch.build_arch(name)
    params = arch.make_params(spec, seed=0)
    model = resnet_oracle.torchvision_model(name, params)
    return resnet_oracle.logits(model, arch.make_inputs(N, spec)).astype(np.float32)


def main(names):
    for name in names:
        out = os.path.join(REPO, "tests", "golden", f"logits_{name}.npz")
        np.savez_compressed(out, logits=golden(name), request_ids=np.arange(N))
        print(out)


if __name__ == "__main__":
    main(sys.argv[1:] or ["resnet50"])
