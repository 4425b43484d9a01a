"""The arch tables and the weight folding (paper_2006_02464_b200/arch.py) against
torchvision itself, on the CPU: the op-list interpreter (oracle/op_interpreter.py) runs
the exact ops / buffers / channel slices / paddings and the exact folded blob layouts the
device plans use, in fp32, and must reproduce torchvision's module on the unfolded
parameters. This pins every zoo arch before any kernel runs (the
reference catalog's densenet169 / inceptionv3, plus resnext50_32x4d / densenet121)."""

import numpy as np
import pytest

from oracle import op_interpreter, resnet_oracle
from paper_2006_02464_b200 import arch

ZOO = ["resnet18", "resnet50", "resnext50_32x4d", "densenet121", "densenet169", "inception_v3"]


@pytest.fixture(scope="module", params=ZOO)
def zoo(request):
    spec = arch.build_arch(request.param)
    params = arch.make_params(spec, seed=3)
    return request.param, spec, params


def test_folded_tables_reproduce_torchvision(zoo):
    name, spec, params = zoo
    x = arch.make_inputs(2, spec, first=5)
    ref = resnet_oracle.logits(resnet_oracle.torchvision_model(name, params), x)
    got = op_interpreter.run(spec, arch.fold(spec, params), x)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 2e-4, (name, err)


def test_bf16_numerics_within_stated_tolerance(zoo):
    """bf16 weights and bf16 activations at every buffer store (the device's storage
    types; fp32 accumulation) stay within the stated parity tolerance (top-1 identical,
    max-abs logit error <= 2% of max |logit|, resnet_oracle.compare)."""
    name, spec, params = zoo
    x = arch.make_inputs(4, spec, first=9)
    ref = resnet_oracle.logits(resnet_oracle.torchvision_model(name, params), x)
    got = op_interpreter.run(spec, arch.fold(spec, params), x, bf16=True)
    c = resnet_oracle.compare(got, ref)
    assert c["ok"], (name, c)


def test_blob_layout(zoo):
    name, spec, params = zoo
    blob = arch.pack_blob(spec, arch.fold(spec, params))
    assert len(blob.locs) == len(spec.layers) <= 192           # kMaxLayers (cw_device.h)
    for lay, (w, b, rows, k, s) in zip(spec.layers, blob.locs):
        if lay.kind != "bn":
            assert rows % 64 == 0 and k % 64 == 0 or lay.layout == "stem4", lay
            assert w % 256 == 0 and w // blob.page_bytes == (w + rows * k * 2 - 1) // blob.page_bytes
        assert (s >= 0) == (lay.pre_bn is not None)
    assert blob.pages * blob.page_bytes >= blob.data.size


def test_reference_catalog_archs_are_buildable():
    for base in ("densenet169", "inceptionv3", "resnet18", "resnet50", "resnet152"):
        spec = arch.build_arch(base)
        assert spec.flops_per_image > 0 and spec.ops[-1]["kind"] == arch.OP_FC
