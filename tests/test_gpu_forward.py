"""End-to-end INFER parity: the worker's CUDA-graph ResNet forward (bf16
tcgen05 kernels, folded BN) against the CPU fp32 oracle on the same seeded
inputs and weights. Tolerance: top-1 identical, max-abs logit error <= 0.02 *
max|logit| (oracle.resnet_oracle.compare)."""

import numpy as np
import pytest

from oracle import resnet_oracle
from paper_2006_02464_b200 import arch
from paper_2006_02464_b200.device import DeviceRuntime

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def r50():
    spec = arch.build_arch("resnet50")
    params = arch.make_params(spec, seed=0)
    blob = arch.pack_blob(spec, arch.fold(spec, params))
    model = resnet_oracle.torchvision_model("resnet50", params)
    return spec, blob, model


@pytest.mark.parametrize("batch", [1, 2, 4, 8, 16])
def test_resnet50_logits_match_oracle(gpu, r50, batch):
    spec, blob, model = r50
    x = arch.make_inputs(batch, spec, first=100 * batch)
    with DeviceRuntime(device=gpu, pages_total=8, io_slots=16) as rt:
        rt.register_arch(0, spec)
        rt.register_blob(0, 0, blob)
        rt.build()
        rt.load(0, [3, 1, 6, 0][:blob.pages])  # non-contiguous pages, header on page 3
        got, ns = rt.infer(0, 3, x)
    ref = resnet_oracle.logits(model, x)
    c = resnet_oracle.compare(got, ref)
    assert c["ok"], c
    assert ns > 0


@pytest.mark.parametrize("name", ["resnet18", "resnet34", "resnet101", "resnet152"])
@pytest.mark.parametrize("batch", [1, 8])
def test_resnet_family_logits_match_oracle(gpu, name, batch):
    """The other torchvision ResNets of the zoo (basic blocks with 3x3 residual convs, deep
    bottleneck stacks whose plans hold 100+ layers) through the same megakernel."""
    spec = arch.build_arch(name)
    params = arch.make_params(spec, seed=1)
    blob = arch.pack_blob(spec, arch.fold(spec, params))
    x = arch.make_inputs(batch, spec, first=7 * batch)
    with DeviceRuntime(device=gpu, pages_total=blob.pages + 2, io_slots=16) as rt:
        rt.register_arch(0, spec, batches=(batch,))
        rt.register_blob(0, 0, blob)
        rt.build()
        rt.load(0, list(range(blob.pages + 1, 0, -1))[:blob.pages])
        got, _ = rt.infer(0, blob.pages + 1, x)
    ref = resnet_oracle.logits(resnet_oracle.torchvision_model(name, params), x)
    c = resnet_oracle.compare(got, ref)
    assert c["ok"], c


@pytest.mark.parametrize("batch", [1, 16])
def test_layer_handoff_repeatable_under_alternating_inputs(gpu, r50, batch):
    """Layer-to-layer handoff stress (the conv layers publish their completion counts with
    a relaxed add after their TMA stores completed, see red_after_bulk_add in mk_infer.cu):
    hundreds of INFERs alternating two inputs must reproduce each input's first logits bit
    for bit. A consumer that read a producer's tile before it landed would see the other
    input's (or an earlier layer's) activations in the reused arena and diverge."""
    spec, blob, _ = r50
    xs = [arch.make_inputs(batch, spec, first=11 + k * batch) for k in range(2)]
    with DeviceRuntime(device=gpu, pages_total=8, io_slots=16) as rt:
        rt.register_arch(0, spec, batches=(batch,))
        rt.register_blob(0, 0, blob)
        rt.build()
        rt.load(0, list(range(blob.pages)))
        first = [rt.infer(0, 0, x)[0].copy() for x in xs]
        assert not np.array_equal(first[0], first[1])
        bad = 0
        for i in range(400 if batch == 1 else 200):
            got, _ = rt.infer(0, 0, xs[i & 1])
            bad += not np.array_equal(got, first[i & 1])
    assert bad == 0, f"{bad} INFERs differ from the first run of their input"


@pytest.mark.parametrize("batch,csize", [(1, 8), (2, 4), (4, 4), (8, 2), (16, 2)])
def test_cluster_split_plans(gpu, r50, batch, csize):
    """Small-batch plans launch the megakernel in thread-block clusters and reduce split-K
    convs through distributed shared memory (no reduce layers): the persistent grid is whole
    clusters, every cluster split-K layer has tasks = tiles x csize on a csize-aligned
    rotation, and back-to-back INFERs (the cluster handshakes' mbarrier phases carry over
    from task to task and INFER to INFER) reproduce the logits bit for bit."""
    spec, blob, model = r50
    x = arch.make_inputs(batch, spec, first=5 * batch)
    with DeviceRuntime(device=gpu, pages_total=8, io_slots=16) as rt:
        rt.register_arch(0, spec, batches=(batch,))
        rt.register_blob(0, 0, blob)
        rt.build()
        rt.load(0, [0, 1, 2, 3][:blob.pages])
        grid, cs = rt.plan_launch(0, batch)
        assert cs == csize and grid % cs == 0 and grid >= 8 * cs
        layers = rt.plan_layers(0, batch)
        csplit = layers[(layers[:, 7] & 2) != 0]
        assert len(csplit) > 0
        assert (csplit[:, 4] == cs).all() and (csplit[:, 2] == 64).all()
        assert not (layers[:, 0] == 6).any()  # no MK_REDUCE layers in a cluster plan
        first, _ = rt.infer(0, 0, x)
        for _ in range(3):
            again, _ = rt.infer(0, 0, x)
            assert np.array_equal(first, again)
    c = resnet_oracle.compare(first, resnet_oracle.logits(model, x))
    assert c["ok"], c
