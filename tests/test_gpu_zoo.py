"""The model zoo on the device (BASELINE configs[3]): ResNeXt-50 32x4d
(grouped 3x3 convs), DenseNet-121/169 (BN+ReLU prologue on the A tiles, concat through
channel-offset stores, BN-pool transitions), Inception-v3 (299x299, im2col stem, 1x7/7x1
and 1x3/3x1 convs, concat branches, avg-pool branches as 3x3 convs), through the same
megakernel, against the frozen golden logits of the CPU fp32 oracle (tests/golden/,
oracle/make_golden_logits.py) and, at other inputs, the live oracle. Tolerance:
resnet_oracle.compare (top-1 identical, max-abs logit error <= 2% of max |logit|).

And the drop-in boundary with the reference's OWN catalog (profiles.py:322-374:
densenet169, inceptionv3, resnet18, resnet50, resnet152): B200Worker(mode="cuda") builds
every model of it and serves LOAD + INFER of each with the golden logits.
"""

import os
import threading
import time

import numpy as np
import pytest

from oracle import resnet_oracle
from paper_2006_02464_b200 import arch, catalog
from paper_2006_02464_b200.device import DeviceRuntime
from paper_2006_02464_b200.wire import Action, ActionKind
from paper_2006_02464_b200.worker import B200Worker

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ZOO = ["resnext50_32x4d", "densenet121", "densenet169", "inception_v3"]


def golden(name):
    return np.load(os.path.join(GOLDEN, f"logits_{name}.npz"))["logits"]


@pytest.fixture(scope="module", params=ZOO)
def net(request, gpu):
    name = request.param
    spec = arch.build_arch(name)
    blob = arch.pack_blob(spec, arch.fold(spec, arch.make_params(spec, seed=0)))
    rt = DeviceRuntime(device=gpu, pages_total=blob.pages + 3, io_slots=16,
                       in_bytes_max=spec.in_c * spec.in_h * spec.in_w * 4)
    rt.__enter__()
    rt.register_arch(0, spec, batches=(1, 2, 8, 16))
    rt.register_blob(0, 0, blob)
    rt.build()
    pages = list(range(blob.pages + 2, 2, -1))[:blob.pages]   # non-contiguous, reversed
    rt.load(0, pages)
    yield name, spec, rt, pages[0]
    rt.__exit__(None, None, None)


@pytest.mark.parametrize("batch", [1, 2, 8, 16])
def test_zoo_matches_frozen_golden_logits(net, batch):
    name, spec, rt, hdr = net
    got, ns = rt.infer(0, hdr, arch.make_inputs(batch, spec))
    c = resnet_oracle.compare(got, golden(name)[:batch])
    assert c["ok"], (name, batch, c)
    assert ns > 0


def test_zoo_matches_live_oracle_other_inputs(net):
    name, spec, rt, hdr = net
    x = arch.make_inputs(8, spec, first=1000)
    got, _ = rt.infer(0, hdr, x)
    params = arch.make_params(spec, seed=0)
    ref = resnet_oracle.logits(resnet_oracle.torchvision_model(name, params), x)
    c = resnet_oracle.compare(got, ref)
    assert c["ok"], (name, c)


def test_zoo_repeatable(net):
    """The same input twice gives bit-identical logits (no stale-buffer or handoff race in
    the concat / prologue paths)."""
    name, spec, rt, hdr = net
    xs = [arch.make_inputs(16, spec, first=k * 16) for k in range(2)]
    first = [rt.infer(0, hdr, x)[0].copy() for x in xs]
    for i in range(40):
        got, _ = rt.infer(0, hdr, xs[i & 1])
        assert np.array_equal(got, first[i & 1]), (name, i)


REF_CATALOG = """page_bytes 16777216
model densenet169
weights_bytes 56500000
weights_transfer_ns 4500000
io_ns 50000 50000
io_bytes 602000 4000
batch 1 5180000
batch 2 6290000
batch 4 8570000
batch 8 12820000
batch 16 21850000
model inceptionv3
weights_bytes 95300000
weights_transfer_ns 7770000
io_ns 50000 50000
io_bytes 1073000 4000
batch 1 4460000
batch 2 6850000
batch 4 10990000
batch 8 16450000
batch 16 26170000
model resnet18
weights_bytes 46700000
weights_transfer_ns 3810000
io_ns 50000 50000
io_bytes 602000 4000
batch 1 1270000
batch 2 1860000
batch 4 2730000
batch 8 4060000
batch 16 7020000
model resnet50
weights_bytes 102300000
weights_transfer_ns 8330000
io_ns 50000 50000
io_bytes 602000 4000
batch 1 2610000
batch 2 3780000
batch 4 5610000
batch 8 9130000
batch 16 15670000
model resnet152
weights_bytes 240900000
weights_transfer_ns 19580000
io_ns 50000 50000
io_bytes 602000 4000
batch 1 7710000
batch 2 11140000
batch 4 16210000
batch 8 26480000
batch 16 44600000
"""


def test_reference_catalog_served_on_device(gpu):
    """profiles.reference_catalog() (the text above is its dumps_catalog output, checked
    against the reference in tests/test_catalog_golden.py) on the cuda worker: every
    model LOADs and serves INFERs of batch 1 and 16 with its golden logits."""
    cat = catalog.parse(REF_CATALOG)
    got = {}
    cv = threading.Condition()

    def send(r):
        with cv:
            got[r.action_id] = r
            cv.notify_all()

    def wait(aid):
        with cv:
            assert cv.wait_for(lambda: aid in got, 120), aid
            return got[aid]

    w = B200Worker(0, cat, None, send, pages_per_gpu=64, mode="cuda", devices=[gpu],
                   epoch_ns=time.time_ns(), keep_outputs=True, input_pool=16)
    names = {0: "densenet169", 1: "inception_v3", 2: "resnet18", 3: "resnet50", 4: "resnet152"}
    try:
        aid = 1
        for m, name in names.items():
            t = time.time_ns() - w.epoch_ns
            w.on_action(Action(aid, ActionKind.LOAD, m, t, t + 10**11))
            assert int(wait(aid).status) == 1, name
            aid += 1
            for b in (1, 16):
                t = time.time_ns() - w.epoch_ns
                w.on_action(Action(aid, ActionKind.INFER, m, t, t + 10**11, tuple(range(b))))
                r = wait(aid)
                assert int(r.status) == 1 and r.device_duration > 0, (name, b)
                deadline = time.time() + 5
                while aid not in w.outputs and time.time() < deadline:
                    time.sleep(0.005)
                c = resnet_oracle.compare(w.outputs[aid], golden(name)[:b])
                assert c["ok"], (name, b, c)
                aid += 1
    finally:
        w.close()
