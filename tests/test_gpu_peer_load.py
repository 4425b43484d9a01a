"""Peer LOAD (`peer_load=True`): a LOAD of a model that another GPU
of the same worker holds resident copies the weights from that GPU's pages
(cudaMemcpyPeerAsync over NVLink) instead of from pinned host memory.

Run here with the worker's two GPU indices mapped onto the one device of the test box
(devices = [g, g]: the peer copy is then a device-to-device copy within one HBM): the source
selection, the header rebuilt for the destination pages, and the source-page fence (the
source GPU may not overwrite pages a peer copy is still reading) are all exercised; only the
NVLink transport itself needs a second GPU."""

import threading
import time

import pytest

from oracle import resnet_oracle
from paper_2006_02464_b200 import arch, catalog
from paper_2006_02464_b200.wire import Action, ActionKind
from paper_2006_02464_b200.worker import B200Worker

pytestmark = pytest.mark.gpu

CAT = """page_bytes 16777216
model resnet50
weights_bytes 102300000
weights_transfer_ns 8330000
io_bytes 602000 4000
batch 1 2610000
batch 8 9130000
replicas resnet50 1
"""


class Collector:
    def __init__(self):
        self.results = {}
        self.cv = threading.Condition()

    def __call__(self, r):
        with self.cv:
            self.results[r.action_id] = r
            self.cv.notify_all()

    def wait(self, aid, timeout=30):
        with self.cv:
            ok = self.cv.wait_for(lambda: aid in self.results, timeout)
        assert ok, f"no result for action {aid}"
        return self.results[aid]


def act(w, col, aid, kind, model, gpu_index, batch=()):
    t = time.time_ns() - w.epoch_ns
    w.on_action(Action(aid, kind, model, t, t + 10**9, tuple(batch), gpu_index))
    return col.wait(aid)


def oracle(first):
    spec = arch.build_arch("resnet50")
    params = arch.make_params(spec, seed=0)
    return resnet_oracle.logits(resnet_oracle.torchvision_model("resnet50", params),
                                arch.make_inputs(8, spec, first=first))


def test_peer_load_copies_from_the_resident_gpu(gpu):
    col = Collector()
    w = B200Worker(0, catalog.parse(CAT), None, col, gpu_count=2, pages_per_gpu=16,
                   mode="cuda", devices=[gpu, gpu], epoch_ns=time.time_ns(), keep_outputs=True,
                   peer_load=True)
    try:
        host = act(w, col, 1, ActionKind.LOAD, 1, 0)      # GPU 0: nothing resident -> host copy
        peer = act(w, col, 2, ActionKind.LOAD, 1, 1)      # GPU 1: model 1 on GPU 0 -> peer copy
        assert int(host.status) == 1 and int(peer.status) == 1
        # 51 MB from HBM vs over the PCIe link (~1 ms): an order of magnitude apart
        assert peer.device_duration * 5 < host.device_duration, (peer, host)
        # the copy on GPU 1 serves INFERs (its header holds GPU 1's own page addresses)
        r = act(w, col, 3, ActionKind.INFER, 1, 1, range(100, 108))
        assert int(r.status) == 1
        time.sleep(0.05)
        c = resnet_oracle.compare(w.outputs[3], oracle(100))
        assert c["ok"], c
        # GPU 0 drops the source copy and reuses its pages for another model (the LOAD waits
        # for the peer copy that read them); both GPUs still compute correct logits
        assert int(act(w, col, 4, ActionKind.UNLOAD, 1, 0).status) == 1
        assert int(act(w, col, 5, ActionKind.LOAD, 0, 0).status) == 1   # host copy (0 nowhere)
        r = act(w, col, 6, ActionKind.INFER, 1, 1, range(200, 208))
        r0 = act(w, col, 7, ActionKind.INFER, 0, 0, range(300, 308))
        assert int(r.status) == 1 and int(r0.status) == 1
        time.sleep(0.05)
        assert resnet_oracle.compare(w.outputs[6], oracle(200))["ok"]
        assert resnet_oracle.compare(w.outputs[7], oracle(300))["ok"]
        assert w.pages(0) == (16 - 7, [(0, 7)]) and w.pages(1) == (16 - 7, [(1, 7)])
    finally:
        w.close()


def test_peer_load_off_by_default_copies_from_host(gpu):
    col = Collector()
    w = B200Worker(0, catalog.parse(CAT), None, col, gpu_count=2, pages_per_gpu=16,
                   mode="cuda", devices=[gpu, gpu], epoch_ns=time.time_ns())
    try:
        a = act(w, col, 1, ActionKind.LOAD, 1, 0)
        b = act(w, col, 2, ActionKind.LOAD, 1, 1)
        assert int(a.status) == 1 and int(b.status) == 1
        # both from host: comparable durations (no D2D shortcut without the option)
        assert b.device_duration * 3 > a.device_duration, (a, b)
    finally:
        w.close()
