"""The B200Worker in cuda mode through its public API (the drop-in boundary):
real LOAD / INFER / UNLOAD on the device, statuses and page accounting identical
to the reference semantics for a timing-independent action sequence, logits
identical (within tolerance) to the CPU oracle, windows enforced on the device."""

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

CAT = """page_bytes 16777216
model resnet50
weights_bytes 102300000
weights_transfer_ns 8330000
io_bytes 602000 4000
batch 1 2610000
batch 2 3780000
batch 4 5610000
batch 8 9130000
batch 16 15670000
replicas resnet50 3
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


@pytest.fixture(scope="module")
def worker(gpu):
    col = Collector()
    w = B200Worker(0, catalog.parse(CAT), None, col, pages_per_gpu=16, mode="cuda",
                   devices=[gpu], epoch_ns=time.time_ns(), keep_outputs=True)
    yield w, col
    w.close()


def now(w):
    return time.time_ns() - w.epoch_ns


def act(w, col, aid, kind, model, batch=(), lo=0, hi=10**9):
    t = now(w)
    w.on_action(Action(aid, kind, model, t + lo, t + hi, tuple(batch), 0))
    return col.wait(aid)


def test_load_infer_unload_pages(worker):
    w, col = worker
    assert w.handshake().pages_total == 16
    r = act(w, col, 1, ActionKind.INFER, 0, (0,))
    assert int(r.status) == 4                       # MODEL_NOT_LOADED
    r = act(w, col, 2, ActionKind.LOAD, 0)
    assert int(r.status) == 1 and r.device_duration > 0 and r.end >= r.start
    assert w.pages() == (16 - 7, [(0, 7)])          # 102.3 MB -> 7 pages (profiles.py:109-111)
    r = act(w, col, 3, ActionKind.LOAD, 0)
    assert int(r.status) == 1 and r.device_duration == 0   # already resident
    r = act(w, col, 4, ActionKind.LOAD, 1)
    assert int(r.status) == 1
    r = act(w, col, 5, ActionKind.LOAD, 2)
    assert int(r.status) == 3                       # OUT_OF_PAGES (2 free < 7)
    r = act(w, col, 6, ActionKind.INFER, 1, range(16))
    assert int(r.status) == 1 and r.device_duration > 0
    r = act(w, col, 7, ActionKind.UNLOAD, 0)
    assert int(r.status) == 1 and w.pages() == (9, [(1, 7)])
    r = act(w, col, 8, ActionKind.UNLOAD, 0)
    assert int(r.status) == 1                       # idempotent
    r = act(w, col, 9, ActionKind.INFER, 0, (0, 1, 2))
    assert int(r.status) == 5                       # batch 3 not in the profile
    r = act(w, col, 10, ActionKind.INFER, 7, (0,))
    assert int(r.status) == 5                       # unknown model


def test_windows_enforced(worker):
    w, col = worker
    act(w, col, 20, ActionKind.LOAD, 1)
    t = now(w)
    w.on_action(Action(21, ActionKind.INFER, 1, t - 10**9, t - 5 * 10**8, (0,), 0))
    assert int(col.wait(21).status) == 2            # latest already passed
    t = now(w)
    w.on_action(Action(22, ActionKind.INFER, 1, t + 30_000_000, t + 10**9, (0,), 0))
    r = col.wait(22)
    assert int(r.status) == 1 and r.start >= t + 30_000_000


def test_infer_logits_match_oracle(worker):
    w, col = worker
    act(w, col, 30, ActionKind.LOAD, 1)
    rids = list(range(40, 48))
    r = act(w, col, 31, ActionKind.INFER, 1, rids)
    assert int(r.status) == 1
    time.sleep(0.05)
    got = w.outputs[31]
    spec = arch.build_arch("resnet50")
    params = arch.make_params(spec, seed=0)
    ref = resnet_oracle.logits(resnet_oracle.torchvision_model("resnet50", params),
                               arch.make_inputs(8, spec, first=40))
    c = resnet_oracle.compare(got, ref)
    assert c["ok"], c


def test_back_to_back_infers_serialize(worker):
    w, col = worker
    act(w, col, 50, ActionKind.LOAD, 1)
    t = now(w)
    for i in range(20):
        w.on_action(Action(100 + i, ActionKind.INFER, 1, t, t + 10**9, tuple(range(4)), 0))
    rs = sorted((col.wait(100 + i) for i in range(20)), key=lambda r: r.start)
    assert all(int(r.status) == 1 for r in rs)
    for a, b in zip(rs, rs[1:]):
        assert b.start >= a.start + a.device_duration   # one Exec at a time


def test_device_gate_window(gpu):
    spec = arch.build_arch("resnet18")
    blob = arch.pack_blob(spec, arch.fold(spec, arch.make_params(spec, 1)))
    with DeviceRuntime(device=gpu, pages_total=4, io_slots=4) as rt:
        rt.register_arch(0, spec, batches=(1,))
        rt.register_blob(0, 0, blob)
        rt.build()
        rt.load(0, [0, 1])
        rt.infer(0, 0, arch.make_inputs(1, spec))
        off = rt.clock_offset
        t = time.time_ns() + off
        rej, t0, t1 = rt.exec_window(0, 1, 0, t + 5_000_000, t + 10**9)
        assert not rej and t0 >= t + 5_000_000 and t1 > t0
        t = time.time_ns() + off
        rej, t0, t1 = rt.exec_window(0, 1, 0, 0, t - 10**6)
        assert rej


def test_native_net_server_cuda(gpu, tmp_path):
    """The controller socket served by cw_net_serve (csrc/net.cpp) on the cuda engine: a raw
    client speaks the wire format (handshake, LOAD, INFERs, UNLOAD) and gets the same
    statuses as through the Python path, with real device durations."""
    import socket

    from paper_2006_02464_b200 import server, wire

    epoch = time.time_ns()
    ports, ready = [], threading.Event()
    t = threading.Thread(target=server.serve, args=("127.0.0.1:0", catalog.parse(CAT)),
                         kwargs=dict(pages_per_gpu=16, epoch_ns=epoch, mode="cuda",
                                     devices=[gpu], telemetry_path=str(tmp_path / "w.csv"),
                                     native=True,
                                     on_ready=lambda p: (ports.append(p), ready.set())),
                         daemon=True)
    t.start()
    assert ready.wait(120)
    s = socket.create_connection(("127.0.0.1", ports[0]))
    hs = wire.recv(s)
    assert isinstance(hs, wire.WorkerHandshake) and hs.pages_total == 16

    def run(aid, kind, model, batch=(), lo=0, hi=10**9):
        t0 = time.time_ns() - epoch
        wire.send(s, Action(aid, kind, model, t0 + lo, t0 + hi, tuple(batch), 0,
                            1 if kind == ActionKind.INFER else 0))
        r = wire.recv(s)
        assert r.action_id == aid
        return r

    assert run(1, ActionKind.INFER, 0, (1,)).status == wire.ResultStatus.MODEL_NOT_LOADED
    r = run(2, ActionKind.LOAD, 0)
    assert r.status == wire.ResultStatus.SUCCESS and r.device_duration > 0
    for aid, b in ((3, 1), (4, 16), (5, 8)):
        r = run(aid, ActionKind.INFER, 0, tuple(range(b)))
        assert r.status == wire.ResultStatus.SUCCESS and 0 < r.device_duration < 5_000_000
    assert run(6, ActionKind.INFER, 0, (1, 2, 3)).status == wire.ResultStatus.MALFORMED_ACTION
    assert run(7, ActionKind.INFER, 0, (1,), lo=-2, hi=-1).status == \
        wire.ResultStatus.REJECTED_TOO_LATE
    assert run(8, ActionKind.UNLOAD, 0).status == wire.ResultStatus.SUCCESS
    s.close()
    t.join(timeout=30)
    rows = open(tmp_path / "w.csv").read().splitlines()
    assert len(rows) == 1 + 8


def test_worker_serves_model_artifact(gpu, tmp_path):
    """Weights from a .cwm model artifact (artifact.py) instead of the built-in random init:
    the served logits are the oracle's for the artifact's parameters."""
    from paper_2006_02464_b200 import artifact

    spec = arch.build_arch("resnet50")
    params = arch.make_params(spec, seed=7)
    artifact.save(str(tmp_path / "resnet50.cwm"), "resnet50",
                  artifact.from_state_dict("resnet50", params))
    col = Collector()
    w = B200Worker(0, catalog.parse(CAT), None, col, pages_per_gpu=16, mode="cuda",
                   devices=[gpu], epoch_ns=time.time_ns(), keep_outputs=True,
                   weights_dir=str(tmp_path))
    try:
        assert int(act(w, col, 1, ActionKind.LOAD, 0).status) == 1
        assert int(act(w, col, 2, ActionKind.INFER, 0, range(8, 12)).status) == 1
        time.sleep(0.05)
        got = w.outputs[2]
    finally:
        w.close()
    ref = resnet_oracle.logits(resnet_oracle.torchvision_model("resnet50", params),
                               arch.make_inputs(4, spec, first=8))
    c = resnet_oracle.compare(got, ref)
    assert c["ok"], c
