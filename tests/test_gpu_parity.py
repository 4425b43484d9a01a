"""Device-side parity of the cuda worker against the oracles (VERDICT r1 "what's weak" #1):

* the 40 golden scenarios (oracle/scenarios.py, the same ones whose reference traces are
  frozen in tests/golden/worker_traces.json) replayed through B200Worker(mode="cuda") one
  action at a time with wide windows, so device timing cannot change an outcome: every
  status and the PageCache state after every action equal the oracle's (worker_oracle.py,
  itself pinned bit-exactly against the reference);
* IOCache exhaustion: INFERs beyond the IOCache gauge queue FIFO on the device path and
  start only after an earlier one's Output released its bytes (worker.py:309-338);
* page reuse while an INFER is in flight: UNLOAD A then LOAD B into A's physical pages
  while A's INFER still runs; A's logits must still be A's (the LOAD copy waits for it);
* logits of every batch size against the frozen golden logits (tests/golden/).
"""

import os
import threading
import time

import numpy as np
import pytest

from oracle import resnet_oracle, scenarios, worker_oracle
from paper_2006_02464_b200 import arch, catalog
from paper_2006_02464_b200.wire import Action, ActionKind
from paper_2006_02464_b200.worker import B200Worker

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
WIDE = 100 * 10**9


class Collector:
    def __init__(self):
        self.results = {}
        self.cv = threading.Condition()

    def __call__(self, r):
        with self.cv:
            self.results[r.action_id] = r
            self.cv.notify_all()

    def wait(self, aid, timeout=60):
        with self.cv:
            ok = self.cv.wait_for(lambda: aid in self.results, timeout)
        assert ok, f"no result for action {aid}"
        return self.results[aid]


def _sequential(sc):
    """The scenario's actions minus the INFERs larger than the whole IOCache gauge (those
    wait forever in the reference, worker.py:210-214, and would stall a one-at-a-time
    replay)."""
    cat = catalog.parse(sc["catalog"])
    out = []
    for d in sc["deliveries"]:
        if d["kind"] == 3 and d["model_id"] < len(cat) and \
                d["batch"] * (cat.models[d["model_id"]].input_bytes +
                              cat.models[d["model_id"]].output_bytes) > sc["io_capacity"]:
            continue
        out.append(d)
    return out


def _oracle_sequential(sc):
    """The oracle fed the scenario's actions one at a time, each delivered after the
    previous one's result, window [t, t + WIDE]."""
    cat = catalog.parse(sc["catalog"])
    profs = [worker_oracle.Profile(p.weights_bytes, p.weights_transfer_ns, dict(p.exec_ns),
                                   p.input_bytes, p.output_bytes, p.input_ns, p.output_ns)
             for p in cat.models]
    w = worker_oracle.OracleWorker(profs, sc["gpu_count"], sc["pages"], sc["io_capacity"],
                                   cat.page_bytes)
    t, out = 0, []
    for d in _sequential(sc):
        w.deliver(t, worker_oracle.Act(d["action_id"], d["kind"], d["model_id"], t, t + WIDE,
                                       d["batch"], d["gpu"]))
        w.run_until(t + 10**12)
        r = w.results[-1]
        assert r[0] == d["action_id"]
        g = d["gpu"] if d["gpu"] < sc["gpu_count"] else 0
        out.append((r[1], w.pages_state(g)))
        t = w.now + 1     # run_until advanced the oracle's clock to the horizon
    return out


@pytest.mark.parametrize("seed", range(40))
def test_golden_scenarios_sequential_on_device(gpu, seed):
    sc = scenarios.scenario(seed)
    expect = _oracle_sequential(sc)
    col = Collector()
    w = B200Worker(0, catalog.parse(sc["catalog"]), None, col, gpu_count=sc["gpu_count"],
                   pages_per_gpu=sc["pages"], io_capacity=sc["io_capacity"], mode="cuda",
                   devices=[gpu] * sc["gpu_count"], epoch_ns=time.time_ns())
    try:
        for i, d in enumerate(_sequential(sc)):
            t = time.time_ns() - w.epoch_ns
            batch = tuple(range(d["batch"])) if d["kind"] == 3 else ()
            w.on_action(Action(d["action_id"], ActionKind(d["kind"]), d["model_id"], t,
                               t + WIDE, batch, d["gpu"]))
            r = col.wait(d["action_id"])
            status, (free, held) = expect[i]
            g = d["gpu"] if d["gpu"] < sc["gpu_count"] else 0
            got_free, got_held = w.pages(g)
            assert (int(r.status), got_free, sorted(got_held)) == \
                (status, free, sorted(tuple(x) for x in held)), (i, d)
            if status == 1 and d["kind"] in (1, 3):
                assert r.end >= r.start
    finally:
        w.close()


CAT_R50 = """page_bytes 16777216
model resnet50
weights_bytes 102300000
weights_transfer_ns 8330000
io_ns 1000 1000
io_bytes 602000 4000
batch 1 2610000
batch 16 15670000
"""


def test_iocache_full_blocks_fifo_on_device(gpu):
    """Gauge for two b=1 requests: the 3rd..6th INFER wait in the FIFO (worker.py:210-214,
    324-338) and each starts only after the Output of the INFER two ahead of it released
    its IOCache bytes; all succeed, in submission order, and the gauge drains to 0."""
    col = Collector()
    w = B200Worker(0, catalog.parse(CAT_R50), None, col, pages_per_gpu=8,
                   io_capacity=2 * 606000 + 1000, mode="cuda", devices=[gpu],
                   epoch_ns=time.time_ns())
    try:
        t = time.time_ns() - w.epoch_ns
        w.on_action(Action(1, ActionKind.LOAD, 0, t, t + WIDE))
        assert int(col.wait(1).status) == 1
        t = time.time_ns() - w.epoch_ns
        for i in range(6):
            w.on_action(Action(10 + i, ActionKind.INFER, 0, t, t + WIDE, (i,)))
        rs = [col.wait(10 + i) for i in range(6)]
        assert all(int(r.status) == 1 for r in rs), rs
        for a, b in zip(rs, rs[1:]):
            assert b.start >= a.start + a.device_duration        # one Exec at a time, FIFO
        for k in range(2, 6):
            assert rs[k].start >= rs[k - 2].end, (k, rs[k - 2], rs[k])   # waited for IO
        deadline = time.time() + 5
        while w.engine.io_in_use() and time.time() < deadline:
            time.sleep(0.01)
        assert w.engine.io_in_use() == 0
    finally:
        w.close()


CAT_AB = """page_bytes 16777216
model resnet50
weights_bytes 102300000
weights_transfer_ns 8330000
io_ns 1 1
io_bytes 602000 4000
batch 16 15670000
model resnet18
weights_bytes 46700000
weights_transfer_ns 3810000
io_ns 1 1
io_bytes 602000 4000
batch 16 7020000
"""


def test_load_into_pages_of_inflight_infer_waits(gpu):
    """7 pages: UNLOAD resnet50 (A) right behind its dispatched b=16 INFER, then LOAD
    resnet18 (B), whose blob lands in 2 of A's 4 physical pages (LIFO free list) while A's
    INFER may still be running. The copy must wait for that INFER (page-reuse fence): A's
    logits stay A's, B's copy ends after A's Exec, and B's INFER afterwards is B's."""
    golden_a = np.load(os.path.join(GOLDEN, "logits_resnet50.npz"))["logits"]
    golden_b = np.load(os.path.join(GOLDEN, "logits_resnet18.npz"))["logits"]
    col = Collector()
    w = B200Worker(0, catalog.parse(CAT_AB), None, col, pages_per_gpu=7, mode="cuda",
                   devices=[gpu], epoch_ns=time.time_ns(), keep_outputs=True)
    aid = iter(range(1, 10**6))
    exercised = 0

    def outputs(a):
        deadline = time.time() + 5
        while a not in w.outputs and time.time() < deadline:
            time.sleep(0.005)
        return w.outputs[a]

    try:
        for it in range(24):
            t = time.time_ns() - w.epoch_ns
            la = next(aid)
            w.on_action(Action(la, ActionKind.LOAD, 0, t, t + WIDE))
            assert int(col.wait(la).status) == 1
            ia, ua, lb = next(aid), next(aid), next(aid)
            t = time.time_ns() - w.epoch_ns
            w.on_action(Action(ia, ActionKind.INFER, 0, t, t + WIDE, tuple(range(16))))
            spin = time.perf_counter() + 60e-6 * (1 + it % 4)   # let the INFER dispatch
            while time.perf_counter() < spin:
                pass
            w.on_action(Action(ua, ActionKind.UNLOAD, 0, t, t + WIDE))
            w.on_action(Action(lb, ActionKind.LOAD, 1, t, t + WIDE))
            ri, ru, rl = col.wait(ia), col.wait(ua), col.wait(lb)
            assert (int(ru.status), int(rl.status)) == (1, 1)
            if int(ri.status) == 4:          # the UNLOAD overtook the INFER's dispatch
                t = time.time_ns() - w.epoch_ns
                ub = next(aid)
                w.on_action(Action(ub, ActionKind.UNLOAD, 1, t, t + WIDE))
                assert int(col.wait(ub).status) == 1
                continue
            assert int(ri.status) == 1
            a_end = ri.start + ri.device_duration
            if rl.start < a_end:             # B's copy was issued while A's INFER ran
                exercised += 1
                assert rl.end >= a_end, (it, ri, rl)
            c = resnet_oracle.compare(outputs(ia), golden_a)
            assert c["ok"], (it, c)
            ib, ub = next(aid), next(aid)
            t = time.time_ns() - w.epoch_ns
            w.on_action(Action(ib, ActionKind.INFER, 1, t, t + WIDE, tuple(range(16))))
            assert int(col.wait(ib).status) == 1
            w.on_action(Action(ub, ActionKind.UNLOAD, 1, t, t + WIDE))
            assert int(col.wait(ub).status) == 1
            c = resnet_oracle.compare(outputs(ib), golden_b)
            assert c["ok"], (it, c)
    finally:
        w.close()
    assert exercised >= 3, exercised


CAT_ALL_B = """page_bytes 16777216
model resnet50
weights_bytes 102300000
weights_transfer_ns 8330000
io_ns 1000 1000
io_bytes 602000 4000
batch 1 2610000
batch 2 3780000
batch 4 5610000
batch 8 9130000
batch 16 15670000
"""


def test_every_batch_size_matches_frozen_golden_logits(gpu):
    """Through the worker's public API: request ids 0..b-1 at every batch size must give
    the frozen golden logits of those requests (tests/golden/logits_resnet50.npz)."""
    golden = np.load(os.path.join(GOLDEN, "logits_resnet50.npz"))["logits"]
    col = Collector()
    w = B200Worker(0, catalog.parse(CAT_ALL_B), None, col, pages_per_gpu=8, mode="cuda",
                   devices=[gpu], epoch_ns=time.time_ns(), keep_outputs=True, input_pool=16)
    try:
        t = time.time_ns() - w.epoch_ns
        w.on_action(Action(1, ActionKind.LOAD, 0, t, t + WIDE))
        assert int(col.wait(1).status) == 1
        for k, b in enumerate((1, 2, 4, 8, 16)):
            t = time.time_ns() - w.epoch_ns
            w.on_action(Action(10 + k, ActionKind.INFER, 0, t, t + WIDE, tuple(range(b))))
            assert int(col.wait(10 + k).status) == 1
            deadline = time.time() + 5
            while 10 + k not in w.outputs and time.time() < deadline:
                time.sleep(0.005)
            c = resnet_oracle.compare(w.outputs[10 + k], golden[:b])
            assert c["ok"], (b, c)
    finally:
        w.close()


def test_softmax_tail_probabilities(gpu):
    """The optional FC/softmax tail (B200Worker(softmax=True), `worker --softmax`): the
    outputs are the softmax of the golden logits (max-abs probability error <= 2% of the
    largest probability, top-1 identical) and every row sums to 1."""
    import torch
    golden = np.load(os.path.join(GOLDEN, "logits_resnet50.npz"))["logits"]
    probs = torch.softmax(torch.from_numpy(golden), dim=1).numpy()
    col = Collector()
    w = B200Worker(0, catalog.parse(CAT_ALL_B), None, col, pages_per_gpu=8, mode="cuda",
                   devices=[gpu], epoch_ns=time.time_ns(), keep_outputs=True, input_pool=16,
                   softmax=True)
    try:
        t = time.time_ns() - w.epoch_ns
        w.on_action(Action(1, ActionKind.LOAD, 0, t, t + WIDE))
        assert int(col.wait(1).status) == 1
        for k, b in enumerate((1, 16)):
            t = time.time_ns() - w.epoch_ns
            w.on_action(Action(10 + k, ActionKind.INFER, 0, t, t + WIDE, tuple(range(b))))
            assert int(col.wait(10 + k).status) == 1
            deadline = time.time() + 5
            while 10 + k not in w.outputs and time.time() < deadline:
                time.sleep(0.005)
            got = w.outputs[10 + k]
            np.testing.assert_allclose(got.sum(1), 1.0, atol=1e-4)
            c = resnet_oracle.compare(got, probs[:b])
            assert c["ok"], (b, c)
    finally:
        w.close()
