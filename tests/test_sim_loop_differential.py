"""B200Worker(mode="sim") and the reference EmulatedWorker on the reference's own SimLoop,
fed the same action stream, emit the same results in the same order.

Unlike tests/test_engine_golden.py (every delivery queued before any engine event), the
deliveries here land on the loop at the same virtual times as engine events (exec / output
/ load completions and wakes on a 0.5 ms grid), so the order in which the loop runs a
delivery against a completion decides which pending action starts: the B200 worker must
schedule one loop callback per engine event, in the reference's loop.call_at order
(worker.py:246, 265, 276, 296). Runs where the read-only reference is mounted.
"""

import os
import random
import sys

import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")

MS = 1_000_000
HALF = MS // 2

# durations on the 0.5 ms grid so completions coincide with deliveries
CATALOG = """\
page_bytes 16777216
model a
weights_bytes 40000000
weights_transfer_ns 1500000
io_ns 500000 500000
io_bytes 602000 4000
batch 1 1000000
batch 2 1500000
batch 4 2000000
model b
weights_bytes 90000000
weights_transfer_ns 2500000
io_ns 500000 1000000
io_bytes 602000 4000
batch 1 500000
batch 2 1000000
batch 4 1500000
replicas b 2
"""


def _stream(seed):
    rng = random.Random(seed)
    out, t = [], 0
    for i in range(rng.randint(20, 120)):
        t += rng.choice([0, 0, HALF, HALF, MS, 2 * MS])
        r = rng.random()
        kind = 3 if r < 0.65 else (1 if r < 0.88 else 2)
        model = rng.randrange(4)
        earliest = max(0, t + rng.choice([-HALF, 0, 0, HALF, MS, 3 * MS]))
        latest = earliest + rng.choice([0, HALF, MS, 2 * MS, 8 * MS, 500 * MS])
        batch = rng.choice([1, 2, 4]) if kind == 3 else 0
        out.append((t, 1 + i, kind, model, earliest, latest, batch))
    return out


def _run(make_worker, ref, stream, pages, io_capacity):
    from sloserve.protocol import Action, ActionKind
    from sloserve.timebase import SimLoop

    loop = SimLoop()
    got = []
    w = make_worker(loop, lambda r: got.append(
        (loop.now(), r.action_id, int(r.status), r.start, r.end, r.device_duration)),
        pages, io_capacity)
    for t, aid, kind, model, lo, hi, b in stream:
        a = Action(aid, ActionKind(kind), model, lo, hi, tuple(range(b)))
        loop.call_at(t, w.on_action, a)
    loop.run_until(10**10)
    if hasattr(w, "close"):
        w.close()
    return got


@pytest.mark.parametrize("seed", range(60))
def test_same_loop_same_results(seed):
    sys.path.insert(0, REF)
    from sloserve.profiles import loads_catalog
    from sloserve.worker import EmulatedWorker

    from paper_2006_02464_b200.worker import B200Worker

    cat = loads_catalog(CATALOG)
    rng = random.Random(1000 + seed)
    pages = rng.choice([3, 6, 12, 40])
    io_capacity = rng.choice([512 * 1024 * 1024, 4 * 606000, 9 * 606000])
    stream = _stream(seed)

    def ref_worker(loop, send, pages, io):
        return EmulatedWorker(0, cat, loop, send, pages_per_gpu=pages, io_capacity=io)

    def b200_worker(loop, send, pages, io):
        return B200Worker(0, cat, loop, send, pages_per_gpu=pages, io_capacity=io, mode="sim")

    ref = _run(ref_worker, None, stream, pages, io_capacity)
    ours = _run(b200_worker, None, stream, pages, io_capacity)
    # (an INFER blocked on the IOCache at the head of the heap can wait forever in the
    # reference, worker.py:237-243: it is never woken; so not every action has a result)
    assert len(ref) >= 10
    assert ours == ref
