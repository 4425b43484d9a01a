"""Native wire codec (csrc/net.cpp) against the Python codec, which is
itself pinned to the reference's bytes (test_wire_golden.py): identical frames, identical
error classes on malformed input, over the golden frames and a seeded fuzz."""

import json
import os
import random

import pytest

from paper_2006_02464_b200 import native_wire as nw
from paper_2006_02464_b200 import wire
from paper_2006_02464_b200.wire import Action, ActionKind, ActionResult, ResultStatus, \
    WorkerHandshake

FRAMES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "wire_frames.json")))


def _py_decode_payload(p):
    try:
        return wire.decode_payload(p)
    except wire.WireError as e:
        return type(e)


def _nat_decode_payload(p):
    try:
        return nw.decode_action(p)
    except wire.WireError as e:
        return type(e)


@pytest.mark.parametrize("i", range(len(FRAMES)))
def test_golden_frames(i):
    f = FRAMES[i]
    frame = bytes.fromhex(f["hex"])
    msg = wire.decode(frame)
    if isinstance(msg, Action):
        assert nw.decode_action(frame[4:]) == msg
    elif isinstance(msg, ActionResult):
        assert nw.encode_result(msg) == frame
    elif isinstance(msg, WorkerHandshake):
        assert nw.encode_handshake(msg) == frame
    else:  # client-side messages never reach the worker: the native decoder refuses them
        with pytest.raises(wire.BadTag):
            nw.decode_action(frame[4:])


def _rand_action(rng):
    kind = ActionKind(rng.randint(1, 3))
    e = rng.randrange(-2**62, 2**62)
    n = rng.randint(1, 20) if kind == ActionKind.INFER else 0
    return Action(rng.randrange(2**64), kind, rng.randrange(2**32), e, e + rng.randrange(2**20),
                  tuple(rng.randrange(2**64) for _ in range(n)), rng.randrange(2**16),
                  rng.randrange(2**62) if kind == ActionKind.INFER else 0)


def test_fuzz_actions_results_handshakes():
    rng = random.Random(5)
    for _ in range(20_000):
        a = _rand_action(rng)
        got = nw.decode_action(wire.encode(a)[4:])
        if len(a.batch) <= 16:
            assert got == a
        else:  # ids past CW_MAX_BATCH are not carried; the engine answers MALFORMED_ACTION
            assert got.batch_size == len(a.batch) or len(got.batch) == 16
            assert got.batch == a.batch[:16]
        st = ResultStatus(rng.randint(1, 5))
        s = rng.randrange(-2**62, 2**62)
        r = ActionResult(rng.randrange(2**64), st, s, s + rng.randrange(2**20),
                         rng.randrange(2**62) if st == 1 else 0)
        assert nw.encode_result(r) == wire.encode(r)
    for _ in range(2_000):
        h = WorkerHandshake(rng.randrange(2**32), rng.randint(1, 2**31), rng.randrange(1, 2**63),
                            tuple(rng.randrange(2**32) for _ in range(rng.randint(0, 30))))
        assert nw.encode_handshake(h) == wire.encode(h)


def test_malformed_payloads_same_error_class():
    rng = random.Random(9)
    for _ in range(20_000):
        p = bytearray(wire.encode(_rand_action(rng))[4:])
        op = rng.randrange(5)
        if op == 0:
            p = p[:rng.randrange(len(p))]                      # truncation
        elif op == 1:
            p += bytes(rng.randint(1, 9))                       # trailing bytes
        elif op == 2:
            p[9] = rng.choice([0, 4, 5, 255])                   # bad kind
        elif op == 3:
            p[rng.randrange(len(p))] = rng.randrange(256)       # random byte
        else:
            p[0] = rng.choice([0, 1, 3, 4, 5, 6, 255])          # other tags
        ref, nat = _py_decode_payload(bytes(p)), _nat_decode_payload(bytes(p))
        if not p or p[0] != 2:
            # not an Action (or empty): the worker side refuses any other message
            assert nat is (wire.Truncated if not p else wire.BadTag), (bytes(p).hex(), nat)
        elif isinstance(ref, type):
            assert nat is ref, (bytes(p).hex(), ref, nat)
        elif len(ref.batch) <= 16:
            assert nat == ref


def test_result_invariants_refused():
    from paper_2006_02464_b200._lib import cw_result, lib
    import ctypes as C
    buf = C.create_string_buffer(nw.RESULT_FRAME)
    bad = cw_result(action_id=1, status=2, start=0, end=0, device_duration=5)  # non-success dur
    assert lib.cw_wire_encode_result(C.byref(bad), buf) == -3
    bad = cw_result(action_id=1, status=1, start=5, end=4, device_duration=0)  # end < start
    assert lib.cw_wire_encode_result(C.byref(bad), buf) == -3
    bad = cw_result(action_id=1, status=9, start=0, end=0, device_duration=0)  # unknown status
    assert lib.cw_wire_encode_result(C.byref(bad), buf) == -3
