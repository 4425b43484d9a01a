"""Python view of the native wire codec (csrc/net.cpp): the same frames as wire.py, built
and parsed in C for the native serving loop (server.serve(native=True)). Used by the tests
to hold the two codecs to identical bytes and identical error classes."""

from __future__ import annotations

import ctypes as C

from . import wire
from ._lib import cw_action, cw_result, lib

RESULT_FRAME = 38
_ERR = {-1: wire.Truncated, -2: wire.BadTag, -3: wire.Invalid}


def decode_action(payload: bytes) -> wire.Action:
    """Payload (tag byte onwards) -> Action; raises the wire.py error class on failure."""
    a = cw_action()
    rc = lib.cw_wire_decode_action(payload, len(payload), C.byref(a))
    if rc:
        raise _ERR.get(rc, wire.WireError)(f"native decode: {rc}")
    n = a.batch_size
    ids = tuple(a.request_ids[i] for i in range(min(n, len(a.request_ids))))
    return wire.Action(a.action_id, wire.ActionKind(a.kind), a.model_id, a.earliest, a.latest,
                       ids, a.gpu_index, a.expected_duration)


def encode_result(r: wire.ActionResult) -> bytes:
    c = cw_result(action_id=r.action_id, status=int(r.status), kind=0, start=r.start, end=r.end,
                  device_duration=r.device_duration, output_ref=-1, pages_free=0)
    buf = C.create_string_buffer(RESULT_FRAME)
    rc = lib.cw_wire_encode_result(C.byref(c), buf)
    if rc < 0:
        raise _ERR.get(rc, wire.WireError)(f"native encode: {rc}")
    return buf.raw[:rc]


def encode_handshake(h: wire.WorkerHandshake) -> bytes:
    ids = tuple(h.models_resident)
    arr = (C.c_uint32 * max(1, len(ids)))(*ids)
    cap = 25 + 4 * len(ids)
    buf = C.create_string_buffer(cap)
    n = lib.cw_wire_encode_handshake(h.worker_id, h.gpu_count, h.pages_total, arr, len(ids), buf,
                                     cap)
    if n < 0:
        raise _ERR.get(n, wire.WireError)(f"native encode: {n}")
    return buf.raw[:n]
