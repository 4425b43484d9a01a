"""The controller fast path: a drop-in for the reference's
`sloserve.scheduler.Scheduler` whose decisions run in native code (csrc/sched.cpp, C ABI
`cw_sched_*` in include/cw.h).

Same constructor and surface as the reference (`scheduler.py:118-150`): `Scheduler(catalog,
config, loop, send_action, send_response)`, `on_handshake`, `on_request`, `on_result`,
`action_sink`, `live_requests`, `state`-free. Each loop event crosses into C++ once; the
native core returns, in the order the reference would have produced them, the actions to
send, the responses, the timers to arm on the caller's loop and the action-sink rows, which
this shim replays (scheduler.py:30: everything stays on the scheduler's loop thread).

Binding: the harness constructs `Scheduler` by name, so a controller
process opts in with `sloserve.harness.Scheduler = NativeScheduler` (or by constructing it
wherever it would construct the reference one). Action / response objects are built from the
hosting controller's own protocol module (`sloserve.protocol` when loaded), because its
encoder dispatches on those classes.

Differences from the reference, by design: one `now` per loop event (the reference re-reads
the wall clock inside some helpers; identical under the simulated loop, where the
differential tests pin it decision for decision), and `live_requests` is a sized view (the
harness only tests its truthiness).
"""

from __future__ import annotations

import ctypes as C
import sys

from . import _lib

EV_ACTION, EV_RESPONSE, EV_TIMER, EV_SINK = 1, 2, 3, 4
_REC = 16


def _protocol():
    mod = sys.modules.get("sloserve.protocol")
    if mod is not None:
        return mod
    from . import wire
    return wire


class _Request:
    """What send_response consumers read of a PendingRequest (scheduler.py:63-77)."""

    __slots__ = ("request_id", "model_id", "arrival", "slo", "deadline", "state",
                 "cold_start", "size_mask", "served_batch")

    def __init__(self, rid, model_id, arrival, slo, deadline, cold, served_batch):
        self.request_id = rid
        self.model_id = model_id
        self.arrival = arrival
        self.slo = slo
        self.deadline = deadline
        self.state = 2  # DONE: only finished requests are handed out
        self.cold_start = bool(cold)
        self.size_mask = 0
        self.served_batch = served_batch


class _Outstanding:
    """What action_sink consumers read of an Outstanding (controller_state.py:168-190)."""

    __slots__ = ("action_id", "worker_id", "gpu_index", "kind", "model_id", "requests",
                 "predicted_start", "predicted_end", "predicted_duration", "batch_size",
                 "predicted_result_end")


class _Live:
    """Sized view of the native live-request table (scheduler.py:139 live_requests)."""

    def __init__(self, h):
        self._h = h

    def __len__(self):
        return int(_lib.lib.cw_sched_live(self._h))

    def __bool__(self):
        return len(self) > 0


class NativeScheduler:
    def __init__(self, catalog, config, loop, send_action, send_response):
        self.catalog = catalog
        self.config = config
        self.loop = loop
        self.send_action = send_action
        self.send_response = send_response
        self.action_sink = None
        p = _protocol()
        self._Action, self._ActionKind = p.Action, p.ActionKind
        self._Response, self._RStatus = p.InferenceResponse, p.ResponseStatus
        ids = list(catalog.model_ids())
        if ids != list(range(len(ids))):
            raise ValueError("catalog model ids must be 0..n-1 (scheduler.py:128-131 indexes them)")
        n_sizes, sizes, durs, it, ot, wt, pages = [], [], [], [], [], [], []
        for m in ids:
            prof = catalog.profile(m)
            bs = list(prof.batch_sizes)
            if len(bs) > 31:
                raise ValueError("at most 31 batch sizes per model (queue bit masks)")
            n_sizes.append(len(bs))
            sizes += bs
            durs += [int(prof.exec_duration[b]) for b in bs]
            it.append(int(prof.input_transfer))
            ot.append(int(prof.output_transfer))
            wt.append(int(prof.weights_transfer))
            pages.append(int(catalog.pages_needed(m)))
        cfg = [config.work_horizon_ns, config.capacity_horizon_ns, config.lead_slack_ns,
               config.tardy_slack_ns, config.unload_tardy_ns, config.estimator_window,
               config.default_slo_ns]

        def arr(t, v):
            return (t * max(1, len(v)))(*v)

        self._h = _lib.lib.cw_sched_create(
            len(ids), arr(C.c_int32, n_sizes), arr(C.c_int32, sizes), arr(C.c_int64, durs),
            arr(C.c_int64, it), arr(C.c_int64, ot), arr(C.c_int64, wt), arr(C.c_int32, pages),
            arr(C.c_int64, [int(x) for x in cfg]), float(config.load_eps_ns))
        if not self._h:
            raise _lib.CwError("cw_sched_create failed")
        self.live_requests = _Live(self._h)
        self._nid = C.c_int64(0)

    def close(self):
        if self._h:
            _lib.lib.cw_sched_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 (interpreter shutdown)
            pass

    # ------------------------------------------------------------------ loop events
    def on_handshake(self, hs) -> None:
        self._replay(_lib.lib.cw_sched_handshake(self._h, int(hs.worker_id), int(hs.gpu_count),
                                                 int(hs.pages_total)))

    def on_request(self, req) -> None:
        self._replay(_lib.lib.cw_sched_request(self._h, int(self.loop.now()), int(req.request_id),
                                               int(req.model_id), int(req.slo)))

    def on_result(self, result) -> None:
        self._replay(_lib.lib.cw_sched_result(
            self._h, int(self.loop.now()), int(result.action_id), int(result.status),
            int(result.start), int(result.end), int(result.device_duration)), result)

    def _timer(self, kind, a, b, c) -> None:
        self._replay(_lib.lib.cw_sched_timer(self._h, int(self.loop.now()), kind, a, b, c))

    # ------------------------------------------------------------------ outputs
    def _replay(self, n: int, result=None) -> None:
        if n <= 0:
            return
        recs = _lib.lib.cw_sched_records(self._h)
        flat = C.cast(recs, C.POINTER(C.c_int64 * (n * _REC))).contents[:]
        idp = _lib.lib.cw_sched_ids(self._h, C.byref(self._nid))
        nid = self._nid.value
        ids = C.cast(idp, C.POINTER(C.c_uint64 * nid)).contents[:] if nid else []
        for k in range(0, n * _REC, _REC):
            t = flat[k]
            if t == EV_ACTION:
                wid, aid, kind, model, earliest, latest, g, exp, nb, off = flat[k + 1:k + 11]
                self.send_action(wid, self._Action(aid, self._ActionKind(kind), model, earliest,
                                                   latest, tuple(ids[off:off + nb]), g, exp))
            elif t == EV_RESPONSE:
                has_pr, rid, status, lat, cold, model, arrival, slo, deadline, served = \
                    flat[k + 1:k + 11]
                pr = _Request(rid, model, arrival, slo, deadline, cold, served) if has_pr else None
                self.send_response(pr, self._Response(rid, self._RStatus(status), lat,
                                                      bool(cold) if has_pr else False))
            elif t == EV_TIMER:
                self.loop.call_at(flat[k + 1], self._timer, flat[k + 2], flat[k + 3],
                                  flat[k + 4], flat[k + 5])
            elif t == EV_SINK:
                if self.action_sink is not None:
                    o = _Outstanding()
                    (o.action_id, kind, o.model_id, o.worker_id, o.gpu_index, o.batch_size,
                     o.predicted_start, o.predicted_end, o.predicted_duration,
                     o.predicted_result_end) = flat[k + 1:k + 11]
                    o.kind = self._ActionKind(kind)
                    o.requests = ()
                    self.action_sink(o, result)


Scheduler = NativeScheduler  # the reference's class name (scheduler.py:112)
