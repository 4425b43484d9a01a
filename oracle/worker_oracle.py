"""Action-semantics oracle — TEST INFRASTRUCTURE ONLY.

A CPU restatement of the reference worker's executor semantics
(pkg/src/sloserve/worker.py) with its own discrete-event clock (the SimLoop
contract, pkg/src/sloserve/timebase.py:55-99: events ordered by (time, seq),
past times clamped to now). Pinned against golden traces produced by the real
reference (oracle/make_golden.py -> tests/golden/worker_traces.json).

Rules restated (line numbers into worker.py):
  on_action        198-219  MALFORMED for unknown model / gpu / batch size; Infer
                            acquires IOCache bytes b*(in+out) or queues FIFO, then
                            joins the Infer heap; Load/Unload join the Load heap.
  executor heap    135-146  pending ordered by (earliest, arrival seq); one busy slot.
  window gate      228-248  reject if now > latest; eff = max(earliest, input_done);
                            reject if eff > latest and eff is known; sleep to eff.
  UNLOAD           250-253  release resident pages; SUCCESS, zero duration.
  LOAD             254-267  resident -> SUCCESS 0; reserve fails -> OUT_OF_PAGES;
                            else copy for weights_transfer, commit on completion.
  INFER            268-278  not resident -> MODEL_NOT_LOADED (releases IO); else
                            touch LRU, run exec_duration[b].
  completions      284-305  executor frees at Exec end; Output b*output_transfer
                            later releases IO, drains blocked inputs, reports
                            start = Exec start, end = Output end.
  PageCache        63-99    pages_free = total - resident - in_transit.
  pages_needed     profiles.py:109-111  max(1, ceil(weights / page_bytes)).
"""

from __future__ import annotations

import heapq
import math
from dataclasses import dataclass, field

NEVER = 1 << 62
LOAD, UNLOAD, INFER = 1, 2, 3
SUCCESS, REJECTED, OUT_OF_PAGES, NOT_LOADED, MALFORMED = 1, 2, 3, 4, 5


@dataclass(frozen=True)
class Profile:
    weights_size: int
    weights_transfer: int
    exec_duration: dict
    input_size: int = 0
    output_size: int = 0
    input_transfer: int = 50_000
    output_transfer: int = 50_000

    def pages(self, page_bytes: int) -> int:
        return max(1, math.ceil(self.weights_size / page_bytes))


@dataclass
class Act:
    action_id: int
    kind: int
    model_id: int
    earliest: int
    latest: int
    batch: int = 0
    gpu: int = 0


@dataclass
class _Device:
    total: int
    io_cap: int
    free: int = 0
    held: dict = field(default_factory=dict)       # model -> pages (resident)
    copying: dict = field(default_factory=dict)    # model -> pages (in transit)
    last_use: dict = field(default_factory=dict)
    io_used: int = 0
    io_queue: list = field(default_factory=list)   # FIFO of blocked Infers
    queues: dict = field(default_factory=lambda: {"load": [], "infer": []})
    busy: dict = field(default_factory=lambda: {"load": False, "infer": False})
    wake_at: dict = field(default_factory=lambda: {"load": NEVER, "infer": NEVER})
    arrivals: int = 0


class OracleWorker:
    def __init__(self, profiles: list[Profile], gpu_count: int = 1, pages_per_gpu: int = 500,
                 io_capacity: int = 512 * 1024 * 1024, page_bytes: int = 16 * 1024 * 1024):
        self.profiles = profiles
        self.page_bytes = page_bytes
        self.devices = [_Device(pages_per_gpu, io_capacity, free=pages_per_gpu)
                        for _ in range(gpu_count)]
        self.now = 0
        self._events: list = []
        self._eseq = 0
        self._input_ready: dict[int, int] = {}
        self.results: list[tuple] = []    # (action_id, status, start, end, dur, pages_free)

    # -- event clock
    def at(self, t: int, fn, *args):
        self._eseq += 1
        heapq.heappush(self._events, (max(t, self.now), self._eseq, fn, args))

    def run_until(self, horizon: int):
        while self._events and self._events[0][0] <= horizon:
            t, _, fn, args = heapq.heappop(self._events)
            self.now = t
            fn(*args)
        self.now = max(self.now, horizon)

    def deliver(self, t: int, act: Act):
        self.at(t, self.receive, act)

    # -- semantics
    def _report(self, act: Act, status: int, start: int, end: int, dur: int):
        dev_free = self.devices[act.gpu].free if act.gpu < len(self.devices) else -1
        self.results.append((act.action_id, status, start, end, dur, dev_free))

    def _io_need(self, act: Act) -> int:
        p = self.profiles[act.model_id]
        return act.batch * (p.input_size + p.output_size)

    def receive(self, act: Act):
        t = self.now
        if not (0 <= act.model_id < len(self.profiles)) or act.gpu >= len(self.devices):
            return self._report(act, MALFORMED, t, t, 0)
        dev = self.devices[act.gpu]
        if act.kind == INFER:
            prof = self.profiles[act.model_id]
            if act.batch not in prof.exec_duration:
                return self._report(act, MALFORMED, t, t, 0)
            need = self._io_need(act)
            if dev.io_used + need <= dev.io_cap:
                dev.io_used += need
                self._input_ready[act.action_id] = t + act.batch * prof.input_transfer
            else:
                dev.io_queue.append(act)
            which = "infer"
        else:
            which = "load"
        dev.arrivals += 1
        heapq.heappush(dev.queues[which], (act.earliest, dev.arrivals, act))
        self._dispatch(act.gpu, which)

    def _dispatch(self, g: int, which: str):
        dev = self.devices[g]
        if dev.busy[which]:
            return
        q = dev.queues[which]
        while q:
            t = self.now
            earliest, _, act = q[0]
            if t > act.latest:
                heapq.heappop(q)
                self._too_late(g, act)
                continue
            ready = earliest
            if act.kind == INFER:
                ready = max(ready, self._input_ready.get(act.action_id, NEVER))
            if ready > act.latest:
                if ready >= NEVER:
                    return
                heapq.heappop(q)
                self._too_late(g, act)
                continue
            if ready > t:
                if ready < dev.wake_at[which]:
                    dev.wake_at[which] = ready
                    self.at(ready, self._wake, g, which)
                return
            heapq.heappop(q)
            prof = self.profiles[act.model_id]
            if act.kind == UNLOAD:
                dev.free += dev.held.pop(act.model_id, 0)
                dev.last_use.pop(act.model_id, None)
                self._report(act, SUCCESS, t, t, 0)
                continue
            if act.kind == LOAD:
                if act.model_id in dev.held:
                    dev.last_use[act.model_id] = t
                    self._report(act, SUCCESS, t, t, 0)
                    continue
                need = prof.pages(self.page_bytes)
                if need > dev.free:
                    self._report(act, OUT_OF_PAGES, t, t, 0)
                    continue
                dev.free -= need
                dev.copying[act.model_id] = need
                dev.busy[which] = True
                self.at(t + prof.weights_transfer, self._copied, g, act, t, prof.weights_transfer)
                return
            if act.model_id not in dev.held:
                self._free_io(dev, act)
                self._report(act, NOT_LOADED, t, t, 0)
                continue
            dev.busy[which] = True
            dev.last_use[act.model_id] = t
            d = prof.exec_duration[act.batch]
            self.at(t + d, self._executed, g, act, t, d)
            return

    def _wake(self, g: int, which: str):
        self.devices[g].wake_at[which] = NEVER
        self._dispatch(g, which)

    def _copied(self, g: int, act: Act, start: int, dur: int):
        dev = self.devices[g]
        dev.held[act.model_id] = dev.copying.pop(act.model_id)
        dev.last_use[act.model_id] = self.now
        dev.busy["load"] = False
        self._report(act, SUCCESS, start, self.now, dur)
        self._dispatch(g, "load")

    def _executed(self, g: int, act: Act, start: int, dur: int):
        self.devices[g].busy["infer"] = False
        out = act.batch * self.profiles[act.model_id].output_transfer
        self.at(self.now + out, self._output_done, g, act, start, dur)
        self._dispatch(g, "infer")

    def _output_done(self, g: int, act: Act, start: int, dur: int):
        dev = self.devices[g]
        self._free_io(dev, act)
        admitted = False
        while dev.io_queue:
            head = dev.io_queue[0]
            need = self._io_need(head)
            if dev.io_used + need > dev.io_cap:
                break
            dev.io_used += need
            dev.io_queue.pop(0)
            self._input_ready[head.action_id] = (
                self.now + head.batch * self.profiles[head.model_id].input_transfer)
            admitted = True
        if admitted:
            self._dispatch(g, "infer")
        self._report(act, SUCCESS, start, self.now, dur)

    def _free_io(self, dev: _Device, act: Act):
        if act.action_id in self._input_ready:
            del self._input_ready[act.action_id]
            dev.io_used -= self._io_need(act)
        elif act in dev.io_queue:
            dev.io_queue.remove(act)

    def _too_late(self, g: int, act: Act):
        if act.kind == INFER:
            self._free_io(self.devices[g], act)
        self._report(act, REJECTED, self.now, self.now, 0)

    def pages_state(self, g: int = 0) -> tuple[int, list]:
        dev = self.devices[g]
        return dev.free, sorted(dev.held.items())
