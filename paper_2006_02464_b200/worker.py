"""B200Worker: drop-in replacement for the reference EmulatedWorker.

Same constructor, `handshake()`, `on_action(action)` and asynchronous
`send_result(ActionResult)` contract as pkg/src/sloserve/worker.py:160-219,
so it can be constructed wherever the reference builds an EmulatedWorker
(harness.py:409-421 in-thread TCP servers, 479-491 in-process wall mode,
550-561 `run_worker_server`), or served over TCP by `server.serve`.

The executor semantics run natively in libcw (csrc/engine.cpp); this class
only marshals actions in and results out.

modes
  "cuda" (default)  real device work on one B200 per gpu_index: LOAD = paged
                    H2D copy of the model's weights, INFER = CUDA-graph forward
                    of the real network on the request inputs, Input/Output =
                    real copies through the IOCache. Wall clock = time.time_ns()
                    minus the loop's epoch (timebase.py:45-52).
  "sim"             the same engine with a virtual clock and the catalog's
                    profiled durations, driven by a reference-style SimLoop
                    (no GPU). Status / page accounting is bit-exact with the
                    reference (tests/test_engine_golden.py).
"""

from __future__ import annotations

import ctypes as C
import functools
import os
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import arch as arch_mod
from . import catalog as catalog_mod
from ._lib import CwError, MAX_BATCH, check, cw_action, cw_engine_config, cw_model_info, \
    cw_result, lib
from .device import DeviceRuntime
from .wire import ActionResult, ResultStatus, WorkerHandshake

DEFAULT_PAGES_PER_GPU = 500
DEFAULT_IO_CAPACITY = 512 * 1024 * 1024


@dataclass
class WorkerActionRecord:
    """Worker telemetry row (same fields as worker.py:120-132)."""
    action_id: int
    kind: int
    model_id: int
    gpu_index: int
    batch_size: int
    status: int
    start: int
    end: int
    device_duration: int


def _as_catalog(catalog) -> catalog_mod.Catalog:
    if isinstance(catalog, catalog_mod.Catalog):
        return catalog
    if hasattr(catalog, "entries"):          # reference ModelCatalog
        return catalog_mod.from_reference(catalog)
    raise TypeError(f"unsupported catalog type {type(catalog).__name__}")


class Engine:
    """Thin owner of a cw_engine handle."""

    def __init__(self, cat: catalog_mod.Catalog, *, mode: str, worker_id: int, gpu_count: int,
                 pages_per_gpu: int, io_capacity: int, epoch_ns: int = 0, devices=None,
                 io_slots: int = 0, in_bytes_max: int = 3 * 224 * 224 * 4,
                 out_bytes_max: int = 4000, peer_load: bool = False):
        self.cat = cat
        bases = cat.bases()
        self.base_index = {b: i for i, b in enumerate(bases)}
        models = (cw_model_info * max(1, len(cat)))()
        for mid, (prof, base) in enumerate(zip(cat.models, cat.base)):
            m = models[mid]
            bi = self.base_index[base]
            m.blob_id = bi if mode == "cuda" else -1
            m.arch_id = bi
            m.pages_needed = cat.pages_needed(mid)
            bs = prof.batch_sizes
            if len(bs) > 8:
                raise CwError(f"model {prof.name}: more than 8 batch sizes")
            if mode == "cuda" and bs[-1] > MAX_BATCH:
                raise CwError(f"model {prof.name}: batch size {bs[-1]} > {MAX_BATCH}")
            m.n_batches = len(bs)
            for i, b in enumerate(bs):
                m.batch_sizes[i] = b
                m.exec_ns[i] = prof.exec_ns[b]
            m.weights_transfer_ns = prof.weights_transfer_ns
            m.input_size, m.output_size = prof.input_bytes, prof.output_bytes
            m.input_transfer_ns, m.output_transfer_ns = prof.input_ns, prof.output_ns
        self._models = models
        self._devices = (C.c_int32 * gpu_count)(*(devices or range(gpu_count)))
        cfg = cw_engine_config()
        cfg.mode = 1 if mode == "cuda" else 0
        cfg.worker_id = worker_id
        cfg.gpu_count = gpu_count
        cfg.n_models = len(cat)
        cfg.pages_per_gpu = pages_per_gpu
        cfg.page_bytes = cat.page_bytes
        cfg.io_capacity = io_capacity
        cfg.epoch_ns = epoch_ns
        cfg.devices = self._devices
        cfg.peer_load = 1 if peer_load else 0
        cfg.models = models
        cfg.io_slots = io_slots
        cfg.in_bytes_max = in_bytes_max
        cfg.out_bytes_max = out_bytes_max
        cfg.executor_cpu, cfg.executor_rt_prio = -1, 0
        if mode == "cuda":  # one pinned (real-time if allowed) executor thread
            cpus = sorted(os.sched_getaffinity(0))
            first = (devices or [0])[0]
            cfg.executor_cpu = cpus[(2 * first + 1) % len(cpus)] if len(cpus) > 1 else -1
            cfg.executor_rt_prio = 10
        self.h = lib.cw_engine_open(C.byref(cfg))
        if not self.h:
            raise CwError(f"cw_engine_open: {lib.cw_last_error().decode()}")
        self._res = (cw_result * 256)()
        self._new_t = (C.c_int64 * 64)()
        self._new_s = (C.c_uint64 * 64)()

    STAT_NAMES = ("dispatched", "host_late", "host_eff_late", "gate_late", "done",
                  "dispatch_delay_sum_ns", "dispatch_delay_max_ns", "gate_late_sum_ns",
                  "gate_late_max_ns", "start_slack_min_ns", "busy_gap_sum_ns",
                  "busy_gap_max_ns", "busy_gaps", "launch_lat_sum_ns", "launch_lat_max_ns",
                  "observe_lat_sum_ns", "observe_lat_max_ns", "clock_resyncs",
                  "clock_step_max_ns")

    def stats(self, gpu: int = 0) -> dict:
        out = (C.c_int64 * 32)()
        n = check(lib.cw_engine_stats(self.h, gpu, out, 32), "stats")
        return dict(zip(self.STAT_NAMES, out[:n]))

    def clock_drift(self, gpu: int = 0) -> int:
        d = C.c_int64()
        check(lib.cw_engine_clock_drift(self.h, gpu, C.byref(d)), "clock_drift")
        return d.value

    def executor_info(self) -> dict:
        cpu, rt = C.c_int32(), C.c_int32()
        lib.cw_engine_executor_info(self.h, C.byref(cpu), C.byref(rt))
        return {"cpu": cpu.value, "sched_fifo": bool(rt.value)}

    def runtime(self, gpu: int) -> DeviceRuntime:
        h = lib.cw_engine_runtime(self.h, gpu)
        if not h:
            raise CwError("engine has no device runtime (sim mode?)")
        return DeviceRuntime(handle=h, page_bytes=self.cat.page_bytes)

    def start(self):
        check(lib.cw_engine_start(self.h), "engine start")

    def close(self):
        if self.h:
            lib.cw_engine_close(self.h)
            self.h = None

    @staticmethod
    def _action(action) -> cw_action:
        a = cw_action()
        a.action_id = action.action_id
        a.kind = int(action.kind)
        a.model_id = action.model_id & 0xFFFFFFFF
        a.gpu_index = action.gpu_index
        batch = tuple(action.batch)
        a.batch_size = len(batch)
        for i, r in enumerate(batch[:MAX_BATCH]):
            a.request_ids[i] = r
        a.earliest = action.earliest
        a.latest = action.latest
        a.expected_duration = getattr(action, "expected_duration", 0)
        return a

    def submit(self, action, at: int = 0):
        check(lib.cw_engine_submit(self.h, C.byref(self._action(action)), at), "submit")

    def sim_deliver(self, action, now: int):
        check(lib.cw_engine_sim_deliver(self.h, C.byref(self._action(action)), now), "sim_deliver")

    def sim_take_new(self) -> list[tuple[int, int]]:
        out = []
        while True:
            n = lib.cw_engine_sim_take_new(self.h, self._new_t, self._new_s, len(self._new_t))
            out += [(self._new_t[i], self._new_s[i]) for i in range(n)]
            if n < len(self._new_t):
                return out

    def sim_run_to(self, t: int, seq: int) -> int:
        return lib.cw_engine_sim_run_to(self.h, t, seq)

    def failed(self) -> bool:
        return bool(self.h) and lib.cw_engine_failed(self.h) == 1

    def poll(self, timeout_us: int = 0) -> list[tuple]:
        n = lib.cw_engine_poll(self.h, self._res, len(self._res), timeout_us)
        if n < 0:
            raise CwError(f"engine failed: {lib.cw_last_error().decode()}")
        return [(r.action_id, r.status, r.start, r.end, r.device_duration, r.output_ref,
                 r.pages_free, r.kind) for r in self._res[:n]]

    def sim_run(self, until: int) -> int:
        return lib.cw_engine_sim_run(self.h, until)

    def next_time(self) -> int:
        return lib.cw_engine_next_time(self.h)

    def pages(self, gpu: int = 0) -> tuple[int, list[tuple[int, int]]]:
        free = C.c_int64()
        n = C.c_int32()
        cap = len(self.cat) + 1
        ms = (C.c_int32 * cap)()
        ps = (C.c_int32 * cap)()
        check(lib.cw_engine_pages(self.h, gpu, C.byref(free), ms, ps, cap, C.byref(n)), "pages")
        return free.value, [(ms[i], ps[i]) for i in range(min(n.value, cap))]

    def io_in_use(self, gpu: int = 0) -> int:
        return lib.cw_engine_io_in_use(self.h, gpu)

    def output(self, gpu: int, ref: int, batch: int, classes: int = 1000) -> np.ndarray:
        out = np.empty((batch, classes), np.float32)
        check(lib.cw_engine_output(self.h, gpu, ref, out.ctypes.data, batch, classes), "output")
        return out


@functools.lru_cache(maxsize=8)
def _random_init_blob(base: str, seed: int, page_bytes: int):
    """Folded, paged blob of the deterministic random-init weights of an arch (shared by
    every worker of the process; the blob is read-only once packed)."""
    spec = arch_mod.build_arch(base)
    return arch_mod.pack_blob(spec, arch_mod.fold(spec, arch_mod.make_params(spec, seed=seed)),
                              page_bytes=page_bytes)


class _WallDriver:
    """Runs a sim-mode engine in wall time when the caller supplies no event loop (the TCP
    server): the engine's own timer queue is the schedule; one thread sleeps until the next
    engine event is close, spins to it, runs the engine up to now and hands the results out
    (outside the lock: send_result may block on a socket)."""

    SPIN_NS = 150_000

    def __init__(self, engine: Engine, now, deliver):
        self.engine, self.now, self.deliver = engine, now, deliver
        self.cv = threading.Condition()
        self.stopped = False
        self.thread = threading.Thread(target=self._run, name="b200-sim-wall", daemon=True)
        self.thread.start()

    def on_action(self, action):
        with self.cv:
            self.engine.sim_deliver(action, self.now())
            self.engine.sim_take_new()
            res = self.engine.poll(0)
            self.cv.notify()
        self.deliver(res)

    def _run(self):
        while True:
            with self.cv:
                if self.stopped:
                    return
                nt, now = self.engine.next_time(), self.now()
                if nt < 0 or nt - now > self.SPIN_NS:
                    self.cv.wait(0.05 if nt < 0 else (nt - now - self.SPIN_NS) / 1e9)
                    continue
            while self.now() < nt:
                pass
            with self.cv:
                self.engine.sim_run(self.now())
                self.engine.sim_take_new()
                res = self.engine.poll(0)
            self.deliver(res)

    def stop(self):
        with self.cv:
            self.stopped = True
            self.cv.notify()
        if self.thread is not threading.current_thread():
            self.thread.join(timeout=2.0)


class B200Worker:
    """Constructor arguments mirror EmulatedWorker (worker.py:164-168); the
    keyword-only tail selects the device side."""

    def __init__(self, worker_id: int, catalog, loop, send_result, gpu_count: int = 1,
                 pages_per_gpu: int = DEFAULT_PAGES_PER_GPU,
                 io_capacity: int = DEFAULT_IO_CAPACITY, jitter=None, seed: int = 0,
                 keep_records: bool = True, *, mode: str = "cuda", devices=None,
                 weights_seed: int = 0, input_pool: int = 64, epoch_ns: int | None = None,
                 keep_outputs: bool = False, poll_results: bool = True,
                 weights_dir: str | None = None, softmax: bool = False,
                 peer_load: bool = False):
        """peer_load (cuda, gpu_count > 1): a LOAD of a model another GPU of this worker holds
        copies the weights from that GPU over NVLink instead of from host memory (SURVEY.md
        §8f rank 3; off by default, see include/cw.h cw_engine_config.peer_load)."""
        if mode not in ("cuda", "sim"):
            raise ValueError(f"mode must be 'cuda' or 'sim', not {mode!r}")
        if jitter is not None and getattr(jitter, "kind", "none") != "none" and \
                getattr(jitter, "sigma", 0.0) != 0.0:
            raise ValueError("jitter injection is an emulation feature; the B200 worker's "
                             "durations are measured on the device")
        self.worker_id = worker_id
        self.catalog = _as_catalog(catalog)
        self.loop = loop
        self.send_result = send_result
        self.gpu_count = gpu_count
        self.pages_per_gpu = pages_per_gpu
        self.mode = mode
        self.keep_records = keep_records
        self.records: list[WorkerActionRecord] = []
        self.outputs: dict[int, np.ndarray] = {}
        self.keep_outputs = keep_outputs
        self._actions: dict[int, tuple] = {}
        self._lock = threading.Lock()
        self._closed = False
        self.failure: str | None = None
        self._driver: _WallDriver | None = None
        cat = self.catalog
        specs = {}
        if mode == "cuda":
            for base in cat.bases():
                # (raises for unsupported nets); softmax: outputs are class probabilities
                specs[base] = arch_mod.build_arch(base, softmax=softmax)
            in_max = max(s.in_c * s.in_h * s.in_w * 4 for s in specs.values())
            out_max = max(s.classes * 4 for s in specs.values())
            per_req = min([p.input_bytes + p.output_bytes for p in cat.models
                           if p.input_bytes + p.output_bytes > 0] or [in_max + out_max])
            io_slots = min(io_capacity // max(per_req, 1) + MAX_BATCH,
                           io_capacity // (in_max + out_max) + 4 * MAX_BATCH)
            if epoch_ns is None:
                clock = getattr(loop, "clock", None)
                epoch_ns = getattr(clock, "epoch_ns", None)
                if epoch_ns is None:
                    epoch_ns = time.time_ns()
        else:
            in_max, out_max, io_slots = 0, 0, 0
            epoch_ns = 0
        self.epoch_ns = epoch_ns
        self.engine = Engine(cat, mode=mode, worker_id=worker_id, gpu_count=gpu_count,
                             pages_per_gpu=pages_per_gpu, io_capacity=io_capacity,
                             epoch_ns=epoch_ns, devices=devices, io_slots=io_slots,
                             in_bytes_max=in_max, out_bytes_max=out_max, peer_load=peer_load)
        self.specs = specs
        if mode == "cuda":
            blobs = {}
            for base, spec in specs.items():
                if weights_dir:  # model artifacts (artifact.py): <dir>/<arch>.cwm
                    from . import artifact
                    name, blob = artifact.load(os.path.join(weights_dir, f"{base}.cwm"))
                    if name != arch_mod.torchvision_name(base) or blob.page_bytes != cat.page_bytes:
                        raise CwError(f"{base}.cwm: arch {name}, page_bytes {blob.page_bytes} "
                                      f"(catalog: {base}, {cat.page_bytes})")
                    blobs[base] = blob
                    continue
                blobs[base] = _random_init_blob(base, weights_seed, cat.page_bytes)
            # synthetic request inputs per input shape (request id r -> image r % input_pool)
            pools = {}
            for spec in specs.values():
                key = (spec.in_c, spec.in_h, spec.in_w)
                if key not in pools:
                    pools[key] = arch_mod.make_inputs(input_pool, spec)
            for g in range(gpu_count):
                rt = self.engine.runtime(g)
                for base, spec in specs.items():
                    bi = self.engine.base_index[base]
                    batches = sorted({b for p, bb in zip(cat.models, cat.base) if bb == base
                                      for b in p.batch_sizes})
                    rt.register_arch(bi, spec, batches=batches)
                    rt.register_blob(bi, bi, blobs[base])
                    rt.set_input_pool(pools[(spec.in_c, spec.in_h, spec.in_w)], bi)
            self.engine.start()
            # poll_results=False: the results are consumed elsewhere (server.serve(native=True)
            # hands the engine to the native serving loop, csrc/net.cpp)
            self._poller = threading.Thread(target=self._poll_loop, name=f"b200-results-{worker_id}",
                                            daemon=True)
            if poll_results:
                self._poller.start()
        elif not hasattr(loop, "call_at"):
            # no event loop to schedule engine events on (server.py): run them in wall time
            self._driver = _WallDriver(self.engine, loop.now, self._deliver)

    # -- protocol surface (worker.py:193-219)
    def handshake(self) -> WorkerHandshake:
        return WorkerHandshake(self.worker_id, self.gpu_count, self.pages_per_gpu,
                               tuple(self.catalog.model_ids()))

    def on_action(self, action) -> None:
        with self._lock:
            self._actions[action.action_id] = (int(action.kind), action.model_id,
                                               action.gpu_index, len(action.batch))
        if self.mode == "cuda":
            if self.failure is not None:
                raise CwError(f"worker stopped after a device error: {self.failure}")
            self.engine.submit(action)
            return
        if self._driver is not None:
            self._driver.on_action(action)
            return
        self.engine.sim_deliver(action, self.loop.now())
        self._after_engine()

    def detach_driver(self):
        """Stop the wall-time driver: a native loop (csrc/net.cpp) drives the engine now."""
        if self._driver is not None:
            self._driver.stop()

    # -- sim mode: every engine event gets its own callback on the caller's loop, scheduled
    # when the engine schedules it (the reference's loop.call_at order, worker.py:246-296)
    def _after_engine(self):
        self._deliver(self.engine.poll(0))
        for t, seq in self.engine.sim_take_new():
            self.loop.call_at(t, self._run_event, t, seq)

    def _run_event(self, t, seq):
        self.engine.sim_run_to(t, seq)
        self._after_engine()

    # -- cuda mode: results arrive on the engine thread
    def _poll_loop(self):
        while not self._closed:
            try:
                res = self.engine.poll(20_000)
            except CwError as exc:     # a device error stopped the engine: no more results
                self.failure = str(exc)
                return
            if res:
                self._deliver(res)

    def _deliver(self, results):
        for aid, status, start, end, dur, ref, _free, kind in results:
            with self._lock:
                info = self._actions.pop(aid, None)
            if info and self.keep_outputs and ref >= 0 and status == 1:
                self.outputs[aid] = self.engine.output(info[2], ref, info[3])
            if self.keep_records and info:
                self.records.append(WorkerActionRecord(aid, info[0], info[1], info[2], info[3],
                                                       status, start, end, dur))
            self.send_result(ActionResult(aid, ResultStatus(status), start, end, dur))

    def pages(self, gpu: int = 0):
        return self.engine.pages(gpu)

    def close(self):
        self._closed = True
        if self._driver is not None:
            self._driver.stop()
        if self.mode == "cuda" and self._poller.is_alive():
            self._poller.join(timeout=1.0)
        self.engine.close()
