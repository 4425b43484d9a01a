"""TCP worker server: the process entry the reference controller connects to.

Same contract as `run_worker_server` (pkg/src/sloserve/harness.py:525-575):
accept one controller connection, send the WorkerHandshake first, then read
Action frames and write ActionResult frames (lock-guarded), and flush a
telemetry CSV on EOF. Differences: the worker id is configurable (the
reference hard-codes 0, harness.py:550, so two external workers collide in
the controller), and the worker is the B200Worker (cuda by default).
"""

from __future__ import annotations

import csv
import os
import socket
import threading
import time

from . import wire
from .timebase import WallClock
from .worker import DEFAULT_IO_CAPACITY, B200Worker, WorkerActionRecord

TELEMETRY_HEADER = ["action_id", "kind", "model_id", "gpu", "batch_size", "status", "start_ns",
                    "end_ns", "device_duration_ns"]


class _EpochOnly:
    """Loop stand-in: the worker only needs the shared epoch (a cuda worker's executor runs
    on the engine thread; a sim worker is driven in wall time from its engine's queue)."""

    def __init__(self, clock: WallClock):
        self.clock = clock

    def now(self) -> int:
        return self.clock.now()


def serve(listen: str, catalog, gpu_count: int = 1, pages_per_gpu: int = 500, jitter=None,
          seed: int = 0, epoch_ns: int | None = None, telemetry_path: str = "",
          io_capacity: int = DEFAULT_IO_CAPACITY, ready_fd: int | None = None, *,
          worker_id: int = 0, devices=None, mode: str = "cuda", weights_seed: int = 0,
          on_ready=None, native: bool = False, weights_dir: str | None = None,
          softmax: bool = False, peer_load: bool = False) -> None:
    """native=True: after the accept, the connection is served by cw_net_serve (csrc/net.cpp):
    frames are decoded into the engine and results encoded back in native threads, with no
    Python on the per-action path."""
    host, port = listen.rsplit(":", 1)
    lsock = socket.socket()
    lsock.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
    lsock.bind((host, int(port)))
    lsock.listen(1)
    bound = lsock.getsockname()[1]
    clock = WallClock(epoch_ns)
    loop = _EpochOnly(clock)
    wlock = threading.Lock()
    conn_box: dict = {}
    pending = {"n": 0}
    done = threading.Condition()

    def send_result(result):
        with wlock:
            c = conn_box.get("conn")
            if c is not None:
                try:
                    wire.send(c, result)
                except OSError:
                    pass
        with done:
            pending["n"] -= 1
            done.notify_all()

    # Build the worker (weights, graphs) before announcing readiness.
    worker = B200Worker(worker_id, catalog, loop, send_result, gpu_count=gpu_count,
                        pages_per_gpu=pages_per_gpu, io_capacity=io_capacity, jitter=jitter,
                        seed=seed, keep_records=bool(telemetry_path), mode=mode, devices=devices,
                        weights_seed=weights_seed, epoch_ns=clock.epoch_ns,
                        poll_results=not native, weights_dir=weights_dir, softmax=softmax,
                        peer_load=peer_load)
    if ready_fd is not None:
        os.write(ready_fd, f"{bound}\n".encode())
        os.close(ready_fd)
    if on_ready is not None:
        on_ready(bound)
    conn, _ = lsock.accept()
    conn.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
    if native:
        _serve_native(worker, conn, lsock, clock, loop, mode, telemetry_path)
        return
    with wlock:
        conn_box["conn"] = conn
        wire.send(conn, worker.handshake())
    try:
        while True:
            try:
                msg = wire.recv(conn)
            except (OSError, wire.WireError):
                break
            if msg is None:
                break
            with done:
                pending["n"] += 1
            worker.on_action(msg)
    finally:
        deadline = time.monotonic() + 2.0
        with done:
            while pending["n"] > 0 and time.monotonic() < deadline:
                done.wait(timeout=0.05)
        with wlock:
            conn_box["conn"] = None
        conn.close()
        lsock.close()
        try:
            worker.close()
        finally:
            if telemetry_path:
                _write_telemetry(telemetry_path, worker.records)


def _serve_native(worker, conn, lsock, clock, loop, mode, telemetry_path) -> None:
    import ctypes as C

    from . import native_wire
    from ._lib import check, cw_net_record, lib

    hs = native_wire.encode_handshake(worker.handshake())
    cap = 1 << 20 if telemetry_path else 0
    recs = (cw_net_record * cap)() if cap else None
    n_recs, n_act = C.c_int64(0), C.c_int64(0)
    try:
        if mode != "cuda":
            worker.detach_driver()  # the native loop drives the sim engine from here on
        check(lib.cw_net_serve(worker.engine.h, conn.fileno(), hs, len(hs), clock.epoch_ns, recs,
                               cap, C.byref(n_recs), C.byref(n_act)), "net_serve")
    finally:
        conn.close()
        lsock.close()
        try:
            worker.close()
        finally:
            if telemetry_path:
                rows = [WorkerActionRecord(r.action_id, r.kind, r.model_id, r.gpu_index,
                                           r.batch_size, r.status, r.start, r.end,
                                           r.device_duration) for r in recs[:n_recs.value]]
                _write_telemetry(telemetry_path, rows)


def _write_telemetry(path: str, records) -> None:
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(TELEMETRY_HEADER)
        for r in list(records):
            w.writerow([r.action_id, r.kind, r.model_id, r.gpu_index, r.batch_size, r.status,
                        r.start, r.end, r.device_duration])
