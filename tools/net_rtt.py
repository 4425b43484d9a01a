"""Controller-socket round trip of zero-duration actions (UNLOAD of a non-resident model:
SUCCESS at once) through server.serve, Python vs native serving loop (profiling helper).
usage: net_rtt.py [n] [sim|cuda]"""
import os
import socket
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2006_02464_b200 import catalog, server, wire  # noqa: E402

CAT = "page_bytes 16777216\nmodel resnet50\nweights_bytes 102300000\nweights_transfer_ns 8330000\n" \
      "io_bytes 602000 4000\nbatch 1 2610000\n"
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
mode = sys.argv[2] if len(sys.argv) > 2 else "sim"
for native in (False, True):
    epoch = time.time_ns()
    ports, ready = [], threading.Event()
    t = threading.Thread(target=server.serve, args=("127.0.0.1:0", catalog.parse(CAT)),
                         kwargs=dict(pages_per_gpu=16, epoch_ns=epoch, mode=mode, native=native,
                                     on_ready=lambda p: (ports.append(p), ready.set())),
                         daemon=True)
    t.start()
    ready.wait(30)
    s = socket.create_connection(("127.0.0.1", ports[0]))
    s.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
    wire.recv(s)
    rtt = []
    for i in range(n):
        now = time.time_ns() - epoch
        t0 = time.perf_counter_ns()
        wire.send(s, wire.Action(i, wire.ActionKind.UNLOAD, 0, now, now + 10**9))
        r = wire.recv(s)
        rtt.append(time.perf_counter_ns() - t0)
        assert r.status == wire.ResultStatus.SUCCESS
    s.close()
    t.join(timeout=15)
    a = np.array(rtt[100:]) / 1e3
    print(f"{mode} {'native' if native else 'python'} net: UNLOAD round trip p50 {np.percentile(a, 50):.1f} us, "
          f"p99 {np.percentile(a, 99):.1f} us, p99.9 {np.percentile(a, 99.9):.1f} us, "
          f"max {a.max():.1f} us (n={len(a)})")
