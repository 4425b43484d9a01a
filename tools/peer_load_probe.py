"""Peer LOAD vs host LOAD durations (measurement helper): a 2-GPU-index worker on the given
devices (default [0, 0]: one physical B200, so the peer copy is a device-to-device copy in
HBM; with two devices it goes over NVLink). Prints LOAD device_duration of each kind.
    python tools/peer_load_probe.py [dev0] [dev1]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_peer_load import CAT, Collector, act  # noqa: E402

from paper_2006_02464_b200 import catalog  # noqa: E402
from paper_2006_02464_b200.wire import ActionKind  # noqa: E402
from paper_2006_02464_b200.worker import B200Worker  # noqa: E402

devs = [int(x) for x in sys.argv[1:3]] or [0, 0]
col = Collector()
w = B200Worker(0, catalog.parse(CAT), None, col, gpu_count=2, pages_per_gpu=16, mode="cuda",
               devices=devs, epoch_ns=time.time_ns(), peer_load=True)
host, peer = [], []
aid = 0
for rep in range(10):
    for g, dst in ((0, host), (1, peer)):
        aid += 1
        r = act(w, col, aid, ActionKind.LOAD, 1, g)
        dst.append(r.device_duration / 1e3)
    for g in (1, 0):
        aid += 1
        act(w, col, aid, ActionKind.UNLOAD, 1, g)
w.close()
host.sort()
peer.sort()
print(f"devices {devs}: 51 MB LOAD from host p50 {host[5]:.0f} us, from the peer GPU p50 "
      f"{peer[5]:.0f} us ({51.06e6 / (peer[5] * 1e-6) / 1e9:.0f} GB/s)")
