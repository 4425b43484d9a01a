"""Exec-time tail of back-to-back INFERs (profiling helper): top outliers and their indices."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2006_02464_b200 import arch  # noqa: E402
from paper_2006_02464_b200.device import DeviceRuntime  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
copies = int(sys.argv[3]) if len(sys.argv) > 3 else 100
spec = arch.build_arch("resnet50")
blob = arch.pack_blob(spec, arch.fold(spec, arch.make_params(spec, 0)))
with DeviceRuntime(pages_total=copies * blob.pages, io_slots=16) as rt:
    rt.register_arch(0, spec, batches=(b,))
    rt.register_blob(0, 0, blob)
    rt.build()
    for c in range(copies):
        rt.load(0, list(range(c * blob.pages, (c + 1) * blob.pages)))
    rt.infer(0, 0, arch.make_inputs(b, spec))
    rng = np.random.default_rng(1)
    for rep in range(3):
        hp = [int(c) * blob.pages for c in rng.integers(0, copies, n)]
        ex, wall = rt.exec_many(0, b, hp)
        ex = ex / 1e3
        top = np.argsort(ex)[-6:][::-1]
        print(f"rep {rep}: p50 {np.median(ex):.1f} p99 {np.percentile(ex, 99):.1f} "
              f"p99.99 {np.percentile(ex, 99.99):.1f} max {ex.max():.1f} us; top (index, us): "
              + ", ".join(f"({i}, {ex[i]:.0f})" for i in top))
