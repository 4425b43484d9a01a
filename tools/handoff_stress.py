"""Layer-handoff race stress (debug helper): INFERs alternating two inputs must reproduce
each input's first logits bit for bit. usage: handoff_stress.py batch iters"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2006_02464_b200 import arch  # noqa: E402
from paper_2006_02464_b200.device import DeviceRuntime  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 16
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
spec = arch.build_arch("resnet50")
blob = arch.pack_blob(spec, arch.fold(spec, arch.make_params(spec, 0)))
xs = [arch.make_inputs(b, spec, first=11 + k * b) for k in range(2)]
with DeviceRuntime(pages_total=8, io_slots=16) as rt:
    rt.register_arch(0, spec, batches=(b,))
    rt.register_blob(0, 0, blob)
    rt.build()
    rt.load(0, list(range(blob.pages)))
    first = [rt.infer(0, 0, x)[0].copy() for x in xs]
    bad = []
    for i in range(iters):
        got, _ = rt.infer(0, 0, xs[i & 1])
        if not np.array_equal(got, first[i & 1]):
            d = np.abs(got - first[i & 1])
            bad.append((i, int((d > 0).sum()), float(d.max())))
print(f"b={b} iters={iters} bad={len(bad)} {bad[:5]}")
