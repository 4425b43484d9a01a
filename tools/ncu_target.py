"""Minimal ncu target: one ResNet-50 copy resident, `reps` graph INFERs of one
batch size on device-resident inputs (profiling helper; run under ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_02464_b200 import arch  # noqa: E402
from paper_2006_02464_b200.device import DeviceRuntime  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
b = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
copies = int(sys.argv[4]) if len(sys.argv) > 4 else 1  # > 2: weights rotate through HBM
spec = arch.build_arch(name)
blob = arch.pack_blob(spec, arch.fold(spec, arch.make_params(spec, 0)))
with DeviceRuntime(pages_total=copies * blob.pages, io_slots=16,
                   in_bytes_max=spec.in_c * spec.in_h * spec.in_w * 4) as rt:
    rt.register_arch(0, spec, batches=(b,))
    rt.register_blob(0, 0, blob)
    rt.build()
    for c in range(copies):
        rt.load(0, list(range(c * blob.pages, (c + 1) * blob.pages)))
    rt.infer(0, 0, arch.make_inputs(b, spec))
    ex, wall = rt.exec_many(0, b, [(i % copies) * blob.pages for i in range(reps)])
    print("exec us", [round(x / 1e3, 1) for x in ex])
