"""Quick per-batch INFER timing on one GPU (device-resident inputs, copies of
ResNet-50 in distinct pages so weights stream from HBM). Profiling helper."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2006_02464_b200 import arch
from paper_2006_02464_b200.device import DeviceRuntime

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
batches = [int(b) for b in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 2, 4, 8, 16]
spec = arch.build_arch(name)
blob = arch.pack_blob(spec, arch.fold(spec, arch.make_params(spec, 0)))
copies = 8
with DeviceRuntime(pages_total=copies * blob.pages, io_slots=16) as rt:
    rt.register_arch(0, spec)
    rt.register_blob(0, 0, blob)
    rt.build()
    for c in range(copies):
        rt.load(0, list(range(c * blob.pages, (c + 1) * blob.pages)))
    x = arch.make_inputs(16, spec)
    rt.infer(0, 0, x)  # fill slots
    out = {}
    for b in batches:
        hp = [(i % copies) * blob.pages for i in range(iters)]
        rt.exec_many(0, b, hp[:20])
        ex, wall = rt.exec_many(0, b, hp)
        n, fl = rt.plan_info(0, b)
        out[b] = dict(p50_us=float(np.median(ex)) / 1e3, p99_us=float(np.percentile(ex, 99)) / 1e3,
                      max_us=float(ex.max()) / 1e3, wall_per_us=wall / iters / 1e3,
                      img_s=b * iters / (wall / 1e9), launches=n,
                      tflops=spec.flops_per_image * b / (np.median(ex) / 1e9) / 1e12)
        print(b, json.dumps(out[b]), flush=True)
