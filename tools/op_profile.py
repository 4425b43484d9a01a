"""Per-op eager timing (CUDA events between launches) with the launch plan,
for one arch and batch. Profiling helper."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2006_02464_b200 import arch
from paper_2006_02464_b200.device import DeviceRuntime

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
batches = [int(b) for b in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 16]
spec = arch.build_arch(name)
blob = arch.pack_blob(spec, arch.fold(spec, arch.make_params(spec, 0)))
names = {0: "stem", 1: "conv", 2: "maxpool", 3: "avgpool", 4: "fc", -1: "fused"}
with DeviceRuntime(pages_total=8 * blob.pages, io_slots=16) as rt:
    rt.register_arch(0, spec)
    rt.register_blob(0, 0, blob)
    rt.build()
    for c in range(8):
        rt.load(0, list(range(c * blob.pages, (c + 1) * blob.pages)))
    rt.infer(0, 0, arch.make_inputs(16, spec))
    for b in batches:
        reps = [rt.profile_ops(0, b, (r % 8) * blob.pages)[0] for r in range(7)]
        ms = np.median(np.stack(reps), axis=0)
        plan = rt.plan_ops(0, b)
        ex, wall = rt.exec_many(0, b, [(i % 8) * blob.pages for i in range(200)])
        print(f"== {name} b={b}: graph exec p50 {np.median(ex)/1e3:.1f} us, eager sum {ms.sum()*1e3:.1f} us")
        for i, (op, t) in enumerate(zip(spec.ops, ms)):
            k, mode, bn, mt, sp, st, kb, pool = plan[i]
            flops = 2 * op["out_h"] * op["out_w"] * op["cout"] * op["kh"] * op["kw"] * op["cin"] * b if op["kind"] == 1 else 0
            tf = flops / (t * 1e-3) / 1e12 if t > 0 and flops else 0
            print(f"{i:3d} {names[int(k)]:7s} {op['cin']:5d}->{op['cout']:5d} k{op['kh']} s{op['stride']} @{op['in_h']:3d} "
                  f"mode{mode:2d} bn{bn:4d} mt{mt:5d} sp{sp:3d} st{st} kb{kb:3d} pool{pool} {t*1e3:8.1f} us {tf:7.1f} TF/s")
