import sys; sys.path.insert(0, ".")
from paper_2006_02464_b200 import arch
from paper_2006_02464_b200.device import DeviceRuntime
import numpy as np
name = sys.argv[1]; b = int(sys.argv[2])
spec = arch.build_arch(name)
blob = arch.pack_blob(spec, arch.fold(spec, arch.make_params(spec, 1)))
with DeviceRuntime(pages_total=8, io_slots=16) as rt:
    rt.register_arch(0, spec, batches=(b,))
    rt.register_blob(0, 0, blob)
    rt.build()
    rt.load(0, list(range(blob.pages)))
    pl = rt.plan_layers(0, b)
    for i, r in enumerate(pl): print(i, [int(x) for x in r])
    out, _ = rt.infer(0, 0, arch.make_inputs(b, spec))
    print("ok", out.shape)
    if len(sys.argv) > 3:
        for _ in range(int(sys.argv[3])):
            out, _ = rt.infer(0, 0, arch.make_inputs(b, spec))
        print("ok2")
