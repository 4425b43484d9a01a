"""Debug one zoo arch on the device: print its plan, run one INFER, compare with the oracle.
    python tools/zoo_debug.py densenet121 [batch]"""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import resnet_oracle
from paper_2006_02464_b200 import arch
from paper_2006_02464_b200.device import DeviceRuntime

name = sys.argv[1]
b = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = arch.build_arch(name)
params = arch.make_params(spec, seed=0)
blob = arch.pack_blob(spec, arch.fold(spec, params))
with DeviceRuntime(device=0, pages_total=blob.pages + 1, io_slots=16,
                   in_bytes_max=spec.in_c * spec.in_h * spec.in_w * 4) as rt:
    rt.register_arch(0, spec, batches=(b,))
    rt.register_blob(0, 0, blob)
    rt.build()
    plan = rt.plan_layers(0, b)
    for i, row in enumerate(plan):
        op = spec.ops[row[6]]
        print(i, "kind", row[0], "mode", row[1], "bn", row[2], "tasks", row[3], "split", row[4],
              "kb", row[5], "op", row[6], "opkind", op["kind"], "cin", op["cin"], "cout", op["cout"],
              "k", (op["kh"], op["kw"]), "flags", op["flags"], flush=True)
    rt.load(0, list(range(blob.pages)))
    x = arch.make_inputs(b, spec)
    got, ns = rt.infer(0, 0, x)
    ref = resnet_oracle.logits(resnet_oracle.torchvision_model(name, params), x)
    print("exec us", ns / 1e3, resnet_oracle.compare(got, ref))
