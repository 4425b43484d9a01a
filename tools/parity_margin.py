"""Logit error margins against the CPU fp32 oracle for one or more library variants
(experiments: CW_LIB per run in a subprocess). Prints rel = max-abs error / max|logit| per
(arch, batch), the quantity the parity tests bound by 0.02.

    python tools/parity_margin.py "resnet18,resnet50" "1,8" libcw.so libcw_x.so
"""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, json
sys.path.insert(0, %(repo)r)
from oracle import resnet_oracle
from paper_2006_02464_b200 import arch
from paper_2006_02464_b200.device import DeviceRuntime
out = {}
for name in %(archs)r:
    spec = arch.build_arch(name)
    params = arch.make_params(spec, seed=1)
    blob = arch.pack_blob(spec, arch.fold(spec, params))
    model = resnet_oracle.torchvision_model(name, params)
    for b in %(batches)r:
        x = arch.make_inputs(b, spec, first=7 * b)
        with DeviceRuntime(pages_total=blob.pages + 2, io_slots=16,
                           in_bytes_max=spec.in_c * spec.in_h * spec.in_w * 4) as rt:
            rt.register_arch(0, spec, batches=(b,))
            rt.register_blob(0, 0, blob)
            rt.build()
            rt.load(0, list(range(blob.pages)))
            got, _ = rt.infer(0, 0, x)
        c = resnet_oracle.compare(got, resnet_oracle.logits(model, x))
        out[f"{name}/{b}"] = round(float(c["rel"]), 5)
print("RESULT" + json.dumps(out))
"""

archs = sys.argv[1].split(",")
batches = [int(b) for b in sys.argv[2].split(",")]
for lib in sys.argv[3:]:
    env = dict(os.environ, CW_LIB=lib)
    r = subprocess.run([sys.executable, "-c", CHILD % dict(repo=REPO, archs=archs, batches=batches)],
                       capture_output=True, text=True, env=env)
    line = [x for x in r.stdout.splitlines() if x.startswith("RESULT")]
    print(lib, json.loads(line[0][6:]) if line else r.stderr[-800:])
