"""Quick A/B of library variants on the device (experiments): per variant (CW_LIB), device
Exec p50 over `n` INFERs at each batch, weights of `copies` model copies rotating through HBM.
    python tools/ab_quick.py resnet50 "1,16" 2000 8 libcw.so libcw_x.so ..."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, json, numpy as np
sys.path.insert(0, %(repo)r)
from paper_2006_02464_b200 import arch
from paper_2006_02464_b200.device import DeviceRuntime
name, batches, n, copies = %(name)r, %(batches)r, %(n)d, %(copies)d
spec = arch.build_arch(name)
blob = arch.pack_blob(spec, arch.fold(spec, arch.make_params(spec, 0)))
out = {}
with DeviceRuntime(pages_total=copies * blob.pages, io_slots=16,
                   in_bytes_max=spec.in_c * spec.in_h * spec.in_w * 4) as rt:
    rt.register_arch(0, spec, batches=tuple(batches))
    rt.register_blob(0, 0, blob)
    rt.build()
    for c in range(copies):
        rt.load(0, list(range(c * blob.pages, (c + 1) * blob.pages)))
    rt.infer(0, 0, arch.make_inputs(max(batches), spec))
    for b in batches:
        hp = [(i %% copies) * blob.pages for i in range(n)]
        rt.exec_many(0, b, hp[:100])
        ex, wall = rt.exec_many(0, b, hp)
        out[b] = {"p50_us": float(np.percentile(ex, 50)) / 1e3, "img_s": b * n / (wall / 1e9)}
print("RESULT" + json.dumps(out))
"""


def main():
    name, batches, n, copies = sys.argv[1], [int(x) for x in sys.argv[2].split(",")], \
        int(sys.argv[3]), int(sys.argv[4])
    res = {}
    for spec in sys.argv[5:]:   # "libcw_x.so" or "libcw_x.so:VAR=1,VAR2=2"
        lib, _, envs = spec.partition(":")
        code = CHILD % {"repo": REPO, "name": name, "batches": batches, "n": n, "copies": copies}
        env = dict(os.environ, CW_LIB=lib)
        for kv in filter(None, envs.split(",")):
            k, v = kv.split("=")
            env[k] = v
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
        res[spec] = json.loads(line[0][6:]) if line else r.stderr[-500:]
        print(spec, res[spec], flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
