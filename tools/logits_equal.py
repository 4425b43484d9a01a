"""Are two library variants' logits bit-identical? (experiments: a rewrite that must not
change numerics). Each CW_LIB runs in a subprocess on the same seeded weights and inputs.

    python tools/logits_equal.py inception_v3 "1,16" libcw_old.so libcw.so
    python tools/logits_equal.py resnet50 "1,16" libcw.so:CW_NO_DENSE_BOX=1 libcw.so
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys
import numpy as np
sys.path.insert(0, %(repo)r)
from paper_2006_02464_b200 import arch
from paper_2006_02464_b200.device import DeviceRuntime
spec = arch.build_arch(%(name)r)
blob = arch.pack_blob(spec, arch.fold(spec, arch.make_params(spec, seed=3)))
out = {}
with DeviceRuntime(pages_total=blob.pages, io_slots=16,
                   in_bytes_max=spec.in_c * spec.in_h * spec.in_w * 4) as rt:
    rt.register_arch(0, spec, batches=tuple(%(batches)r))
    rt.register_blob(0, 0, blob)
    rt.build()
    rt.load(0, list(range(blob.pages)))
    for b in %(batches)r:
        out[str(b)] = rt.infer(0, 0, arch.make_inputs(b, spec, first=7))[0]
np.savez(%(path)r, **out)
"""


def main():
    name, batches = sys.argv[1], [int(x) for x in sys.argv[2].split(",")]
    libs = sys.argv[3:]
    res = {}
    with tempfile.TemporaryDirectory() as tmp:
        for i, spec in enumerate(libs):
            lib, _, envs = spec.partition(":")
            env = dict(os.environ, CW_LIB=lib)
            for kv in filter(None, envs.split(",")):
                k, v = kv.split("=")
                env[k] = v
            path = os.path.join(tmp, f"{i}.npz")
            code = CHILD % {"repo": REPO, "name": name, "batches": batches, "path": path}
            r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
            if r.returncode:
                print(spec, "failed:", r.stderr[-800:])
                return 1
            res[spec] = dict(np.load(path))
    ok = True
    for b in batches:
        a, z = res[libs[0]][str(b)], res[libs[-1]][str(b)]
        same = np.array_equal(a, z)
        ok &= same
        print(f"{name} b={b}: {'bit-identical' if same else 'DIFFER'} "
              f"(max |diff| {float(np.max(np.abs(a.astype(np.float64) - z))):.3g})")
    return 0 if ok else 2


if __name__ == "__main__":
    sys.exit(main())
