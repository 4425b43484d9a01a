"""Stem check on the device (debug helper): one INFER, then the NHWC4 input buffer and the
stem + max-pool output buffer read back and compared with torch (conv1 + bn1 + relu +
maxpool of the oracle model on the same bf16-rounded input).
    python tools/stem_debug.py [arch] [batch]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import resnet_oracle  # noqa: E402
from paper_2006_02464_b200 import arch  # noqa: E402
from paper_2006_02464_b200.device import DeviceRuntime  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
b = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = arch.build_arch(name)
params = arch.make_params(spec, seed=1)
blob = arch.pack_blob(spec, arch.fold(spec, params))
spec.ops = spec.ops[:3]  # input conversion, stem conv, its max pool (fused): BUF_X0 = output
x = arch.make_inputs(b, spec, first=7 * b)
with DeviceRuntime(pages_total=blob.pages + 1, io_slots=16) as rt:
    rt.register_arch(0, spec, batches=(b,))
    rt.register_blob(0, 0, blob)
    rt.build()
    rt.load(0, list(range(blob.pages)))
    rt.infer(0, 0, x)
    pw = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    hp, wp = 224 + 6, 224 + 2 * pw
    inp = np.zeros((b, hp, wp, 4), np.uint16)
    rt.buffer_io(0, arch.BUF_IM2COL, inp, False)
    out = np.zeros((b, 56, 56, 64), np.uint16)
    rt.buffer_io(0, arch.BUF_X0, out, False)


def bf(a):
    return (a.astype(np.uint32) << 16).view(np.float32)


xin = bf(inp)[:, 3:3 + 224, pw:pw + 224, :3]            # NHWC
ref_in = torch.tensor(x).permute(0, 2, 3, 1).to(torch.bfloat16).float().numpy()
print("input max abs diff", float(np.abs(xin - ref_in).max()),
      "pad nonzero", int((inp[:, :3] != 0).sum() + (inp[:, :, :pw] != 0).sum()))
model = resnet_oracle.torchvision_model(name, params).eval()
with torch.no_grad():
    t = torch.tensor(ref_in).permute(0, 3, 1, 2)
    y = model.maxpool(model.relu(model.bn1(model.conv1(t)))).permute(0, 2, 3, 1).numpy()
got = bf(out)
d = np.abs(got - y)
print("stem out max abs diff", float(d.max()), "ref max", float(np.abs(y).max()))
bad = np.argwhere(d > 0.05 * max(1e-6, float(np.abs(y).max())))
print("bad count", len(bad))
if len(bad):
    rows = sorted(set(int(v) for v in bad[:, 1]))
    cols = sorted(set(int(v) for v in bad[:, 2]))
    chans = sorted(set(int(v) for v in bad[:, 3]))
    print("rows", rows[:20], "cols", cols[:20], "chans", chans[:20])
