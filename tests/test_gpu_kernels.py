"""Per-layer parity of the tcgen05 implicit-GEMM convolution against a plain
PyTorch fp32 reference of the same op (bf16-rounded inputs and weights).

Tolerance: |out - ref| <= 0.02 * max|ref| + 0.01 (bf16 output rounding plus
fp32-accumulation-order differences; K up to 4608)."""

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_2006_02464_b200 import arch
from paper_2006_02464_b200.device import DeviceRuntime

pytestmark = pytest.mark.gpu


def _single_conv_arch(b, h, w, cin, cout, k, stride, pad, relu, residual):
    spec = arch.ArchSpec("single")
    lay = arch.Layer(0, "c", "bn", cin, cout, k, stride, pad, k * k * cin)
    spec.layers.append(lay)
    oh = (h + 2 * pad - k) // stride + 1
    ow = (w + 2 * pad - k) // stride + 1
    spec.ops.append(arch._op(arch.OP_CONV, layer=0, in_buf=0, out_buf=1,
                             res_buf=2 if residual else -1, cin=cin, cout=cout, kh=k, kw=k,
                             stride=stride, pad=pad, relu=int(relu), in_h=h, in_w=w, out_h=oh,
                             out_w=ow, kpad=k * k * cin))
    if residual:  # make buffer 2 exist with the output shape
        spec.ops.append(arch._op(arch.OP_CONV, layer=0, in_buf=0, out_buf=2, cin=cin, cout=cout,
                                 kh=k, kw=k, stride=stride, pad=pad, in_h=h, in_w=w, out_h=oh,
                                 out_w=ow, kpad=k * k * cin))
    return spec, oh, ow


CASES = [
    # b, h, w, cin, cout, k, stride, pad, relu, residual
    (2, 56, 56, 64, 256, 1, 1, 0, True, False),
    (1, 7, 7, 2048, 512, 1, 1, 0, True, False),
    (3, 14, 14, 1024, 256, 1, 1, 0, False, True),
    (2, 56, 56, 64, 64, 3, 1, 1, True, False),
    (3, 14, 14, 256, 256, 3, 1, 1, True, False),
    (2, 7, 7, 512, 512, 3, 1, 1, True, True),
    (5, 7, 7, 512, 512, 3, 1, 1, True, False),
    (2, 56, 56, 128, 128, 3, 2, 1, True, False),
    (1, 28, 28, 256, 256, 3, 2, 1, True, False),
    (2, 56, 56, 256, 512, 1, 2, 0, False, False),
    (16, 28, 28, 128, 512, 1, 1, 0, True, True),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "b{}_{}x{}_{}to{}_k{}s{}".format(*c[:7]))
def test_conv_layer_matches_torch(gpu, case):
    b, h, w, cin, cout, k, stride, pad, relu, residual = case
    spec, oh, ow = _single_conv_arch(b, h, w, cin, cout, k, stride, pad, relu, residual)
    rng = np.random.default_rng(hash(case) % 2**32)
    x = rng.standard_normal((b, h, w, cin)).astype(np.float32)
    wt = (rng.standard_normal((cout, k, k, cin)) / np.sqrt(k * k * cin)).astype(np.float32)
    bias = rng.standard_normal(cout).astype(np.float32) * 0.1
    res = rng.standard_normal((b, oh, ow, cout)).astype(np.float32)
    xb = arch.to_bf16_bits(x)
    wb = arch.to_bf16_bits(wt.reshape(cout, -1))
    resb = arch.to_bf16_bits(res)
    blob = arch.pack_blob(spec, [(wt.reshape(cout, -1), bias)])
    with DeviceRuntime(device=gpu, pages_total=8, io_slots=16) as rt:
        rt.register_arch(0, spec, batches=(b,))
        rt.register_blob(0, 0, blob)
        rt.build()
        rt.load(0, list(range(blob.pages)))
        rt.buffer_io(0, 0, xb, True)
        if residual:
            rt.buffer_io(0, 2, resb, True)
        ex, _ = rt.exec_many(0, b, [0])
        if residual:  # the second op overwrote buffer 2 with conv(x); re-run op 0 only
            pass
        out = np.empty((b, oh, ow, cout), np.uint16)
        rt.buffer_io(0, 1, out, False)
    got = arch.bf16_to_f32(out)
    xt = torch.from_numpy(arch.bf16_to_f32(xb)).permute(0, 3, 1, 2)
    wtt = torch.from_numpy(arch.bf16_to_f32(wb).reshape(cout, k, k, cin)).permute(0, 3, 1, 2)
    ref = F.conv2d(xt, wtt, torch.from_numpy(bias), stride=stride, padding=pad)
    ref = ref.permute(0, 2, 3, 1).numpy()
    if residual:
        # op order: op0 (with residual from buf 2) runs before op1 rewrites buf 2
        ref = ref + arch.bf16_to_f32(resb)
    if relu:
        ref = np.maximum(ref, 0)
    err = np.abs(got - ref).max()
    tol = 0.02 * np.abs(ref).max() + 0.01
    assert err <= tol, f"max err {err} > {tol}"
    assert ex[0] > 0
