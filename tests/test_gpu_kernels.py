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


def _up(x, m=64):
    return (x + m - 1) // m * m


def _single_conv_arch(b, h, w, cin, cout, k, stride, pad, relu, residual, kw=None, pad_w=None):
    kh, kw = k, (k if kw is None else kw)
    ph, pw = pad, (pad if pad_w is None else pad_w)
    spec = arch.ArchSpec("single")
    kpad = kh * kw * _up(cin)
    lay = arch.Layer(0, "c", "bn", cin, cout, kh, kw, stride, ph, pw, kpad, cout_pad=_up(cout))
    spec.layers.append(lay)
    oh = (h + 2 * ph - kh) // stride + 1
    ow = (w + 2 * pw - kw) // stride + 1
    common = dict(cin=cin, cout=cout, kh=kh, kw=kw, stride=stride, pad=ph, pad_w=pw, in_h=h,
                  in_w=w, out_h=oh, out_w=ow, kpad=kpad, in_ctot=cin, out_ctot=cout,
                  cout_pad=_up(cout))
    spec.ops.append(arch._op(arch.OP_CONV, layer=0, in_buf=0, out_buf=1,
                             res_buf=2 if residual else -1, relu=int(relu), **common))
    if residual:  # make buffer 2 exist with the output shape
        spec.ops.append(arch._op(arch.OP_CONV, layer=0, in_buf=0, out_buf=2, **common))
    return spec, oh, ow, kpad


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
    # zoo shapes: real Cin / Cout not multiples of 64 (zero-filled channel blocks, clipped
    # stores), asymmetric kernels and paddings (Inception 1x7 / 7x1 / 1x3), valid convs
    (2, 35, 35, 48, 64, 5, 1, 2, True, False),
    (2, 73, 73, 80, 192, 3, 1, 0, True, False),
    (3, 17, 17, 160, 96, (1, 7), 1, (0, 3), True, False),
    (3, 17, 17, 160, 192, (7, 1), 1, (3, 0), True, False),
    (2, 8, 8, 384, 384, (1, 3), 1, (0, 1), True, False),
    (2, 35, 35, 288, 384, 3, 2, 0, True, False),
    (4, 35, 35, 288, 48, 1, 1, 0, True, False),
]


def _case_id(c):
    k = c[5] if isinstance(c[5], tuple) else (c[5], c[5])
    return "b{}_{}x{}_{}to{}_k{}x{}s{}".format(*c[:5], *k, c[6])


@pytest.mark.parametrize("case", CASES, ids=_case_id)
def test_conv_layer_matches_torch(gpu, case):
    b, h, w, cin, cout, k, stride, pad, relu, residual = case
    kh, kw = k if isinstance(k, tuple) else (k, k)
    ph, pw = pad if isinstance(pad, tuple) else (pad, pad)
    spec, oh, ow, kpad = _single_conv_arch(b, h, w, cin, cout, kh, stride, ph, relu, residual,
                                           kw=kw, pad_w=pw)
    rng = np.random.default_rng(abs(hash(str(case))) % 2**32)
    x = rng.standard_normal((b, h, w, cin)).astype(np.float32)
    wt = (rng.standard_normal((cout, kh, kw, cin)) / np.sqrt(kh * kw * cin)).astype(np.float32)
    bias = rng.standard_normal(cout).astype(np.float32) * 0.1
    res = rng.standard_normal((b, oh, ow, cout)).astype(np.float32)
    xb = arch.to_bf16_bits(x)
    wb = arch.to_bf16_bits(wt.reshape(cout, -1))
    resb = arch.to_bf16_bits(res)
    # device layout: [cout_pad][taps][cin_pad], zero-padded
    wdev = np.zeros((_up(cout), kh * kw, _up(cin)), np.float32)
    wdev[:cout, :, :cin] = wt.reshape(cout, kh * kw, cin)
    bdev = np.zeros(_up(cout), np.float32)
    bdev[:cout] = bias
    blob = arch.pack_blob(spec, [(wdev.reshape(_up(cout), kpad), bdev, None)])
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
    wtt = torch.from_numpy(arch.bf16_to_f32(wb).reshape(cout, kh, kw, cin)).permute(0, 3, 1, 2)
    ref = F.conv2d(xt, wtt, torch.from_numpy(bias), stride=stride, padding=(ph, pw))
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
