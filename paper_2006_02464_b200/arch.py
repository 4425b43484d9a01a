"""Model artifacts for the B200 worker: architecture tables, deterministic
random-init parameters, BatchNorm folding and the 16 MiB-paged weight blob.

This is the artifact side of the paper's model compilation step (PAPER.md
§5.1: weights + per-batch kernels + memory metadata). The
reference ships profiles only (pkg/src/sloserve/profiles.py:1-8, "profiles are
plain data files that stand in for compiled models"); here a catalog base name
maps to a real network. The zoo: the reference catalog's own architectures
(profiles.py:322-374: densenet169, inceptionv3, resnet18, resnet50, resnet152)
and BASELINE.json configs[3]'s (resnet50/152, resnext50_32x4d, densenet121,
inception_v3), all following the torchvision definitions, with parameters named
exactly like torchvision's state_dict so the CPU oracle loads them into
torchvision's own modules.

An arch is a list of ops over workspace buffers (NHWC bf16). Every conv reads
`cin` channels of a buffer whose channel stride is `in_ctot` and writes `cout`
channels at channel offset `out_coff` of a buffer of stride `out_ctot` (concat =
several convs writing disjoint channel slices of one buffer: Inception blocks,
DenseNet blocks). Device shapes are padded for the tensor cores: the weights of
a conv are [cout_pad][kpad] with cout_pad = cout rounded up to 64 and K laid out
tap-major with the channels of every tap padded to a multiple of 64 (zeros; the
activation loads clip at `cin` and fill zeros).

Blob layout (all offsets are blob byte offsets; blob offset o lives in blob
page o // page_bytes at in-page offset o % page_bytes):
    [0, 64 KiB)   header, filled at LOAD with the page-resolved tensor maps
    tensors       per layer: folded weights bf16 [cout_pad][kpad], folded bias fp32
                  [cout_pad], and for layers with a BatchNorm on their INPUT
                  (DenseNet's pre-activation, applied in the consumer) fp32 scale and
                  shift [cin_pad]; 256-byte aligned, never straddling a page.
"""

from __future__ import annotations

import zlib
from dataclasses import dataclass, field

import numpy as np

HEADER_BYTES = 65536
BN_EPS = 1e-5

# op kinds (mirror CwOp in csrc/runtime.h and cw_op in include/cw.h)
OP_STEM, OP_CONV, OP_MAXPOOL, OP_AVGPOOL, OP_FC, OP_IM2COL, OP_BNPOOL, OP_SOFTMAX = range(8)
# op flags
F_GROUPED64 = 1   # grouped conv, groups within 64-channel blocks (ResNeXt): K = taps x 64
F_PRE_BN = 2      # BatchNorm + ReLU applied to the A operand in shared memory (DenseNet)

# Workspace buffer ids of the ResNets (other archs allocate ids as they go).
BUF_IM2COL, BUF_STEM, BUF_X0, BUF_X1, BUF_T1, BUF_T2, BUF_DS, BUF_POOL = range(8)


def _up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


@dataclass
class Layer:
    """One header entry: a weight-bearing layer (conv / fc), or a BatchNorm applied by
    a SIMT op (DenseNet transition / final norm: kind "bn")."""
    index: int
    name: str            # torchvision module name of the conv / fc ("" for kind "bn")
    bn: str | None       # BatchNorm folded into this layer's OUTPUT (None: none / fc)
    cin: int             # input channels of the torchvision weight (per conv, not per group)
    cout: int
    kh: int = 1
    kw: int = 1
    stride: int = 1
    pad_h: int = 0
    pad_w: int = 0
    kpad: int = 0        # stored K
    layout: str = "rsc"  # "rsc" | "stem4" | "im2col" | "avg3" | "g64" | "fc" | "none"
    groups: int = 1
    bn_eps: float = BN_EPS
    pre_bn: str | None = None   # BatchNorm (+ReLU) on this layer's input: scale/shift stored
    kind: str = "conv"          # "conv" | "fc" | "bn"
    cout_pad: int = 0

    @property
    def k(self) -> int:          # square kernels (ResNet tables)
        return self.kh

    @property
    def has_weights(self) -> bool:
        return self.kind != "bn"


@dataclass
class ArchSpec:
    name: str
    in_c: int = 3
    in_h: int = 224
    in_w: int = 224
    classes: int = 1000
    layers: list[Layer] = field(default_factory=list)
    ops: list[dict] = field(default_factory=list)
    flops_per_image: int = 0   # algorithmic (torchvision definition), conv + fc
    n_bufs: int = 0

    def op_structs(self):
        from . import _lib  # lazily: the tables themselves load no native code
        arr = (_lib.cw_op * len(self.ops))()
        for i, op in enumerate(self.ops):
            for k, v in op.items():
                setattr(arr[i], k, int(v))
        return arr


def _op(kind, **kw):
    d = dict(kind=kind, layer=-1, in_buf=-1, out_buf=-1, res_buf=-1, cin=0, cout=0, kh=1, kw=1,
             stride=1, pad=0, relu=0, in_h=0, in_w=0, out_h=0, out_w=0, kpad=0, pad_w=0,
             in_ctot=0, out_ctot=0, out_coff=0, cout_pad=0, flags=0, pre_layer=-1)
    d.update(kw)
    return d


class _Builder:
    """Shared bookkeeping of the arch tables: layers, ops, buffers, FLOPs."""

    def __init__(self, spec: ArchSpec, first_buf: int = 0):
        self.spec = spec
        self.flops = 0
        self.next_buf = first_buf

    def buf(self) -> int:
        b = self.next_buf
        self.next_buf += 1
        return b

    def layer(self, name, bn, cin, cout, kh, kw, stride, ph, pw, layout="rsc", groups=1,
              eps=BN_EPS, pre_bn=None, kind="conv", cin_read=None, kpad=None) -> Layer:
        cr = cin if cin_read is None else cin_read
        if kpad is None:
            if layout == "g64":
                kpad = kh * kw * 64
            elif kind == "fc":
                kpad = cin
            elif kind == "bn":
                kpad = 0
            else:
                kpad = kh * kw * _up(cr, 64)
        lay = Layer(len(self.spec.layers), name, bn, cin, cout, kh, kw, stride, ph, pw, kpad,
                    layout, groups, eps, pre_bn, kind,
                    _up(cout, 64) if kind != "bn" else 0)
        self.spec.layers.append(lay)
        return lay

    def conv(self, name, bn, cin, cout, k, stride, pad, h, w, in_buf, out_buf, relu,
             res_buf=-1, *, kw=None, pad_w=None, in_ctot=0, out_ctot=0, out_coff=0,
             eps=BN_EPS, layout="rsc", groups=1, pre_bn=None, flops_k=None):
        """A conv (+ folded BN) (+ residual) (+ ReLU) op; returns the output (h, w)."""
        kh, kw = k, (k if kw is None else kw)
        ph, pw = pad, (pad if pad_w is None else pad_w)
        oh = (h + 2 * ph - kh) // stride + 1
        ow = (w + 2 * pw - kw) // stride + 1
        lay = self.layer(name, bn, cin, cout, kh, kw, stride, ph, pw, layout, groups, eps, pre_bn)
        flags = (F_GROUPED64 if layout == "g64" else 0) | (F_PRE_BN if pre_bn else 0)
        self.spec.ops.append(_op(
            OP_CONV, layer=lay.index, in_buf=in_buf, out_buf=out_buf, res_buf=res_buf,
            cin=cin, cout=cout, kh=kh, kw=kw, stride=stride, pad=ph, pad_w=pw, relu=relu,
            in_h=h, in_w=w, out_h=oh, out_w=ow, kpad=lay.kpad, in_ctot=in_ctot or cin,
            out_ctot=out_ctot or cout, out_coff=out_coff, cout_pad=lay.cout_pad, flags=flags,
            pre_layer=lay.index if pre_bn else -1))
        taps = kh * kw if flops_k is None else flops_k
        self.flops += 2 * oh * ow * cout * taps * (cin // groups)
        return oh, ow

    def maxpool(self, in_buf, out_buf, c, h, w, k=3, stride=2, pad=1, in_ctot=0, out_ctot=0,
                out_coff=0):
        oh = (h + 2 * pad - k) // stride + 1
        ow = (w + 2 * pad - k) // stride + 1
        self.spec.ops.append(_op(OP_MAXPOOL, in_buf=in_buf, out_buf=out_buf, cin=c, cout=c,
                                 kh=k, kw=k, stride=stride, pad=pad, pad_w=pad, in_h=h,
                                 in_w=w, out_h=oh, out_w=ow, in_ctot=in_ctot or c,
                                 out_ctot=out_ctot or c, out_coff=out_coff))
        return oh, ow

    def avgpool(self, in_buf, out_buf, c, h, w, pre_bn=None):
        pre = -1
        if pre_bn:
            pre = self.layer("", None, c, c, 1, 1, 1, 0, 0, "none", pre_bn=pre_bn,
                             kind="bn").index
        self.spec.ops.append(_op(OP_AVGPOOL, in_buf=in_buf, out_buf=out_buf, cin=c, cout=c,
                                 in_h=h, in_w=w, out_h=1, out_w=1, in_ctot=c,
                                 pre_layer=pre, flags=F_PRE_BN if pre_bn else 0))

    def fc(self, name, in_buf, feat, classes=1000):
        lay = self.layer(name, None, feat, classes, 1, 1, 1, 0, 0, "fc", kind="fc")
        self.spec.ops.append(_op(OP_FC, layer=lay.index, in_buf=in_buf, cin=feat, cout=classes,
                                 kpad=lay.kpad, cout_pad=lay.cout_pad))
        self.flops += 2 * feat * classes

    def finish(self):
        self.spec.flops_per_image = self.flops
        self.spec.n_bufs = self.next_buf
        return self.spec


# ---------------------------------------------------------------------------- ResNet / ResNeXt

_RESNETS = {
    "resnet18": ("basic", [2, 2, 2, 2], 1, 64),
    "resnet34": ("basic", [3, 4, 6, 3], 1, 64),
    "resnet50": ("bottleneck", [3, 4, 6, 3], 1, 64),
    "resnet101": ("bottleneck", [3, 4, 23, 3], 1, 64),
    "resnet152": ("bottleneck", [3, 8, 36, 3], 1, 64),
    "resnext50_32x4d": ("bottleneck", [3, 4, 6, 3], 32, 4),
}


def _resnet(name: str) -> ArchSpec:
    block, counts, groups, base_width = _RESNETS[name]
    spec = ArchSpec(name)
    B = _Builder(spec, first_buf=8)
    # Stem: the input stage converts fp32 NCHW to bf16 NHWC4 rows (channel 3 = 0, zero
    # pixels either side); the 7x7/s2 conv reads overlapping 8-pixel row windows of those
    # rows, K = 7 kernel rows x (8 pixels x 4 channels) = 224; the 3x3/s2 max pool is fused.
    h = w = 224
    spec.ops.append(_op(OP_STEM, out_buf=BUF_IM2COL, in_h=h, in_w=w, out_h=112, out_w=112,
                        kpad=224, cin=3))
    stem = B.layer("conv1", "bn1", 3, 64, 7, 7, 2, 3, 3, "stem4", kpad=224)
    spec.ops.append(_op(OP_CONV, layer=stem.index, in_buf=BUF_IM2COL, out_buf=BUF_STEM, cin=4,
                        cout=64, kh=7, kw=7, stride=2, pad=3, pad_w=3, relu=1, in_h=224,
                        in_w=224, out_h=112, out_w=112, kpad=224, in_ctot=4, out_ctot=64,
                        cout_pad=64))
    B.flops += 2 * 112 * 112 * 64 * 147
    B.maxpool(BUF_STEM, BUF_X0, 64, 112, 112)
    h = w = 56
    x = BUF_X0
    inplanes = 64
    expansion = 4 if block == "bottleneck" else 1
    for li, (planes, n) in enumerate(zip([64, 128, 256, 512], counts)):
        width = int(planes * (base_width / 64.0)) * groups
        for bi in range(n):
            stride = 2 if (li > 0 and bi == 0) else 1
            pre = f"layer{li + 1}.{bi}"
            y = BUF_X1 if x == BUF_X0 else BUF_X0
            has_ds = stride != 1 or inplanes != planes * expansion
            if block == "bottleneck":
                B.conv(f"{pre}.conv1", f"{pre}.bn1", inplanes, width, 1, 1, 0, h, w, x, BUF_T1, 1)
                oh, ow = B.conv(f"{pre}.conv2", f"{pre}.bn2", width, width, 3, stride, 1, h, w,
                                BUF_T1, BUF_T2, 1, layout="g64" if groups > 1 else "rsc",
                                groups=groups)
                if has_ds:
                    B.conv(f"{pre}.downsample.0", f"{pre}.downsample.1", inplanes,
                           planes * 4, 1, stride, 0, h, w, x, BUF_DS, 0)
                B.conv(f"{pre}.conv3", f"{pre}.bn3", width, planes * 4, 1, 1, 0, oh, ow, BUF_T2,
                       y, 1, res_buf=BUF_DS if has_ds else x)
            else:
                oh, ow = B.conv(f"{pre}.conv1", f"{pre}.bn1", inplanes, planes, 3, stride, 1, h,
                                w, x, BUF_T1, 1)
                if has_ds:
                    B.conv(f"{pre}.downsample.0", f"{pre}.downsample.1", inplanes, planes, 1,
                           stride, 0, h, w, x, BUF_DS, 0)
                B.conv(f"{pre}.conv2", f"{pre}.bn2", planes, planes, 3, 1, 1, oh, ow, BUF_T1, y,
                       1, res_buf=BUF_DS if has_ds else x)
            inplanes = planes * expansion
            x = y
            h, w = oh, ow
    B.avgpool(x, BUF_POOL, inplanes, h, w)
    B.fc("fc", BUF_POOL, inplanes)
    return B.finish()


# ---------------------------------------------------------------------------- DenseNet

_DENSENETS = {"densenet121": (32, (6, 12, 24, 16), 64),
              "densenet169": (32, (6, 12, 32, 32), 64)}


def _densenet(name: str) -> ArchSpec:
    """torchvision DenseNet-BC (bn_size 4): pre-activation dense layers. norm1+ReLU of a
    dense layer is applied to the concatenated block features inside the consumer conv
    (F_PRE_BN: BN+ReLU on the A tile in shared memory); norm2 folds into conv1's output;
    conv2's 32 channels are written at their channel offset of the block buffer (the
    concat); a transition is BN+ReLU+2x2 average pool (one SIMT op) then the 1x1 conv
    (pooling first is exact: the conv is linear)."""
    growth, blocks, c0 = _DENSENETS[name]
    spec = ArchSpec(name)
    B = _Builder(spec, first_buf=8)
    ctots = []
    c = c0
    for i, n in enumerate(blocks):
        ctots.append(c + n * growth)
        c = (c + n * growth) // 2
    blk = B.buf()
    spec.ops.append(_op(OP_STEM, out_buf=BUF_IM2COL, in_h=224, in_w=224, out_h=112, out_w=112,
                        kpad=224, cin=3))
    stem = B.layer("features.conv0", "features.norm0", 3, c0, 7, 7, 2, 3, 3, "stem4", kpad=224)
    spec.ops.append(_op(OP_CONV, layer=stem.index, in_buf=BUF_IM2COL, out_buf=BUF_STEM, cin=4,
                        cout=c0, kh=7, kw=7, stride=2, pad=3, pad_w=3, relu=1, in_h=224,
                        in_w=224, out_h=112, out_w=112, kpad=224, in_ctot=4, out_ctot=c0,
                        cout_pad=64))
    B.flops += 2 * 112 * 112 * c0 * 147
    h = w = 56
    B.maxpool(BUF_STEM, blk, c0, 112, 112, out_ctot=ctots[0])
    t1 = B.buf()
    c = c0
    for bi, n in enumerate(blocks):
        ctot = ctots[bi]
        for li in range(n):
            pre = f"features.denseblock{bi + 1}.denselayer{li + 1}"
            B.conv(f"{pre}.conv1", f"{pre}.norm2", c, 4 * growth, 1, 1, 0, h, w, blk, t1, 1,
                   in_ctot=ctot, pre_bn=f"{pre}.norm1")
            B.conv(f"{pre}.conv2", None, 4 * growth, growth, 3, 1, 1, h, w, t1, blk, 0,
                   out_ctot=ctot, out_coff=c)
            c += growth
        if bi + 1 < len(blocks):
            tr = f"features.transition{bi + 1}"
            pooled = B.buf()
            lay = B.layer("", None, ctot, ctot, 1, 1, 1, 0, 0, "none", pre_bn=f"{tr}.norm",
                          kind="bn")
            spec.ops.append(_op(OP_BNPOOL, in_buf=blk, out_buf=pooled, cin=ctot, cout=ctot,
                                kh=2, kw=2, stride=2, in_h=h, in_w=w, out_h=h // 2,
                                out_w=w // 2, in_ctot=ctot, out_ctot=ctot, pre_layer=lay.index,
                                flags=F_PRE_BN))
            h, w = h // 2, w // 2
            nxt = B.buf()
            B.conv(f"{tr}.conv", None, ctot, ctot // 2, 1, 1, 0, h, w, pooled, nxt, 0,
                   out_ctot=ctots[bi + 1])
            B.flops += 0   # (torchvision pools after the conv: same FLOPs at 1/4 the pixels x4)
            B.flops += 2 * h * w * (ctot // 2) * ctot * 3   # conv at full resolution = 4x
            blk = nxt
            c = ctot // 2
    pool = B.buf()
    B.avgpool(blk, pool, c, h, w, pre_bn="features.norm5")
    B.fc("classifier", pool, c)
    return B.finish()


# ---------------------------------------------------------------------------- Inception-v3

def _inception_v3(name: str) -> ArchSpec:
    """torchvision Inception3 (eval: no aux head, transform_input False), 299x299 input.
    BasicConv2d = conv + BN(eps 0.001) + ReLU, folded. Branch outputs are written at their
    channel offsets of the block buffer (the concat). The branch pools (avg 3x3/s1/p1,
    count_include_pad) followed by a 1x1 conv run as ONE 3x3 conv with the 1x1 weights / 9
    on every tap (layout "avg3": both are linear). The first conv (3 channels, 3x3/s2) runs
    on an im2col tile (K = 27 -> 64) built from the fp32 request images by a SIMT op."""
    spec = ArchSpec(name, in_h=299, in_w=299)
    B = _Builder(spec, first_buf=8)
    E = 0.001

    def bc(nm, cin, cout, k, stride, pad, h, w, ib, ob, kw=None, pad_w=None, in_ctot=0,
           out_ctot=0, out_coff=0, layout="rsc"):
        return B.conv(f"{nm}.conv", f"{nm}.bn", cin, cout, k, stride, pad, h, w, ib, ob, 1,
                      kw=kw, pad_w=pad_w, in_ctot=in_ctot, out_ctot=out_ctot, out_coff=out_coff,
                      eps=E, layout=layout, flops_k=1 if layout == "avg3" else None)

    # stem
    col = B.buf()
    spec.ops.append(_op(OP_IM2COL, out_buf=col, cin=3, cout=64, kh=3, kw=3, stride=2, pad=0,
                        in_h=299, in_w=299, out_h=149, out_w=149, kpad=64))
    lay = B.layer("Conv2d_1a_3x3.conv", "Conv2d_1a_3x3.bn", 3, 32, 3, 3, 2, 0, 0, "im2col",
                  eps=E, kpad=64)
    a = B.buf()
    spec.ops.append(_op(OP_CONV, layer=lay.index, in_buf=col, out_buf=a, cin=64, cout=32,
                        relu=1, in_h=149, in_w=149, out_h=149, out_w=149, kpad=64, in_ctot=64,
                        out_ctot=32, cout_pad=64))
    B.flops += 2 * 149 * 149 * 32 * 27
    b = B.buf()
    h, w = bc("Conv2d_2a_3x3", 32, 32, 3, 1, 0, 149, 149, a, b)
    c = B.buf()
    h, w = bc("Conv2d_2b_3x3", 32, 64, 3, 1, 1, h, w, b, c)
    d = B.buf()
    h, w = B.maxpool(c, d, 64, h, w, 3, 2, 0)
    e = B.buf()
    h, w = bc("Conv2d_3b_1x1", 64, 80, 1, 1, 0, h, w, d, e)
    f = B.buf()
    h, w = bc("Conv2d_4a_3x3", 80, 192, 3, 1, 0, h, w, e, f)
    x = B.buf()
    h, w = B.maxpool(f, x, 192, h, w, 3, 2, 0)
    cin = 192

    def block_a(nm, x, cin, pool_features, h, w):
        ctot = 224 + pool_features
        y = B.buf()
        bc(f"{nm}.branch1x1", cin, 64, 1, 1, 0, h, w, x, y, out_ctot=ctot, out_coff=0)
        t = B.buf()
        bc(f"{nm}.branch5x5_1", cin, 48, 1, 1, 0, h, w, x, t)
        bc(f"{nm}.branch5x5_2", 48, 64, 5, 1, 2, h, w, t, y, out_ctot=ctot, out_coff=64)
        t1, t2 = B.buf(), B.buf()
        bc(f"{nm}.branch3x3dbl_1", cin, 64, 1, 1, 0, h, w, x, t1)
        bc(f"{nm}.branch3x3dbl_2", 64, 96, 3, 1, 1, h, w, t1, t2)
        bc(f"{nm}.branch3x3dbl_3", 96, 96, 3, 1, 1, h, w, t2, y, out_ctot=ctot, out_coff=128)
        bc(f"{nm}.branch_pool", cin, pool_features, 3, 1, 1, h, w, x, y, out_ctot=ctot,
           out_coff=224, layout="avg3")
        return y, ctot

    def block_b(nm, x, cin, h, w):
        ctot = 384 + 96 + cin
        y = B.buf()
        oh, ow = bc(f"{nm}.branch3x3", cin, 384, 3, 2, 0, h, w, x, y, out_ctot=ctot)
        t1, t2 = B.buf(), B.buf()
        bc(f"{nm}.branch3x3dbl_1", cin, 64, 1, 1, 0, h, w, x, t1)
        bc(f"{nm}.branch3x3dbl_2", 64, 96, 3, 1, 1, h, w, t1, t2)
        bc(f"{nm}.branch3x3dbl_3", 96, 96, 3, 2, 0, h, w, t2, y, out_ctot=ctot, out_coff=384)
        B.maxpool(x, y, cin, h, w, 3, 2, 0, in_ctot=cin, out_ctot=ctot, out_coff=480)
        return y, ctot, oh, ow

    def block_c(nm, x, cin, c7, h, w):
        ctot = 768
        y = B.buf()
        bc(f"{nm}.branch1x1", cin, 192, 1, 1, 0, h, w, x, y, out_ctot=ctot)
        t1, t2 = B.buf(), B.buf()
        bc(f"{nm}.branch7x7_1", cin, c7, 1, 1, 0, h, w, x, t1)
        bc(f"{nm}.branch7x7_2", c7, c7, 1, 1, 0, h, w, t1, t2, kw=7, pad_w=3)
        bc(f"{nm}.branch7x7_3", c7, 192, 7, 1, 3, h, w, t2, y, kw=1, pad_w=0, out_ctot=ctot,
           out_coff=192)
        u1, u2, u3, u4 = B.buf(), B.buf(), B.buf(), B.buf()
        bc(f"{nm}.branch7x7dbl_1", cin, c7, 1, 1, 0, h, w, x, u1)
        bc(f"{nm}.branch7x7dbl_2", c7, c7, 7, 1, 3, h, w, u1, u2, kw=1, pad_w=0)
        bc(f"{nm}.branch7x7dbl_3", c7, c7, 1, 1, 0, h, w, u2, u3, kw=7, pad_w=3)
        bc(f"{nm}.branch7x7dbl_4", c7, c7, 7, 1, 3, h, w, u3, u4, kw=1, pad_w=0)
        bc(f"{nm}.branch7x7dbl_5", c7, 192, 1, 1, 0, h, w, u4, y, kw=7, pad_w=3, out_ctot=ctot,
           out_coff=384)
        bc(f"{nm}.branch_pool", cin, 192, 3, 1, 1, h, w, x, y, out_ctot=ctot, out_coff=576,
           layout="avg3")
        return y, ctot

    def block_d(nm, x, cin, h, w):
        ctot = 320 + 192 + cin
        y = B.buf()
        t = B.buf()
        bc(f"{nm}.branch3x3_1", cin, 192, 1, 1, 0, h, w, x, t)
        oh, ow = bc(f"{nm}.branch3x3_2", 192, 320, 3, 2, 0, h, w, t, y, out_ctot=ctot)
        u1, u2, u3 = B.buf(), B.buf(), B.buf()
        bc(f"{nm}.branch7x7x3_1", cin, 192, 1, 1, 0, h, w, x, u1)
        bc(f"{nm}.branch7x7x3_2", 192, 192, 1, 1, 0, h, w, u1, u2, kw=7, pad_w=3)
        bc(f"{nm}.branch7x7x3_3", 192, 192, 7, 1, 3, h, w, u2, u3, kw=1, pad_w=0)
        bc(f"{nm}.branch7x7x3_4", 192, 192, 3, 2, 0, h, w, u3, y, out_ctot=ctot, out_coff=320)
        B.maxpool(x, y, cin, h, w, 3, 2, 0, in_ctot=cin, out_ctot=ctot, out_coff=512)
        return y, ctot, oh, ow

    def block_e(nm, x, cin, h, w):
        ctot = 2048
        y = B.buf()
        bc(f"{nm}.branch1x1", cin, 320, 1, 1, 0, h, w, x, y, out_ctot=ctot)
        t = B.buf()
        bc(f"{nm}.branch3x3_1", cin, 384, 1, 1, 0, h, w, x, t)
        bc(f"{nm}.branch3x3_2a", 384, 384, 1, 1, 0, h, w, t, y, kw=3, pad_w=1, out_ctot=ctot,
           out_coff=320)
        bc(f"{nm}.branch3x3_2b", 384, 384, 3, 1, 1, h, w, t, y, kw=1, pad_w=0, out_ctot=ctot,
           out_coff=704)
        u1, u2 = B.buf(), B.buf()
        bc(f"{nm}.branch3x3dbl_1", cin, 448, 1, 1, 0, h, w, x, u1)
        bc(f"{nm}.branch3x3dbl_2", 448, 384, 3, 1, 1, h, w, u1, u2)
        bc(f"{nm}.branch3x3dbl_3a", 384, 384, 1, 1, 0, h, w, u2, y, kw=3, pad_w=1,
           out_ctot=ctot, out_coff=1088)
        bc(f"{nm}.branch3x3dbl_3b", 384, 384, 3, 1, 1, h, w, u2, y, kw=1, pad_w=0,
           out_ctot=ctot, out_coff=1472)
        bc(f"{nm}.branch_pool", cin, 192, 3, 1, 1, h, w, x, y, out_ctot=ctot, out_coff=1856,
           layout="avg3")
        return y, ctot

    x, cin = block_a("Mixed_5b", x, cin, 32, h, w)
    x, cin = block_a("Mixed_5c", x, cin, 64, h, w)
    x, cin = block_a("Mixed_5d", x, cin, 64, h, w)
    x, cin, h, w = block_b("Mixed_6a", x, cin, h, w)
    for nm, c7 in (("Mixed_6b", 128), ("Mixed_6c", 160), ("Mixed_6d", 160), ("Mixed_6e", 192)):
        x, cin = block_c(nm, x, cin, c7, h, w)
    x, cin, h, w = block_d("Mixed_7a", x, cin, h, w)
    x, cin = block_e("Mixed_7b", x, cin, h, w)
    x, cin = block_e("Mixed_7c", x, cin, h, w)
    pool = B.buf()
    B.avgpool(x, pool, cin, h, w)
    B.fc("fc", pool, cin)
    return B.finish()


_BUILDERS = {**{n: _resnet for n in _RESNETS}, **{n: _densenet for n in _DENSENETS},
             "inception_v3": _inception_v3}
# catalog base names -> torchvision model names (the reference catalog spells Inception-v3
# "inceptionv3", profiles.py:331)
ALIASES = {"inceptionv3": "inception_v3", "resnext50": "resnext50_32x4d"}
SUPPORTED = tuple(_BUILDERS) + tuple(ALIASES)


def torchvision_name(name: str) -> str:
    return ALIASES.get(name, name)


def build_arch(name: str, softmax: bool = False) -> ArchSpec:
    """Layer table + op list of a torchvision-definition network (catalog base name).
    softmax=True appends the softmax tail: the request outputs are class probabilities
    instead of logits."""
    tv = torchvision_name(name)
    if tv not in _BUILDERS:
        raise KeyError(f"no B200 implementation for architecture {name!r} "
                       f"(supported: {', '.join(SUPPORTED)})")
    spec = _BUILDERS[tv](tv)
    spec.name = tv
    if softmax:
        spec.ops.append(_op(OP_SOFTMAX, cin=spec.classes, cout=spec.classes))
    return spec


# ---------------------------------------------------------------------------- parameters

def _rng(seed: int, name: str) -> np.random.Generator:
    return np.random.default_rng([seed, zlib.crc32(name.encode())])


def _bn_params(p: dict, seed: int, name: str, c: int) -> None:
    rb = _rng(seed, name)
    p[f"{name}.weight"] = rb.uniform(0.5, 1.0, c).astype(np.float32)
    p[f"{name}.bias"] = (rb.standard_normal(c) * 0.1).astype(np.float32)
    p[f"{name}.running_mean"] = (rb.standard_normal(c) * 0.1).astype(np.float32)
    p[f"{name}.running_var"] = rb.uniform(0.75, 1.25, c).astype(np.float32)


def make_params(spec: ArchSpec, seed: int = 0) -> dict[str, np.ndarray]:
    """Random-init parameters in torchvision state_dict naming (fp32).

    conv: Kaiming-normal fan_out (torchvision's init); BatchNorm eval statistics
    randomized so folding is exercised: gamma~U[0.5,1], beta~N(0,0.1),
    mean~N(0,0.1), var~U[0.75,1.25]; fc: U(+-1/sqrt(fan_in)).
    """
    p: dict[str, np.ndarray] = {}
    for lay in spec.layers:
        if lay.pre_bn:
            _bn_params(p, seed, lay.pre_bn, lay.cin)
        if lay.kind == "bn":
            continue
        r = _rng(seed, lay.name)
        if lay.kind == "fc":
            bound = 1.0 / np.sqrt(lay.cin)
            p[f"{lay.name}.weight"] = r.uniform(-bound, bound, (lay.cout, lay.cin)).astype(np.float32)
            p[f"{lay.name}.bias"] = r.uniform(-bound, bound, (lay.cout,)).astype(np.float32)
            continue
        kh, kw = (1, 1) if lay.layout == "avg3" else (lay.kh, lay.kw)
        std = np.sqrt(2.0 / (lay.cout * kh * kw))
        p[f"{lay.name}.weight"] = (r.standard_normal((lay.cout, lay.cin // lay.groups, kh, kw))
                                   * std).astype(np.float32)
        if lay.bn:
            _bn_params(p, seed, lay.bn, lay.cout)
    return p


def _bn_affine(params, name, eps):
    g = params[f"{name}.weight"].astype(np.float64)
    beta = params[f"{name}.bias"].astype(np.float64)
    mu = params[f"{name}.running_mean"].astype(np.float64)
    var = params[f"{name}.running_var"].astype(np.float64)
    scale = g / np.sqrt(var + eps)
    return scale, beta - mu * scale


def fold(spec: ArchSpec, params: dict[str, np.ndarray]) -> list[tuple]:
    """Fold eval-mode BatchNorm into each conv (in float64).

    Returns per layer (W [cout_pad][kpad] fp32 or None, bias [cout_pad] fp32 or None,
    pre [2][cin_pad] fp32 scale/shift or None) in the device K order:
      rsc    W[co, (r*KW + s)*cin_pad + c] = w[co, c, r, s] * gamma/sqrt(var+eps)
      stem4  W[co, r*32 + (s+1)*4 + c] (window pixel 0 and channel 3 zero), matching the
             NHWC4 row windows the stem conv reads
      im2col W[co, (r*KW + s)*cin + c], K zero-padded to 64
      avg3   a 1x1 conv after a 3x3/s1/p1 average pool: 3x3 taps of w[co, c] / 9
      g64    grouped conv: W[co, (r*KW + s)*64 + c'] for the 64 input channels of co's
             64-channel block (zero outside co's group)
    """
    out = []
    for lay in spec.layers:
        pre = None
        if lay.pre_bn:
            s, t = _bn_affine(params, lay.pre_bn, lay.bn_eps)
            cp = _up(lay.cin, 64)
            pre = np.zeros((2, cp), np.float32)
            pre[0, :lay.cin], pre[1, :lay.cin] = s, t
        if lay.kind == "bn":
            out.append((None, None, pre))
            continue
        w = params[f"{lay.name}.weight"].astype(np.float64)
        if lay.kind == "fc":
            wpad = np.zeros((lay.cout_pad, lay.kpad), np.float64)
            wpad[:lay.cout] = w
            b = np.zeros(lay.cout_pad, np.float64)
            b[:lay.cout] = params[f"{lay.name}.bias"]
            out.append((wpad.astype(np.float32), b.astype(np.float32), pre))
            continue
        if lay.bn:
            scale, shift = _bn_affine(params, lay.bn, lay.bn_eps)
        else:
            scale, shift = np.ones(lay.cout), np.zeros(lay.cout)
        w = w * scale[:, None, None, None]           # [cout][cin/g][kh][kw]
        wpad = np.zeros((lay.cout_pad, lay.kpad), np.float64)
        if lay.layout == "stem4":
            w4 = wpad[:lay.cout].reshape(lay.cout, lay.kh, 8, 4)
            w4[:, :, 1:, :lay.cin] = w.transpose(0, 2, 3, 1)
        elif lay.layout == "im2col":
            wk = w.transpose(0, 2, 3, 1).reshape(lay.cout, -1)
            wpad[:lay.cout, :wk.shape[1]] = wk
        elif lay.layout == "avg3":
            cp = _up(lay.cin, 64)
            w3 = wpad[:lay.cout].reshape(lay.cout, 9, cp)
            w3[:, :, :lay.cin] = (w[:, :, 0, 0] / 9.0)[:, None, :]
        elif lay.layout == "g64":
            gw = lay.cin // lay.groups                 # channels per group
            taps = lay.kh * lay.kw
            wg = wpad[:lay.cout].reshape(lay.cout, taps, 64)
            for co in range(lay.cout):
                g0 = (co // gw) * gw                   # first input channel of co's group
                c0 = g0 % 64                           # ... within co's 64-channel block
                wg[co, :, c0:c0 + gw] = w[co].reshape(gw, taps).T
        else:
            cp = _up(lay.cin, 64)
            wt = wpad[:lay.cout].reshape(lay.cout, lay.kh * lay.kw, cp)
            wt[:, :, :lay.cin] = w.transpose(0, 2, 3, 1).reshape(lay.cout, lay.kh * lay.kw,
                                                                  lay.cin)
        b = np.zeros(lay.cout_pad, np.float64)
        b[:lay.cout] = shift
        out.append((wpad.astype(np.float32), b.astype(np.float32), pre))
    return out


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit patterns (uint16), round to nearest even."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


@dataclass
class Blob:
    data: np.ndarray          # uint8, page-structured
    locs: list[tuple[int, int, int, int, int]]   # (w_off, b_off, rows, k, s_off) per layer
    pages: int
    page_bytes: int

    def loc_structs(self):
        from . import _lib
        arr = (_lib.cw_tensor_loc * len(self.locs))()
        for i, (w, b, r, k, s) in enumerate(self.locs):
            arr[i].w_off, arr[i].b_off, arr[i].rows, arr[i].k, arr[i].s_off = w, b, r, k, s
        return arr


def pack_blob(spec: ArchSpec, folded, page_bytes: int = 16 * 1024 * 1024) -> Blob:
    """Bin-pack folded tensors into page-sized segments (no tensor straddles a page)."""
    pieces = []
    off = HEADER_BYTES

    def place(nbytes: int) -> int:
        nonlocal off
        off = (off + 255) // 256 * 256
        if nbytes > page_bytes:
            raise ValueError(f"tensor of {nbytes} B exceeds the {page_bytes} B page")
        if off // page_bytes != (off + nbytes - 1) // page_bytes:
            off = (off // page_bytes + 1) * page_bytes
        at = off
        off += nbytes
        return at

    locs = []
    for lay, (w, b, pre) in zip(spec.layers, folded):
        wo = bo = so = -1
        rows = k = 0
        if w is not None:
            wb = to_bf16_bits(w).tobytes()
            bb = b.astype(np.float32).tobytes()
            wo, bo = place(len(wb)), place(len(bb))
            pieces += [(wo, wb), (bo, bb)]
            rows, k = lay.cout_pad, lay.kpad
        if pre is not None:
            sb = pre.astype(np.float32).tobytes()
            so = place(len(sb))
            pieces.append((so, sb))
        locs.append((wo, bo, rows, k, so))
    data = np.zeros(off, np.uint8)
    for at, buf in pieces:
        data[at:at + len(buf)] = np.frombuffer(buf, np.uint8)
    pages = (off + page_bytes - 1) // page_bytes
    return Blob(data, locs, pages, page_bytes)


def weights_bytes(spec: ArchSpec) -> int:
    """Folded parameter bytes (bf16 weights at real K + fp32 bias + pre-BN scale/shift)."""
    n = 0
    for lay in spec.layers:
        if lay.kind == "conv":
            taps = 1 if lay.layout == "avg3" else lay.kh * lay.kw
            n += lay.cout * taps * (lay.cin // lay.groups) * 2 + lay.cout * 4
        elif lay.kind == "fc":
            n += lay.cout * lay.cin * 2 + lay.cout * 4
        if lay.pre_bn:
            n += lay.cin * 8
    return n


def make_inputs(n: int, spec: ArchSpec, first: int = 0) -> np.ndarray:
    """Synthetic request inputs: image i = N(0,1) fp32 [C][H][W] from default_rng(i)."""
    return np.stack([np.random.default_rng(first + i).standard_normal(
        (spec.in_c, spec.in_h, spec.in_w), dtype=np.float32) for i in range(n)])
