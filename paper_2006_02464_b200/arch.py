"""Model artifacts for the B200 worker: architecture tables, deterministic
random-init parameters, BatchNorm folding and the 16 MiB-paged weight blob.

This is the artifact side of the paper's model compilation step (PAPER.md
§5.1: weights + per-batch kernels + memory metadata). The
reference ships profiles only (pkg/src/sloserve/profiles.py:1-8, "profiles are
plain data files that stand in for compiled models"); here a catalog base name
(`resnet50`, ...) maps to a real network.

Networks follow the torchvision ResNet definitions (v1.5: stride on the 3x3
conv of the bottleneck), with parameters named exactly like torchvision's
state_dict so the CPU oracle can load them into torchvision's own modules.

Blob layout (all offsets are blob byte offsets; blob offset o lives in blob
page o // page_bytes at in-page offset o % page_bytes):
    [0, 64 KiB)   header, filled at LOAD with the page-resolved tensor maps
    tensors       per layer: folded weights bf16 [Cout][K] (K = KH*KW*Cin,
                  tap-major / channel-minor, zero-padded to a multiple of 64),
                  folded bias fp32 [Cout]; 256-byte aligned, never straddling a page.
"""

from __future__ import annotations

import zlib
from dataclasses import dataclass, field

import numpy as np

HEADER_BYTES = 65536
BN_EPS = 1e-5

OP_STEM, OP_CONV, OP_MAXPOOL, OP_AVGPOOL, OP_FC = 0, 1, 2, 3, 4

# Workspace buffer ids.
BUF_IM2COL, BUF_STEM, BUF_X0, BUF_X1, BUF_T1, BUF_T2, BUF_DS, BUF_POOL = range(8)


@dataclass
class Layer:
    """One weight-bearing layer (a header index)."""
    index: int
    name: str            # torchvision module name of the conv / fc
    bn: str | None       # torchvision module name of its BatchNorm (None for fc)
    cin: int
    cout: int
    k: int               # kernel size (square)
    stride: int
    pad: int
    kpad: int            # stored K
    layout: str = "rsc"  # K order: "rsc" = (r, s, c); "stem4" = (r, q, c4), see fold()


@dataclass
class ArchSpec:
    name: str
    in_c: int = 3
    in_h: int = 224
    in_w: int = 224
    classes: int = 1000
    layers: list[Layer] = field(default_factory=list)
    ops: list[dict] = field(default_factory=list)
    flops_per_image: int = 0   # algorithmic (unpadded K), conv + fc

    def op_structs(self):
        from . import _lib  # lazily: the tables themselves load no native code
        arr = (_lib.cw_op * len(self.ops))()
        for i, op in enumerate(self.ops):
            for k, v in op.items():
                setattr(arr[i], k, int(v))
        return arr


_RESNETS = {
    "resnet18": ("basic", [2, 2, 2, 2]),
    "resnet34": ("basic", [3, 4, 6, 3]),
    "resnet50": ("bottleneck", [3, 4, 6, 3]),
    "resnet101": ("bottleneck", [3, 4, 23, 3]),
    "resnet152": ("bottleneck", [3, 8, 36, 3]),
}

SUPPORTED = tuple(_RESNETS)


def _op(kind, **kw):
    d = dict(kind=kind, layer=-1, in_buf=-1, out_buf=-1, res_buf=-1, cin=0, cout=0, kh=1, kw=1,
             stride=1, pad=0, relu=0, in_h=0, in_w=0, out_h=0, out_w=0, kpad=0, reserved=0)
    d.update(kw)
    return d


def build_arch(name: str) -> ArchSpec:
    """Layer table + op list of a torchvision-definition ResNet."""
    if name not in _RESNETS:
        raise KeyError(f"no B200 implementation for architecture {name!r} "
                       f"(supported: {', '.join(SUPPORTED)})")
    block, counts = _RESNETS[name]
    spec = ArchSpec(name)
    flops = 0

    def add_layer(lname, bn, cin, cout, k, stride, pad, kpad=None, layout="rsc"):
        kp = kpad if kpad is not None else k * k * cin
        assert kp % 64 == 0 or layout == "stem4", (lname, kp)
        lay = Layer(len(spec.layers), lname, bn, cin, cout, k, stride, pad, kp, layout)
        spec.layers.append(lay)
        return lay

    def conv(lname, bn, cin, cout, k, stride, pad, h, w, in_buf, out_buf, relu, res_buf=-1):
        nonlocal flops
        oh = (h + 2 * pad - k) // stride + 1
        ow = (w + 2 * pad - k) // stride + 1
        lay = add_layer(lname, bn, cin, cout, k, stride, pad)
        spec.ops.append(_op(OP_CONV, layer=lay.index, in_buf=in_buf, out_buf=out_buf,
                            res_buf=res_buf, cin=cin, cout=cout, kh=k, kw=k, stride=stride,
                            pad=pad, relu=relu, in_h=h, in_w=w, out_h=oh, out_w=ow,
                            kpad=lay.kpad))
        flops += 2 * oh * ow * cout * k * k * cin
        return oh, ow

    # Stem: the input stage converts fp32 NCHW to bf16 NHWC4 rows (channel 3 = 0,
    # zero pixels either side); the 7x7/s2 conv reads overlapping 8-pixel row
    # windows of those rows, K = 7 kernel rows x (8 pixels x 4 channels) = 224.
    h = w = 224
    spec.ops.append(_op(OP_STEM, out_buf=BUF_IM2COL, in_h=h, in_w=w, out_h=112, out_w=112,
                        kpad=224, cin=3))
    stem = add_layer("conv1", "bn1", 3, 64, 7, 2, 3, kpad=224, layout="stem4")
    spec.ops.append(_op(OP_CONV, layer=stem.index, in_buf=BUF_IM2COL, out_buf=BUF_STEM, cin=4,
                        cout=64, kh=7, kw=7, stride=2, pad=3, relu=1, in_h=224, in_w=224,
                        out_h=112, out_w=112, kpad=224))
    flops += 2 * 112 * 112 * 64 * 147
    spec.ops.append(_op(OP_MAXPOOL, in_buf=BUF_STEM, out_buf=BUF_X0, cin=64, in_h=112, in_w=112,
                        out_h=56, out_w=56))
    h = w = 56
    x = BUF_X0
    inplanes = 64
    expansion = 4 if block == "bottleneck" else 1
    for li, (planes, n) in enumerate(zip([64, 128, 256, 512], counts)):
        for bi in range(n):
            stride = 2 if (li > 0 and bi == 0) else 1
            pre = f"layer{li + 1}.{bi}"
            y = BUF_X1 if x == BUF_X0 else BUF_X0
            has_ds = stride != 1 or inplanes != planes * expansion
            if block == "bottleneck":
                conv(f"{pre}.conv1", f"{pre}.bn1", inplanes, planes, 1, 1, 0, h, w, x, BUF_T1, 1)
                oh, ow = conv(f"{pre}.conv2", f"{pre}.bn2", planes, planes, 3, stride, 1, h, w,
                              BUF_T1, BUF_T2, 1)
                if has_ds:
                    conv(f"{pre}.downsample.0", f"{pre}.downsample.1", inplanes, planes * 4, 1,
                         stride, 0, h, w, x, BUF_DS, 0)
                conv(f"{pre}.conv3", f"{pre}.bn3", planes, planes * 4, 1, 1, 0, oh, ow, BUF_T2, y,
                     1, res_buf=BUF_DS if has_ds else x)
            else:
                oh, ow = conv(f"{pre}.conv1", f"{pre}.bn1", inplanes, planes, 3, stride, 1, h, w,
                              x, BUF_T1, 1)
                if has_ds:
                    conv(f"{pre}.downsample.0", f"{pre}.downsample.1", inplanes, planes, 1, stride,
                         0, h, w, x, BUF_DS, 0)
                conv(f"{pre}.conv2", f"{pre}.bn2", planes, planes, 3, 1, 1, oh, ow, BUF_T1, y, 1,
                     res_buf=BUF_DS if has_ds else x)
            inplanes = planes * expansion
            x = y
            h, w = oh, ow
    feat = inplanes
    spec.ops.append(_op(OP_AVGPOOL, in_buf=x, out_buf=BUF_POOL, cin=feat, in_h=h, in_w=w,
                        out_h=1, out_w=1))
    fc = add_layer("fc", None, feat, 1000, 1, 1, 0, kpad=feat)
    spec.ops.append(_op(OP_FC, layer=fc.index, in_buf=BUF_POOL, cin=feat, cout=1000))
    flops += 2 * feat * 1000
    spec.flops_per_image = flops
    return spec


# ---------------------------------------------------------------------------- parameters

def _rng(seed: int, name: str) -> np.random.Generator:
    return np.random.default_rng([seed, zlib.crc32(name.encode())])


def make_params(spec: ArchSpec, seed: int = 0) -> dict[str, np.ndarray]:
    """Random-init parameters in torchvision state_dict naming (fp32).

    conv: Kaiming-normal fan_out (torchvision's init); BatchNorm eval statistics
    randomized so folding is exercised: gamma~U[0.5,1], beta~N(0,0.1),
    mean~N(0,0.1), var~U[0.75,1.25]; fc: U(+-1/sqrt(fan_in)).
    """
    p: dict[str, np.ndarray] = {}
    for lay in spec.layers:
        r = _rng(seed, lay.name)
        if lay.bn is None:
            bound = 1.0 / np.sqrt(lay.cin)
            p[f"{lay.name}.weight"] = r.uniform(-bound, bound, (lay.cout, lay.cin)).astype(np.float32)
            p[f"{lay.name}.bias"] = r.uniform(-bound, bound, (lay.cout,)).astype(np.float32)
            continue
        std = np.sqrt(2.0 / (lay.cout * lay.k * lay.k))
        p[f"{lay.name}.weight"] = (r.standard_normal((lay.cout, lay.cin, lay.k, lay.k)) * std
                                   ).astype(np.float32)
        rb = _rng(seed, lay.bn)
        p[f"{lay.bn}.weight"] = rb.uniform(0.5, 1.0, lay.cout).astype(np.float32)
        p[f"{lay.bn}.bias"] = (rb.standard_normal(lay.cout) * 0.1).astype(np.float32)
        p[f"{lay.bn}.running_mean"] = (rb.standard_normal(lay.cout) * 0.1).astype(np.float32)
        p[f"{lay.bn}.running_var"] = rb.uniform(0.75, 1.25, lay.cout).astype(np.float32)
    return p


def fold(spec: ArchSpec, params: dict[str, np.ndarray]) -> list[tuple[np.ndarray, np.ndarray]]:
    """Fold eval-mode BatchNorm into each conv (in float64).

    Returns per layer (W [Cout][K] fp32 in the device K order, bias [Cout] fp32):
    W[co, (r*KW + s)*Cin + c] = w[co, c, r, s] * gamma/sqrt(var+eps), zero-padded to kpad.
    Stem ("stem4"): W[co, r*32 + (s+1)*4 + c] (window pixel 0 and channel 3 are zero),
    matching the NHWC4 row windows the stem conv reads.
    """
    out = []
    for lay in spec.layers:
        w = params[f"{lay.name}.weight"].astype(np.float64)
        if lay.bn is None:
            wk = w
            b = params[f"{lay.name}.bias"].astype(np.float64)
        else:
            g = params[f"{lay.bn}.weight"].astype(np.float64)
            beta = params[f"{lay.bn}.bias"].astype(np.float64)
            mu = params[f"{lay.bn}.running_mean"].astype(np.float64)
            var = params[f"{lay.bn}.running_var"].astype(np.float64)
            scale = g / np.sqrt(var + BN_EPS)
            wk = (w * scale[:, None, None, None]).transpose(0, 2, 3, 1).reshape(lay.cout, -1)
            b = beta - mu * scale
        wpad = np.zeros((lay.cout, lay.kpad), np.float64)
        if lay.layout == "stem4":
            w4 = wpad.reshape(lay.cout, lay.k, 8, 4)
            w4[:, :, 1:, :lay.cin] = wk.reshape(lay.cout, lay.k, lay.k, lay.cin)
        else:
            wpad[:, :wk.shape[1]] = wk
        out.append((wpad.astype(np.float32), b.astype(np.float32)))
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
    locs: list[tuple[int, int, int, int]]   # (w_off, b_off, rows, k) per layer
    pages: int
    page_bytes: int

    def loc_structs(self):
        from . import _lib
        arr = (_lib.cw_tensor_loc * len(self.locs))()
        for i, (w, b, r, k) in enumerate(self.locs):
            arr[i].w_off, arr[i].b_off, arr[i].rows, arr[i].k = w, b, r, k
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
    for lay, (w, b) in zip(spec.layers, folded):
        wb = to_bf16_bits(w).tobytes()
        bb = b.astype(np.float32).tobytes()
        wo = place(len(wb))
        bo = place(len(bb))
        pieces.append((wo, wb))
        pieces.append((bo, bb))
        locs.append((wo, bo, lay.cout, lay.kpad))
    data = np.zeros(off, np.uint8)
    for at, buf in pieces:
        data[at:at + len(buf)] = np.frombuffer(buf, np.uint8)
    pages = (off + page_bytes - 1) // page_bytes
    return Blob(data, locs, pages, page_bytes)


def weights_bytes(spec: ArchSpec) -> int:
    """Folded parameter bytes on the device (bf16 weights at real K + fp32 bias)."""
    n = 0
    for lay in spec.layers:
        k_real = lay.k * lay.k * lay.cin if lay.bn is not None else lay.cin
        n += lay.cout * k_real * 2 + lay.cout * 4
    return n


def make_inputs(n: int, spec: ArchSpec, first: int = 0) -> np.ndarray:
    """Synthetic request inputs: image i = N(0,1) fp32 [C][H][W] from default_rng(i)."""
    return np.stack([np.random.default_rng(first + i).standard_normal(
        (spec.in_c, spec.in_h, spec.in_w), dtype=np.float32) for i in range(n)])
