"""CPU interpreter of an arch's op list on its FOLDED device weights — TEST INFRASTRUCTURE.

Runs the exact tables the device plans are built from (arch.build_arch ops, buffers,
channel offsets/strides of the concats, paddings, pre-BN prologues, grouped 64-channel
blocks, the avg-pool-as-3x3-conv trick, the im2col stem, the fused stem pool) with the
exact folded weight layouts the blob holds (arch.fold: stem4 / rsc / im2col / avg3 / g64),
in fp32 torch on NCHW tensors. tests/test_arch_tables.py holds it equal to torchvision's
own module (oracle/resnet_oracle.py) on the unfolded parameters: that pins the tables and
the folding on the CPU, before any kernel runs. With bf16=True the activations are rounded
to bf16 at every buffer store and the weights are the blob's bf16 values (the device's
numerics up to accumulation order), to size the device tolerance.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

from paper_2006_02464_b200 import arch as A


def _weights(lay, w: np.ndarray) -> torch.Tensor:
    """Folded [cout_pad][kpad] -> torch conv weight [cout][cin_eff][kh][kw]."""
    cp = lambda c: (c + 63) // 64 * 64  # noqa: E731
    if lay.layout == "stem4":
        w4 = w[:lay.cout].reshape(lay.cout, lay.kh, 8, 4)[:, :, 1:, :lay.cin]  # [co][r][s][c]
        return torch.from_numpy(np.ascontiguousarray(w4.transpose(0, 3, 1, 2)))
    if lay.layout == "im2col":
        wk = w[:lay.cout, :lay.kh * lay.kw * lay.cin].reshape(lay.cout, lay.kh, lay.kw, lay.cin)
        return torch.from_numpy(np.ascontiguousarray(wk.transpose(0, 3, 1, 2)))
    if lay.layout == "g64":
        taps = lay.kh * lay.kw
        full = np.zeros((lay.cout, lay.cin, lay.kh, lay.kw), np.float32)
        wg = w[:lay.cout].reshape(lay.cout, taps, 64)
        for co in range(lay.cout):
            b0 = (co // 64) * 64
            full[co, b0:b0 + 64] = wg[co].T.reshape(64, lay.kh, lay.kw)
        return torch.from_numpy(full)
    taps = lay.kh * lay.kw
    wt = w[:lay.cout].reshape(lay.cout, lay.kh, lay.kw, cp(lay.cin))[:, :, :, :lay.cin]
    return torch.from_numpy(np.ascontiguousarray(wt.transpose(0, 3, 1, 2)))


def run(spec: A.ArchSpec, folded, images: np.ndarray, bf16: bool = False) -> np.ndarray:
    x_in = torch.from_numpy(np.ascontiguousarray(images, dtype=np.float32))
    n = x_in.shape[0]
    bufs: dict[int, torch.Tensor] = {}

    def rnd(t):
        return t.to(torch.bfloat16).to(torch.float32) if bf16 else t

    def wts(i):
        w, b, pre = folded[i]
        if bf16 and w is not None:
            w = A.bf16_to_f32(A.to_bf16_bits(w))
        return w, b, pre

    def store(buf, ctot, coff, val, h, w):
        if buf not in bufs or tuple(bufs[buf].shape) != (n, ctot, h, w):
            bufs[buf] = torch.zeros(n, ctot, h, w)   # (ResNet buffers are reused per stage)
        bufs[buf][:, coff:coff + val.shape[1]] = rnd(val)

    ops = spec.ops
    i = 0
    while i < len(ops):
        op = ops[i]
        k = op["kind"]
        if k == A.OP_STEM:
            bufs[op["out_buf"]] = rnd(x_in)                      # NCHW fp32 -> bf16 rows
        elif k == A.OP_IM2COL:
            bufs[op["out_buf"]] = rnd(x_in)                      # the conv unfolds it
        elif k == A.OP_CONV:
            lay = spec.layers[op["layer"]]
            w, b, pre = wts(op["layer"])
            src = bufs[op["in_buf"]]
            if lay.layout not in ("stem4", "im2col"):
                src = src[:, :op["cin"]]
            if pre is not None:
                src = rnd(torch.relu(src * torch.from_numpy(pre[0, :op["cin"]])[None, :, None, None]
                                     + torch.from_numpy(pre[1, :op["cin"]])[None, :, None, None]))
            wt = _weights(lay, w)
            ph, pw = op["pad"], op["pad_w"]
            stride = op["stride"]
            if lay.layout == "im2col":
                stride, ph, pw = lay.stride, lay.pad_h, lay.pad_w
            if lay.layout == "stem4":
                stride, ph, pw = 2, 3, 3
            y = F.conv2d(F.pad(src, (pw, pw, ph, ph)), wt, stride=stride)
            y = y + torch.from_numpy(b[:lay.cout])[None, :, None, None]
            if op["res_buf"] >= 0:
                y = y + bufs[op["res_buf"]][:, :lay.cout]
            if op["relu"]:
                y = torch.relu(y)
            if lay.layout == "stem4":
                y = rnd(y)
                nxt = ops[i + 1]                                 # the fused 3x3/s2/p1 max pool
                y = F.max_pool2d(y, 3, 2, 1)
                store(nxt["out_buf"], nxt["out_ctot"], nxt["out_coff"], y, *y.shape[2:])
                i += 2
                continue
            store(op["out_buf"], op["out_ctot"], op["out_coff"], y, *y.shape[2:])
        elif k == A.OP_MAXPOOL:
            src = bufs[op["in_buf"]][:, :op["cin"]]
            y = F.max_pool2d(src, op["kh"], op["stride"], op["pad"])
            store(op["out_buf"], op["out_ctot"], op["out_coff"], y, *y.shape[2:])
        elif k == A.OP_BNPOOL:
            _, _, pre = wts(op["pre_layer"])
            src = bufs[op["in_buf"]][:, :op["cin"]]
            c = op["cin"]
            y = torch.relu(src * torch.from_numpy(pre[0, :c])[None, :, None, None]
                           + torch.from_numpy(pre[1, :c])[None, :, None, None])
            y = F.avg_pool2d(y, 2, 2)
            store(op["out_buf"], op["out_ctot"], 0, y, *y.shape[2:])
        elif k == A.OP_AVGPOOL:
            src = bufs[op["in_buf"]][:, :op["cin"]]
            if op["pre_layer"] >= 0:
                _, _, pre = wts(op["pre_layer"])
                c = op["cin"]
                src = torch.relu(src * torch.from_numpy(pre[0, :c])[None, :, None, None]
                                 + torch.from_numpy(pre[1, :c])[None, :, None, None])
            bufs[op["out_buf"]] = src.mean(dim=(2, 3))           # fp32 pooled features
        elif k == A.OP_FC:
            lay = spec.layers[op["layer"]]
            w, b, _ = wts(op["layer"])
            feat = bufs[op["in_buf"]]
            out = feat @ torch.from_numpy(w[:lay.cout, :lay.cin]).T + torch.from_numpy(b[:lay.cout])
            return out.numpy()
        i += 1
    raise RuntimeError("op list has no FC")
