"""On-disk model artifact (a model is its weights
blob, the page map the worker loads it by, and the per-batch graph metadata).

A `.cwm` file is the device weight blob exactly as LOAD copies it page by page, preceded by
a JSON header:

    b"CWM1"  u32 header_len  header (UTF-8 JSON)  zero pad to 4096  blob (pages x page_bytes)

    header = {"arch": "resnet50", "page_bytes": 16777216, "pages": 4, "blob_bytes": N,
              "layers": [name, ...], "locs": [[w_off, b_off, rows, k], ...],
              "crc32": crc32(blob)}

`locs` is the page map (where each layer's folded bf16 weights and fp32 bias sit; no tensor
straddles a page, arch.pack_blob); the per-batch graph is not stored: it is rebuilt from
the arch tables (`arch.build_arch`) when the worker builds its plans. Weights come from a
torchvision-named state dict (numpy arrays, e.g. an .npz) and are BatchNorm-folded here.
"""

from __future__ import annotations

import json
import struct
import zlib
from typing import Mapping

import numpy as np

from . import arch as arch_mod

MAGIC = b"CWM1"
ALIGN = 4096


class ArtifactError(ValueError):
    pass


def from_state_dict(arch_name: str, state_dict: Mapping[str, np.ndarray],
                    page_bytes: int = 16 * 1024 * 1024) -> arch_mod.Blob:
    """Fold and pack a torchvision-named state dict (conv weights + BatchNorm statistics)."""
    spec = arch_mod.build_arch(arch_name)
    bn_keys = ("weight", "bias", "running_mean", "running_var")
    need = []
    for lay in spec.layers:
        if lay.kind != "bn":
            need.append(f"{lay.name}.weight")
        if lay.kind == "fc":
            need.append(f"{lay.name}.bias")
        for bn in (lay.bn, lay.pre_bn):
            if bn:
                need += [f"{bn}.{f}" for f in bn_keys]
    missing = [k for k in need if k not in state_dict]
    if missing:
        raise ArtifactError(f"{arch_name}: state dict lacks {missing[:4]}"
                            f"{' ...' if len(missing) > 4 else ''}")
    params = {k: np.asarray(v, dtype=np.float32) for k, v in state_dict.items()}
    return arch_mod.pack_blob(spec, arch_mod.fold(spec, params), page_bytes=page_bytes)


def save(path: str, arch_name: str, blob: arch_mod.Blob) -> None:
    spec = arch_mod.build_arch(arch_name)
    if len(blob.locs) != len(spec.layers):
        raise ArtifactError("blob does not match the architecture")
    data = np.ascontiguousarray(blob.data, dtype=np.uint8)
    hdr = json.dumps({"arch": spec.name, "page_bytes": blob.page_bytes, "pages": blob.pages,
                      "blob_bytes": int(data.size), "layers": [l.name for l in spec.layers],
                      "locs": [list(map(int, l)) for l in blob.locs],
                      "crc32": zlib.crc32(data.tobytes())}).encode()
    head = MAGIC + struct.pack("<I", len(hdr)) + hdr
    pad = (-len(head)) % ALIGN
    with open(path, "wb") as f:
        f.write(head + b"\0" * pad)
        f.write(data.tobytes())


def load(path: str) -> tuple[str, arch_mod.Blob]:
    with open(path, "rb") as f:
        raw = f.read()
    if raw[:4] != MAGIC or len(raw) < 8:
        raise ArtifactError(f"{path}: not a CWM1 model artifact")
    (n,) = struct.unpack_from("<I", raw, 4)
    try:
        h = json.loads(raw[8:8 + n])
    except ValueError as e:
        raise ArtifactError(f"{path}: bad header ({e})") from None
    start = (8 + n + ALIGN - 1) // ALIGN * ALIGN
    data = np.frombuffer(raw, np.uint8, count=h["blob_bytes"], offset=start).copy() \
        if len(raw) >= start + h["blob_bytes"] else None
    if data is None:
        raise ArtifactError(f"{path}: truncated blob")
    if zlib.crc32(data.tobytes()) != h["crc32"]:
        raise ArtifactError(f"{path}: blob checksum mismatch")
    spec = arch_mod.build_arch(h["arch"])
    if h["layers"] != [l.name or l.pre_bn for l in spec.layers]:
        raise ArtifactError(f"{path}: layer table does not match arch {h['arch']}")
    locs = [tuple(l) for l in h["locs"]]
    for (w, b, rows, k, so), lay in zip(locs, spec.layers):
        if lay.kind != "bn" and (rows != lay.cout_pad or k != lay.kpad or
                                 max(w, b) >= data.size):
            raise ArtifactError(f"{path}: page map entry for {lay.name} is inconsistent")
        if (so >= 0) != (lay.pre_bn is not None) or so >= data.size:
            raise ArtifactError(f"{path}: input-BatchNorm entry for {lay.name} is inconsistent")
    if h["pages"] * h["page_bytes"] < data.size:
        raise ArtifactError(f"{path}: blob larger than its pages")
    return h["arch"], arch_mod.Blob(data, locs, h["pages"], h["page_bytes"])
