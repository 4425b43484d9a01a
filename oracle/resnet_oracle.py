"""CPU fp32 numerics oracle for INFER — TEST INFRASTRUCTURE ONLY.

The reference computes no INFER outputs: its Exec is a sleep
(pkg/src/sloserve/worker.py:273-277) and SPEC.md:98 lists "accuracy of any
inference output" as a non-goal. The original arithmetic lived in TVM v0.7
kernels and model-zoo weights that do not ship, so
logits parity is UNPINNED against the reference itself. This oracle is the
stated restatement: the torchvision definition of the same network (the
paper's model zoo was ResNet-50 et al.), evaluated in fp32
on the CPU in eval mode with the UNFOLDED random-init parameters and BatchNorm
statistics, i.e. the exact model whose folded bf16 form the worker runs.
"""

from __future__ import annotations

import numpy as np
import torch
import torchvision


ALIASES = {"inceptionv3": "inception_v3", "resnext50": "resnext50_32x4d"}


def torchvision_model(arch_name: str, params: dict[str, np.ndarray]) -> torch.nn.Module:
    """torchvision's own module for the arch (catalog names accepted), loaded with `params`.
    Inception-v3's auxiliary classifier (training only; not evaluated in eval mode) keeps
    torchvision's own init."""
    name = ALIASES.get(arch_name, arch_name)
    kw = {"aux_logits": True, "init_weights": False} if name == "inception_v3" else {}
    model = getattr(torchvision.models, name)(weights=None, **kw)
    sd = model.state_dict()
    new = {}
    for k, v in sd.items():
        if k.endswith("num_batches_tracked") or (k.startswith("AuxLogits.") and k not in params):
            new[k] = v
        else:
            new[k] = torch.from_numpy(np.ascontiguousarray(params[k]))
    model.load_state_dict(new)
    return model.eval()


@torch.no_grad()
def logits(model: torch.nn.Module, images: np.ndarray, threads: int | None = None) -> np.ndarray:
    if threads:
        torch.set_num_threads(threads)
    x = torch.from_numpy(np.ascontiguousarray(images, dtype=np.float32))
    return model(x).numpy()


def compare(got: np.ndarray, ref: np.ndarray) -> dict:
    """Tolerance (stated in DESIGN.md): top-1 identical on every request and
    max|got - ref| <= 0.02 * max|ref|."""
    err = float(np.abs(got - ref).max())
    scale = float(np.abs(ref).max())
    top_ok = bool((got.argmax(1) == ref.argmax(1)).all())
    return {"max_abs": err, "max_ref": scale, "rel": err / scale, "top1_equal": top_ok,
            "ok": top_ok and err <= 0.02 * scale}
