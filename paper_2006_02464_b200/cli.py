"""Worker command line, flag-compatible with `sloserve worker`
(pkg/src/sloserve/cli.py:140-152) plus the B200 additions.

    python -m paper_2006_02464_b200 worker --listen HOST:PORT --catalog FILE
        [--gpus N] [--pages N] [--clock wall] [--jitter none] [--seed N]
        [--epoch-ns N] [--telemetry FILE]
        [--worker-id N] [--devices 0,1,...] [--mode cuda|sim] [--weights-seed N]
        [--native-net] [--weights DIR] [--softmax]
    python -m paper_2006_02464_b200 pack --arch resnet50 (--state-dict SD.npz | --random-seed N)
        --out resnet50.cwm
"""

from __future__ import annotations

import argparse
import sys

from . import catalog as catalog_mod
from . import server


def _parse_jitter(text: str):
    if text not in ("", "none"):
        kind, _, sigma = text.partition(":")
        if kind != "lognormal" or float(sigma) != 0.0:
            raise SystemExit("worker: jitter injection is emulation-only; the B200 worker "
                             "reports measured device durations")
    return None


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2006_02464_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("worker", help="serve a B200 worker over TCP")
    p.add_argument("--listen", required=True, help="host:port (port 0 for ephemeral)")
    p.add_argument("--catalog", required=True)
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--pages", type=int, default=500)
    p.add_argument("--clock", choices=["sim", "wall"], default="wall")
    p.add_argument("--jitter", default="none")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--epoch-ns", type=int, default=None)
    p.add_argument("--telemetry", default="")
    p.add_argument("--ready-fd", type=int, default=-1, help=argparse.SUPPRESS)
    p.add_argument("--worker-id", type=int, default=0)
    p.add_argument("--devices", default="", help="comma-separated CUDA devices, one per gpu")
    p.add_argument("--mode", choices=["cuda", "sim"], default="cuda")
    p.add_argument("--weights-seed", type=int, default=0)
    p.add_argument("--native-net", action="store_true",
                   help="serve the controller socket from native threads (csrc/net.cpp)")
    p.add_argument("--weights", default="",
                   help="directory of <arch>.cwm model artifacts (default: random-init weights)")
    p.add_argument("--peer-load", action="store_true",
                   help="with --gpus > 1: LOAD from another GPU holding the model (NVLink)")
    p.add_argument("--softmax", action="store_true",
                   help="INFER outputs class probabilities (softmax tail) instead of logits")
    k = sub.add_parser("pack", help="fold + pack a torchvision-named state dict (.npz) into a "
                                    ".cwm model artifact")
    k.add_argument("--arch", required=True)
    k.add_argument("--state-dict", default="", help=".npz of named arrays (torchvision naming)")
    k.add_argument("--random-seed", type=int, default=None,
                   help="pack random-init weights instead (make_params seed)")
    k.add_argument("--page-bytes", type=int, default=16 * 1024 * 1024)
    k.add_argument("--out", required=True)
    args = ap.parse_args(argv)
    if args.cmd == "pack":
        return _pack(args)
    if args.clock == "sim":
        print("worker: simulated clock mode only makes sense in-process", file=sys.stderr)
        return 2
    devices = [int(d) for d in args.devices.split(",")] if args.devices else None
    server.serve(args.listen, catalog_mod.load(args.catalog), args.gpus, args.pages,
                 _parse_jitter(args.jitter), args.seed, args.epoch_ns,
                 telemetry_path=args.telemetry,
                 ready_fd=args.ready_fd if args.ready_fd >= 0 else None,
                 worker_id=args.worker_id, devices=devices, mode=args.mode,
                 weights_seed=args.weights_seed, native=args.native_net,
                 weights_dir=args.weights or None, softmax=args.softmax,
                 peer_load=args.peer_load)
    return 0


def _pack(args) -> int:
    import numpy as np

    from . import arch, artifact
    if args.state_dict:
        with np.load(args.state_dict) as z:
            sd = {k: z[k] for k in z.files}
    elif args.random_seed is not None:
        sd = arch.make_params(arch.build_arch(args.arch), seed=args.random_seed)
    else:
        print("pack: --state-dict or --random-seed is required", file=sys.stderr)
        return 2
    blob = artifact.from_state_dict(args.arch, sd, page_bytes=args.page_bytes)
    artifact.save(args.out, args.arch, blob)
    print(f"{args.out}: {args.arch}, {blob.pages} pages of {blob.page_bytes} B")
    return 0


if __name__ == "__main__":
    sys.exit(main())
