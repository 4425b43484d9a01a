"""Worker command line, flag-compatible with `sloserve worker`
(pkg/src/sloserve/cli.py:140-152) plus the B200 additions.

    python -m paper_2006_02464_b200 worker --listen HOST:PORT --catalog FILE
        [--gpus N] [--pages N] [--clock wall] [--jitter none] [--seed N]
        [--epoch-ns N] [--telemetry FILE]
        [--worker-id N] [--devices 0,1,...] [--mode cuda|sim] [--weights-seed N]
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
    args = ap.parse_args(argv)
    if args.clock == "sim":
        print("worker: simulated clock mode only makes sense in-process", file=sys.stderr)
        return 2
    devices = [int(d) for d in args.devices.split(",")] if args.devices else None
    server.serve(args.listen, catalog_mod.load(args.catalog), args.gpus, args.pages,
                 _parse_jitter(args.jitter), args.seed, args.epoch_ns,
                 telemetry_path=args.telemetry,
                 ready_fd=args.ready_fd if args.ready_fd >= 0 else None,
                 worker_id=args.worker_id, devices=devices, mode=args.mode,
                 weights_seed=args.weights_seed, native=args.native_net)
    return 0


if __name__ == "__main__":
    sys.exit(main())
