"""Diagnose the configs[2] e2e leg: one cuda B200 worker served in-process (native net loop,
no Python on its action path) behind the unmodified reference controller (baseline/_ref),
then the worker's executor counters, the globaltimer drift since open, and the
controller's predicted-vs-actual INFER start times.

    python tools/e2e_diag.py [--seconds 20] [--rate 2500] [--pages 8000] [--copies 1000]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import bench_e2e  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=20)
    ap.add_argument("--rate", type=float, default=2500)
    ap.add_argument("--pages", type=int, default=8000)
    ap.add_argument("--copies", type=int, default=1000)
    ap.add_argument("--kind", default="trace", choices=["trace", "cold"])
    ap.add_argument("--out", default="gpurun_out/e2e_diag.json")
    args = ap.parse_args()
    harness, workload, profiles = bench_e2e.sloserve()
    from paper_2006_02464_b200 import catalog, server

    cat = bench_e2e.catalog_text("b200", args.copies)
    epoch = time.time_ns() + 40_000_000_000
    box = {}
    ready = threading.Event()

    def on_ready(port):
        box["port"] = port
        ready.set()

    orig = server.B200Worker

    def keep(*a, **kw):
        w = orig(*a, **kw)
        box["worker"] = w
        return w

    server.B200Worker = keep
    t = threading.Thread(target=server.serve, args=("127.0.0.1:0", catalog.parse(cat)),
                         kwargs=dict(pages_per_gpu=args.pages, epoch_ns=epoch, mode="cuda",
                                     devices=[0], native=True, on_ready=on_ready), daemon=True)
    t.start()
    assert ready.wait(120)
    w = box["worker"]
    time.sleep(max(0.0, (epoch - time.time_ns()) / 1e9))
    h = int(args.seconds * 1e9)
    if args.kind == "trace":
        groups = [bench_e2e.trace_group(workload, args.copies, args.rate, h, 1)[0]]
    else:
        groups = [bench_e2e.cold_group(workload, args.copies, args.rate)]
    cfg = harness.ExperimentConfig(
        name="diag", mode="wall", transport="tcp", horizon_ns=h, catalog_text=cat,
        workers=[harness.WorkerSpec(address=f"127.0.0.1:{box['port']}")], epoch_ns=epoch,
        groups=groups, keep_request_records=False, keep_action_records=True)
    res = harness.run_experiment(cfg)
    stats = w.engine.stats(0)
    drift = w.engine.clock_drift(0)
    rows = [r for r in res.sink.action_rows if r[1] == "infer"]
    ok = np.array([r[10] - r[7] for r in rows if r[6] == "success"], np.int64)
    rej = np.array([r[10] - r[7] for r in rows if r[6] == "rejected_too_late"], np.int64)
    dur_err = np.array([r[12] - r[9] for r in rows if r[6] == "success"], np.int64)

    def q(a):
        if len(a) == 0:
            return None
        return {p: float(np.percentile(a, p)) / 1e3 for p in (1, 10, 50, 90, 99)}

    n = max(stats["dispatched"], 1)
    derived = {"busy_gap_mean_us": stats["busy_gap_sum_ns"] / max(stats["busy_gaps"], 1) / 1e3,
               "launch_lat_mean_us": stats["launch_lat_sum_ns"] / n / 1e3,
               "observe_lat_mean_us": stats["observe_lat_sum_ns"] / n / 1e3,
               "dispatch_delay_mean_us": stats["dispatch_delay_sum_ns"] / n / 1e3}
    out = {"derived": derived, "summary": {k: v for k, v in res.summary.to_dict().items() if k != "intervals"},
           "engine_stats": stats, "clock_drift_us": drift / 1e3,
           "start_minus_predicted_us_ok": q(ok), "start_minus_predicted_us_rejected": q(rej),
           "device_minus_predicted_duration_us": q(dur_err),
           "n_ok": int(len(ok)), "n_rej": int(len(rej))}
    s = json.dumps(out, indent=1)
    print(s)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        f.write(s)
    os._exit(0)


if __name__ == "__main__":
    main()
