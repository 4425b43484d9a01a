"""The same wall-clock experiment behind the reference controller twice — once with its own
Scheduler, once with NativeScheduler (csrc/sched.cpp) in its place — against B200 worker
processes over TCP (bench_e2e.run_leg). Measurement helper for SURVEY §8(f) rank 1.

    python tools/ctl_compare.py cold|hot [seconds]

cold: configs[1] (1000 ResNet-50 copies, 500 pages, 1000 req/s open loop uniform over copies)
hot:  16 copies resident, 15k req/s open loop: the controller, not the GPU, is the limit
"""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench_e2e  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "hot"
    secs = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0
    h = int(secs * 1e9)
    if which == "cold":
        copies, pages, rate = 1000, 500, 1000.0
        group = lambda wl: [bench_e2e.cold_group(wl, copies, rate)]  # noqa: E731
    else:
        copies, pages, rate = 16, 8000, 15000.0
        group = lambda wl: [wl.ClientGroup(kind="open", model_ids=list(range(copies)),  # noqa: E731
                                           slo_ns=bench_e2e.SLO_NS, rate=rate, name="hot")]
    out = {"workload": which, "seconds": secs, "copies": copies, "pages": pages, "rate": rate}
    for name, native in (("reference_scheduler", False), ("native_scheduler", True)):
        r = bench_e2e.run_leg("b200", group, copies, pages, h, [0], 120.0, native_sched=native)
        out[name] = {k: r[k] for k in ("goodput_rps", "offered_rps", "satisfaction", "mean_batch",
                                       "rejected_too_late", "latency_p99_ms", "actions",
                                       "cold_starts", "wall_s")}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
