"""Controller throughput: the reference harness in simulated mode (reference EmulatedWorkers,
open-loop clients) run once with the reference Scheduler and once with NativeScheduler in its
place; reports wall seconds and requests handled per wall second for each, and checks that
the two produced the same summary (decision-for-decision parity on this workload).

    python tools/sched_throughput.py [rate_rps] [horizon_s] [gpus] [models]

Needs the reference sloserve package importable (baseline/_ref or /root/reference/pkg/src).
Profiling / measurement helper (bench.py runs the same comparison as its `controller` leg).
"""
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
for p in (os.path.join(REPO, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(p, "sloserve")):
        sys.path.insert(0, p)
        break


def run(rate=20000.0, horizon_s=1.0, gpus=8, models=64, slo_ms=100):
    import sloserve.harness as harness
    import sloserve.workload as workload

    from paper_2006_02464_b200.native_scheduler import NativeScheduler

    def cfg():
        return harness.ExperimentConfig(
            name="ctl", mode="sim", horizon_ns=int(horizon_s * 1e9),
            replicate=[("resnet50", models)],
            workers=[harness.WorkerSpec(gpu_count=gpus, pages_per_gpu=500)],
            keep_request_records=False, keep_action_records=False,
            groups=[workload.ClientGroup(kind="open", rate=rate,
                                         model_ids=list(range(5, 5 + models)),
                                         slo_ns=slo_ms * 1_000_000)])

    out = {}
    orig = harness.Scheduler
    try:
        for name, sched in (("reference", orig), ("native", NativeScheduler)):
            harness.Scheduler = sched
            t0 = time.perf_counter()
            res = harness.run_experiment(cfg())
            dt = time.perf_counter() - t0
            tot = res.summary.totals
            out[name] = {"wall_s": dt, "arrivals": tot["arrivals"],
                         "requests_per_wall_s": tot["arrivals"] / dt, "totals": tot,
                         "goodput_rps": res.summary.goodput_rps}
    finally:
        harness.Scheduler = orig
    out["same_summary"] = out["reference"]["totals"] == out["native"]["totals"]
    out["speedup"] = out["reference"]["wall_s"] / out["native"]["wall_s"]
    out["config"] = {"rate_rps": rate, "horizon_s": horizon_s, "gpus": gpus, "models": models,
                     "slo_ms": slo_ms, "mode": "sim (reference harness, EmulatedWorker)"}
    return out


if __name__ == "__main__":
    a = [float(x) for x in sys.argv[1:]]
    r = run(*(a[:1] or [20000.0]), *(a[1:2] or [1.0]), *[int(x) for x in a[2:4]])
    print(json.dumps(r, indent=1))
