"""The controller fast path (csrc/sched.cpp via native_scheduler.NativeScheduler) against the
reference scheduler it replaces (sloserve/scheduler.py + controller_state.py).

The reference harness runs the same simulated experiment twice — once with its own
Scheduler, once with NativeScheduler in its place — and every request row (id, model,
arrival, deadline, status, latency, served batch, cold start), every action row (id, kind,
model, worker, gpu, batch, status, predicted start / result end / duration, worker start /
end / duration) and the summary totals must be identical: decision-for-decision parity,
including the float load statistics and the tie orders. Workloads cover closed and open
loops, replayed synthetic traces, eviction-heavy page pressure, several workers and GPUs,
lognormal duration jitter (estimator updates, rejected-too-late retries) and network delay.
Skipped where the read-only reference is not mounted (it is test infrastructure only).
"""

import ctypes as C
import os
import random
import sys

import pytest

from paper_2006_02464_b200 import _lib

REF = "/root/reference/pkg/src"


def test_fsum_matches_cpython_sum():
    """The load statistics sum floats with CPython 3.12's compensated sum(): bit-exact."""
    rng = random.Random(7)
    for n in [1, 2, 3, 5, 8, 17, 64]:
        for _ in range(200):
            xs = [rng.choice([1.0, 1e-3, 1e9, 1e16]) * rng.uniform(-1, 1) for _ in range(n)]
            arr = (C.c_double * n)(*xs)
            assert _lib.lib.cw_sched_fsum(arr, n) == sum(xs), xs
    assert _lib.lib.cw_sched_fsum((C.c_double * 1)(0.0), 0) == sum([])


@pytest.fixture(scope="module")
def sloserve():
    if not os.path.isdir(REF):
        pytest.skip("reference not mounted")
    sys.path.insert(0, REF)
    import sloserve.harness as harness
    import sloserve.workload as workload
    import sloserve.worker as worker
    return harness, workload, worker


def _run(harness, cfg, native, monkeypatch):
    from paper_2006_02464_b200.native_scheduler import NativeScheduler
    if native:
        monkeypatch.setattr(harness, "Scheduler", NativeScheduler)
    else:
        monkeypatch.undo()
    res = harness.run_experiment(cfg)
    return res.sink.request_rows, res.sink.action_rows, res.summary.to_dict()


def _configs(harness, workload, worker):
    trace = workload.gen_synthetic_trace(12, 2, seed=3)
    return {
        "closed_evictions": harness.ExperimentConfig(
            name="a", mode="sim", horizon_ns=2_000_000_000, replicate=[("resnet50", 6)],
            workers=[harness.WorkerSpec(gpu_count=1, pages_per_gpu=30)],
            groups=[workload.ClientGroup(kind="closed", concurrency=8,
                                         model_ids=[2, 5, 6, 7, 8, 9], slo_ns=100_000_000)]),
        "open_two_workers_jitter": harness.ExperimentConfig(
            name="b", mode="sim", seed=5, horizon_ns=2_000_000_000,
            replicate=[("resnet50", 8)], net_delay_ns=200_000,
            jitter=worker.JitterSpec(kind="lognormal", sigma=0.2),
            workers=[harness.WorkerSpec(gpu_count=2, pages_per_gpu=40),
                     harness.WorkerSpec(gpu_count=1, pages_per_gpu=60)],
            groups=[workload.ClientGroup(kind="open", rate=1500.0,
                                         model_ids=list(range(5, 13)), slo_ns=50_000_000),
                    workload.ClientGroup(kind="closed", concurrency=4, model_ids=[3],
                                         slo_ns=25_000_000)]),
        "replay_trace_cold": harness.ExperimentConfig(
            name="c", mode="sim", seed=1, horizon_ns=3_000_000_000,
            replicate=[("resnet50", 40)],
            workers=[harness.WorkerSpec(gpu_count=2, pages_per_gpu=50)],
            groups=[workload.ClientGroup(kind="replay", trace=trace, scale=30.0,
                                         model_ids=list(range(5, 45)), slo_ns=100_000_000)]),
        "tight_slo_mixed": harness.ExperimentConfig(
            name="d", mode="sim", seed=9, horizon_ns=2_000_000_000,
            jitter=worker.JitterSpec(kind="lognormal", sigma=0.5),
            workers=[harness.WorkerSpec(gpu_count=1, pages_per_gpu=20)],
            groups=[workload.ClientGroup(kind="open", rate=800.0, model_ids=[0, 1, 2, 3, 4],
                                         slo_ns=12_000_000),
                    workload.ClientGroup(kind="open", rate=300.0, model_ids=[2, 4],
                                         slo_ns=400_000_000, stagger_ns=300_000_000,
                                         assign="uniform_active")]),
    }


@pytest.mark.parametrize("case", ["closed_evictions", "open_two_workers_jitter",
                                  "replay_trace_cold", "tight_slo_mixed"])
def test_native_scheduler_matches_reference_decision_for_decision(sloserve, monkeypatch, case):
    harness, workload, worker = sloserve
    cfg = _configs(harness, workload, worker)[case]
    ref_req, ref_act, ref_sum = _run(harness, cfg, False, monkeypatch)
    cfg = _configs(harness, workload, worker)[case]
    nat_req, nat_act, nat_sum = _run(harness, cfg, True, monkeypatch)
    assert len(ref_req) > 100 and len(ref_act) > 20
    assert nat_act == ref_act
    assert nat_req == ref_req
    assert nat_sum == ref_sum
