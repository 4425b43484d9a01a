"""Drop-in checks with the reference controller (only where the read-only
reference is mounted, i.e. the build container; skipped elsewhere):

* In-process sim: the reference harness (scheduler + clients) driving the
  B200Worker in sim mode yields the same experiment summary as with the
  reference EmulatedWorker.
* Wall clock over TCP: the unmodified reference controller connects to our
  server (sim-mode engine in wall time) by address and completes a workload.
"""

import os
import sys
import threading

import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")


@pytest.fixture(scope="module")
def sloserve():
    sys.path.insert(0, REF)
    import sloserve.harness as harness
    import sloserve.workload as workload
    return harness, workload


def _config(harness, workload, **kw):
    cfg = harness.ExperimentConfig(
        name="t", mode="sim", horizon_ns=2_000_000_000, replicate=[("resnet50", 4)],
        workers=[harness.WorkerSpec(gpu_count=1, pages_per_gpu=30)],
        groups=[workload.ClientGroup(kind="closed", concurrency=8, model_ids=[2, 5, 6, 7],
                                     slo_ns=100_000_000)],
        **kw)
    return cfg


def test_sim_harness_with_b200_sim_worker_matches_reference(sloserve, monkeypatch):
    harness, workload = sloserve
    ref = harness.run_experiment(_config(harness, workload)).summary.to_dict()

    from paper_2006_02464_b200.worker import B200Worker

    def factory(wid, catalog, loop, send_result, **kw):
        kw.pop("jitter", None)
        return B200Worker(wid, catalog, loop, send_result, mode="sim", **kw)

    monkeypatch.setattr(harness, "EmulatedWorker", factory)
    ours = harness.run_experiment(_config(harness, workload)).summary.to_dict()
    assert ours["totals"] == ref["totals"]
    assert abs(ours["goodput_rps"] - ref["goodput_rps"]) <= 0.01 * ref["goodput_rps"]


@pytest.mark.parametrize("native", [False, True], ids=["python-net", "native-net"])
def test_reference_controller_over_tcp(sloserve, tmp_path, native):
    """native-net: the connection is served by cw_net_serve (csrc/net.cpp), which also runs
    the sim engine's event loop in wall time."""
    harness, workload = sloserve
    import time

    from paper_2006_02464_b200 import catalog, server
    from sloserve import profiles

    cat_text = profiles.dumps_catalog(profiles.reference_catalog())
    epoch = time.time_ns() + 500_000_000
    ports = []
    ready = threading.Event()
    t = threading.Thread(target=server.serve, args=("127.0.0.1:0", catalog.parse(cat_text)),
                         kwargs=dict(pages_per_gpu=100, epoch_ns=epoch, mode="sim",
                                     worker_id=0, telemetry_path=str(tmp_path / "w.csv"),
                                     native=native,
                                     on_ready=lambda p: (ports.append(p), ready.set())),
                         daemon=True)
    t.start()
    assert ready.wait(30)
    cfg = harness.ExperimentConfig(
        name="tcp", mode="wall", transport="tcp", horizon_ns=1_500_000_000, catalog_text=cat_text,
        workers=[harness.WorkerSpec(address=f"127.0.0.1:{ports[0]}")], epoch_ns=epoch,
        groups=[workload.ClientGroup(kind="open", rate=100.0, model_ids=[3], slo_ns=100_000_000)])
    res = harness.run_experiment(cfg)
    s = res.summary
    assert s.offered_rps * 1.5 > 50
    assert s.satisfaction >= 0.9, s.to_dict()
    t.join(timeout=60)  # the reference harness drops its reader socket ~10 s after the run
    assert (tmp_path / "w.csv").exists()
    rows = open(tmp_path / "w.csv").read().splitlines()
    assert rows[0].startswith("action_id,kind") and len(rows) > 50
