"""N > 1 path (replicas only): one independent worker per GPU,
requests (not tensors) sharded by the controller, no data-path collective.

* gloo world_size 2: each rank runs its own native engine (sim device) on its
  own shard of a seeded action stream, exactly as `bench.py --gpus N` does on
  B200s; the only cross-rank traffic is bench.py's timing reduction
  (max over ranks) and the request-count sum. Shard results must equal the
  single-process run of the same shards.
* two external TCP workers with distinct --worker-id behind the unmodified
  reference controller (the reference hard-codes worker id 0,
  harness.py:550, so this is the configuration that needs our server).
"""

import os
import socket
import sys
import threading

import pytest
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg/src"


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _shard_results(rank: int, world: int):
    """Run scenario shards rank, rank+world, ... through the native engine (sim)."""
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    from helpers import run_engine, scenario
    out = []
    for i in range(rank, 8, world):
        r = run_engine(scenario(i))
        out.append((i, len(r["results"]), sum(x[1] == 1 for x in r["results"]),
                    [f[0] for f in r["final"]]))
    return out


def _worker(rank: int, world: int, port: int, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, REPO)
    import bench
    d = bench.Dist()
    assert d.dist.get_backend() == "gloo"   # no NCCL: replicas exchange no tensors
    res = _shard_results(rank, world)
    d.barrier()
    n_ok = d.sum(float(sum(r[2] for r in res)))
    t_max = d.max(float(rank + 1))  # bench.py reports the max over ranks of the timed region
    q.put((rank, res, n_ok, t_max))
    d.close()


def test_replicas_gloo_world_size_2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    got = []
    while len(got) < world:
        try:
            got.append(q.get(timeout=5))
        except queue.Empty:
            assert all(p.is_alive() or p.exitcode == 0 for p in procs), "a rank died"
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    by_rank = {g[0]: g for g in got}
    # shards equal the single-process engine on the same scenarios
    single = {r[0]: r for r in _shard_results(0, 1)}
    total_ok = 0
    for rank in range(world):
        for shard in by_rank[rank][1]:
            assert tuple(shard) == tuple(single[shard[0]])
            total_ok += shard[2]
    # the cross-rank reductions bench.py uses
    assert all(g[2] == total_ok for g in got)
    assert all(g[3] == float(world) for g in got)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_two_external_workers_distinct_ids_behind_reference_controller(tmp_path):
    sys.path.insert(0, REF)
    import time

    import sloserve.harness as harness
    import sloserve.workload as workload
    from sloserve import profiles

    from paper_2006_02464_b200 import catalog, server

    cat_text = profiles.dumps_catalog(profiles.reference_catalog())
    epoch = time.time_ns() + 800_000_000
    ports = {}
    threads = []
    for wid in (0, 1):
        ready = threading.Event()
        t = threading.Thread(
            target=server.serve, args=("127.0.0.1:0", catalog.parse(cat_text)),
            kwargs=dict(pages_per_gpu=20, epoch_ns=epoch, mode="sim", worker_id=wid,
                        telemetry_path=str(tmp_path / f"w{wid}.csv"),
                        on_ready=lambda p, wid=wid, ev=ready: (ports.__setitem__(wid, p), ev.set())),
            daemon=True)
        t.start()
        assert ready.wait(30)
        threads.append(t)
    cfg = harness.ExperimentConfig(
        name="tcp2", mode="wall", transport="tcp", horizon_ns=1_500_000_000,
        catalog_text=cat_text, epoch_ns=epoch,
        workers=[harness.WorkerSpec(address=f"127.0.0.1:{ports[w]}") for w in (0, 1)],
        # all five reference models (35 pages) cannot fit one 20-page worker
        groups=[workload.ClientGroup(kind="open", rate=300.0, model_ids=[0, 1, 2, 3, 4],
                                     slo_ns=100_000_000)])
    res = harness.run_experiment(cfg)
    assert res.summary.satisfaction >= 0.9, res.summary.to_dict()
    for t in threads:
        t.join(timeout=30)
    assert not any(t.is_alive() for t in threads), "worker servers did not shut down"
    # both workers executed actions (requests were sharded across them)
    rows = [sum(1 for _ in open(tmp_path / f"w{w}.csv")) - 1 for w in (0, 1)]
    assert all(r > 0 for r in rows), rows


@pytest.mark.skipif(not os.path.isdir(os.path.join(REPO, "baseline", "_ref", "sloserve")),
                    reason="baseline/_ref (reference install) missing")
def test_bench_controller_leg_two_workers_sim():
    """bench.py's configs[2] leg as it runs at N=2: the unmodified reference controller
    (baseline/_ref) replays the synthetic trace against two worker processes with distinct
    ids (sim engines here, one cuda worker per GPU on the box); both receive INFERs."""
    sys.path.insert(0, REPO)
    import bench_e2e
    h = 3_000_000_000
    r = bench_e2e.run_leg(
        "b200-sim", lambda wl: [bench_e2e.trace_group(wl, 50, 400.0, h, 1)[0]],
        50, 200, h, [0, 1], startup_s=20.0)
    assert r["workers"] == 2 and r["infer_actions"] > 100
    assert r["satisfaction"] > 0.9, r
    assert r["totals"]["over_slo"] == 0
