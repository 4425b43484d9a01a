"""Controller-driven legs of bench.py (BASELINE.json configs[2] and configs[1]).

The UNMODIFIED reference controller -- `sloserve` installed from /root/reference/pkg into
baseline/_ref (git-ignored; it travels to the GPU box with the snapshot) -- runs its own
wall-clock experiment (harness._run_wall, pkg/src/sloserve/harness.py:458-513: Scheduler,
ClientManager, TelemetrySink) against external worker processes over TCP
(transport="tcp", WorkerSpec(address=...), harness.py:466-477), and scores it with its own
`summarize` (harness.py:247-291). Nothing of this repo is imported into the controller
process except this file.

Workers, one process per GPU, each started from its own CLI:
  b200       python -m paper_2006_02464_b200 worker --native-net --devices D --worker-id R
             (the drop-in: real LOAD / INFER / UNLOAD on the B200)
  reference  python -m sloserve.cli worker (the reference EmulatedWorker: waits out the
             catalog's V100-profiled durations, pkg/src/sloserve/worker.py:1-9)

Both arms see the same trace, SLO, model set, page budget and weights_bytes (so identical
page accounting); their catalogs differ only in the profiled durations the controller
seeds its estimators with (B200-measured vs the reference's V100 rows, profiles.py:354-363).
"""

from __future__ import annotations

import os
import select
import subprocess
import sys
import tempfile
import time

REPO = os.path.dirname(os.path.abspath(__file__))
REF_SITE = os.path.join(REPO, "baseline", "_ref")
SLO_NS = 100_000_000


def sloserve():
    """The reference package from baseline/_ref (pip --target install of /root/reference/pkg)."""
    if not os.path.isdir(os.path.join(REF_SITE, "sloserve")):
        raise RuntimeError("baseline/_ref/sloserve missing: run `python -m pip install --no-index "
                           "--no-build-isolation --no-deps --target baseline/_ref <copy of "
                           "/root/reference/pkg>` in the build container")
    if REF_SITE not in sys.path:
        sys.path.insert(0, REF_SITE)
    import sloserve.harness as harness
    import sloserve.profiles as profiles
    import sloserve.workload as workload
    return harness, workload, profiles


# ResNet-50 rows. weights_bytes is the reference catalog's (102.3 MB -> 7 pages,
# profiles.py:355) in both, so page accounting is identical; the B200 row's durations are
# this repo's measured device times (BENCH_r01 / profiles/r1_bench_line.json: Exec p50 b=1
# 272 us .. b=16 530 us, LOAD copy ~1 ms, per-request input copy ~25 us), rounded up: the
# controller only seeds its p99-of-10 estimators with them (controller_state.py:19-44).
B200_RESNET50 = """model resnet50
weights_bytes 102300000
weights_transfer_ns 1300000
io_ns 30000 3000
io_bytes 602000 4000
batch 1 300000
batch 2 330000
batch 4 380000
batch 8 460000
batch 16 600000
"""


def catalog_text(kind: str, copies: int) -> str:
    harness, workload, profiles = sloserve()
    if kind in ("b200", "b200-sim"):
        body = "page_bytes 16777216\n" + B200_RESNET50
    else:
        # the reference catalog's own resnet50 record (V100 numbers, profiles.py:354-363)
        text = profiles.dumps_catalog(profiles.reference_catalog())
        recs = text.split("\nmodel ")
        body = recs[0].split("\n")[0] + "\n" + "model " + next(
            r for r in recs[1:] if r.startswith("resnet50\n")).rstrip("\n") + "\n"
    return body + (f"replicas resnet50 {copies - 1}\n" if copies > 1 else "")


def start_worker(kind: str, catalog_path: str, pages: int, epoch_ns: int, device: int = 0,
                 worker_id: int = 0, telemetry: str = "", timeout_s: float = 300.0):
    """Launch one worker process; returns (Popen, port) once it listens."""
    r, w = os.pipe()
    env = dict(os.environ)
    if kind in ("b200", "b200-sim"):  # b200-sim: the same worker, sim engine (CPU tests)
        cmd = [sys.executable, "-m", "paper_2006_02464_b200", "worker", "--native-net",
               "--worker-id", str(worker_id)]
        cmd += ["--mode", "sim"] if kind == "b200-sim" else ["--devices", str(device)]
        env["PYTHONPATH"] = REPO + os.pathsep + env.get("PYTHONPATH", "")
    else:
        cmd = [sys.executable, "-m", "sloserve.cli", "worker"]
        env["PYTHONPATH"] = REF_SITE + os.pathsep + env.get("PYTHONPATH", "")
    cmd += ["--listen", "127.0.0.1:0", "--catalog", catalog_path, "--pages", str(pages),
            "--epoch-ns", str(epoch_ns), "--ready-fd", str(w)]
    if telemetry:
        cmd += ["--telemetry", telemetry]
    proc = subprocess.Popen(cmd, pass_fds=(w,), env=env, cwd=REPO)
    os.close(w)
    ready, _, _ = select.select([r], [], [], timeout_s)
    line = os.read(r, 64).decode().strip() if ready else ""
    os.close(r)
    if not line:
        proc.kill()
        raise RuntimeError(f"{kind} worker did not come up within {timeout_s:.0f} s")
    return proc, int(line)


def trace_group(workload, copies: int, rate: float, horizon_ns: int, seed: int):
    """configs[2]: gen_synthetic_trace (workload.py:151-187) over `copies` workloads mapped
    round-robin onto the copies, replayed (ClientGroup kind="replay") and scaled so that
    the expected arrival rate over the horizon is `rate`."""
    trace = workload.gen_synthetic_trace(copies, 1, seed)
    per_min = sum(c for _, m, c in trace if m == 0)
    scale = rate * 60.0 / max(per_min, 1)
    return workload.ClientGroup(kind="replay", model_ids=list(range(copies)), slo_ns=SLO_NS,
                                trace=trace, scale=scale, name="maf-synthetic"), scale


def cold_group(workload, copies: int, rate: float):
    """configs[1] (Fig. 6 analog): open-loop Poisson arrivals spread
    uniformly over all copies (assign="uniform_active", workload.py:251-261)."""
    return workload.ClientGroup(kind="open", model_ids=list(range(copies)), slo_ns=SLO_NS,
                                rate=rate, assign="uniform_active", name="uniform-cold")


def run_controller(addresses, cat_text: str, epoch_ns: int, horizon_ns: int, groups,
                   seed: int = 0, native_sched: bool = False) -> dict:
    """native_sched: the controller runs this repo's NativeScheduler (the reference
    Scheduler's decisions in C++) in place of sloserve.scheduler.Scheduler;
    everything else (harness, clients, wire, summarize) stays the reference's."""
    harness, workload, profiles = sloserve()
    ref_sched = harness.Scheduler
    if native_sched:
        from paper_2006_02464_b200.native_scheduler import NativeScheduler
        harness.Scheduler = NativeScheduler
    try:
        return _run_controller(harness, addresses, cat_text, epoch_ns, horizon_ns, groups, seed)
    finally:
        harness.Scheduler = ref_sched


def _run_controller(harness, addresses, cat_text, epoch_ns, horizon_ns, groups, seed):
    cfg = harness.ExperimentConfig(
        name="bench", seed=seed, mode="wall", transport="tcp", horizon_ns=horizon_ns,
        catalog_text=cat_text, workers=[harness.WorkerSpec(address=a) for a in addresses],
        epoch_ns=epoch_ns, groups=groups, keep_request_records=False,
        keep_action_records=True)
    t0 = time.time()
    res = harness.run_experiment(cfg)
    wall = time.time() - t0
    s = res.summary
    status = {}
    batches = []
    for row in res.sink.action_rows:
        kind, st = row[1], row[6]
        status[f"{kind}:{st}"] = status.get(f"{kind}:{st}", 0) + 1
        if kind == "infer" and st == "success":
            batches.append(row[5])
    loads = status.get("load:success", 0)
    infers = max(1, len(batches))
    mean_b = sum(batches) / infers if batches else 0.0
    return {
        "goodput_rps": s.goodput_rps, "offered_rps": s.offered_rps,
        "satisfaction": s.satisfaction, "totals": s.totals, "cold_starts": s.cold_starts,
        "latency_p50_ms": (s.latency_p50 or 0) / 1e6, "latency_p99_ms": (s.latency_p99 or 0) / 1e6,
        "latency_max_ms": (s.latency_max or 0) / 1e6, "mean_batch": mean_b,
        "actions": status, "infer_actions": len(batches), "loads": loads,
        "rejected_too_late": sum(v for k, v in status.items() if k.endswith("rejected_too_late")),
        "underprediction_fraction": s.underprediction_fraction,
        "overprediction_fraction": s.overprediction_fraction,
        "horizon_s": horizon_ns / 1e9, "wall_s": wall,
        "h2d_bytes_per_infer": mean_b * 602112 + loads * 54e6 / infers,
        "d2h_bytes_per_infer": mean_b * 4000,
    }


_READY_S: dict = {}  # observed worker startup time per (kind, catalog size), seconds


def run_leg(kind: str, group_fn, copies: int, pages: int, horizon_ns: int, devices,
            startup_s: float, seed: int = 0, workdir: str | None = None,
            cat_text: str | None = None, native_sched: bool = False) -> dict:
    """Start one worker per device, run the reference controller against all of them for
    `horizon_ns`, score with summarize. `group_fn(workload)` builds the client groups;
    `cat_text` overrides the ResNet-50 x `copies` catalog."""
    harness, workload, profiles = sloserve()
    workdir = workdir or tempfile.mkdtemp(prefix="cw_bench_")
    cat = cat_text if cat_text is not None else catalog_text(kind, copies)
    cat_path = os.path.join(workdir, f"catalog_{kind}.txt")
    with open(cat_path, "w") as f:
        f.write(cat)
    # One shared CLOCK_REALTIME epoch, set in the future so it is "now" when the controller
    # starts, after the workers have built their plans (an old epoch would
    # back-date the first arrivals). The lead is the startup time observed for the same kind
    # of worker earlier in this process (+50 %), else `startup_s`.
    key = (kind, len(cat))
    lead = min(startup_s, 1.5 * _READY_S[key] + 3.0) if key in _READY_S else startup_s
    t_launch = time.time()
    epoch = time.time_ns() + int(lead * 1e9)
    procs, addrs = [], []
    try:
        for i, dev in enumerate(devices):
            p, port = start_worker(kind, cat_path, pages, epoch, dev, i,
                                   timeout_s=max(startup_s, 300.0))
            procs.append(p)
            addrs.append(f"127.0.0.1:{port}")
        _READY_S[key] = max(_READY_S.get(key, 0.0), time.time() - t_launch)
        wait = epoch - time.time_ns()
        if wait > 0:
            time.sleep(wait / 1e9)
        groups = group_fn(workload)
        out = run_controller(addrs, cat, epoch, horizon_ns, groups, seed, native_sched)
    finally:
        # the harness closes its sockets but its reader threads keep them open for a while
        # (the worker would see EOF ~10 s later): the counts come from the controller's own
        # action rows, so stop the workers now
        for p in procs:
            p.terminate()
        for p in procs:
            try:
                p.wait(timeout=20)
            except subprocess.TimeoutExpired:
                p.kill()
    out["workers"] = len(devices)
    out["epoch_lead_s"] = lead
    out["epoch_late_s"] = max(0.0, -wait / 1e9)
    out["worker_kind"] = kind
    return out
