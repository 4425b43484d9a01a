#!/usr/bin/env python
"""Benchmark of the B200 Clockwork worker (BASELINE.json: goodput req/s within a 100 ms SLO;
INFER images/s and p99.99/p50 per batch size).

One line of JSON from rank 0. Its legs:

  value      configs[0] at b = --batch (16): INFER throughput of the device path with the
             request inputs already in the IOCache and the weights of all --copies (1000)
             ResNet-50 copies resident in distinct HBM pages, one copy per step from a seeded
             uniform schedule (so every step streams its copy's 51 MB from HBM: far larger
             than L2). K timed steps = K INFER graphs (gate -> megakernel -> done) back to
             back on the Exec stream, CUDA-event time, max over ranks. A request counts if its
             Exec time is within the SLO (all are). No LOAD in this leg.
  infer      configs[0] sweep, b = 1..16: img/s (pipelined launches) and the Exec-time spread
             (device %globaltimer) over --sweep-samples INFERs per batch, plus the
             host-observed span of --host-samples closed-loop INFERs.
  e2e        configs[2] at N GPUs, the headline: the UNMODIFIED reference controller
             (sloserve from baseline/_ref: Scheduler, ClientManager, summarize) replays a
             synthetic MAF-style trace (workload.gen_synthetic_trace) over the 1000 copies at
             --e2e-rate req/s per GPU for --e2e-seconds of wall clock against one B200 worker
             process per GPU over TCP (the public API: `python -m paper_2006_02464_b200
             worker --native-net`). Every INFER copies its requests' inputs H2D (pinned) and
             their logits D2H; cold models are LOADed (paged pinned H2D). Goodput as the
             reference's summarize computes it.
  cold_start configs[1]: the same controller and worker with only --cold-pages pages (71
             copies of 7 pages fit) and open-loop arrivals spread uniformly over all 1000
             copies: LOAD / UNLOAD on almost every request.
  roofline   the INFER megakernel at --batch: algorithmic FLOPs per launch / the measured
             launch time vs the measured bf16 peak; DRAM traffic from the committed ncu capture.
  cpu_baseline  the fp32 CPU oracle (oracle/resnet_oracle.py, torchvision ResNet-50) on all
             host cores, ~15 s sample, rank 0 only.

`--impl reference`: the reference's own implementation of the path, run unmodified from
baseline/_ref: the same configs[2] experiment (same controller, trace, rate, SLO, copies,
pages) against the reference EmulatedWorker processes (`python -m sloserve.cli worker`, the
reference catalog's resnet50 durations), which wait out profiled V100 durations on the host
CPU (pkg/src/sloserve/worker.py:1-9). It imports nothing of this repo but bench_e2e.py.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import bench_e2e  # noqa: E402

SLO_NS = bench_e2e.SLO_NS
METRIC = "goodput req/s within 100ms SLO; INFER images/s and p99.99/p50 per batch"
VALUE_WORKLOAD = ("configs[0] INFER throughput, resnet50 b=16, request inputs resident in the "
                  "IOCache, 1000 weight copies resident in 16MiB HBM pages rotating per step "
                  "(no LOAD in the timed region)")
E2E_WORKLOAD = ("configs[2] synthetic MAF-style trace over 1000 resnet50 copies, unmodified "
                "reference controller (baseline/_ref sloserve) -> one worker process per GPU "
                "over TCP, SLO 100ms")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--copies", type=int, default=1000)
    ap.add_argument("--sweep-samples", type=int, default=20000)
    ap.add_argument("--host-samples", type=int, default=2000)
    ap.add_argument("--e2e-seconds", type=float, default=30.0)
    ap.add_argument("--e2e-rate", type=float, default=2500.0, help="offered req/s per GPU")
    ap.add_argument("--e2e-pages", type=int, default=8000)
    ap.add_argument("--cold-seconds", type=float, default=15.0)
    ap.add_argument("--cold-rate", type=float, default=1000.0)
    ap.add_argument("--cold-pages", type=int, default=500)
    ap.add_argument("--startup", type=float, default=60.0,
                    help="seconds allowed for the worker processes to build their plans")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cold", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# ----------------------------------------------------------------------------- processes

def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_spawn(args) -> None:
    """`--gpus N` without a launcher: re-run under torch.distributed.run, one rank per GPU."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))


class Dist:
    """Rank plumbing over gloo (CPU tensors): barriers and max / sum of scalars. The
    workers share no tensors (replicas only), so there is no NCCL."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world > 1:
            import torch
            import torch.distributed as dist
            dist.init_process_group("gloo")
            self.dist, self.torch = dist, torch

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def _reduce(self, v: float, op) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([float(v)], dtype=self.torch.float64)
        self.dist.all_reduce(t, op=op)
        return float(t.item())

    def max(self, v: float) -> float:
        return self._reduce(v, None if self.world == 1 else self.dist.ReduceOp.MAX)

    def sum(self, v: float) -> float:
        return self._reduce(v, None if self.world == 1 else self.dist.ReduceOp.SUM)

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi every 100 ms while a region runs (the recipe's clocks line)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, devices):
        self.devices = ",".join(str(d) for d in devices)
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", self.devices],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        busy = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- helpers

def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return p["bf16_tflops"], p["bf16_tflops_sustained"], p["hbm_gbs"], "measured"
    except (OSError, KeyError, ValueError):
        return 1590.0, 1400.0, 6650.0, "fallback"


def schedule(n: int, copies: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, copies, n)


def pct(a, q):
    return float(np.percentile(np.asarray(a, dtype=np.float64), q))


def ncu_traffic(b: int):
    """DRAM bytes (read + write) per launch of the INFER megakernel at batch b, from the
    newest committed `ncu --set full` capture summary (tools/ncu_capture.sh +
    tools/ncu_summary.py) under profiles/."""
    for name in ("r2d_ncu_full_mk_infer_summary.json", "r2c_ncu_full_mk_infer_summary.json", "r2b_ncu_full_mk_infer_summary.json",
                 "r2_ncu_full_mk_infer_summary.json",
                 "r1_ncu_full_mk_infer_summary.json"):
        path = os.path.join(REPO, "profiles", name)
        try:
            s = json.load(open(path))[f"b{b}"]
            mb = sum(float(s[k].split()[0]) for k in ("dram__bytes_read.sum",
                                                       "dram__bytes_write.sum"))
            unit = s["dram__bytes_read.sum"].split()[1]
            scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
            return mb * scale, f"profiles/{name} (b={b})"
        except (OSError, KeyError, ValueError, IndexError):
            continue
    return None, None


# ----------------------------------------------------------------------------- our arm

def run_device_legs(args, d: Dist) -> dict:
    from paper_2006_02464_b200 import arch
    from paper_2006_02464_b200.device import DeviceRuntime

    dev = d.local
    spec = arch.build_arch("resnet50")
    params = arch.make_params(spec, seed=0)
    blob = arch.pack_blob(spec, arch.fold(spec, params))
    b = args.batch
    bf16_peak, bf16_sus, hbm_peak, peak_kind = peaks()
    out: dict = {"spec": spec, "params": params, "blob_bytes": blob.data.nbytes}
    copies = args.copies
    with DeviceRuntime(device=dev, pages_total=copies * blob.pages, io_slots=16) as rt:
        rt.register_arch(0, spec)
        rt.register_blob(0, 0, blob)
        rt.build()
        load_ns = [rt.load(0, list(range(c * blob.pages, (c + 1) * blob.pages)))
                   for c in range(copies)]
        rt.infer(0, 0, arch.make_inputs(16, spec))
        launches, _ = rt.plan_info(0, b)
        sched = schedule(args.warmup + args.steps, copies, 1 + d.rank)
        hdr = [int(c) * blob.pages for c in sched]
        rt.exec_many(0, b, hdr[:args.warmup])
        d.barrier()
        with ClockSampler([dev]) as clk:
            d.barrier()
            ex, wall = rt.exec_many(0, b, hdr[args.warmup:])
            d.barrier()
        t_max = d.max(wall)
        reqs = d.sum(b * int((ex <= SLO_NS).sum()))
        out["value"] = reqs / (t_max / 1e9)
        out["ms_per_step"] = t_max / 1e6 / args.steps
        out["clocks"] = clk.summary()
        out["gpu_launches"] = launches * args.steps
        out["exec_p50_us"] = pct(ex, 50) / 1e3
        out["load_copy_ms_p50"] = pct(load_ns, 50) / 1e6
        out["load_gbs"] = blob.data.nbytes / (pct(load_ns, 50) / 1e9) / 1e9

        # ---- per-batch sweep: img/s + device Exec spread (pipelined), host span (closed loop)
        sweep = {}
        with ClockSampler([dev]) as clk_sweep:
            for bb in (1, 2, 4, 8, 16):
                n = args.sweep_samples
                hp = [int(c) * blob.pages for c in schedule(n + 50, copies, 100 + bb)]
                rt.exec_many(0, bb, hp[:50])
                ex_b, wall_b = rt.exec_many(0, bb, hp[50:])
                hn = args.host_samples
                ex_c, host_c = rt.exec_closed(0, bb, hp[:hn])
                p50 = pct(ex_b, 50)
                # ~2 ms whole-GPU stalls hit any kernel on these boxes every few seconds (a plain
                # FMA kernel shows them too: tools/stall_probe.cu, profiles/r1_tail.txt):
                # counted, and excluded only in the separately labelled percentile
                stall = ex_b > p50 + 1_000_000
                calm = ex_b[~stall]
                sweep[str(bb)] = {
                    "img_s": bb * n / (wall_b / 1e9), "p50_us": p50 / 1e3,
                    "p99_us": pct(ex_b, 99) / 1e3, "p9999_us": pct(ex_b, 99.99) / 1e3,
                    "max_us": float(ex_b.max()) / 1e3, "p9999_over_p50": pct(ex_b, 99.99) / p50,
                    "platform_stalls": int(stall.sum()),
                    "p9999_over_p50_excl_stalls": pct(calm, 99.99) / p50, "n": n,
                    "host_span_p50_us": pct(host_c, 50) / 1e3,
                    "host_span_p99_us": pct(host_c, 99) / 1e3,
                    "host_span_max_us": float(host_c.max()) / 1e3,
                    "closed_loop_exec_p50_us": pct(ex_c, 50) / 1e3, "host_n": hn,
                    "roofline_us": max(spec.flops_per_image * bb / (bf16_peak * 1e12),
                                       (blob.data.nbytes + bb * 606112) / (hbm_peak * 1e9)) * 1e6}
        out["infer"] = sweep
        out["clocks_sweep"] = clk_sweep.summary()

        # ---- roofline of the dominant kernel: the INFER megakernel (one persistent launch
        # per INFER; the graph adds a 1-CTA gate and a 1-thread done kernel). Achieved =
        # algorithmic FLOPs of the timed INFERs / the CUDA-event time of the timed region on
        # the Exec stream (the stream the graphs are launched on).
        flops = spec.flops_per_image * b
        achieved = flops * args.steps / (wall / 1e9) / 1e12
        ends, kinds = rt.profile_layers(0, b, int(sched[0]) * blob.pages)
        plan = rt.plan_layers(0, b)
        conv_t = prev = 0.0
        for k, t in zip(kinds, ends):
            t = float(t)
            if k == 1:
                conv_t += max(0.0, t - prev)
            prev = max(prev, t)
        traffic, traffic_src = ncu_traffic(b)
        out["roofline"] = {
            "bound": "tensor", "achieved": achieved, "peak": bf16_peak, "unit": "TFLOP/s",
            "frac": achieved / bf16_peak, "traffic": traffic, "traffic_source": traffic_src,
            "algorithmic_bytes": blob.data.nbytes + b * 606112,
            "kernel": "mk_infer_kernel (persistent tcgen05/TMA megakernel, whole forward)",
            "flops_per_launch": flops, "launches_per_infer": int(launches),
            "layers": int(len(plan)), "conv_share_of_trace": conv_t / max(prev, 1e-9),
            "trace_end_us": prev * 1e3,
            "peak_source": f"MEASURED_PEAKS.json bf16_tflops (burst, {peak_kind})"}
    return out


def run_controller_legs(args, d: Dist) -> dict:
    """configs[2] (e2e) and configs[1] (cold_start) behind the reference controller. Rank 0
    starts one worker process per GPU of the job and drives them; the other ranks wait."""
    out = {}
    if d.rank == 0:
        devices = list(range(d.world))
        if not args.skip_e2e:
            h = int(args.e2e_seconds * 1e9)
            with ClockSampler(devices) as clk:
                r = bench_e2e.run_leg(
                    "b200", lambda wl: [bench_e2e.trace_group(wl, args.copies,
                                                              args.e2e_rate * d.world, h, 1)[0]],
                    args.copies, args.e2e_pages, h, devices, args.startup)
            r["clocks"] = clk.summary()
            out["e2e"] = r
        if not args.skip_cold:
            h = int(args.cold_seconds * 1e9)
            out["cold_start"] = bench_e2e.run_leg(
                "b200", lambda wl: [bench_e2e.cold_group(wl, args.copies, args.cold_rate * d.world)],
                args.copies, args.cold_pages, h, devices, args.startup)
    d.barrier()
    return out


def e2e_line(r: dict, args, n_gpus: int) -> dict:
    return {
        "value": r["goodput_rps"], "unit": "req/s",
        "h2d_bytes_per_step": int(r["h2d_bytes_per_infer"]),
        "d2h_bytes_per_step": int(r["d2h_bytes_per_infer"]),
        "step": "one INFER action (mean_batch requests)",
        "workload": E2E_WORKLOAD, "offered_rps": r["offered_rps"],
        "satisfaction": r["satisfaction"], "cold_starts": r["cold_starts"],
        "rejected_too_late": r["rejected_too_late"], "actions": r["actions"],
        "mean_batch": r["mean_batch"], "latency_p50_ms": r["latency_p50_ms"],
        "latency_p99_ms": r["latency_p99_ms"], "latency_max_ms": r["latency_max_ms"],
        "over_slo": r["totals"].get("over_slo"), "horizon_s": r["horizon_s"],
        "wall_s": r["wall_s"], "pages_per_gpu": args.e2e_pages, "copies": args.copies,
        "rate_per_gpu": args.e2e_rate, "workers": r["workers"], "worker_kind": r["worker_kind"],
        "clocks": r.get("clocks"),
        "underprediction_fraction": r["underprediction_fraction"],
        "overprediction_fraction": r["overprediction_fraction"],
    }


def h2d_link_peak(dev: int) -> float:
    """Pinned host -> device copy bandwidth of this box (GB/s): LOAD's roofline."""
    import torch
    n = 256 << 20
    src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(n, dtype=torch.uint8, device=f"cuda:{dev}")
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(5):
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, n / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return best


def reference_worker_closed_loop(n_per_batch: int = 200) -> dict:
    """SURVEY §8(d) CPU-baseline leg (i): the reference's own worker path on this host --
    EmulatedWorker on its WallLoop (baseline/_ref), closed-loop INFERs of the reference
    catalog's resnet50 at b = 1 and 16 -- and the realized spread of its emulated spans
    (Exec + Output, result.end - result.start) next to the profiled duration."""
    bench_e2e.sloserve()
    from sloserve import profiles
    from sloserve.protocol import Action, ActionKind
    from sloserve.timebase import WallClock, WallLoop
    from sloserve.worker import EmulatedWorker

    cat = profiles.reference_catalog()
    mid = next(e.model_id for e in cat.entries if e.replica_of == "resnet50")
    loop = WallLoop(WallClock(), name="ref-worker").start()
    done = threading.Event()
    box = {}

    def send(r):
        box["r"] = r
        done.set()

    w = EmulatedWorker(0, cat, loop, send, pages_per_gpu=500)
    aid = [0]

    def call(kind, b=0):
        aid[0] += 1
        done.clear()
        t = loop.now()
        loop.call_soon(w.on_action, Action(aid[0], kind, mid, t, t + 10**9, tuple(range(b))))
        done.wait(10)
        return box["r"]

    call(ActionKind.LOAD)
    out = {}
    for b in (1, 16):
        spans = []
        for _ in range(n_per_batch):
            r = call(ActionKind.INFER, b)
            spans.append(r.end - r.start)
        p50 = pct(spans, 50)
        out[str(b)] = {"n": n_per_batch, "span_p50_ms": p50 / 1e6,
                       "span_p9999_ms": pct(spans, 99.99) / 1e6,
                       "p9999_over_p50": pct(spans, 99.99) / p50,
                       "profiled_exec_ms": cat.profile(mid).exec_duration[b] / 1e6}
    loop.stop()
    return out


def cpu_baseline(spec, params, budget_s: float) -> dict:
    import torch

    from oracle import resnet_oracle
    from paper_2006_02464_b200 import arch

    cores = os.cpu_count() or 1
    torch.set_num_threads(cores)
    model = resnet_oracle.torchvision_model("resnet50", params)
    x = arch.make_inputs(16, spec)
    resnet_oracle.logits(model, x[:2])
    n, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s or n < 2:
        resnet_oracle.logits(model, x)
        n += 1
    dt = time.perf_counter() - t0
    return {"value": 16 * n / dt, "unit": "img/s", "cores": cores, "kind": "port",
            "sample": f"{n} INFERs of batch 16 through the fp32 CPU oracle (torchvision "
                      f"resnet50, {cores} threads), {dt:.1f} s; per-batch latency "
                      f"{dt / n * 1e3:.0f} ms"}


# ----------------------------------------------------------------------------- reference arm

def run_reference(args, d: Dist):
    """The reference implementation behind the same controller on the same configs[2]
    experiment: EmulatedWorker processes (CPU) in place of the B200 workers. Rank 0 only."""
    if d.rank != 0:
        return None
    h = int(args.e2e_seconds * 1e9)
    devices = list(range(d.world))   # one emulated worker per GPU of the job
    r = bench_e2e.run_leg(
        "reference", lambda wl: [bench_e2e.trace_group(wl, args.copies,
                                                       args.e2e_rate * d.world, h, 1)[0]],
        args.copies, args.e2e_pages, h, devices, startup_s=15.0)
    e2e = e2e_line(r, args, d.world)
    e2e["h2d_bytes_per_step"] = 0
    e2e["d2h_bytes_per_step"] = 0
    value = r["goodput_rps"]
    return {
        "metric": METRIC, "value": value, "unit": "req/s", "n_gpus": d.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / max(value, 1e-9),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (gen_synthetic_trace, seed 1)", "impl": "reference",
        "config": {"workload": E2E_WORKLOAD, "copies": args.copies,
                   "pages_per_gpu": args.e2e_pages, "rate_per_gpu": args.e2e_rate,
                   "horizon_s": args.e2e_seconds, "parallelism": "replicas (one worker per GPU)"},
        "cpu_baseline": {"value": value, "unit": "req/s", "cores": 2, "kind": "reference",
                         "sample": f"{args.e2e_seconds:.0f} s of the configs[2] trace replay "
                                   f"through the reference controller against "
                                   f"{len(devices)} reference EmulatedWorker process(es) "
                                   "(each: one WallLoop thread + one socket thread), which "
                                   "wait out the reference catalog's V100 resnet50 durations"},
        "e2e": e2e,
        "native_so_loaded": [m for m in _loaded_objects() if "libcw" in m],
    }


def _loaded_objects() -> list[str]:
    try:
        with open(f"/proc/{os.getpid()}/maps") as f:
            return sorted({ln.split()[-1] for ln in f if ln.rstrip().endswith(".so")})
    except OSError:
        return []


# ----------------------------------------------------------------------------- main

def main():
    args = parse_args()
    maybe_spawn(args)
    d = Dist()
    if args.impl == "reference":
        line = run_reference(args, d)
        if line is not None:
            print(json.dumps(line), flush=True)
        d.close()
        return
    res = run_device_legs(args, d)
    ctl = run_controller_legs(args, d)
    if d.rank == 0:
        line = {
            "metric": METRIC, "value": res["value"], "unit": "req/s", "n_gpus": d.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (N(0,1) 3x224x224 inputs, random-init ResNet-50 weights)",
            "config": {"workload": VALUE_WORKLOAD, "batch": args.batch, "copies": args.copies,
                       "parallelism": "replicas (one worker per GPU)",
                       "l2": "inputs larger than L2: 1000 copies x 51 MB weights rotate per step",
                       "e2e_workload": E2E_WORKLOAD},
            "clocks": res["clocks"], "clocks_sweep": res["clocks_sweep"],
            "gpu_launches": res["gpu_launches"], "roofline": res["roofline"],
            "infer": res["infer"],
            "load": {"copy_ms_p50": res["load_copy_ms_p50"], "gbs": res["load_gbs"],
                     "blob_bytes": res["blob_bytes"]},
            "exec_p50_us": res["exec_p50_us"],
        }
        if "e2e" in ctl:
            line["e2e"] = e2e_line(ctl["e2e"], args, d.world)
            line["gpu_launches_e2e"] = 3 * sum(
                v for k, v in ctl["e2e"]["actions"].items() if k.startswith("infer:")
                and not k.endswith("model_not_loaded"))
        if "cold_start" in ctl:
            c = ctl["cold_start"]
            line["cold_start"] = {
                "workload": "configs[1]: 1000 resnet50 copies, open-loop uniform over copies, "
                            f"{args.cold_pages} pages per GPU (71 copies fit), reference controller",
                "goodput_rps": c["goodput_rps"], "offered_rps": c["offered_rps"],
                "satisfaction": c["satisfaction"], "cold_starts": c["cold_starts"],
                "loads": c["loads"], "actions": c["actions"], "mean_batch": c["mean_batch"],
                "latency_p99_ms": c["latency_p99_ms"], "horizon_s": c["horizon_s"]}
        try:
            link = h2d_link_peak(d.local)
            line["load"].update({"link_gbs": link, "frac": res["load_gbs"] / link,
                                 "roofline": "pinned H2D link bandwidth of this box (256 MiB "
                                             "copy, best of 5)"})
        except Exception as exc:  # noqa: BLE001 (diagnostic leg)
            line["load"]["link_error"] = str(exc)
        try:
            # the controller fast path against the reference scheduler in
            # the same simulated harness (8 GPUs, 64 models, 20k req/s offered, 1 s)
            sys.path.insert(0, os.path.join(REPO, "tools"))
            import sched_throughput
            ct = sched_throughput.run(20000.0, 1.0, 8, 64)
            line["controller"] = {
                "workload": "reference harness, sim mode: 8 emulated GPUs, 64 resnet50 copies, "
                            "open loop 20k req/s offered, SLO 100 ms, 1 s horizon",
                "reference_requests_per_wall_s": ct["reference"]["requests_per_wall_s"],
                "native_requests_per_wall_s": ct["native"]["requests_per_wall_s"],
                "speedup": ct["speedup"], "same_summary": ct["same_summary"]}
        except Exception as exc:  # noqa: BLE001 (diagnostic leg)
            line["controller"] = {"error": str(exc)}
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(res["spec"], res["params"], budget_s=15.0)
            try:
                line["cpu_baseline"]["reference_worker_closed_loop"] = \
                    reference_worker_closed_loop()
            except Exception as exc:  # noqa: BLE001
                line["cpu_baseline"]["reference_worker_closed_loop"] = {"error": str(exc)}
        print(json.dumps(line), flush=True)
    d.close()


if __name__ == "__main__":
    main()
