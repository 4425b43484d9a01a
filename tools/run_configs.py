"""BASELINE.json configs[3] (mixed zoo) and configs[4] (SLO sweep with isolation) on the GPU,
behind the unmodified reference controller (baseline/_ref), for the B200 worker and the
reference EmulatedWorker. Writes one JSON (default profiles/r2_configs.json).

    python tools/run_configs.py [--seconds 20] [--out profiles/r2_configs.json]

Steps:
 1. B200 catalog rows, measured: for every zoo arch, device Exec p99 at b = 1..16 (200
    INFERs each, 1000... copies not needed: weights of one copy, L2 flushed by the others'
    absence is irrelevant at these sizes) and the LOAD copy time; written as catalog rows
    (durations +10 %) that seed the controller's estimators ("B200 rows for
    the zoo are new data"). weights_bytes are the reference catalog's where it has the arch
    (profiles.py:322-374), else the fp32 parameter bytes.
 2. configs[3]: ResNet-50/152, ResNeXt-50, DenseNet-121, Inception-v3, 20 copies each,
    open-loop per-model-group clients with per-model SLOs of 10-100 ms (B200 worker).
 3. reference-catalog zoo (densenet169, inceptionv3, resnet18/50/152 x 20 copies, SLOs
    10-100 ms): both arms, the reference worker with the reference catalog's V100 rows.
 4. configs[4]: SLO sweep 10-500 ms with request-level isolation (Fig. 8
    analog): latency-sensitive open-loop clients (200 r/s over 10 ResNet-50 copies, SLO
    swept) next to closed-loop batch clients (concurrency 16 on 5 other copies, SLO 1 s):
    both arms, 1 GPU.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import bench_e2e  # noqa: E402

REF_WEIGHTS = {"densenet169": 56_500_000, "inceptionv3": 95_300_000, "resnet18": 46_700_000,
               "resnet50": 102_300_000, "resnet152": 240_900_000}
BATCHES = (1, 2, 4, 8, 16)


def measure_rows(bases, pages_per=None):
    """Device-measured catalog rows (B200) for the given catalog base names."""
    from paper_2006_02464_b200 import arch
    from paper_2006_02464_b200.device import DeviceRuntime
    rows, meas = [], {}
    for base in bases:
        spec = arch.build_arch(base)
        params = arch.make_params(spec, seed=0)
        blob = arch.pack_blob(spec, arch.fold(spec, params))
        with DeviceRuntime(device=0, pages_total=blob.pages, io_slots=16,
                           in_bytes_max=spec.in_c * spec.in_h * spec.in_w * 4) as rt:
            rt.register_arch(0, spec)
            rt.register_blob(0, 0, blob)
            rt.build()
            load_ns = [rt.load(0, list(range(blob.pages))) for _ in range(5)]
            rt.set_input_pool(arch.make_inputs(16, spec), 0)
            rt.infer(0, 0, arch.make_inputs(16, spec))
            ex = {}
            for b in BATCHES:
                e, _ = rt.exec_many(0, b, [0] * 200)
                ex[b] = int(np.percentile(e, 99))
        wbytes = REF_WEIGHTS.get(base, 4 * sum(
            v.size for k, v in params.items() if "running" not in k))
        in_bytes = spec.in_c * spec.in_h * spec.in_w * 4
        io_in = 1073000 if base == "inceptionv3" else 602000
        meas[base] = {"exec_p99_us": {b: v / 1e3 for b, v in ex.items()},
                      "load_ms": float(np.median(load_ns)) / 1e6, "blob_bytes": blob.data.nbytes,
                      "flops": spec.flops_per_image}
        rows.append(f"model {base}\nweights_bytes {wbytes}\n"
                    f"weights_transfer_ns {int(np.median(load_ns) * 1.1)}\n"
                    f"io_ns {max(1000, int(in_bytes / 25e9 * 1e9))} 3000\n"
                    f"io_bytes {io_in} 4000\n" +
                    "".join(f"batch {b} {int(ex[b] * 1.1)}\n" for b in BATCHES))
    return rows, meas


def ref_rows(bases):
    harness, workload, profiles = bench_e2e.sloserve()
    text = profiles.dumps_catalog(profiles.reference_catalog())
    recs = {r.split("\n", 1)[0]: "model " + r.rstrip("\n") + "\n" for r in text.split("\nmodel ")[1:]}
    return [recs[b] for b in bases]


def catalog(rows, bases, copies):
    return ("page_bytes 16777216\n" + "".join(rows) +
            "".join(f"replicas {b} {copies - 1}\n" for b in bases))


def model_ids(cat_text):
    from paper_2006_02464_b200 import catalog as C
    cat = C.parse(cat_text)
    out = {}
    for mid, base in enumerate(cat.base):
        out.setdefault(base, []).append(mid)
    return out


def zoo_groups(ids, slos, rates):
    def fn(workload):
        return [workload.ClientGroup(kind="open", model_ids=ids[b], slo_ns=int(slos[b] * 1e6),
                                     rate=rates[b], name=f"{b}-{slos[b]}ms") for b in ids]
    return fn


def run(kind, cat_text, groups, pages, seconds, startup):
    h = int(seconds * 1e9)
    r = bench_e2e.run_leg(kind, groups, 0, pages, h, [0], startup, cat_text=cat_text)
    r.pop("totals", None)
    return r


def per_group(kind, cat_text, groups_fn, pages, seconds, startup):
    """Like run(), but with the per-client-group summary (request rows kept)."""
    harness, workload, profiles = bench_e2e.sloserve()
    import tempfile
    h = int(seconds * 1e9)
    workdir = tempfile.mkdtemp(prefix="cw_cfg_")
    cat_path = os.path.join(workdir, "cat.txt")
    open(cat_path, "w").write(cat_text)
    epoch = time.time_ns() + int(startup * 1e9)
    proc, port = bench_e2e.start_worker(kind, cat_path, pages, epoch, 0, 0, timeout_s=startup)
    try:
        time.sleep(max(0.0, (epoch - time.time_ns()) / 1e9))
        groups = groups_fn(workload)
        cfg = harness.ExperimentConfig(
            name="cfg", mode="wall", transport="tcp", horizon_ns=h, catalog_text=cat_text,
            workers=[harness.WorkerSpec(address=f"127.0.0.1:{port}")], epoch_ns=epoch,
            groups=groups, keep_request_records=True, keep_action_records=True)
        res = harness.run_experiment(cfg)
    finally:
        proc.terminate()
        proc.wait(timeout=20)
    s = res.summary
    by = {}
    for g in groups:
        ids = set(g.model_ids)
        rows = [r for r in res.sink.request_rows if r[1] in ids and r[2] < h]
        ok = sum(1 for r in rows if r[4] == "ok")
        lat = sorted(r[5] for r in rows if r[4] == "ok")
        by[g.name] = {"offered": len(rows), "ok": ok, "goodput_rps": ok / seconds,
                      "satisfaction": ok / max(1, len(rows)),
                      "latency_p99_ms": (lat[int(0.99 * (len(lat) - 1))] / 1e6) if lat else None,
                      "slo_ms": g.slo_ns / 1e6}
    return {"goodput_rps": s.goodput_rps, "offered_rps": s.offered_rps,
            "satisfaction": s.satisfaction, "cold_starts": s.cold_starts,
            "over_slo": s.totals["over_slo"], "groups": by}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=20.0)
    ap.add_argument("--startup", type=float, default=150.0)
    ap.add_argument("--out", default=os.path.join(REPO, "profiles", "r2_configs.json"))
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    out = {"seconds": args.seconds}
    zoo = ["resnet50", "resnet152", "resnext50", "densenet121", "inceptionv3"]
    refzoo = ["densenet169", "inceptionv3", "resnet18", "resnet50", "resnet152"]
    allb = sorted(set(zoo + refzoo))
    rows, meas = measure_rows(allb)
    row = dict(zip(allb, rows))
    out["b200_rows_measured"] = meas
    out["b200_catalog_rows"] = "".join(row[b] for b in allb)
    copies = 20
    if not args.only or "zoo" in args.only:
        cat = catalog([row[b] for b in zoo], zoo, copies)
        ids = model_ids(cat)
        slos = {"resnet50": 25, "resnet152": 50, "resnext50": 25, "densenet121": 100,
                "inceptionv3": 10}
        rates = {b: 300.0 for b in zoo}
        out["configs3_mixed_zoo_b200"] = per_group("b200", cat, zoo_groups(ids, slos, rates),
                                                   2000, args.seconds, args.startup)
    if not args.only or "refzoo" in args.only:
        slos = {"densenet169": 100, "inceptionv3": 50, "resnet18": 10, "resnet50": 25,
                "resnet152": 100}
        rates = {b: 100.0 for b in refzoo}
        for kind, rws in (("b200", [row[b] for b in refzoo]), ("reference", ref_rows(refzoo))):
            cat = catalog(rws, refzoo, copies)
            out[f"reference_catalog_zoo_{kind}"] = per_group(
                kind, cat, zoo_groups(model_ids(cat), slos, rates), 2000, args.seconds,
                args.startup if kind == "b200" else 15)
    if not args.only or "slo" in args.only:
        sweep = {}
        for kind in ("b200", "reference"):
            rws = [row["resnet50"]] if kind == "b200" else ref_rows(["resnet50"])
            cat = catalog(rws, ["resnet50"], 15)
            for slo in (10, 25, 50, 100, 250, 500):
                def groups(workload, slo=slo):
                    return [workload.ClientGroup(kind="open", model_ids=list(range(10)),
                                                 slo_ns=slo * 1_000_000, rate=200.0,
                                                 name="latency-sensitive"),
                            workload.ClientGroup(kind="closed", model_ids=list(range(10, 15)),
                                                 slo_ns=1_000_000_000, concurrency=16,
                                                 name="batch")]
                sweep[f"{kind}_slo{slo}"] = per_group(kind, cat, groups, 500, args.seconds / 2,
                                                      args.startup if kind == "b200" else 15)
        out["configs4_slo_sweep"] = sweep
    json.dump(out, open(args.out, "w"), indent=1)
    print(json.dumps(out)[:3000])


if __name__ == "__main__":
    main()
