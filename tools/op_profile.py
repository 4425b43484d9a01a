"""Per-layer timeline of the INFER megakernel (device trace: when each plan
layer's last task finished, relative to Exec start) with the plan, for one
arch and batch sizes. Profiling helper."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2006_02464_b200 import arch  # noqa: E402
from paper_2006_02464_b200.device import DeviceRuntime  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
batches = [int(b) for b in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 16]
spec = arch.build_arch(name)
blob = arch.pack_blob(spec, arch.fold(spec, arch.make_params(spec, 0)))
names = {1: "conv", 2: "input", 3: "maxpool", 4: "avgpool", 5: "fc", 6: "reduce"}
with DeviceRuntime(pages_total=8 * blob.pages, io_slots=16,
                   in_bytes_max=spec.in_c * spec.in_h * spec.in_w * 4) as rt:
    rt.register_arch(0, spec)
    rt.register_blob(0, 0, blob)
    rt.build()
    for c in range(8):
        rt.load(0, list(range(c * blob.pages, (c + 1) * blob.pages)))
    rt.infer(0, 0, arch.make_inputs(16, spec))
    for b in batches:
        reps = [rt.profile_layers(0, b, (r % 8) * blob.pages)[0] for r in range(9)]
        ends = np.median(np.stack(reps), axis=0)
        plan = rt.plan_layers(0, b)
        ex, wall = rt.exec_many(0, b, [(i % 8) * blob.pages for i in range(200)])
        print(f"== {name} b={b}: exec p50 {np.median(ex) / 1e3:.1f} us, "
              f"trace end {ends.max() * 1e3:.1f} us, {len(plan)} layers")
        prev = 0.0
        for i, (pl, t) in enumerate(zip(plan, ends)):
            kind, mode, bn, tasks, sp, kb, opi, pool = (int(x) for x in pl)
            op = spec.ops[opi]
            flops = 0
            if kind == 1:
                k = 147 if op["kh"] == 7 else op["kh"] * op["kw"] * op["cin"]
                flops = 2 * op["out_h"] * op["out_w"] * op["cout"] * k * b
            dt = (t - prev) * 1e3
            tf = flops / (dt * 1e-6) / 1e12 if dt > 0 and flops else 0
            print(f"{i:3d} {names.get(kind, '?'):7s} {op['cin']:5d}->{op['cout']:5d} k{op['kh']} "
                  f"s{op['stride']} @{op['in_h']:3d} mode{mode:2d} bn{bn:4d} tasks{tasks:5d} "
                  f"sp{sp:3d} kb{kb:3d} pool{pool} end {t * 1e3:8.1f} us  +{dt:6.1f} us "
                  f"{tf:7.1f} TF/s")
            prev = max(prev, t)

    # Fine-grained view of the last profiled INFER: per layer, over the SMs with
    # work, the median time of inputs-ready (producer), first-tile-landed (MMA),
    # first-accumulator-ready (epilogue) and done, relative to the layer's start
    # (the previous layer's end).
    if "--detail" in sys.argv:
        for b in batches:
            rt.profile_layers(0, b, 0)
            plan = rt.plan_layers(0, b)
            tr, _, clk = rt.last_trace(len(plan))
            ok = clk[:, 2] > clk[:, 0]
            mhz = (clk[ok, 3] - clk[ok, 1]) / ((clk[ok, 2] - clk[ok, 0]) / 1e3)
            print(f"SM clock during the megakernel: median {np.median(mhz):.0f} MHz "
                  f"(min {mhz.min():.0f}, max {mhz.max():.0f}); kernel span "
                  f"{(clk[ok, 2].max() - clk[ok, 0].min()) / 1e3:.1f} us")
            print(f"== detail b={b}: us since previous layer end (median over SMs with work / max)")
            prev = 0
            for i, pl in enumerate(plan):
                row = tr[i]
                done = row[:, 0]
                act = done >= 0
                if not act.any():
                    continue
                def med(k):
                    v = row[act, k]
                    v = v[v >= 0]
                    return (np.median(v) - prev) / 1e3 if len(v) else float("nan")
                end = done[act].max()
                print(f"{i:3d} {names.get(int(pl[0]), '?'):7s} tasks{int(pl[3]):5d} sms{int(act.sum()):4d} "
                      f"in {med(1):7.1f} land {med(3):7.1f} acc {med(2):7.1f} "
                      f"done {(np.median(done[act]) - prev) / 1e3:7.1f} / {(end - prev) / 1e3:7.1f}")
                prev = max(prev, end)
