"""Single-conv megakernel probe (profiling helper): one conv layer of a given
shape, one INFER traced; reports the per-k-block rate of the MMA pipeline
(first accumulator ready - first tile landed) / k-blocks of the first task, and
the layer time. CW_FORCE_BN / CW_FORCE_SPLIT override the planner."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2006_02464_b200 import arch  # noqa: E402
from paper_2006_02464_b200.device import DeviceRuntime  # noqa: E402


def run(b, h, cin, cout, k, stride):
    pad = k // 2
    spec = arch.ArchSpec("probe")
    spec.layers.append(arch.Layer(0, "c", "bn", cin, cout, k, k, stride, pad, pad, k * k * cin,
                                  cout_pad=cout))
    oh = (h + 2 * pad - k) // stride + 1
    spec.ops.append(arch._op(arch.OP_CONV, layer=0, in_buf=0, out_buf=1, cin=cin, cout=cout, kh=k,
                             kw=k, stride=stride, pad=pad, relu=1, in_h=h, in_w=h, out_h=oh,
                             out_w=oh, kpad=k * k * cin))
    rng = np.random.default_rng(0)
    wt = rng.standard_normal((cout, k * k * cin)).astype(np.float32) * 0.01
    blob = arch.pack_blob(spec, [(wt, np.zeros(cout, np.float32), None)])
    with DeviceRuntime(pages_total=8, io_slots=16) as rt:
        rt.register_arch(0, spec, batches=(b,))
        rt.register_blob(0, 0, blob)
        rt.build()
        rt.load(0, list(range(blob.pages)))
        for _ in range(3):
            rt.profile_layers(0, b, 0)
        res = []
        for _ in range(5):
            ends, _ = rt.profile_layers(0, b, 0)
            plan = rt.plan_layers(0, b)
            tr, _, clk = rt.last_trace(len(plan))
            ok = clk[:, 2] > clk[:, 0]
            mhz = float(np.median((clk[ok, 3] - clk[ok, 1]) / ((clk[ok, 2] - clk[ok, 0]) / 1e3)))
            row = tr[0]
            act = row[:, 0] >= 0
            land = np.median(row[act, 3])
            acc = np.median(row[act, 2][row[act, 2] >= 0]) if (row[act, 2] >= 0).any() else np.nan
            inp = np.median(row[act, 1])
            done = np.median(row[act, 0])
            res.append((ends[-1] * 1e3, (acc - land) / 1e3, mhz, inp / 1e3, land / 1e3, acc / 1e3,
                        done / 1e3, row[act, 0].max() / 1e3))
        kind, mode, bn, tasks, sp, kb, _, _ = (int(x) for x in plan[0])
        t, span, mhz, inp, land, acc, done, dmax = np.median(np.array(res), axis=0)
        kb_task = -(-kb // sp)
        flops = 2.0 * b * oh * oh * cout * k * k * cin
        print(f"b{b} {h}x{h} {cin}->{cout} k{k}s{stride}: bn {bn} split {sp} tasks {tasks} "
              f"kb/task {kb_task}: layer {t:6.1f} us ({flops / t / 1e6:6.1f} TF/s), "
              f"first task MMA pipe {span:5.2f} us = {span / kb_task:5.3f} us/kb "
              f"= {span / kb_task * mhz:5.0f} cycles/kb at {mhz:.0f} MHz\n"
              f"    since kernel start: inputs ready {inp:.1f}, first tile {land:.1f}, first acc "
              f"{acc:.1f}, done median {done:.1f} / max {dmax:.1f} us", flush=True)


for case in sys.argv[1:]:
    run(*[int(x) for x in case.split(",")])
