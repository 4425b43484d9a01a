"""Summarise the ncu --set full captures of the INFER megakernel (gpurun_out/ncu_mk_b*.raw.csv,
written by tools/ncu_capture.sh) into profiles/<round>_ncu_full_mk_infer_summary.json, and the
launch list of the bench run into profiles/<round>_ncu_launches_bench.csv (profiling helper)."""
import csv
import json
import os
import shutil
import sys

ROUND = sys.argv[1] if len(sys.argv) > 1 else "r1"
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(HERE, "gpurun_out")
WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__icc_request_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "launch__shared_mem_per_block_dynamic",
]
summary = {"how": "ncu --set full --clock-control none -k regex:mk_infer -s 6 -c 1 "
                  "python tools/ncu_target.py resnet50 <b> 8 4 (weights rotate over 4 copies)"}
def one(path):
    rows = list(csv.reader(open(path)))
    head, units, vals = rows[0], rows[1], rows[2]
    return {n: f"{vals[head.index(n)]} {units[head.index(n)]}".strip() for n in WANT if n in head}


for b in (16, 1):
    path = os.path.join(OUT, f"ncu_mk_b{b}.raw.csv")
    if os.path.exists(path):
        summary[f"b{b}"] = one(path)
for f in sorted(os.listdir(OUT)):
    if f.startswith("ncu_mk_") and f.endswith("_b16.raw.csv") and f != "ncu_mk_b16.raw.csv":
        summary[f[len("ncu_mk_"):-len(".raw.csv")]] = one(os.path.join(OUT, f))
os.makedirs(os.path.join(HERE, "profiles"), exist_ok=True)
with open(os.path.join(HERE, "profiles", f"{ROUND}_ncu_full_mk_infer_summary.json"), "w") as f:
    json.dump(summary, f, indent=1)
src = os.path.join(OUT, "ncu_launches_bench.csv")
if os.path.exists(src):
    shutil.copy(src, os.path.join(HERE, "profiles", f"{ROUND}_ncu_launches_bench.csv"))
print(json.dumps(summary, indent=1))
