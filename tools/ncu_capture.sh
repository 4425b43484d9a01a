# ncu evidence for the INFER megakernel (run under gpurun, one GPU):
#  1) --set full capture of mk_infer at b=16 and b=1 for ResNet-50 (weights rotating over 4
#     copies, so they stream from HBM as in the bench) and at b=16 for the zoo archs,
#  2) the launch list of a short bench run (device legs only).
set -x
for b in 16 1; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:mk_infer -s 6 -c 1 \
    -o gpurun_out/ncu_mk_b$b python tools/ncu_target.py resnet50 $b 8 4 > gpurun_out/ncu_mk_b$b.log 2>&1
  ncu -i gpurun_out/ncu_mk_b$b.ncu-rep --page raw --csv > gpurun_out/ncu_mk_b$b.raw.csv 2>/dev/null
done
for a in ${CW_NCU_ZOO:-}; do
  timeout 900 ncu --set full --clock-control none -k regex:mk_infer -s 6 -c 1 \
    -o gpurun_out/ncu_mk_${a}_b16 python tools/ncu_target.py $a 16 8 2 > gpurun_out/ncu_mk_${a}.log 2>&1
  ncu -i gpurun_out/ncu_mk_${a}_b16.ncu-rep --page raw --csv > gpurun_out/ncu_mk_${a}_b16.raw.csv 2>/dev/null
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/ncu_launches_bench.csv python bench.py --steps 3 --warmup 3 \
  --sweep-samples 20 --host-samples 20 --copies 40 --no-cpu-baseline --skip-e2e --skip-cold \
  > gpurun_out/ncu_launches_bench.log 2>&1
