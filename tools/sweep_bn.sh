# bn sweep (split 1 and the planner's choice) of single conv layers (profiling helper)
for shape in ${SHAPES}; do
  timeout 60 python tools/conv_probe.py $shape 2>&1 | grep "^b" | sed 's/first task.*//;s/^/planner: /'
  for bn in 64 128 256; do
    CW_FORCE_BN=$bn CW_FORCE_SPLIT=${SPLIT:-1} timeout 60 python tools/conv_probe.py $shape 2>&1 | grep "^b" | sed 's/first task.*//'
  done
done
