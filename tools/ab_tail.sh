# A/B of megakernel build variants on one box (profiling helper): alternating tail_probe runs
for r in 1 2; do
  for lib in ${LIBS:-libcw.so}; do
    for b in ${BATCHES:-16 1}; do
      echo "$lib b=$b $(CW_LIB=$lib timeout 300 python tools/tail_probe.py $b ${N:-3000} 2>&1 | grep -o 'p50 [0-9.]*' | tr '\n' ' ')"
    done
  done
done
