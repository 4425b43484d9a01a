# A/B of megakernel build variants (profiling helper): conv probe + full-network exec p50,
# variants interleaved over ROUNDS rounds. usage: LIBS="libcw.so libcw_x.so" bash tools/ab_libs.sh
for r in $(seq ${ROUNDS:-2}); do
  for lib in ${LIBS:-libcw.so}; do
    echo "=== $lib round $r"
    CW_LIB=$lib timeout 120 python tools/conv_probe.py ${PROBES:-16,56,64,256,1,1} 2>&1 | grep "^b"
    CW_LIB=$lib timeout 300 python tools/op_profile.py ${ARCH:-resnet50} ${BATCHES:-1,16} 2>&1 | grep "exec p50"
  done
done
