# A/B of megakernel build variants (profiling helper): conv probes + full-network exec times
for lib in ${LIBS:-libcw.so}; do
  echo "=== $lib"
  CW_LIB=$lib timeout 120 python tools/conv_probe.py 16,14,256,256,3,1 16,28,128,128,3,1 16,56,64,256,1,1 2>&1 | grep -v "^$" | grep "^b"
  CW_LIB=$lib timeout 300 python tools/op_profile.py resnet50 1,16 2>&1 | grep "exec p50"
done
