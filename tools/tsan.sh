#!/bin/bash
# ThreadSanitizer build + run of the worker's host threads (tools/tsan_engine_test.cpp): every
# host translation unit of libcw compiled with -fsanitize=thread, linked into a test program
# that drives the sim-mode engine through the native serving loop. CPU only (no GPU needed).
# Output: build/tsan/tsan.log (the committed copy: profiles/r2_tsan_engine.log).
set -e
cd "$(dirname "$0")/.."
OUT=build/tsan
mkdir -p $OUT
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="-O1 -g -std=c++17 -Xcompiler -fsanitize=thread,-fPIC -I paper_2006_02464_b200/csrc -I include"
for f in engine.cpp capi_engine.cpp net.cpp capi_rt.cpp tmap.cpp; do
  $NVCC $ARCH $FLAGS -x cu -c paper_2006_02464_b200/csrc/$f -o $OUT/$f.o
done
for f in runtime.cu simt_kernels.cu mk_infer.cu; do
  $NVCC $ARCH $FLAGS -c paper_2006_02464_b200/csrc/$f -o $OUT/$f.o
done
g++ -fsanitize=thread -g -O1 -std=c++17 -I include -c tools/tsan_engine_test.cpp -o $OUT/test.o
$NVCC $ARCH -o $OUT/tsan_engine_test $OUT/*.o -Xcompiler -fsanitize=thread -cudart static \
  -lpthread -lrt -ldl
TSAN_OPTIONS="halt_on_error=0 report_signal_unsafe=0" $OUT/tsan_engine_test 2>&1 | tee $OUT/tsan.log
echo "tsan warnings: $(grep -c 'WARNING: ThreadSanitizer' $OUT/tsan.log)"
