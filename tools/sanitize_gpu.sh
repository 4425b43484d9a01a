#!/bin/bash
# compute-sanitizer runs of the INFER megakernel (run under gpurun, one GPU): memcheck,
# racecheck (shared-memory hazards: the ring / staging buffers / BN-prologue tiles) and
# synccheck (barrier usage) on one INFER per case (below). Built with the waits' timeout raised (instrumented runs are slow).
# Logs: gpurun_out/sanitize_<tool>_<arch>.log
set -x
cd "$(dirname "$0")/.."
CW_BUILD_TAG=san CW_NVCC_DEFS="-DCW_TIMEOUT_NS=600000000000ull" python -c "
import sys; sys.path.insert(0, '.')
from paper_2006_02464_b200 import build; build.build(verbose=True)"
# CASES: arch:batch pairs (default ResNet-18 b=1, DenseNet-121 b=1, ResNet-50 b=16: the
# fused shortcuts, the row-staged stem with several tasks per CTA, 2-CTA cluster split-K)
for case in ${CASES:-resnet18:1 densenet121:1 resnet50:16}; do
  arch=${case%%:*}; b=${case##*:}
  for tool in memcheck racecheck synccheck; do
    CW_LIB=libcw_san.so timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool \
      --print-limit 50 python tools/ncu_target.py $arch $b 1 1 \
      > gpurun_out/sanitize_${tool}_${arch}_b${b}.log 2>&1
    tail -3 gpurun_out/sanitize_${tool}_${arch}_b${b}.log
  done
done
