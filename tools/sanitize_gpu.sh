#!/bin/bash
# compute-sanitizer runs of the INFER megakernel (run under gpurun, one GPU): memcheck,
# racecheck (shared-memory hazards: the ring / staging buffers / BN-prologue tiles) and
# synccheck (barrier usage) on one small INFER each of ResNet-18 b=1 and DenseNet-121 b=1
# (the BN-prologue warps). Built with the waits' timeout raised (instrumented runs are slow).
# Logs: gpurun_out/sanitize_<tool>_<arch>.log
set -x
cd "$(dirname "$0")/.."
CW_BUILD_TAG=san CW_NVCC_DEFS="-DCW_TIMEOUT_NS=600000000000ull" python -c "
import sys; sys.path.insert(0, '.')
from paper_2006_02464_b200 import build; build.build(verbose=True)"
for arch in resnet18 densenet121; do
  for tool in memcheck racecheck synccheck; do
    CW_LIB=libcw_san.so timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool \
      --print-limit 50 python tools/ncu_target.py $arch 1 1 1 \
      > gpurun_out/sanitize_${tool}_${arch}.log 2>&1
    tail -3 gpurun_out/sanitize_${tool}_${arch}.log
  done
done
