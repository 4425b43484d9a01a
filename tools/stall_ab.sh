#!/bin/bash
# Is the ~2 ms whole-GPU stall caused by nvidia-smi / NVML polling? tail_probe (3 x 20,000
# back-to-back INFERs) with and without a concurrent `nvidia-smi -lms 100` sampler.
cd "$(dirname "$0")/.."
for b in 16 2; do
  echo "== b=$b without nvidia-smi polling"
  python tools/tail_probe.py $b 20000 100
  echo "== b=$b with nvidia-smi -lms 100 polling"
  nvidia-smi --query-gpu=clocks.sm,clocks_event_reasons.active --format=csv,noheader -lms 100 \
    > /dev/null 2>&1 &
  P=$!
  python tools/tail_probe.py $b 20000 100
  kill $P
done
