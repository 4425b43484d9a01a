# A/B of planner environment settings on one box (profiling helper): alternating tail_probe runs
# usage: ENVS="CW_SPLIT_US=4 CW_SPLIT_US=6" bash tools/ab_envs.sh
for r in 1 2; do
  for e in ${ENVS:-X=0}; do
    for b in ${BATCHES:-16 1}; do
      echo "$e b=$b $(env $e timeout 300 python tools/tail_probe.py $b ${N:-2000} 2>&1 | grep -o 'p50 [0-9.]*' | tr '\n' ' ')"
    done
  done
done
