# A/B of runtime env settings (profiling helper): conv probes + full-network exec times.
# usage: ENVS="CW_KPACK=1;CW_KPACK=2" bash tools/ab_env.sh
IFS=';' read -ra SETS <<< "${ENVS:-X=0}"
for e in "${SETS[@]}"; do
  echo "=== $e"
  env $e timeout 120 python tools/conv_probe.py ${PROBES:-16,14,256,256,3,1 16,28,128,128,3,1 16,56,64,256,1,1 16,56,64,64,3,1} 2>&1 | grep -v "^$" | grep "^b"
  env $e timeout 300 python tools/op_profile.py resnet50 1,16 2>&1 | grep "exec p50"
done
