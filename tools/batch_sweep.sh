# whole-network exec time per batch size under env settings (profiling helper)
IFS=';' read -ra SETS <<< "${ENVS:-X=0}"
for e in "${SETS[@]}"; do
  echo "=== $e"; env $e timeout 300 python tools/op_profile.py resnet50 1,2,4,8,16 2>&1 | grep "exec p50"
done
