for f in 0 1 2 4 6; do
  for bn in 64 128 256; do
  echo "== flags $f bn $bn"
  CW_FORCE_BN=$bn CW_MK_FLAGS=$f timeout 120 python tools/conv_probe.py 16,14,256,256,3,1 16,28,128,128,3,1 2>&1 | grep -v "^$"
  done
done
