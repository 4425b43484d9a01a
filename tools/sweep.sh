# bn x split sweep of single conv layers (profiling helper)
for shape in ${SHAPES:-16,14,256,256,3,1 16,28,128,128,3,1 16,56,64,64,3,1 16,14,1024,256,1,1 16,7,512,512,3,1}; do
  for bn in 64 128 256; do
    for sp in 1 2 4 8; do
      CW_FORCE_BN=$bn CW_FORCE_SPLIT=$sp timeout 60 python tools/conv_probe.py $shape 2>&1 | grep "^b" | sed 's/first task.*//'
    done
  done
done
