C="16,14,256,256,3,1 16,14,256,1024,1,1 16,56,64,64,3,1 16,56,64,256,1,1"
for bn in 64 256; do echo "== BN$bn"; CW_FORCE_BN=$bn timeout 100 python tools/conv_probe.py $C; done
