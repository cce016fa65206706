for v in u16_mb2 u12_mb2 u16_mb1 u4_mb4; do SKT_LIB_PATH=tools/libsketch_$v.so timeout 300 python tools/dense_ceiling.py > gpurun_out/ceil_$v.json 2>&1; echo v=$v; cat gpurun_out/ceil_$v.json; done
