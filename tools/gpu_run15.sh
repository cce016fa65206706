mkdir -p gpurun_out
SKT_CSR_KERNEL=lane timeout 600 python -m pytest tests/test_gpu_core.py -x -q -m gpu -k "csr or golden" > gpurun_out/t15.log 2>&1; echo rc_t=$?; tail -3 gpurun_out/t15.log
for c in c4 c2; do SKT_CSR_KERNEL=lane python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/bench_${c}_lane.json 2> gpurun_out/bench_${c}_lane.err; echo rc_$c=$?; done
SKT_CSR_KERNEL=lane python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_c4.log 2>&1 && \
SKT_CSR_KERNEL=lane ncu --set full --clock-control none --import-source on -k regex:csr_ -s 3 -c 1 -o gpurun_out/prof_c4_lane python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1; echo rc_ncu=$?
