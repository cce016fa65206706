mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_core.py -x -q -m gpu -k "csr or golden or shift" > gpurun_out/t12.log 2>&1; echo rc_t=$?; tail -3 gpurun_out/t12.log
for c in c4 c2; do python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo rc_$c=$?;
SKT_CSR_GTILE=0 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/bench_${c}_nog.json 2> gpurun_out/bench_${c}_nog.err; done
python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:csr_ -s 3 -c 1 -o gpurun_out/prof_c4h python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1; echo rc_ncu=$?
