mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_core.py -x -q -m gpu -k "dense or golden or structure or unit" > gpurun_out/t6.log 2>&1; echo rc_t=$?; tail -3 gpurun_out/t6.log
timeout 300 python tools/dense_ceiling.py > gpurun_out/ceiling_tma.json 2>&1; cat gpurun_out/ceiling_tma.json
SKT_DENSE_TMA=0 timeout 300 python tools/dense_ceiling.py > gpurun_out/ceiling_ldg.json 2>&1; cat gpurun_out/ceiling_ldg.json
python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo rc_c3=$?
python bench.py --config c1 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo rc_c1=$?
