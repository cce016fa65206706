mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_core.py -x -q -m gpu -k "wide or csr or golden" > gpurun_out/t11.log 2>&1; echo rc_t=$?; tail -15 gpurun_out/t11.log
python bench.py --config c5 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo rc_c5=$?; tail -3 gpurun_out/bench_c5.err
