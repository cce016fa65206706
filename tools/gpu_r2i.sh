cd $GRAFT_REPO_ROOT
F=gpurun_out/r2i; mkdir -p $F
timeout 300 python -m pytest tests/test_gpu_wide.py tests/test_gpu_buckets.py tests/test_gpu_fullsize.py tests/test_gpu_core.py -k "wide or colsweep or config5 or bucket or csr" -q -x > $F/pytest.log 2>&1; echo rc_pytest=$?
python bench.py --config c5 --no-e2e --no-cpu-baseline > $F/bench_c5.json 2> $F/bench_c5.err; echo rc_c5=$?
SKT_CSR_WIDE=colblock python bench.py --config c5 --no-e2e --no-cpu-baseline > $F/bench_c5_colblock.json 2>&1
timeout 900 nsys --version > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/launches_c5.csv python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $F/ncu_launch.log 2>&1; echo rc_ncu=$?
