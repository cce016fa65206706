# column-sweep kernel (config 5 deterministic): parity tests, bench, ncu
cd $GRAFT_REPO_ROOT
F=gpurun_out/r2e; mkdir -p $F
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_buckets.py tests/test_gpu_fullsize.py -q -x > $F/pytest.log 2>&1; echo rc_pytest=$?
python bench.py --config c5 --no-e2e --no-cpu-baseline > $F/bench_c5.json 2> $F/bench_c5.err; echo rc_c5=$?
python bench.py --config c5 --fast --no-e2e --no-cpu-baseline > $F/bench_c5_fast.json 2> $F/bench_c5_fast.err; echo rc_c5f=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_colsweep_kernel -s 2 -c 1 -o /tmp/prof_cs -f python bench.py --config c5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $F/ncu.log 2>&1; echo rc_ncu=$?
ncu -i /tmp/prof_cs.ncu-rep --page details --csv > $F/prof_cs.details.csv 2>&1
ncu -i /tmp/prof_cs.ncu-rep --page raw --csv > $F/prof_cs.raw.csv 2>&1
