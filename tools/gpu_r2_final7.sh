# last pass of the round after the csr_quad slot-group change: all GPU tests, smoke,
# config 4 (bench, e2e, ncu), headline bench
cd $GRAFT_REPO_ROOT; rm -rf gpurun_out/*
F=gpurun_out/final7; mkdir -p $F
timeout 1500 python -m pytest tests/ -q -m gpu > $F/pytest_gpu.log 2>&1; echo rc_pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.log 2>&1; echo rc_smoke=$?
python bench.py > $F/bench_c3.json 2> $F/bench_c3.err; echo rc_bench=$?
python bench.py --config c4 > $F/bench_c4.json 2> $F/bench_c4.err; echo rc_c4=$?
python bench.py --config c2 > $F/bench_c2.json 2> $F/bench_c2.err; echo rc_c2=$?
timeout 900 tools/ref_tests_shim.sh run -q > $F/ref_shim.log 2>&1; echo rc_refshim=$?
bash tools/gpu_ncu_one.sh c4 csr_quad_kernel c4_quad > $F/ncu_quad.log 2>&1; echo rc_ncu_quad=$?
rm -f gpurun_out/ncu_one/c4_quad.ncu-rep
