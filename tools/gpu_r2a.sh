cd $GRAFT_REPO_ROOT
F=gpurun_out/r2a; mkdir -p $F
nproc > $F/nproc.txt; free -g > $F/free.txt
timeout 1500 python -m pytest tests/ -q -m gpu -x --durations=15 > $F/pytest_gpu.log 2>&1; echo rc_pytest=$?
timeout 900 tools/ref_tests_shim.sh run -q -x > $F/ref_shim.log 2>&1; echo rc_refshim=$?
python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.log 2>&1; echo rc_smoke=$?
python bench.py > $F/bench_c3.json 2> $F/bench_c3.err; echo rc_bench=$?
