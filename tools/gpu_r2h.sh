# full GPU suite + CSR e2e (device canonical check) + reference test suite via the shim
cd $GRAFT_REPO_ROOT
F=gpurun_out/r2h; mkdir -p $F
timeout 1200 python -m pytest tests/ -q -m gpu -x > $F/pytest_gpu.log 2>&1; echo rc_pytest=$?
for c in c2 c4 c5; do python bench.py --config $c --no-cpu-baseline > $F/bench_$c.json 2> $F/bench_$c.err; echo rc_$c=$?; done
timeout 900 tools/ref_tests_shim.sh run -q > $F/ref_shim.log 2>&1; echo rc_refshim=$?
