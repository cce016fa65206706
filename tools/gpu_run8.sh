mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/t8.log 2>&1; echo rc_t=$?; tail -5 gpurun_out/t8.log
for c in c3 c4 c2 c1; do python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo rc_$c=$?; done
