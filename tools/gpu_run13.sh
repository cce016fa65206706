mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu > gpurun_out/t13.log 2>&1; echo rc_t=$?; tail -2 gpurun_out/t13.log
for c in c4 c2 c5; do python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo rc_$c=$?; done
