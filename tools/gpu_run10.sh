mkdir -p gpurun_out
python bench.py --config c4 --kernel lev --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/bench_lev_tc.json 2> gpurun_out/bench_lev_tc.err; echo rc=$?
SKT_LEV_TC=0 python bench.py --config c4 --kernel lev --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_lev_cc.json 2> gpurun_out/bench_lev_cc.err; echo rc=$?
python bench.py --config c4 --kernel lev --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_lev.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lev_tc -s 3 -c 1 -o gpurun_out/prof_lev python bench.py --config c4 --kernel lev --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_lev.log 2>&1; echo rc_ncu=$?
