# round-1 measurement pass: tests, smoke, headline bench, reference arm, other configs, ncu evidence
mkdir -p gpurun_out/final
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/final/pytest_gpu.log 2>&1; echo rc_pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo rc_smoke=$?
python bench.py > gpurun_out/final/bench_c3.json 2> gpurun_out/final/bench_c3.err; echo rc_bench=$?
python bench.py --impl reference > gpurun_out/final/ref_c3.json 2> gpurun_out/final/ref_c3.err; echo rc_ref=$?
for c in c1 c2 c4 c5; do python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err; echo rc_$c=$?; done
python bench.py --config c4 --kernel lev --no-e2e --no-cpu-baseline > gpurun_out/final/bench_c4_lev.json 2> gpurun_out/final/bench_c4_lev.err; echo rc_lev=$?
python bench.py --config c5 --exact --no-e2e --no-cpu-baseline > gpurun_out/final/bench_c5_exact.json 2> gpurun_out/final/bench_c5_exact.err; echo rc_c5x=$?
timeout 300 python tools/srht_time.py > gpurun_out/final/srht_time.txt 2>&1; echo rc_srht=$?
timeout 300 tools/gather_bench > gpurun_out/final/gather_bench.txt 2>&1; echo rc_gather=$?
nproc > gpurun_out/final/nproc.txt; nvidia-smi -q | head -40 > gpurun_out/final/nvsmi.txt
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final/ncu_launch.log 2>&1; echo rc_ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:apply_dense -s 3 -c 1 -o gpurun_out/final/prof_c3 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final/ncu_full.log 2>&1; echo rc_ncu2=$?
python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:csr_ -s 3 -c 1 -o gpurun_out/final/prof_c4 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final/ncu_c4.log 2>&1; echo rc_ncu3=$?
python bench.py --config c4 --kernel lev --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final/plain_lev.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lev_tc3 -s 3 -c 1 -o gpurun_out/final/prof_lev python bench.py --config c4 --kernel lev --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final/ncu_lev.log 2>&1; echo rc_ncu4=$?
