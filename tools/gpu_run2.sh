set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo rc_c3=$?
python bench.py --config c4 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo rc_c4=$?
python bench.py --config c2 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo rc_c2=$?
python bench.py --config c1 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo rc_c1=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_c3.json 2> gpurun_out/ref_c3.err; echo rc_ref=$?
nproc > gpurun_out/nproc.txt
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_ncu.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu1.log 2>&1; echo rc_ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:apply_dense -s 3 -c 1 -o gpurun_out/prof_c3 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo rc_ncu2=$?
