# round-1 measurement pass: tests, smoke, headline bench, reference arm, other
# configs, ncu evidence (reports stay in /tmp on the box; raw / details CSVs
# come back in gpurun_out/final)
mkdir -p gpurun_out/final
cd $GRAFT_REPO_ROOT
F=gpurun_out/final
timeout 1200 python -m pytest tests/ -q -m gpu > $F/pytest_gpu.log 2>&1; echo rc_pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.log 2>&1; echo rc_smoke=$?
python bench.py > $F/bench_c3.json 2> $F/bench_c3.err; echo rc_bench=$?
python bench.py --impl reference > $F/ref_c3.json 2> $F/ref_c3.err; echo rc_ref=$?
for c in c1 c2 c4 c5; do python bench.py --config $c --no-e2e --no-cpu-baseline > $F/bench_$c.json 2> $F/bench_$c.err; echo rc_$c=$?; done
python bench.py --config c4 --kernel lev --no-e2e --no-cpu-baseline > $F/bench_c4_lev.json 2> $F/bench_c4_lev.err; echo rc_lev=$?
python bench.py --config c5 --exact --no-e2e --no-cpu-baseline > $F/bench_c5_exact.json 2> $F/bench_c5_exact.err; echo rc_c5x=$?
timeout 900 python bench.py --config c5 --kernel lowrank > $F/lowrank_c5.json 2> $F/lowrank_c5.err; echo rc_lowrank=$?
nproc > $F/nproc.txt; nvidia-smi -q | head -40 > $F/nvsmi.txt
cap() {  # name regex bench-args...
  name=$1; rx=$2; shift 2
  ncu --set full --clock-control none --import-source on -k regex:$rx -s 3 -c 1 -o /tmp/prof_$name -f python bench.py "$@" --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $F/ncu_$name.log 2>&1
  echo rc_ncu_$name=$?
  ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > $F/prof_${name}.raw.csv 2>&1
  ncu -i /tmp/prof_$name.ncu-rep --page details --csv > $F/prof_${name}.details.csv 2>&1
}
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $F/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $F/ncu_launch.log 2>&1; echo rc_ncu_launch=$?
cap c3 "dense_g4|apply_dense"
cap c4 "csr_" --config c4
cap c4_lev "lev_tc3" --config c4 --kernel lev
