# round-2 bench hygiene pass: headline (finiteness scan timed, numpy e2e),
# full-matrix reference arm, CSR e2e + cpu baselines
cd $GRAFT_REPO_ROOT
F=gpurun_out/r2b; mkdir -p $F
python bench.py > $F/bench_c3.json 2> $F/bench_c3.err; echo rc_bench=$?
timeout 900 python bench.py --impl reference --steps 16 --warmup 3 > $F/ref_c3.json 2> $F/ref_c3.err; echo rc_ref=$?
for c in c1 c2 c4; do python bench.py --config $c > $F/bench_$c.json 2> $F/bench_$c.err; echo rc_$c=$?; done
python bench.py --config c5 > $F/bench_c5.json 2> $F/bench_c5.err; echo rc_c5=$?
python bench.py --config c5 --exact > $F/bench_c5_exact.json 2> $F/bench_c5_exact.err; echo rc_c5x=$?
for c in c1 c2 c4 c5; do timeout 600 python bench.py --impl reference --config $c --steps 5 --warmup 3 > $F/ref_$c.json 2> $F/ref_$c.err; echo rc_ref_$c=$?; done
