# round-2 measurement pass: tests, smoke, headline bench + reference arm, the
# other configs, K5 fp32/fp64, torchrun N=1, the reference suite through the
# shim, and the ncu launch list + full capture of the headline kernel
cd $GRAFT_REPO_ROOT; rm -rf gpurun_out/*
F=gpurun_out/final6; mkdir -p $F
nproc > $F/nproc.txt; nvidia-smi -q | head -40 > $F/nvsmi.txt
timeout 1500 python -m pytest tests/ -q -m gpu > $F/pytest_gpu.log 2>&1; echo rc_pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.log 2>&1; echo rc_smoke=$?
python bench.py > $F/bench_c3.json 2> $F/bench_c3.err; echo rc_bench=$?
timeout 900 python bench.py --impl reference --steps 16 --warmup 3 > $F/ref_c3.json 2> $F/ref_c3.err; echo rc_ref=$?
for c in c1 c2 c4 c5; do python bench.py --config $c > $F/bench_$c.json 2> $F/bench_$c.err; echo rc_$c=$?; done
python bench.py --config c5 --fast --no-e2e --no-cpu-baseline > $F/bench_c5_fast.json 2> $F/bench_c5_fast.err; echo rc_c5f=$?
python bench.py --config c4 --kernel lev --no-e2e --no-cpu-baseline > $F/bench_c4_lev.json 2> $F/bench_c4_lev.err; echo rc_lev=$?
python bench.py --config c4 --kernel lev --lev-f64 --no-e2e --no-cpu-baseline > $F/bench_c4_lev64.json 2> $F/bench_c4_lev64.err; echo rc_lev64=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 3 > $F/bench_c3_torchrun1.json 2> $F/bench_c3_torchrun1.err; echo rc_trun=$?
timeout 900 tools/ref_tests_shim.sh run -q > $F/ref_shim.log 2>&1; echo rc_refshim=$?
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $F/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $F/ncu_launch.log 2>&1; echo rc_ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_g4 -s 3 -c 1 -o /tmp/prof_c3 -f python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $F/ncu_c3.log 2>&1; echo rc_ncu_c3=$?
ncu -i /tmp/prof_c3.ncu-rep --page raw --csv > $F/prof_c3.raw.csv 2>&1
ncu -i /tmp/prof_c3.ncu-rep --page details --csv > $F/prof_c3.details.csv 2>&1
timeout 300 python tools/csr_window_ab.py --skip-small > $F/window_ab.log 2>&1; echo rc_window=$?
timeout 300 python tools/csr_window_ab.py --skip-small --kernel cta > $F/cta_ab.log 2>&1; echo rc_cta=$?
bash tools/gpu_fine_ncu.sh > $F/fine_ncu.log 2>&1; echo rc_fine_ncu=$?
for m in partition colblock; do SKT_CSR_WIDE=$m timeout 300 python tools/wide_ab.py > $F/wide_ab_$m.log 2>&1; done; timeout 300 python tools/wide_ab.py > $F/wide_ab_fine.log 2>&1; echo rc_wide_ab=$?
bash tools/gpu_ncu_one.sh c4 csr_quad_kernel c4_quad > $F/ncu_quad.log 2>&1; echo rc_ncu_quad=$?
rm -f gpurun_out/ncu_one/c4_quad.ncu-rep
SKT_CSR_KERNEL=tile python bench.py --config c4 --no-e2e --no-cpu-baseline > $F/bench_c4_tile.json 2> $F/bench_c4_tile.err; echo rc_c4_tile=$?
