# csr_sweep (windowed row order) on config 4: timings and one ncu capture
cd $GRAFT_REPO_ROOT
F=gpurun_out/r2d; mkdir -p $F
for sh in 1 2; do for R in 16 32; do SKT_CSR_SHIFT=$sh SKT_SWEEP_R=$R python bench.py --config c4 --no-e2e --no-cpu-baseline --steps 20 > $F/sweep_s${sh}_R$R.json 2>$F/sweep_s${sh}_R$R.err; echo rc_s${sh}_R$R=$?; done; done
SKT_CSR_SHIFT=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_sweep -s 3 -c 1 -o /tmp/prof_sweep -f python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $F/ncu_sweep.log 2>&1; echo rc_ncu=$?
ncu -i /tmp/prof_sweep.ncu-rep --page raw --csv > $F/prof_sweep.raw.csv 2>&1
ncu -i /tmp/prof_sweep.ncu-rep --page details --csv > $F/prof_sweep.details.csv 2>&1
ncu -i /tmp/prof_sweep.ncu-rep --page source --csv > $F/prof_sweep.source.csv 2>&1
