# launch-time list and ncu --set full of the two fine-block kernels of config 5
cd $GRAFT_REPO_ROOT
F=gpurun_out/fine; mkdir -p $F
python bench.py --config c5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $F/plain.json 2> $F/plain.err || { echo plain failed; tail -5 $F/plain.err; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:csr_ -s 30 -c 12 --csv --log-file $F/launches.csv \
  python bench.py --config c5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $F/ncu_launch.log 2>&1
for k in scatter accum; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_fine_$k -s 3 -c 1 -o $F/fine_$k -f \
    python bench.py --config c5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $F/ncu_$k.log 2>&1; echo rc_$k=$?
  ncu -i $F/fine_$k.ncu-rep --page details --csv > $F/fine_$k.details.csv 2>&1
  ncu -i $F/fine_$k.ncu-rep --page raw --csv > $F/fine_$k.raw.csv 2>&1
  rm -f $F/fine_$k.ncu-rep
done
cat $F/plain.json
