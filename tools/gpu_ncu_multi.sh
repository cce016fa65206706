# ncu --set full of several kernels of one bench command (one capture each)
#   tools/gpu_ncu_multi.sh NAME "regex1 regex2 ..." bench-args...
cd $GRAFT_REPO_ROOT
name=$1; rxs=$2; shift 2
F=gpurun_out/ncu_$name; mkdir -p $F
for rx in $rxs; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 1 -c 1 -o /tmp/prof_$rx -f python bench.py "$@" --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $F/ncu_$rx.log 2>&1; echo rc_$rx=$?
  ncu -i /tmp/prof_$rx.ncu-rep --page raw --csv > $F/$rx.raw.csv 2>&1
  ncu -i /tmp/prof_$rx.ncu-rep --page source --csv > $F/$rx.sass.csv 2>&1
done
