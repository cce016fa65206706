# ncu --set full of one kernel of one config: bash tools/gpu_ncu_one.sh <config> <kernel regex> <name> [bench args]
cd $GRAFT_REPO_ROOT
c=$1; k=$2; n=$3; shift 3
F=gpurun_out/ncu_one; mkdir -p $F
python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline "$@" > $F/plain_$n.json 2> $F/plain_$n.err || { echo plain failed; tail -5 $F/plain_$n.err; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $F/$n -f \
  python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline "$@" > $F/ncu_$n.log 2>&1; echo rc=$?
ncu -i $F/$n.ncu-rep --page details --csv > $F/$n.details.csv 2>&1
ncu -i $F/$n.ncu-rep --page source --csv --print-source sass > $F/$n.sass.csv 2>&1
ncu -i $F/$n.ncu-rep --page raw --csv > $F/$n.raw.csv 2>&1
[ $(stat -c %s $F/$n.ncu-rep) -gt 40000000 ] && rm -f $F/$n.ncu-rep
