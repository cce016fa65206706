# one ncu --set full capture of a kernel + its CUDA-source-level table
#   tools/gpu_ncu_src.sh NAME KERNEL_REGEX bench-args...
cd $GRAFT_REPO_ROOT
name=$1; rx=$2; shift 2
F=gpurun_out/ncu_$name; mkdir -p $F
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 2 -c 1 -o /tmp/prof_$name -f python bench.py "$@" --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $F/ncu.log 2>&1; echo rc_ncu=$?
ncu -i /tmp/prof_$name.ncu-rep --page details --csv > $F/details.csv 2>&1
ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > $F/raw.csv 2>&1
ncu -i /tmp/prof_$name.ncu-rep --page source --print-source cuda --csv > $F/source_cuda.csv 2>&1
ncu -i /tmp/prof_$name.ncu-rep --page source --csv > $F/source_sass.csv 2>&1
