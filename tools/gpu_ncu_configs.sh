# ncu --set full of the dominant kernel of configs 1, 2, 4, 5 (one capture each;
# each only after the same bench command exited 0 without ncu), details + raw pages
cd $GRAFT_REPO_ROOT
F=gpurun_out/ncu_cfg; mkdir -p $F
cap() {  # name config regex
  python bench.py --config $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $F/plain_$1.log 2>&1 || { echo plain_$1 failed; return; }
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s 3 -c 1 -o /tmp/prof_$1 -f \
    python bench.py --config $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $F/ncu_$1.log 2>&1; echo rc_$1=$?
  ncu -i /tmp/prof_$1.ncu-rep --page details --csv > $F/$1.details.csv 2>&1
  ncu -i /tmp/prof_$1.ncu-rep --page raw --csv > $F/$1.raw.csv 2>&1
}
cap c1_apply_dense c1 apply_dense_kernel
cap c2_csr_group c2 csr_group_kernel
cap c4_csr_tile c4 csr_tile_kernel
cap c5_part_scatter c5 csr_part_scatter_kernel
cap c5_part_accum c5 csr_part_accum_kernel
