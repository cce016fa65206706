# ncu source-level capture of the K5 v2 kernel in tools/lev_prof (run on the GPU box)
set -e
mkdir -p gpurun_out
timeout 200 tools/lev_prof > gpurun_out/lev_prof.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lev_tc2 -c 1 -o gpurun_out/lev_tc2 -f tools/lev_prof > gpurun_out/lev_ncu.log 2>&1
echo done
