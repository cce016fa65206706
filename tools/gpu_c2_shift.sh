# kernel time of config 2 under plan group sizes: bash tools/gpu_c2_shift.sh <shift> ...
cd $GRAFT_REPO_ROOT
for v in "$@"; do
  if [ $v = auto ]; then L=""; else L="SKT_CSR_SHIFT=$v"; fi
  env $L python bench.py --config c2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('shift $v', d['roofline']['kernel_ms'], d['roofline']['frac'])"
done
