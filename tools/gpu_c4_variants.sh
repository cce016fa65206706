# kernel time of config 4 under build variants: bash tools/gpu_c4_variants.sh <variant|base> ...
cd $GRAFT_REPO_ROOT
for v in "$@"; do
  if [ $v = base ]; then L=""; else L="SKT_LIB_PATH=tools/libsketch_$v.so"; fi
  env $L python bench.py --config c4 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['roofline']['kernel_ms'], d['roofline']['frac'])"
done
