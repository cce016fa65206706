# fp64 tensor-core K5 (lev_dmma): parity, timing vs the CUDA-core kernel, ncu
cd $GRAFT_REPO_ROOT
F=gpurun_out/r2g; mkdir -p $F
timeout 900 python -m pytest tests/test_gpu_core.py -q -x -k "lev" > $F/pytest.log 2>&1; echo rc_pytest=$?
python bench.py --config c4 --kernel lev --lev-f64 --no-e2e --no-cpu-baseline > $F/lev64.json 2> $F/lev64.err; echo rc_lev64=$?
SKT_LEV_DMMA=0 python bench.py --config c4 --kernel lev --lev-f64 --no-e2e --no-cpu-baseline > $F/lev64_cuda_core.json 2> $F/lev64_cc.err; echo rc_lev64cc=$?
python bench.py --config c4 --kernel lev --no-e2e --no-cpu-baseline > $F/lev32.json 2> $F/lev32.err; echo rc_lev32=$?
