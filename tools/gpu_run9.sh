mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_core.py -x -q -m gpu -k "lev" > gpurun_out/t9.log 2>&1; echo rc_t=$?; tail -25 gpurun_out/t9.log
