set -x
timeout 900 python -m pytest tests/test_gpu_fuzz.py -x -q > gpurun_out/t_fuzz.log 2>&1; echo tests rc=$?
