set -x
timeout 900 python -m pytest tests/test_gpu_diamond.py -x -q > gpurun_out/t_diamond.log 2>&1; echo tests rc=$?
