set -x
timeout 1500 python -m pytest tests/test_gpu_memopt.py -x -q -s > gpurun_out/r02b_memopt.log 2>&1; echo memopt rc=$?
