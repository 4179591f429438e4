set -x
timeout 900 python -m pytest tests/test_gpu_search.py tests/test_gpu_interleave.py -x -q > gpurun_out/t_search.log 2>&1; echo search rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not 94B_bench" > gpurun_out/t_c.log 2>&1; echo tests rc=$?
