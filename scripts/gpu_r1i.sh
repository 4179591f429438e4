set -x
timeout 1200 python -m pytest tests/test_gpu_memopt.py tests/test_gpu_search.py -x -q > gpurun_out/t_memopt2.log 2>&1; echo memopt rc=$?
timeout 600 python bench.py --steps 5 > gpurun_out/bench_f3b.log 2>&1; echo bench rc=$?
