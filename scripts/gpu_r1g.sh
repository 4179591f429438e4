set -x
timeout 900 python -m pytest tests/test_gpu_search.py tests/test_gpu_timeline.py -x -q > gpurun_out/t_search.log 2>&1; echo search rc=$?
python bench.py --steps 5 > gpurun_out/bench_f2.log 2>&1; echo bench rc=$?
