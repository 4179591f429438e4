set -x
timeout 900 python -m pytest tests/test_gpu_memopt.py tests/test_gpu_pipeline.py tests/test_gpu_search.py -x -q > gpurun_out/t_f3e.log 2>&1; echo tests rc=$?
timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bench_f3e.log 2>&1; echo bench rc=$?
