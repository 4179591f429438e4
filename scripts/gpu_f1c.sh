set -x
timeout 900 python -m pytest tests/test_gpu_interleave.py tests/test_gpu_search.py -x -q > gpurun_out/t_f1c.log 2>&1; echo tests rc=$?
timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bench_f1c.log 2>&1; echo bench rc=$?
python bench.py --config 12B --steps 5 --no-cpu-baseline > gpurun_out/bench_f1c_12B.log 2>&1; echo bench12 rc=$?
