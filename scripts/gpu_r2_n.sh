# round 2: the per-rank-order kernel in one large block per SM, BUILD without counters -- parity + f1 numbers
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02n_build.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_interleave.py tests/test_gpu_search.py tests/test_gpu_timeline.py tests/test_gpu_memopt.py tests/test_gpu_diamond.py tests/test_gpu_fuzz.py -x -q > gpurun_out/r02n_tests.log 2>&1; echo tests rc=$?
for cfg in 94B T2V 12B; do
  timeout 900 python bench.py --config $cfg --no-e2e --no-cpu-baseline > gpurun_out/r02n_bench_$cfg.log 2>&1; echo $cfg rc=$?
done
