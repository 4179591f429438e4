# round 2: f1 O(1) neighbour adds for every group width (G < 32 too): parity + f1 numbers per config
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02k_build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests/test_gpu_interleave.py tests/test_gpu_search.py tests/test_gpu_diamond.py tests/test_gpu_fuzz.py tests/test_gpu_timeline.py -x -q > gpurun_out/r02k_tests.log 2>&1; echo tests rc=$?
for cfg in 12B 37B T2V; do
  timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline --f3-count 0 --f2-rounds 0 > gpurun_out/r02k_bench_$cfg.log 2>&1; echo $cfg rc=$?
done
timeout 900 python -m pytest tests/test_gpu_memopt.py -x -q -k "raises_the_makespan_bound or bench_size" > gpurun_out/r02k_memopt.log 2>&1; echo memopt rc=$?
