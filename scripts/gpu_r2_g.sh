# round 2: f1 kernel with ready-set summaries + O(1) neighbour adds + consumer-ready slots; tests + f1/f2 numbers
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02g_build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_interleave.py tests/test_gpu_search.py tests/test_gpu_timeline.py tests/test_gpu_memopt.py tests/test_gpu_diamond.py -x -q -k "not full_size and not bench_size" > gpurun_out/r02g_tests.log 2>&1; echo tests rc=$?
timeout 900 python bench.py --no-e2e --no-cpu-baseline --f3-count 0 > gpurun_out/r02g_bench.log 2>&1; echo bench rc=$?
