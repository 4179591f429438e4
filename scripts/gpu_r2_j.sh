# round 2: parity of the packed-count scorer (incl. full 94B population), f3 bound / 1,024 samples,
# exploration policies, pipeline; default bench with the f2 policy comparison
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02j_build.log 2>&1; echo build rc=$?
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_memopt.py tests/test_gpu_search.py tests/test_gpu_pipeline.py tests/test_gpu_fuzz.py -x -q -s > gpurun_out/r02j_tests.log 2>&1; echo tests rc=$?
timeout 900 python bench.py > gpurun_out/r02j_bench.log 2>&1; echo bench rc=$?
