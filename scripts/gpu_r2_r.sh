# round 2: host-view end-to-end path with chunks ramping up from 1/8 (a short unoverlapped first copy)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02r_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q > gpurun_out/r02r_tests.log 2>&1; echo tests rc=$?
timeout 900 python bench.py > gpurun_out/r02r_bench_94B.log 2>&1; echo bench rc=$?
