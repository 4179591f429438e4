# round 2: the ready-set f1 kernel (dip_order.cu) and everything built on it vs the oracle
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02c_build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_interleave.py -x -q -s -k "not bench_size_full" > gpurun_out/r02c_f1.log 2>&1; echo f1 rc=$?
timeout 900 python -m pytest tests/test_gpu_search.py tests/test_gpu_timeline.py tests/test_gpu_memopt.py -x -q -s -k "orders or search or timeline" > gpurun_out/r02c_f2.log 2>&1; echo f2 rc=$?
timeout 900 python -m pytest tests/test_gpu_diamond.py tests/test_gpu_fuzz.py tests/test_gpu_pipeline.py -x -q > gpurun_out/r02c_misc.log 2>&1; echo misc rc=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.log 2>&1; echo smoke rc=$?
