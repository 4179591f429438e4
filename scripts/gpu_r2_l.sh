set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02l_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fuzz.py -x -q > gpurun_out/r02l_fuzz.log 2>&1; echo fuzz rc=$?
