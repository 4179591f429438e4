# round 2: f3 per-rank ILP on the GPU (parity incl. branch and bound), full-population parity, smoke
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02a_build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests/test_gpu_memopt.py -x -q -s > gpurun_out/r02a_memopt.log 2>&1; echo memopt rc=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -s -k full_population > gpurun_out/r02a_fullpop.log 2>&1; echo fullpop rc=$?
timeout 900 python -m pytest tests/test_gpu_interleave.py -x -q -s -k bench_size_full > gpurun_out/r02a_f1full.log 2>&1; echo f1full rc=$?
