set -x
timeout 2400 python -m pytest tests/ -x -q -m gpu > gpurun_out/t_full2.log 2>&1; echo tests rc=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > gpurun_out/bench_full2.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --config 12B > gpurun_out/bench_full2_12B.log 2>&1; echo bench12 rc=$?
