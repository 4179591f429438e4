set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests/ -x -q -m gpu > gpurun_out/t_final.log 2>&1; echo tests rc=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_final_ref.log 2>&1; echo ref rc=$?
