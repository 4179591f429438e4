set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not 94B_bench" > gpurun_out/t_b.log 2>&1; echo tests rc=$?
python __graft_entry__.py > gpurun_out/smoke_b.log 2>&1; echo smoke rc=$?
python bench.py --per-gpu 262144 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_b.log 2>&1; echo bench rc=$?
python bench.py --per-gpu 131072 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dip_eval -s 3 -c 1 -o gpurun_out/prof_94B_b python bench.py --per-gpu 131072 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_b.log 2>&1; echo ncu rc=$?
