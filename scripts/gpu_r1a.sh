set -x
python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
python bench.py > gpurun_out/bench_94B.log 2>&1; echo bench rc=$?
python bench.py --config 12B > gpurun_out/bench_12B.log 2>&1; echo bench12 rc=$?
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
python bench.py --per-gpu 131072 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --per-gpu 131072 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dip_eval -s 3 -c 1 -o gpurun_out/prof_94B python bench.py --per-gpu 131072 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
