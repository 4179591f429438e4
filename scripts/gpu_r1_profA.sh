# round-1 evidence (A): default bench lines (94B, 12B) and the ncu launch list of the bench command
set -x
python bench.py > gpurun_out/bench_default.log 2>&1; echo bench rc=$?
python bench.py --config 12B > gpurun_out/bench_12B.log 2>&1; echo bench12 rc=$?
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu rc=$?
