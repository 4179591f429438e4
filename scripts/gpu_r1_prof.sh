# round-1 evidence: default bench line, its ncu launch list, one full capture of the scorer kernel
set -x
python bench.py > gpurun_out/bench_default.log 2>&1; echo bench rc=$?
python bench.py --config 12B > gpurun_out/bench_12B.log 2>&1; echo bench12 rc=$?
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1 && \
python bench.py --per-gpu 131072 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dip_eval -s 3 -c 1 -o gpurun_out/prof_r01_94B \
    python bench.py --per-gpu 131072 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
