# round-1 evidence (C): one ncu --set full capture of the f3 selection kernel (94B, 16384 schedules)
set -x
python bench.py --per-gpu 16384 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --f1-count 0 --f2-rounds 0 > gpurun_out/plain_f3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dip_memopt -c 1 -o gpurun_out/prof_r01_f3_94B \
    python bench.py --per-gpu 16384 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --f1-count 0 --f2-rounds 0 > gpurun_out/ncu_f3.log 2>&1; echo ncu rc=$?
