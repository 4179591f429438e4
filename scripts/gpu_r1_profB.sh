# round-1 evidence (B): one ncu --set full capture of the scorer kernel (94B, 131072 candidates per launch)
set -x
python bench.py --per-gpu 131072 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 --f2-rounds 0 > gpurun_out/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dip_eval -s 3 -c 1 -o gpurun_out/prof_r01_94B \
    python bench.py --per-gpu 131072 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 --f2-rounds 0 > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
