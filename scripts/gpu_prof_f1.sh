# one ncu --set full capture of the f1 interleaving kernel (94B, 65536 candidates)
set -x
python bench.py --per-gpu 65536 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --f3-count 0 --f2-rounds 0 > gpurun_out/plain_f1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dip_eval_kernel -s 6 -c 1 -o gpurun_out/prof_r01_f1_94B \
    python bench.py --per-gpu 65536 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --f3-count 0 --f2-rounds 0 > gpurun_out/ncu_f1.log 2>&1; echo ncu rc=$?
