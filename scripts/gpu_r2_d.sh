# round 2: default bench (94B) with the new f1 / f3, ubench; ncu --set full of the f1 build kernel
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02d_build.log 2>&1; echo build rc=$?
timeout 900 python bench.py > gpurun_out/r02d_bench.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --config 12B --f2-rounds 4 > gpurun_out/r02d_bench12.log 2>&1; echo bench12 rc=$?
python bench.py --per-gpu 65536 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --f3-count 0 --f2-rounds 0 > gpurun_out/r02d_plain_f1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dip_order_kernel -s 2 -c 1 -o gpurun_out/prof_r02_f1_94B \
    python bench.py --per-gpu 65536 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --f3-count 0 --f2-rounds 0 > gpurun_out/r02d_ncu_f1.log 2>&1; echo ncu rc=$?
