# round 2: ncu --set full of the record scorer, channel rings vs per-segment state (94B, 131072 per launch)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02f_build.log 2>&1
A="--per-gpu 131072 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 --f2-rounds 0"
python bench.py $A > gpurun_out/r02f_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dip_eval_kernel -s 3 -c 1 -o gpurun_out/prof_r02_ring_94B python bench.py $A > gpurun_out/r02f_ncu_ring.log 2>&1; echo ring rc=$?
DIP_SCORER=segment timeout 900 ncu --set full --clock-control none --import-source on -k regex:dip_order_kernel -s 3 -c 1 -o gpurun_out/prof_r02_seg_94B python bench.py $A > gpurun_out/r02f_ncu_seg.log 2>&1; echo seg rc=$?
timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q > gpurun_out/r02f_pipeline.log 2>&1; echo pipeline rc=$?
timeout 900 python bench.py --f1-count 0 --f3-count 0 --f2-rounds 0 --no-cpu-baseline > gpurun_out/r02f_bench_e2e.log 2>&1; echo bench rc=$?
