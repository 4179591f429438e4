# round 2: f1 selection walk takes two positions per pass
# -- quick gate, parity, f1 numbers, f1 capture
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02y_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_interleave.py -x -q -k "paper_pins or gating or bad or toy" > gpurun_out/r02y_quick.log 2>&1; rc=$?; echo quick rc=$rc
[ $rc -eq 0 ] || exit 1
timeout 1500 python -m pytest tests/test_gpu_interleave.py tests/test_gpu_search.py tests/test_gpu_memopt.py tests/test_gpu_timeline.py tests/test_gpu_fuzz.py tests/test_gpu_diamond.py -x -q > gpurun_out/r02y_tests.log 2>&1; echo tests rc=$?
for cfg in 94B T2V 12B; do
  timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline > gpurun_out/r02y_bench_$cfg.log 2>&1; echo $cfg rc=$?
done
B="--per-gpu 65536 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --f3-count 0 --f2-rounds 0"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dip_order_kernel -s 2 -c 1 -o gpurun_out/prof_r02y_f1_94B python bench.py $B > gpurun_out/r02y_ncu_f1.log 2>&1; echo ncu f1 rc=$?
