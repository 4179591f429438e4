# round 2: f1 (placed-direction re-derive) and f3 (shorter bisection) -- parity, bench, ncu of f1 and f3
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02i_build.log 2>&1; echo build rc=$?
timeout 1200 python -m pytest tests/test_gpu_interleave.py tests/test_gpu_search.py tests/test_gpu_memopt.py tests/test_gpu_timeline.py tests/test_gpu_diamond.py tests/test_gpu_fuzz.py -x -q > gpurun_out/r02i_tests.log 2>&1; echo tests rc=$?
timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r02i_bench.log 2>&1; echo bench rc=$?
A="--per-gpu 65536 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --f2-rounds 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dip_order_kernel -s 2 -c 1 -o gpurun_out/prof_r02_f1b_94B python bench.py $A --f3-count 0 > gpurun_out/r02i_ncu_f1.log 2>&1; echo ncu f1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dip_memopt_kernel -s 2 -c 1 -o gpurun_out/prof_r02_f3_94B python bench.py $A --f1-count 0 > gpurun_out/r02i_ncu_f3.log 2>&1; echo ncu f3 rc=$?
