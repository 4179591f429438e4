# round 2: small order-kernel launches (f2's rounds) spread over every SM with fewer warps per block
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02u_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_interleave.py -x -q -k "paper_pins or gating or bad or toy" > gpurun_out/r02u_quick.log 2>&1; rc=$?; echo quick rc=$rc
[ $rc -eq 0 ] || exit 1
timeout 1500 python -m pytest tests/test_gpu_interleave.py tests/test_gpu_search.py tests/test_gpu_memopt.py tests/test_gpu_timeline.py -x -q > gpurun_out/r02u_tests.log 2>&1; echo tests rc=$?
for cfg in 94B 12B T2V; do
  DIP_SEARCH_PROFILE=1 timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline > gpurun_out/r02u_bench_$cfg.log 2>&1; echo $cfg rc=$?
done
