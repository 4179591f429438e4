# round 2: f1 places on several ranks per step (conservative ring lookahead; shuffles outside the
# per-group branches) + f3 warm start's block-max argmax -- a quick gate first, then parity, f1 / f3
# numbers, lookahead depth A/B (DIP_ORDER_NIT 2 / 3 / 5) and an f1 capture
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02p_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_interleave.py -x -q -k "paper_pins or gating or bad or toy" > gpurun_out/r02p_quick.log 2>&1; rc=$?; echo quick rc=$rc
[ $rc -eq 0 ] || exit 1
for n in 2 5; do
  python -c "from paper_2504_14145_b200 import build as b; b.build(force=True, defines=['DIP_ORDER_NIT=$n'], out='paper_2504_14145_b200/libdip_nit$n.so')" >> gpurun_out/r02p_build.log 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_interleave.py tests/test_gpu_search.py tests/test_gpu_memopt.py tests/test_gpu_timeline.py tests/test_gpu_fuzz.py -x -q > gpurun_out/r02p_tests.log 2>&1; echo tests rc=$?
for cfg in 94B T2V 12B; do
  timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline > gpurun_out/r02p_bench_$cfg.log 2>&1; echo $cfg rc=$?
done
for n in 2 5; do
  DIP_LIB=paper_2504_14145_b200/libdip_nit$n.so timeout 600 python bench.py --config 94B --no-e2e --no-cpu-baseline --f3-count 0 --f2-rounds 0 > gpurun_out/r02p_bench_94B_nit$n.log 2>&1; echo nit$n rc=$?
done
B="--per-gpu 65536 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --f3-count 0 --f2-rounds 0"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dip_order_kernel -s 2 -c 1 -o gpurun_out/prof_r02p_f1_94B python bench.py $B > gpurun_out/r02p_ncu_f1.log 2>&1; echo ncu f1 rc=$?
