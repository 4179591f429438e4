# round-2 final evidence on one B200: pytest -m gpu, smoke, every config's bench line, reference arm,
# ncu launch list of the default bench, ncu --set full of the scorer and of f1
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fin_build.log 2>&1; echo build rc=$?
timeout 3000 python -m pytest tests/ -q -m gpu > gpurun_out/fin_tests.log 2>&1; echo tests rc=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo smoke rc=$?
for cfg in 94B toy 12B 37B T2V; do
  timeout 900 python bench.py --config $cfg > gpurun_out/fin_bench_$cfg.log 2>&1; echo bench $cfg rc=$?
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_bench_ref.log 2>&1; echo ref rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --f2-rounds 2 > gpurun_out/fin_ncu_launches.log 2>&1; echo launches rc=$?
A="--per-gpu 131072 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 --f2-rounds 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dip_eval_kernel -s 3 -c 1 -o gpurun_out/prof_fin_94B python bench.py $A > gpurun_out/fin_ncu_scorer.log 2>&1; echo ncu scorer rc=$?
B="--per-gpu 65536 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --f3-count 0 --f2-rounds 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dip_order_kernel -s 2 -c 1 -o gpurun_out/prof_fin_f1_94B python bench.py $B > gpurun_out/fin_ncu_f1.log 2>&1; echo ncu f1 rc=$?
