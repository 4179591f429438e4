# round 2 evidence: full GPU test suite, smoke, every BASELINE.json config at N=1 (bench lines),
# the ncu launch list of the default bench command
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02h_build.log 2>&1; echo build rc=$?
timeout 2400 python -m pytest tests/ -q -m gpu > gpurun_out/r02h_tests.log 2>&1; echo tests rc=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; echo smoke rc=$?
for cfg in toy 12B 37B T2V 94B; do
  timeout 900 python bench.py --config $cfg > gpurun_out/r02h_bench_$cfg.log 2>&1; echo bench $cfg rc=$?
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02h_bench_ref.log 2>&1; echo ref rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --f2-rounds 2 > gpurun_out/r02h_ncu_launches.log 2>&1; echo launches rc=$?
