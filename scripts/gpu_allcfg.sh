# every BASELINE.json config at N = 1 (default K / W, all side measurements)
set -x
for c in toy 12B 37B T2V 94B; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_cfg_$c.log 2>&1; echo $c rc=$?
done
