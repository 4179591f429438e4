set -x
for hc in 32768 131072 262144; do
python bench.py --steps 5 --no-cpu-baseline --f1-count 0 --f3-count 0 --f2-rounds 0 --host-chunk $hc > gpurun_out/bench_hc$hc.log 2>&1; echo hc $hc rc=$?
done
