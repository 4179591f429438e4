set -x
python bench.py --steps 5 > gpurun_out/bench_f1.log 2>&1; echo bench rc=$?
python bench.py --config 12B --steps 5 > gpurun_out/bench_f1_12B.log 2>&1; echo bench rc=$?
