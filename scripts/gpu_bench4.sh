set -x
timeout 600 python bench.py > gpurun_out/bench_r1z.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --config 12B > gpurun_out/bench_r1z_12B.log 2>&1; echo bench12 rc=$?
