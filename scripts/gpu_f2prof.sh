set -x
DIP_SEARCH_PROFILE=1 timeout 600 python bench.py --steps 2 --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 > gpurun_out/f2prof.log 2>&1; echo rc=$?
DIP_SEARCH_PROFILE=1 timeout 600 python bench.py --config 12B --steps 2 --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 > gpurun_out/f2prof12.log 2>&1; echo rc=$?
