# round 2: f2 search phase split (DIP_SEARCH_PROFILE: select / build / gpu / backprop wall times)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02t_build.log 2>&1
nproc > gpurun_out/r02t_nproc.txt
for cfg in 94B 12B; do
  DIP_SEARCH_PROFILE=1 timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 > gpurun_out/r02t_bench_$cfg.log 2>&1; echo $cfg rc=$?
done
