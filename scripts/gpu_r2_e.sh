# round 2: A/B of the record scorer -- channel rings (default) vs per-segment state (DIP_SCORER=segment)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02e_build.log 2>&1; echo build rc=$?
DIP_SCORER=segment timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not full_population" > gpurun_out/r02e_parity_seg.log 2>&1; echo parity_seg rc=$?
for cfg in 94B 12B T2V; do
  timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 --f2-rounds 0 > gpurun_out/r02e_ring_$cfg.log 2>&1
  DIP_SCORER=segment timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 --f2-rounds 0 > gpurun_out/r02e_seg_$cfg.log 2>&1
done
DIP_SCORER=segment timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_population and 94B" > gpurun_out/r02e_fullpop_seg.log 2>&1; echo fullpop_seg rc=$?
