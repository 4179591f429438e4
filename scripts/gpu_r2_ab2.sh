# round 2: scorer A/B -- base (packed shuffles) vs + kept-packed counters, 32-bit bit-row offsets and
# single-index slot addressing; parity of the new loop
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab2_build.log 2>&1
A="--steps 5 --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 --f2-rounds 0"
for rep in 1 2; do
  for v in base new; do
    if [ $v = new ]; then L=paper_2504_14145_b200/libdip.so; else L=paper_2504_14145_b200/libdip_base.so; fi
    DIP_LIB=$L timeout 600 python bench.py $A > gpurun_out/ab2_${v}_$rep.log 2>&1; echo $v $rep rc=$?
    DIP_LIB=$L timeout 600 python bench.py --config 12B $A > gpurun_out/ab2_${v}_12B_$rep.log 2>&1
  done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_timeline.py tests/test_gpu_diamond.py tests/test_gpu_memopt.py -x -q -k "not bench_size" > gpurun_out/ab2_parity.log 2>&1; echo parity rc=$?
