set -x
DIP_LIB=paper_2504_14145_b200/libdip_c8.so timeout 900 python -m pytest tests/test_gpu_interleave.py tests/test_gpu_search.py tests/test_gpu_diamond.py tests/test_gpu_fuzz.py -x -q > gpurun_out/ab_par_c8.log 2>&1; echo par c8 rc=$?
for rep in 1 2; do
  for v in base c8; do
    if [ $v = base ]; then L=paper_2504_14145_b200/libdip.so; else L=paper_2504_14145_b200/libdip_$v.so; fi
    DIP_LIB=$L python bench.py --steps 2 --no-e2e --no-cpu-baseline --f3-count 0 --f2-rounds 0 > gpurun_out/ab6_${v}_$rep.log 2>&1; echo bench $v $rep rc=$?
  done
done
