set -x
DIP_LIB=paper_2504_14145_b200/libdip_f3t.so timeout 900 python -m pytest tests/test_gpu_memopt.py tests/test_gpu_pipeline.py tests/test_gpu_diamond.py tests/test_gpu_fuzz.py tests/test_gpu_search.py -x -q > gpurun_out/ab_par_f3t.log 2>&1; echo par f3t rc=$?
for rep in 1 2; do
  for v in base f3t; do
    if [ $v = base ]; then L=paper_2504_14145_b200/libdip.so; else L=paper_2504_14145_b200/libdip_$v.so; fi
    DIP_LIB=$L python bench.py --steps 2 --no-e2e --no-cpu-baseline --f1-count 0 --f2-rounds 0 > gpurun_out/ab8_${v}_$rep.log 2>&1; echo bench $v $rep rc=$?
  done
done
