set -x
DIP_LIB=paper_2504_14145_b200/libdip_kx.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_diamond.py tests/test_gpu_fuzz.py tests/test_gpu_timeline.py -x -q > gpurun_out/ab_par_kx.log 2>&1; echo par kx rc=$?
for rep in 1 2; do
  for v in base kx; do
    if [ $v = base ]; then L=paper_2504_14145_b200/libdip.so; else L=paper_2504_14145_b200/libdip_$v.so; fi
    DIP_LIB=$L python bench.py --steps 5 --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 --f2-rounds 0 > gpurun_out/ab10_${v}_$rep.log 2>&1; echo bench $v $rep rc=$?
  done
done
DIP_LIB=paper_2504_14145_b200/libdip_kx.so python bench.py --config 12B --steps 5 --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 --f2-rounds 0 > gpurun_out/ab10_kx_12B.log 2>&1
python bench.py --config 12B --steps 5 --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 --f2-rounds 0 > gpurun_out/ab10_base_12B.log 2>&1
