# round 2: scorer micro-variant A/B (packed count shuffles, clamped row load), 94B and 12B, two reps
set -x
A="--steps 5 --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 --f2-rounds 0"
for rep in 1 2; do
  for v in base pack clamp both; do
    if [ $v = base ]; then L=paper_2504_14145_b200/libdip.so; else L=paper_2504_14145_b200/libdip_$v.so; fi
    DIP_LIB=$L timeout 600 python bench.py $A > gpurun_out/r02ab_${v}_$rep.log 2>&1; echo $v $rep rc=$?
  done
done
for v in base pack both; do
  if [ $v = base ]; then L=paper_2504_14145_b200/libdip.so; else L=paper_2504_14145_b200/libdip_$v.so; fi
  DIP_LIB=$L timeout 600 python bench.py --config 12B $A > gpurun_out/r02ab_${v}_12B.log 2>&1
done
DIP_LIB=paper_2504_14145_b200/libdip_both.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not full_population" > gpurun_out/r02ab_par_both.log 2>&1; echo par rc=$?
