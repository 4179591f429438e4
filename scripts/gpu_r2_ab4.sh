# round 2: scorer channel-ring depth A/B (D = 4 default vs 2 vs 8), with up to 24 warps per block
set -x
A="--steps 5 --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 --f2-rounds 0"
for rep in 1 2; do
  for v in d4 d2 d8; do
    if [ $v = d4 ]; then L=paper_2504_14145_b200/libdip.so; else L=paper_2504_14145_b200/libdip_$v.so; fi
    DIP_LIB=$L timeout 600 python bench.py $A > gpurun_out/ab4_${v}_$rep.log 2>&1; echo $v $rep rc=$?
    DIP_LIB=$L timeout 600 python bench.py --config T2V $A > gpurun_out/ab4_${v}_T2V_$rep.log 2>&1
  done
done
DIP_LIB=paper_2504_14145_b200/libdip_d2.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not full_population" > gpurun_out/ab4_parity_d2.log 2>&1; echo par2 rc=$?
