# A/B of scorer-loop variants (DIP_KV bits): parity on each, then alternating bench runs
set -x
for v in kv1 kv3 kv5 kv7; do
  DIP_LIB=paper_2504_14145_b200/libdip_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/ab_par_$v.log 2>&1; echo par $v rc=$?
done
for rep in 1 2; do
  for v in base kv1 kv3 kv5 kv7; do
    if [ $v = base ]; then L=paper_2504_14145_b200/libdip.so; else L=paper_2504_14145_b200/libdip_$v.so; fi
    DIP_LIB=$L python bench.py --steps 5 --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 --f2-rounds 0 > gpurun_out/ab_${v}_$rep.log 2>&1; echo bench $v $rep rc=$?
  done
done
