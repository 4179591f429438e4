# round 2: scorer occupancy A/B -- up to 8 warps per block (3 blocks/SM) vs up to 24 (one large block)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab3_build.log 2>&1
A="--steps 5 --no-e2e --no-cpu-baseline --f1-count 0 --f3-count 0 --f2-rounds 0"
for rep in 1 2; do
  for w in 8 24 12; do
    DIP_MAXWPB=$w timeout 600 python bench.py $A > gpurun_out/ab3_w${w}_$rep.log 2>&1; echo $w $rep rc=$?
    DIP_MAXWPB=$w timeout 600 python bench.py --config 12B $A > gpurun_out/ab3_w${w}_12B_$rep.log 2>&1
    DIP_MAXWPB=$w timeout 600 python bench.py --config T2V $A > gpurun_out/ab3_w${w}_T2V_$rep.log 2>&1
  done
done
DIP_MAXWPB=24 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not full_population" > gpurun_out/ab3_parity.log 2>&1; echo parity rc=$?
