# round 2: the scorer with D = 2 rings and one large block per SM -- every record-scorer parity suite
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02m_build.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_timeline.py tests/test_gpu_diamond.py tests/test_gpu_memopt.py tests/test_gpu_pipeline.py -x -q -s > gpurun_out/r02m_parity.log 2>&1; echo parity rc=$?
for cfg in 94B 37B T2V 12B; do
  timeout 900 python bench.py --config $cfg > gpurun_out/r02m_bench_$cfg.log 2>&1; echo $cfg rc=$?
done
