# 4-GPU checks on the round-2 start tree: the NCCL argmin worker (4 ranks, RESULT line kept),
# bench at N=2 and N=4 (94B, 1,048,576 candidates per GPU)
set -x
nvidia-smi topo -m > gpurun_out/r02_topo4.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02_build.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tests/workers/multi_gpu_argmin.py > gpurun_out/r02_multi4.log 2>&1; echo multi rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 4 --steps 5 --warmup 3 --f2-rounds 0 > gpurun_out/r02_bench_n4.log 2>&1; echo bench4 rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --f2-rounds 0 > gpurun_out/r02_bench_n2.log 2>&1; echo bench2 rc=$?
