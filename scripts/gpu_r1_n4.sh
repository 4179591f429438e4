# 4-GPU checks: NCCL argmin test (4 ranks), bench at N=4 and its reference arm
set -x
nvidia-smi topo -m > gpurun_out/topo4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/t_multi4.log 2>&1; echo multi rc=$?
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench_n4.log 2>&1; echo bench4 rc=$?
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_n4.log 2>&1; echo ref4 rc=$?
