# round-2 final evidence on a 4×B200 box: the 4-rank NCCL argmin test, bench at N = 2 and N = 4
set -x
nvidia-smi topo -m > gpurun_out/fin4_topo.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fin4_build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/fin4_multi_test.log 2>&1; echo multi rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 tests/workers/multi_gpu_argmin.py > gpurun_out/fin4_multi4.log 2>&1; echo multi4 rc=$?
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/fin4_bench_n4.log 2>&1; echo bench4 rc=$?
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/fin4_bench_n2.log 2>&1; echo bench2 rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 4 --impl reference --steps 3 --warmup 1 > gpurun_out/fin4_bench_ref_n4.log 2>&1; echo ref4 rc=$?
