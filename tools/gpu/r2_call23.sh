# two GPUs: the NCCL consensus tests and the bench at N=2
timeout 1200 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/r2c23_multigpu.log 2>&1
echo "rc=$?" >> gpurun_out/r2c23_multigpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2c23_bench_n2.json 2> gpurun_out/r2c23_bench_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 --no-ttt > gpurun_out/r2c23_ref_n2.json 2> gpurun_out/r2c23_ref_n2.err
