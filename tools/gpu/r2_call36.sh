# N=2 / N=4 bench lines with the native host coordinator in e2e; multi-GPU tests at N=4;
# one ncu --set full capture of the bench's own (quarter-GPU) DMMA Hv launch on one GPU
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2c36_bench_n2.json 2> gpurun_out/r2c36_bench_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r2c36_bench_n4.json 2> gpurun_out/r2c36_bench_n4.err
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -x > gpurun_out/r2c36_mgpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2c36_mgpu.log
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dmma_pass_kernel --launch-skip 300 -c 1 -o gpurun_out/r2c36_bench_dmma python bench.py --no-cpu --no-ttt --steps 2 --warmup 3 > gpurun_out/r2c36_ncu.log 2>&1
