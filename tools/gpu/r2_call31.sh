# four GPUs: headline bench at N=4 and N=2, cfg3 weak scaling at N=2 / N=4
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r2c31_bench_n4.json 2> gpurun_out/r2c31_bench_n4.err
echo "rc=$?" >> gpurun_out/r2c31_bench_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 bench.py --config cfg3 --gpus 4 --steps 10 --warmup 3 > gpurun_out/r2c31_cfg3_n4.json 2> gpurun_out/r2c31_cfg3_n4.err
echo "rc=$?" >> gpurun_out/r2c31_cfg3_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --config cfg3 --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2c31_cfg3_n2.json 2> gpurun_out/r2c31_cfg3_n2.err
echo "rc=$?" >> gpurun_out/r2c31_cfg3_n2.err
timeout 600 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/r2c31_multigpu.log 2>&1
echo "rc=$?" >> gpurun_out/r2c31_multigpu.log
