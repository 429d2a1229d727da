# N=2 / N=4 bench lines with both time-to-target thresholds
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 > gpurun_out/r2c59_n2.json 2> gpurun_out/r2c59_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29572 bench.py --gpus 4 > gpurun_out/r2c59_n4.json 2> gpurun_out/r2c59_n4.err
nproc > gpurun_out/r2c59_nproc.txt
