# NCCL all-reduce sweep on 2 and 4 GPUs (BASELINE.md §2 denominator)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 tools/prof/nccl_sweep.py > gpurun_out/r2c60_nccl_n2.json 2> gpurun_out/r2c60_nccl_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29582 tools/prof/nccl_sweep.py > gpurun_out/r2c60_nccl_n4.json 2> gpurun_out/r2c60_nccl_n4.err
