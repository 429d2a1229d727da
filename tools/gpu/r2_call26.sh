export PYTHONFAULTHANDLER=1
timeout -s INT 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --steps 10 --warmup 3 --no-ttt > gpurun_out/r2c26_n2_nottt.json 2> gpurun_out/r2c26_n2_nottt.err
echo "rc=$?" >> gpurun_out/r2c26_n2_nottt.err
timeout -s INT 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2c26_n2.json 2> gpurun_out/r2c26_n2.err
echo "rc=$?" >> gpurun_out/r2c26_n2.err
