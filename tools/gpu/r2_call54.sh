# final verification on 2 GPUs: whole GPU suite (incl. 2-rank NCCL tests), smoke, N=1 and N=2 bench lines
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2c54_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c54_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2c54_smoke.log 2>&1
timeout 900 python bench.py --no-cpu > gpurun_out/r2c54_bench_n1.json 2> gpurun_out/r2c54_bench_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 > gpurun_out/r2c54_bench_n2.json 2> gpurun_out/r2c54_bench_n2.err
