# e2e split (workers_solve vs host coordinator per rank) at N=4 and N=2, default vs passive OpenMP waits
for pol in default PASSIVE; do
  if [ $pol = default ]; then unset OMP_WAIT_POLICY; else export OMP_WAIT_POLICY=$pol; fi
  NADMM_BENCH_E2E_PROFILE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu --no-ttt > gpurun_out/r2c39_n4_$pol.json 2> gpurun_out/r2c39_n4_$pol.err
  NADMM_BENCH_E2E_PROFILE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-ttt > gpurun_out/r2c39_n2_$pol.json 2> gpurun_out/r2c39_n2_$pol.err
done
nproc > gpurun_out/r2c39_nproc.txt
