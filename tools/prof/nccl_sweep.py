"""NVLink 5 / NVSwitch all-reduce sweep: ncclAllReduce of float64 buffers from 8 B to
256 MiB on N GPUs of one box, CUDA-event time per call (max over ranks), algorithmic and bus
bandwidth (busbw = algbw x 2 (N - 1) / N, nccl-tests convention). The consensus loop's own buffer
(d + 1 doubles plus the per-rank stat slots, ~221 KB at the bench workload) is in the sweep.
usage: python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/prof/nccl_sweep.py"""
import json
import os

import torch
import torch.distributed as dist


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sizes = [8 << k for k in range(0, 26, 1)] + [221_192]  # 8 B .. 256 MiB, + the consensus buffer
    out = []
    for nbytes in sorted(set(sizes)):
        n = max(1, nbytes // 8)
        x = torch.ones(n, dtype=torch.float64, device="cuda")
        reps = 50 if nbytes <= (4 << 20) else 10
        for _ in range(5):
            dist.all_reduce(x)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            dist.all_reduce(x)
        e1.record()
        e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / reps], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        us = float(t.item()) * 1e3
        alg = n * 8 / (us * 1e-6) / 1e9
        out.append({"bytes": n * 8, "us": us, "algbw_gbs": alg, "busbw_gbs": alg * 2 * (world - 1) / world})
    if rank == 0:
        print(json.dumps({"n_gpus": world, "nccl": ".".join(map(str, torch.cuda.nccl.version())), "sweep": out}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
