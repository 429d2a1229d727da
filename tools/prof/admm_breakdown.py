"""Where an outer ADMM iteration's time goes (bench workload, N = 1, device-resident loop):
with / without the per-iteration F(z) evaluation, vs the Newton graphs alone (worker solves)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1807_07132_b200 as nadmm  # noqa: E402

N_TOTAL, P, C, LAM, NODES = 55_556, 3072, 10, 1e-3, 8
ctx = nadmm.Context(0)
Xtr, ytr, _, _ = nadmm.generate_synthetic(N_TOTAL, P, C, 1.0, 1.0, 0)
owner = nadmm.partition_owner(len(ytr), NODES)
shards = [nadmm.Dataset.dense(Xtr[owner == i], ytr[owner == i], C, ctx=ctx) for i in range(NODES)]
stream = torch.cuda.ExternalStream(ctx.stream)


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.synchronize()
    t0 = time.perf_counter()
    e0.record(stream)
    fn(reps)
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps, (time.perf_counter() - t0) * 1e3 / reps


for ev in (True, False):
    cfg = nadmm.AdmmConfig(n_workers=NODES, lam=LAM, penalty=nadmm.PenaltyPolicy(kind="spectral"),
                           stopping=nadmm.StoppingConfig(max_outer_iters=100000))
    s = nadmm.AdmmSession(shards, cfg, nadmm.EvalContext(eval_objective=ev, ignore_convergence=True))
    s.step(3)
    dev, host = timed(lambda r: s.step(r), 10)
    print(f"outer iteration, eval_objective={ev}: {dev:.3f} ms device, {host:.3f} ms host", flush=True)
    s.close()

workers = [nadmm.Worker(sh) for sh in shards]
d = shards[0].weight_dim()
z, y = np.zeros(d), np.zeros(d)


def solves(r):
    for _ in range(r):
        for w in workers:
            w.solve(1.0, z, y, nadmm.NewtonConfig(), 1)


dev, host = timed(solves, 5)
print(f"8 worker solves through the ABI (host z/y, x back): {dev:.3f} ms device, {host:.3f} ms host")
