import sys, os
sys.path.insert(0, os.getcwd())
mode = sys.argv[1]
if mode == "torch":
    import torch
    torch.cuda.set_device(0)
import numpy as np
import paper_1807_07132_b200 as nadmm
Xtr, ytr, _, _ = nadmm.generate_synthetic(int(sys.argv[2]), int(sys.argv[3]), 10, 3.0, 1.0, 0)
owner = nadmm.partition_owner(len(ytr), 8)
ctx = nadmm.Context(0)
shards = [nadmm.Dataset.dense(Xtr[owner == i], ytr[owner == i], 10, ctx=ctx) for i in range(8)]
cfg = nadmm.AdmmConfig(n_workers=8, lam=1e-3)
s = nadmm.AdmmSession(shards, cfg, nadmm.EvalContext(eval_objective=True, ignore_convergence=True))
print(mode, sys.argv[2:], "steps", s.step(3), s.metrics[-1]["train_objective"], flush=True)
