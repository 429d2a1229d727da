"""Bench workload (8 nodes, SPS) to theta <= 1e-3: outer iterations and device time (one GPU)."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1807_07132_b200 as nadmm  # noqa: E402

f_star = json.loads((Path(__file__).resolve().parents[2] / "profiles" / "r2_fstar.json").read_text())["f_star"]
Xtr, ytr, Xte, yte = nadmm.generate_synthetic(55_556, 3072, 10, 1.0, 1.0, 0)
owner = nadmm.partition_owner(len(ytr), 8)
ctx = nadmm.Context(0)
parts = [nadmm.Dataset.dense(Xtr[owner == i], ytr[owner == i], 10, ctx=ctx) for i in range(8)]
for target, cap in [(0.05, 300), (1e-2, 2000), (1e-3, 6000)]:
    cfg = nadmm.AdmmConfig(n_workers=8, lam=1e-3, penalty=nadmm.PenaltyPolicy(kind="spectral"),
                           stopping=nadmm.StoppingConfig(max_outer_iters=cap))
    s = nadmm.AdmmSession(parts, cfg, nadmm.EvalContext(True, f_star, target))
    t0 = time.perf_counter()
    s.step(cap)
    wall = time.perf_counter() - t0
    r = s.result()
    rows = r.metrics
    hit = [m for m in rows if m["theta"] <= target]
    print(json.dumps({"target": target, "iters": hit[0]["iteration"] if hit else None,
                      "seconds": hit[0]["wall_seconds"] if hit else None, "final_theta": rows[-1]["theta"],
                      "ran": len(rows), "wall": wall}), flush=True)
    s.close()
