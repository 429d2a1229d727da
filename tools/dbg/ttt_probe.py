"""Probe: theta trajectory of Newton-ADMM on the cfg2 workload for a few data/penalty settings."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1807_07132_b200 as nadmm  # noqa: E402

N_TOTAL, P, C, LAM, NODES = 55_556, 3072, 10, 1e-3, 8
ctx = nadmm.Context(0)
for sep in [float(a) for a in sys.argv[1:]] or [1.0, 3.0]:
    Xtr, ytr, Xte, yte = nadmm.generate_synthetic(N_TOTAL, P, C, sep, 1.0, 0)
    owner = nadmm.partition_owner(len(ytr), NODES)
    shards = [nadmm.Dataset.dense(Xtr[owner == i], ytr[owner == i], C, ctx=ctx) for i in range(NODES)]
    full = nadmm.Dataset.dense(Xtr, ytr, C, ctx=ctx)
    d = (C - 1) * P
    t0 = time.time()
    ref = nadmm.newton_solve(nadmm.make_softmax_objective(full, LAM), np.zeros(d),
                             nadmm.NewtonConfig(cg_tol=1e-10, cg_max_iters=200, grad_tol=1e-10, newton_max_iters=60))
    fstar = ref.trace[-1].objective
    print(f"sep={sep} F*={fstar:.6g} newton iters={len(ref.trace)} ({time.time() - t0:.1f}s)", flush=True)
    for kind in ("fixed", "spectral"):
        cfg = nadmm.AdmmConfig(n_workers=NODES, lam=LAM, penalty=nadmm.PenaltyPolicy(kind=kind),
                               stopping=nadmm.StoppingConfig(max_outer_iters=300))
        s = nadmm.AdmmSession(shards, cfg, nadmm.EvalContext(True, fstar, 0.0, True))
        s.step(300)
        r = s.result()
        rows = r.metrics
        th = [x["theta"] for x in rows]
        hit = [x for x in rows if x["theta"] <= 0.05]
        hit3 = [x for x in rows if x["theta"] <= 1e-3]
        conv = [x["iteration"] for x in rows if x.get("converged")]
        print(f"  {kind:9s} theta@1,5,10,30,100,300 = " + ", ".join(f"{th[k - 1]:.3g}" for k in (1, 5, 10, 30, 100, 300) if k <= len(th)) +
              f" | <=0.05 at it {hit[0]['iteration'] if hit else None} t={hit[0]['wall_seconds'] if hit else None}"
              f" | <=1e-3 at {hit3[0]['iteration'] if hit3 else None} | rho[0]={r.rho[0]:.3g}"
              f" acc={nadmm.accuracy(nadmm.predict(nadmm.Dataset.dense(Xte, yte, C, ctx=ctx), r.z), yte):.4f}"
              f" first-converged-flag-it={conv[0] if conv else None}", flush=True)
        s.close()
    for sh in shards:
        sh.close()
    full.close()
