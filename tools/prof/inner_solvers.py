"""Newton-CG vs L-BFGS as the ADMM workers' inner solver (the paper's Fig. 1-style
comparison) and synchronous mini-batch SGD with the Appendix's step-size sweep (§8f #4; Fig. 2-style)
on the bench workload: CIFAR-shaped 50,000 x 3,072, C = 10, 8 ADMM nodes on one GPU,
SPS penalty, lambda = 1e-3. Reports time-to-target theta = (F - F*)/F* <= 0.05 and time per outer
iteration. usage: python tools/prof/inner_solvers.py [max_outer_iters]"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_1807_07132_b200 as nadmm  # noqa: E402


def main(max_outer: int):
    ctx = nadmm.Context(0)
    Xtr, ytr, _, _, owner = bench.make_data()
    C, lam, nodes = bench.C, bench.LAM, bench.NODES
    shards = [nadmm.Dataset.dense(Xtr[owner == i], ytr[owner == i], C, ctx=ctx) for i in range(nodes)]
    full = nadmm.Dataset.dense(Xtr, ytr, C, ctx=ctx)
    d = full.weight_dim()
    ref = nadmm.newton_solve(nadmm.make_softmax_objective(full, lam), np.zeros(d),
                             nadmm.NewtonConfig(cg_tol=1e-10, cg_max_iters=200, grad_tol=1e-10, newton_max_iters=60))
    fstar = ref.trace[-1].objective
    full.close()
    sps = nadmm.PenaltyPolicy(kind="spectral")
    out = []
    for solver, inner in [("newton", 1), ("lbfgs", 1), ("lbfgs", 5), ("lbfgs", 10)]:
        cfg = nadmm.AdmmConfig(n_workers=nodes, lam=lam, penalty=sps, inner_iters=inner, inner_solver=solver,
                               stopping=nadmm.StoppingConfig(max_outer_iters=max_outer))
        for s in shards:  # fresh warm starts per run
            nadmm.Worker(s)
        r = nadmm.run_admm(shards, cfg, nadmm.EvalContext(True, fstar, bench.THETA_TARGET))
        rows = r.metrics
        hit = [m for m in rows if m["theta"] == m["theta"] and m["theta"] <= bench.THETA_TARGET]
        line = {"inner_solver": solver, "inner_iters": inner, "outer_iters": r.iterations,
                "time_to_target_s": hit[0]["wall_seconds"] if hit else None,
                "ttt_outer_iters": hit[0]["iteration"] if hit else None,
                "final_theta": rows[-1]["theta"] if rows else None,
                "ms_per_outer_iter": 1e3 * rows[-1]["wall_seconds"] / len(rows) if rows else None,
                "fn_evals_total": int(sum(m["fn_evals"] for m in rows)),
                "cg_iters_total": int(sum(m["cg_iters"] for m in rows))}
        print(json.dumps(line), flush=True)
        out.append(line)
    # sync-SGD: batch 100 per worker, ceil(n / (m N)) steps per epoch, eta swept by decades
    n_total = sum(s.n() for s in shards)
    for eta in [1e-4, 1e-3, 1e-2, 1e-1, 1.0, 10.0]:
        cfg = nadmm.SgdConfig(eta=eta, batch=100, epochs=5, seed=0)
        try:
            r = nadmm.sync_sgd(shards, cfg, lam)
        except nadmm.SolverError as e:
            print(json.dumps({"solver": "sync_sgd", "eta": eta, "diverged": str(e)}), flush=True)
            continue
        thetas = [(m["train_objective"] - fstar) / fstar for m in r.metrics]
        line = {"solver": "sync_sgd", "eta": eta, "batch": 100, "epochs": r.epochs,
                "steps_per_epoch": r.metrics[0]["inner_iterations"] if r.metrics else None,
                "messages_per_epoch": r.metrics[0]["messages"] if r.metrics else None,
                "theta_per_epoch": thetas, "seconds": r.metrics[-1]["wall_seconds"] if r.metrics else None,
                "n_total": n_total}
        print(json.dumps(line), flush=True)
        out.append(line)
    return out


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 100)
