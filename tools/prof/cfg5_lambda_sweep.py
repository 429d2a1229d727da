"""cfg5 lambda sweep (large dense 4M x 2048, C = 100, lambda in {1e-5, 1e-4, 1e-3, 1e-2}
with the spectral penalty): the 8 row-shard nodes (500,000 x 2,048 each, per-node seeds
mix_seed(0, node), built once) on one B200, `iters` Newton-ADMM outer iterations per lambda with F(z)
evaluated every iteration. Reports per lambda the device time per outer iteration, Hv/s, and the
per-iteration objective, residuals and mean penalty (the SPS adaptation). No F* (SURVEY: per-
iteration timing for cfg4/5; a full-data reference solve would need the 65 GB matrix on one host).
usage: python tools/prof/cfg5_lambda_sweep.py [iters]"""
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_1807_07132_b200 as nadmm  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    workload, kind, p, C_, _, nodes, rows = bench.CONFIGS["cfg5"]
    ctx = nadmm.Context(0)
    t0 = time.perf_counter()
    shards = [bench.config_shard(nadmm, "cfg5", i, kind, p, C_, rows, ctx)[0] for i in range(nodes)]
    gen_s = time.perf_counter() - t0
    stream = torch.cuda.ExternalStream(ctx.stream)
    out = []
    for lam in (1e-5, 1e-4, 1e-3, 1e-2):
        cfg = nadmm.AdmmConfig(n_workers=nodes, lam=lam, penalty=nadmm.PenaltyPolicy(kind="spectral"),
                               stopping=nadmm.StoppingConfig(max_outer_iters=iters))
        sess = nadmm.AdmmSession(shards, cfg, nadmm.EvalContext(eval_objective=True, ignore_convergence=True))
        ctx.reset_stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        done = sess.step(iters)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        st = ctx.stats()
        rows_m = sess.result().metrics
        sess.close()
        keep = ("iteration", "train_objective", "primal_norm", "dual_norm", "rho_mean", "cg_iters")
        out.append({"lambda": lam, "outer_iters": done, "ms_per_outer_iter": ms / max(done, 1),
                    "hv_per_s": st["hv_products"] / (ms * 1e-3),
                    "metrics": [{k: m.get(k) for k in keep} for m in rows_m]})
        print(json.dumps({"lambda": lam, "ms_per_outer_iter": out[-1]["ms_per_outer_iter"],
                          "hv_per_s": out[-1]["hv_per_s"], "final": out[-1]["metrics"][-1] if rows_m else None}),
              file=sys.stderr, flush=True)
    # importing bench routes fd 1 to stderr (library banners); its emit() writes the real stdout
    bench.emit({"workload": workload + " (lambda sweep)", "nodes": nodes, "rows_per_node": shards[0].n(),
                "generation_s": gen_s, "iters_per_lambda": iters, "sweep": out})


if __name__ == "__main__":
    main()
