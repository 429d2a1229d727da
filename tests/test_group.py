"""Node-group DMMA passes (csrc/dmma_group.cuh; opt-in NADMM_GROUP=1): the local nodes' Newton
iterations as one graph of full-GPU group launches must reproduce the oracle's ADMM loop, and the
WorkerPool round must match the reference's worker solves. Runs in a subprocess because the opt-in
switch is read once per process."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r'''
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import oracle
import paper_1807_07132_b200 as nadmm
port = oracle.Port()
out = {}
# ADMM over 4 DMMA nodes (p = 784 and 3072 layouts), spectral penalty
for p, n in [(784, 3000), (3072, 1800)]:
    N, C = 4, 10
    Xtr, ytr, _, _ = port.generate_synthetic(n, p, C, separation=3.0, noise=1.0, seed=4)
    owner = port.partition_owner(len(ytr), N)
    parts_o = [oracle.Shard(Xtr[owner == i], ytr[owner == i], C) for i in range(N)]
    parts_g = [nadmm.Dataset.dense(Xtr[owner == i], ytr[owner == i], C) for i in range(N)]
    ro = port.admm_run(parts_o, oracle.admm_cfg(n_workers=N, lam=1e-3, penalty="spectral", max_outer_iters=6))
    cfg = nadmm.AdmmConfig(n_workers=N, lam=1e-3, penalty=nadmm.PenaltyPolicy(kind="spectral"),
                           stopping=nadmm.StoppingConfig(max_outer_iters=6))
    rg = nadmm.run_admm(parts_g, cfg, nadmm.EvalContext(eval_objective=True))
    out[str(p)] = dict(it=[rg.iterations, ro["iterations"]],
                       z=float(np.abs(rg.z - ro["z"]).max() / np.abs(ro["z"]).max()),
                       f=max(abs(a["train_objective"] - b["train_objective"]) / abs(b["train_objective"])
                             for a, b in zip(rg.metrics, ro["metrics"])),
                       trace=all(a["cg_iters"] == b["cg_iters"] and a["fn_evals"] == b["fn_evals"]
                                 for a, b in zip(rg.metrics, ro["metrics"])))
    st = parts_g[0].ctx.stats()
# WorkerPool round through the group path vs the reference's worker solves
ref = oracle.ref()
rng = np.random.default_rng(15)
parts = [(rng.normal(size=(300 + 40 * i, 3072)) * 0.02, (np.arange(300 + 40 * i) % 10 + 1).astype(np.int32)) for i in range(4)]
ws = [nadmm.Worker(nadmm.Dataset.dense(X, y, 10)) for X, y in parts]
rws = [ref.dataset(oracle.Shard(X, y, 10)).worker() for X, y in parts]
d = 9 * 3072
errs, same = [], True
for k in range(2):
    z = rng.normal(size=d) * 0.01
    ys = [rng.normal(size=d) * 0.01 for _ in ws]
    rho = [1.0, 0.5, 2.0, 1.5]
    xs, sts = nadmm.workers_solve(ws, rho, z, ys)
    for i in range(4):
        xr, sr = rws[i].solve(rho[i], z, ys[i])
        errs.append(float(np.abs(xs[i] - xr).max() / np.abs(xr).max()))
        same = same and (sts[i].cg_iters, sts[i].fn_evals, sts[i].flags) == (sr["cg_iters"], sr["fn_evals"], sr["flags"])
out["workers"] = dict(err=max(errs), same=same)
print(json.dumps(out))
'''


def test_node_group_matches_oracle():
    env = dict(os.environ, NADMM_GROUP="1", NADMM_DMMA_VERBOSE="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "node group" in r.stderr  # the group path actually ran
    out = json.loads(r.stdout.strip().splitlines()[-1])
    for p in ("784", "3072"):
        o = out[p]
        assert o["it"][0] == o["it"][1] and o["trace"]
        assert o["z"] <= 1e-9 and o["f"] <= 1e-9
    assert out["workers"]["same"] and out["workers"]["err"] <= 1e-10
