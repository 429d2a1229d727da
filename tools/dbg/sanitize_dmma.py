"""Small fused-DMMA Hv / cache passes for compute-sanitizer (racecheck / synccheck): one p = 768, C = 10
shard (cluster layout: DSMEM exchange, mbarrier rings), products checked against the oracle port."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import oracle  # noqa: E402
import paper_1807_07132_b200 as nadmm  # noqa: E402

rng = np.random.default_rng(3)
n, p, C = 200, 768, 10
X = rng.normal(size=(n, p)) / np.sqrt(p)
y = (np.arange(n) % C + 1).astype(np.int32)
ds = nadmm.Dataset.dense(X, y, C)
sh = oracle.Shard(X, y, C)
port = oracle.Port()
w = rng.normal(size=sh.d) * 0.1
v = rng.normal(size=sh.d)
h = nadmm.hessian_vec(ds, w, v, 1e-3)
ho = port.hessian_vec(sh, w, v, 1e-3)
g = nadmm.gradient(ds, w, 1e-3)
err = max(np.abs(h - ho).max() / np.abs(ho).max(), np.abs(g - port.gradient(sh, w, 1e-3)).max() / np.abs(g).max())
print(f"sanitize run ok: rel err {err:.2e}")  # (no grid-barrier solver kernels: racecheck may serialise CTAs)
