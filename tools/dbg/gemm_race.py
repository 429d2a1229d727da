"""Debug: two-GEMM Hv race hunt (n sweep, class counts, feature counts)."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import oracle  # noqa: E402
import paper_1807_07132_b200 as nadmm  # noqa: E402

port = oracle.Port()
rel = lambda a, b: np.abs(a - b).max() / np.abs(b).max()
for n, p, C in [(40000, 2048, 100), (60000, 2048, 21), (60000, 200, 100), (60000, 64, 100), (40000, 2048, 3)]:
    rng = np.random.default_rng(1)
    X = rng.normal(size=(n, p)) / np.sqrt(p)
    y = (np.arange(n) % C + 1).astype(np.int32)
    ds = nadmm.Dataset.dense(X, y, C)
    sh = oracle.Shard(X, y, C)
    w = rng.normal(size=sh.d) * 0.3
    v = rng.normal(size=sh.d)
    hg = nadmm.hessian_vec(ds, w, v, 1e-3)
    hg2 = nadmm.hessian_vec(ds, w, v, 1e-3)
    hp = port.hessian_vec(sh, w, v, 1e-3)
    g1 = nadmm.gradient(ds, w * 1.01, 1e-3)
    gp = port.gradient(sh, w * 1.01, 1e-3)
    print(f"n={n} p={p} C={C} poison={os.environ.get('NADMM_GEMM_POISON_U')}: hv {rel(hg, hp):.2e} nan {np.isnan(hg).sum()} "
          f"repeat {np.array_equal(hg, hg2)} grad {rel(g1, gp):.2e}", flush=True)
    ds.close()
