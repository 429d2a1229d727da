"""Debug: two-GEMM path Hv / gradient vs the oracle port at growing n (C = 100, p = 2048)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import oracle  # noqa: E402
import paper_1807_07132_b200 as nadmm  # noqa: E402

port = oracle.Port()
for n, p, C in [(389, 2048, 100), (1500, 2048, 100), (5000, 2048, 100), (20000, 2048, 100), (20000, 200, 100),
                (20000, 2048, 21), (3000, 2048, 100)]:
    rng = np.random.default_rng(n + p)
    X = rng.normal(size=(n, p)) / 45
    y = (np.arange(n) % C + 1).astype(np.int32)
    ds = nadmm.Dataset.dense(X, y, C)
    sh = oracle.Shard(X, y, C)
    w = rng.normal(size=sh.d) * 0.01
    v = rng.normal(size=sh.d)
    g = nadmm.gradient(ds, w, 1e-3)
    go = port.gradient(sh, w, 1e-3)
    h = nadmm.hessian_vec(ds, w, v, 1e-3)
    ho = port.hessian_vec(sh, w, v, 1e-3)
    rg = np.abs(g - go).max() / np.abs(go).max()
    rh = np.abs(h - ho).max() / np.abs(ho).max()
    bad = np.abs(h - ho).reshape(C - 1, p)
    print(f"n={n} p={p} C={C}: grad {rg:.2e} hv {rh:.2e}  worst class {bad.max(1).argmax()} feature "
          f"{bad.max(0).argmax()}", flush=True)
    ds.close()
