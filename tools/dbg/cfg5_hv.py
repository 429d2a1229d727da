"""Debug: cfg5-sized (125,000 x 2,048, C = 100) Hv: GPU vs the port vs the reference build."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import oracle  # noqa: E402
import paper_1807_07132_b200 as nadmm  # noqa: E402

port, ref = oracle.Port(), oracle.ref()
for n_total in [int(sys.argv[1])] if len(sys.argv) > 1 else [22_223, 138_889]:
    Xtr, ytr, _, _ = ref.generate_synthetic(n_total, 2048, 100, 3.0, 1.0, port.mix_seed(0, 0))
    ds = nadmm.Dataset.dense(Xtr, ytr, 100)
    sh = oracle.Shard(Xtr, ytr, 100)
    rd = ref.dataset(sh)
    rng = np.random.default_rng(5)
    d = sh.d
    w = rng.normal(size=d) * 0.01
    v = rng.normal(size=d)
    t = time.time()
    hg = nadmm.hessian_vec(ds, w, v, 1e-3)
    hr = rd.hessian_vec(w, v, 1e-3)
    hp = port.hessian_vec(sh, w, v, 1e-3)
    rel = lambda a, b: np.abs(a - b).max() / np.abs(b).max()
    c = nadmm.stable_exp_cache(ds, w)
    lg, rm, al, pr = port.cache(sh, w)
    print(f"n={len(ytr)}: gpu-ref {rel(hg, hr):.2e} gpu-port {rel(hg, hp):.2e} ref-port {rel(hr, hp):.2e} "
          f"P gpu-port {rel(c.probs, pr):.2e} logits {rel(c.logits, lg):.2e} ({time.time() - t:.0f} s)", flush=True)
    bad = np.abs(hg - hp).reshape(99, 2048)
    print("  worst classes", np.argsort(bad.max(1))[-5:], "worst features", np.argsort(bad.max(0))[-5:])
    rows_bad = np.abs(c.probs - pr).max(1)
    print("  rows with P err > 1e-12:", np.nonzero(rows_bad > 1e-12)[0][:20], (rows_bad > 1e-12).sum())
