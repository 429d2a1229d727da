"""Debug: two-GEMM Hv vs the port across n at C = 100, p = 2048 (generator data), repeatability."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import oracle  # noqa: E402
import paper_1807_07132_b200 as nadmm  # noqa: E402

port, ref = oracle.Port(), oracle.ref()
rel = lambda a, b: np.abs(a - b).max() / np.abs(b).max()
Xall, yall, _, _ = ref.generate_synthetic(138_889, 2048, 100, 3.0, 1.0, port.mix_seed(0, 0))
for n in [int(a) for a in sys.argv[1:]] or [30000, 40000, 60000, 90000, 125000]:
    Xtr, ytr = Xall[:n], yall[:n]
    ds = nadmm.Dataset.dense(Xtr, ytr, 100)
    sh = oracle.Shard(Xtr, ytr, 100)
    rng = np.random.default_rng(5)
    w = rng.normal(size=sh.d) * 0.01
    v = rng.normal(size=sh.d)
    hg = nadmm.hessian_vec(ds, w, v, 1e-3)
    hg2 = nadmm.hessian_vec(ds, w, v, 1e-3)
    hp = port.hessian_vec(sh, w, v, 1e-3)
    gg = nadmm.gradient(ds, w, 1e-3)
    gp = port.gradient(sh, w, 1e-3)
    print(f"n={n} [{os.environ.get('NADMM_DISABLE_GEMM', 'gemm')}]: hv {rel(hg, hp):.2e} repeat-identical "
          f"{np.array_equal(hg, hg2)} grad {rel(gg, gp):.2e}", flush=True)
    ds.close()
