"""Where the fixed cost of one DMMA pass goes: per-CTA globaltimer stamps from a trace build.
usage: NADMM_LIB=tools/prof/var_trace.so python tools/prof/dmma_kstamps.py N P C"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1807_07132_b200 as nadmm  # noqa: E402
from paper_1807_07132_b200 import _lib as L  # noqa: E402

n, p, K1 = (int(a) for a in sys.argv[1:4])
rng = np.random.default_rng(0)
X = rng.normal(size=(n, p)) / np.sqrt(p)
y = (np.arange(n) % K1 + 1).astype(np.int32)
ds = nadmm.Dataset.dense(X, y, K1)
w, v = rng.normal(size=ds.weight_dim()) * 0.01, rng.normal(size=ds.weight_dim())
for _ in range(5):
    nadmm.hessian_vec(ds, w, v)
buf = (C.c_longlong * (256 * 8))()
L.lib().nadmm_debug_dmma_kstamps(buf)
t = np.array(buf, dtype=np.int64).reshape(256, 8)
live = t[:, 0] > 0
t = t[live]
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
names = ["entry", "setup", "TMA#1", "tile0 in", "last B", "partial", "cl sync", "exit"]
print(f"{len(t)} CTAs; us since the first CTA entered (min / median / max over CTAs):")
for k, nm in enumerate(names):
    col = rel[:, k]
    print(f"  {nm:9s} {col.min():8.2f} {np.median(col):8.2f} {col.max():8.2f}")
