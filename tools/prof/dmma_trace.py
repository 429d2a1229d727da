"""Per-tile timeline of the fused DMMA pass (CTA 0), from a trace build of the library.
usage: NADMM_LIB=tools/prof/libnadmm_trace.so python tools/prof/dmma_trace.py N P C"""
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
for _ in range(3):
    nadmm.hessian_vec(ds, w, v)
buf = (C.c_longlong * (64 * 16))()
L.lib().nadmm_debug_dmma_trace(buf)
t = np.array(buf, dtype=np.int64).reshape(64, 16)
t0 = t[0, 0]
names = ["A start", "A done", "push got", "push done", "rbar ok", "epi done", "U ok(Bst)", "B done"]
print("tile " + " ".join(f"{x:>9s}" for x in names))
for i in range(24):
    print(f"{i:4d} " + " ".join(f"{(t[i, k] - t0):9d}" for k in range(8)))
d = np.diff(t[4:40, 7])
print("steady cycles per tile (B done to B done):", float(np.median(d)))
for a, b, nm in [(1, 2, "A done -> pusher got"), (2, 3, "push time"), (3, 4, "push done -> rbar"), (4, 5, "epilogue"),
                 (5, 6, "epi done -> B start (same tile)"), (6, 7, "B time"), (0, 1, "A time"),
                 (4, 8, "epi: full wait"), (8, 9, "epi: pass1"), (9, 11, "epi: credits"), (11, 12, "epi: pass2"),
                 (2, 13, "push: credit wait"), (13, 14, "push: partial sums"), (14, 3, "push: bulk copies")]:
    print(f"{nm:32s} median {float(np.median(t[4:40, b] - t[4:40, a])):9.0f} cycles")
