"""Per-node timeline of one Newton iteration graph replay (the ADMM worker solve of the bench's
node 0 shard), from event marks captured into the graph. Aggregated by mark name.
usage: NADMM_GRAPH_TIMELINE=1 python tools/prof/graph_timeline.py [N P C]"""
import ctypes as C
import os
import sys
from collections import OrderedDict
from pathlib import Path

import numpy as np

os.environ.setdefault("NADMM_GRAPH_TIMELINE", "1")
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1807_07132_b200 as nadmm  # noqa: E402
from paper_1807_07132_b200 import _lib as L  # noqa: E402

n, p, K1 = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (6250, 3072, 10)
Xtr, ytr, _, _ = nadmm.generate_synthetic(n * 10 // 9 + 1, p, K1, 1.0, 1.0, 0)
ds = nadmm.Dataset.dense(Xtr[:n], ytr[:n], K1)
w = nadmm.Worker(ds)
d = ds.weight_dim()
rng = np.random.default_rng(0)
fn = L.lib().nadmm_debug_graph_timeline
fn.restype = C.c_int
fn.argtypes = [C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_char_p), C.c_int]
agg = OrderedDict()
reps = 5
for r in range(reps + 2):
    w.solve(1.0, rng.normal(size=d) * 1e-3, np.zeros(d), nadmm.NewtonConfig(), 1)
    ms = (C.c_float * 512)()
    names = (C.c_char_p * 512)()
    k = fn(ds.handle, ms, names, 512)
    if r < 2:
        continue
    for i in range(k):
        nm = names[i].decode()
        t, c = agg.get(nm, (0.0, 0))
        agg[nm] = (t + ms[i], c + 1)
tot = sum(t for t, _ in agg.values()) / reps
print(f"shard {n}x{p} C={K1}: one Newton iteration graph = {tot * 1e3:.1f} us (mean of {reps} replays)")
for nm, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"  {nm:26s} {t / reps * 1e3:8.1f} us/iter  {100 * t / reps / tot:5.1f}%  ({c // reps} per iter, "
          f"{t / c * 1e3:6.1f} us each)")
