"""Host-side cost of one nadmm_worker_solve on a tiny shard (device work ~0): Python wrapper vs raw
ctypes call, to size the e2e leg's per-node turnaround."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1807_07132_b200 as nadmm  # noqa: E402
from paper_1807_07132_b200 import _lib as L  # noqa: E402

Xtr, ytr, _, _ = nadmm.generate_synthetic(2000, 3072, 10, 1.0, 1.0, 0)
ds = nadmm.Dataset.dense(Xtr[:64], ytr[:64], 10)
w = nadmm.Worker(ds)
d = ds.weight_dim()
z = torch.zeros(d, dtype=torch.float64).pin_memory().numpy()
y = torch.zeros(d, dtype=torch.float64).pin_memory().numpy()
x = torch.zeros(d, dtype=torch.float64).pin_memory().numpy()
cfg = nadmm.NewtonConfig()
for _ in range(5):
    w.solve(1.0, z, y, cfg, 1, out=x)
t0 = time.perf_counter()
for _ in range(200):
    w.solve(1.0, z, y, cfg, 1, out=x)
t1 = time.perf_counter()
c = cfg.to_c()
st = L.InnerStats()
lib = L.lib()
zp, yp, xp = (a.ctypes.data_as(C.POINTER(C.c_double)) for a in (z, y, x))
t2 = time.perf_counter()
for _ in range(200):
    lib.nadmm_worker_solve(w.handle, 1.0, zp, yp, C.byref(c), 1, xp, C.byref(st))
t3 = time.perf_counter()
print(f"Worker.solve (python wrapper): {(t1 - t0) / 200 * 1e6:.1f} us per call; raw ctypes: {(t3 - t2) / 200 * 1e6:.1f} us "
      f"(64-row shard, d={d})")
