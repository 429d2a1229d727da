"""Repeated shard Hessian-vector products on device-resident data (profiling driver).
usage: python tools/prof/hv_loop.py N P C REPS"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1807_07132_b200 as nadmm
from paper_1807_07132_b200 import _lib as L

n, p, K1, reps = (int(a) for a in sys.argv[1:5])
rng = np.random.default_rng(0)
X = rng.normal(size=(n, p)) / np.sqrt(p)
y = (np.arange(n) % K1 + 1).astype(np.int32)
ctx = nadmm.Context(0)
ds = nadmm.Dataset.dense(X, y, K1, ctx=ctx)
d = ds.weight_dim()
import torch

w = torch.tensor(rng.normal(size=d) * 0.01, device="cuda")
v = torch.tensor(rng.normal(size=d), device="cuda")
hv = torch.zeros(d, dtype=torch.float64, device="cuda")
lib = L.lib()
assert lib.nadmm_set_point_dev(ds.handle, C.c_void_p(w.data_ptr())) == 0
ctx.synchronize()
st = torch.cuda.ExternalStream(ctx.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(3):
    lib.nadmm_hessian_vec_dev(ds.handle, C.c_void_p(v.data_ptr()), 0.0, C.c_void_p(hv.data_ptr()))
ctx.synchronize()
e0.record(st)
for r in range(reps):
    lib.nadmm_hessian_vec_dev(ds.handle, C.c_void_p(v.data_ptr()), 0.0, C.c_void_p(hv.data_ptr()))
e1.record(st)
e1.synchronize()
ms = e0.elapsed_time(e1) / reps
gb = (8 * n * p + 8 * n * (K1 - 1) + 16 * p * (K1 - 1)) / 1e9
print(f"n={n} p={p} C={K1}: {ms*1e3:.1f} us per Hv (incl. finalize), {gb/ms*1e3:.0f} GB/s algorithmic")
