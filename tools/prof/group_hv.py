"""Node-group DMMA Hv pass vs per-shard passes (whole-GPU layouts), CUDA events, no solver tails.
usage: python tools/prof/group_hv.py [nodes] [rows] [p]"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1807_07132_b200 as nadmm  # noqa: E402
from paper_1807_07132_b200 import _lib as L  # noqa: E402

nodes = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 6250
p = int(sys.argv[3]) if len(sys.argv) > 3 else 3072
ctx = nadmm.Context(0)
rng = np.random.default_rng(0)
shards = []
for i in range(nodes):
    X = rng.normal(size=(rows, p)) / np.sqrt(p)
    shards.append(nadmm.Dataset.dense(X, (np.arange(rows) % 10 + 1).astype(np.int32), 10, ctx=ctx))
d = 9 * p
vs = [torch.tensor(rng.normal(size=d), device="cuda") for _ in range(nodes)]
lib = L.lib()
for s in shards:  # a cache (P) on every shard
    lib.nadmm_set_point_dev(s.handle, C.c_void_p(torch.zeros(d, dtype=torch.float64, device="cuda").data_ptr()))
hs = (C.c_void_p * nodes)(*[s.handle for s in shards])
vp = (C.c_void_p * nodes)(*[v.data_ptr() for v in vs])
mg, ms = C.c_float(), C.c_float()
rc = lib.nadmm_debug_group_hv(hs, nodes, vp, 10, C.byref(mg), C.byref(ms))
nbytes = 8 * rows * p + 8 * rows * 9 + 16 * p * 9
print(f"rc={rc} nodes={nodes} rows={rows} p={p}: group {mg.value * 1e3:.1f} us ({nodes * nbytes / (mg.value * 1e-3) / 1e9:.0f} GB/s)"
      f"  {nodes} single passes {ms.value * 1e3:.1f} us ({nodes * nbytes / (ms.value * 1e-3) / 1e9:.0f} GB/s)", flush=True)
