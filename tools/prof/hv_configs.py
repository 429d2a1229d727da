"""Hv timing at the per-GPU shard shapes of every BASELINE config, device-resident
data, CUDA events; algorithmic bytes per SURVEY §8d. usage: python tools/prof/hv_configs.py [cfg ...]"""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1807_07132_b200 as nadmm  # noqa: E402
from paper_1807_07132_b200 import _lib as L  # noqa: E402
import torch  # noqa: E402

HBM = 6527.5


def dense_bytes(n, p, K):
    return 8 * n * p + 8 * n * K + 16 * p * K


def sparse_bytes(n, p, K, nnz):
    return 2 * (12 * nnz + 4 * (n + 1)) + 24 * n * K + 16 * p * K


def time_hv(ds, reps):
    lib = L.lib()
    d = ds.weight_dim()
    rng = np.random.default_rng(0)
    w = torch.tensor(rng.normal(size=d) * 0.01, device="cuda")
    v = torch.tensor(rng.normal(size=d), device="cuda")
    hv = torch.zeros(d, dtype=torch.float64, device="cuda")
    assert lib.nadmm_set_point_dev(ds.handle, C.c_void_p(w.data_ptr())) == 0
    st = torch.cuda.ExternalStream(ds.ctx.stream)
    for _ in range(2):
        assert lib.nadmm_hessian_vec_dev(ds.handle, C.c_void_p(v.data_ptr()), 0.0, C.c_void_p(hv.data_ptr())) == 0
    ds.ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        lib.nadmm_hessian_vec_dev(ds.handle, C.c_void_p(v.data_ptr()), 0.0, C.c_void_p(hv.data_ptr()))
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def report(name, shape, ms, nbytes, flops):
    gbs = nbytes / ms / 1e6
    print(f"{name:8s} {shape:34s} {ms * 1e3:9.1f} us/Hv  {gbs:7.0f} GB/s ({gbs / HBM:.2f} of HBM)  "
          f"{flops / ms / 1e9:6.2f} TFLOP/s", flush=True)


def main(cfgs):
    ctx = nadmm.Context(0)
    rng = np.random.default_rng(1)
    if "1" in cfgs:
        n, p, C1 = 60000, 784, 10
        X = rng.normal(size=(n, p)) / 28
        ds = nadmm.Dataset.dense(X, (np.arange(n) % C1 + 1).astype(np.int32), C1, ctx=ctx)
        report("cfg1", f"dense {n}x{p} C={C1}", time_hv(ds, 20), dense_bytes(n, p, C1 - 1), 4 * n * p * (C1 - 1))
        ds.close()
    if "2" in cfgs:
        n, p, C1 = 6250, 3072, 10
        X = rng.normal(size=(n, p)) / 55
        ds = nadmm.Dataset.dense(X, (np.arange(n) % C1 + 1).astype(np.int32), C1, ctx=ctx)
        report("cfg2", f"dense {n}x{p} C={C1}", time_hv(ds, 20), dense_bytes(n, p, C1 - 1), 4 * n * p * (C1 - 1))
        ds.close()
    if "3" in cfgs:
        n, p, C1 = 1375000, 28, 2
        X = rng.normal(size=(n, p))
        ds = nadmm.Dataset.dense(X, (np.arange(n) % C1 + 1).astype(np.int32), C1, ctx=ctx)
        report("cfg3", f"dense {n}x{p} C={C1}", time_hv(ds, 20), dense_bytes(n, p, C1 - 1), 4 * n * p * (C1 - 1))
        ds.close()
    if "4" in cfgs:
        n, p, C1, nnz_row = 125000, 1300000, 20, 650
        t0 = time.time()
        ip, ix, vv, y = nadmm.generate_sparse(n, p, C1, nnz_row, 0)
        print(f"  (sparse fixture generated in {time.time() - t0:.1f} s)", flush=True)
        ds = nadmm.Dataset.sparse(ip, ix, vv, y, C1, p, ctx=ctx)
        nnz = int(ip[-1])
        report("cfg4", f"CSR {n}x{p} nnz/row={nnz_row} C={C1}", time_hv(ds, 5), sparse_bytes(n, p, C1 - 1, nnz),
               4 * nnz * (C1 - 1))
        ds.close()
    if "5full" in cfgs:
        n, p, C1 = 500000, 2048, 100  # the full per-GPU cfg5 shard (8.2 GB of X)
        X = np.empty((n, p))
        for r0 in range(0, n, 50000):
            X[r0:r0 + 50000] = rng.normal(size=(min(50000, n - r0), p)) / 45
        ds = nadmm.Dataset.dense(X, (np.arange(n) % C1 + 1).astype(np.int32), C1, ctx=ctx)
        del X
        report("cfg5", f"dense {n}x{p} C={C1}", time_hv(ds, 3), dense_bytes(n, p, C1 - 1), 4 * n * p * (C1 - 1))
        ds.close()
    if "5" in cfgs:
        n, p, C1 = 125000, 2048, 100  # a quarter of the 500,000-row cfg5 shard (time scales with n)
        X = rng.normal(size=(n, p)) / 45
        ds = nadmm.Dataset.dense(X, (np.arange(n) % C1 + 1).astype(np.int32), C1, ctx=ctx)
        report("cfg5/4", f"dense {n}x{p} C={C1}", time_hv(ds, 3), dense_bytes(n, p, C1 - 1), 4 * n * p * (C1 - 1))
        ds.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["1", "2", "3", "4", "5"])
