"""Handle lifetimes: a context outlives its shards / communicators and a shard its workers / ADMM
sessions whatever order the handles are freed in (finalizers run in arbitrary order when a Python
process exits with objects still held, e.g. by a failed test's traceback)."""
import subprocess
import sys
import textwrap
from pathlib import Path

import numpy as np
import pytest

import paper_1807_07132_b200 as nadmm

ROOT = Path(__file__).resolve().parents[1]


def _data(n=300, p=40, C=4, seed=0):
    X, y, _, _ = nadmm.generate_synthetic(n + 10, p, C, 1.0, 1.0, seed)
    return X[:n], y[:n]


@pytest.mark.gpu
def test_free_in_any_order():
    X, y = _data()
    for order in ("ctx_first", "shard_first", "worker_last"):
        ctx = nadmm.Context(0)
        ds = nadmm.Dataset.dense(X, y, 4, ctx=ctx)
        ds2 = nadmm.Dataset.dense(X, y, 4, ctx=ctx)
        w = nadmm.Worker(ds)
        sess = nadmm.AdmmSession([ds2], nadmm.AdmmConfig(n_workers=1, lam=1e-3))
        d = ds.weight_dim()
        x, _ = w.solve(1.0, np.zeros(d), np.zeros(d), nadmm.NewtonConfig(), 1)
        sess.step(2)
        if order == "ctx_first":
            ctx.close()  # deferred: shards, worker and session still work
            x2, _ = w.solve(1.0, np.zeros(d), np.zeros(d), nadmm.NewtonConfig(), 1)
            assert np.isfinite(x2).all()
            sess.step(1)
            ds.close()
            ds2.close()
            w.close()
            sess.close()
        elif order == "shard_first":
            ds.close()  # deferred until the worker goes
            ds2.close()
            sess.step(1)
            w.close()
            sess.close()
            ctx.close()
        else:
            sess.close()
            ctx.close()
            ds2.close()
            ds.close()
            w.close()
        assert np.isfinite(x).all()


@pytest.mark.gpu
def test_process_exit_with_live_handles():
    code = textwrap.dedent(
        f"""
        import sys, gc
        sys.path.insert(0, {str(ROOT)!r})
        import numpy as np
        import paper_1807_07132_b200 as nadmm
        X, y, _, _ = nadmm.generate_synthetic(310, 40, 4, 1.0, 1.0, 0)
        ctx = nadmm.Context(0)
        ds = nadmm.Dataset.dense(X[:300], y[:300], 4, ctx=ctx)
        w = nadmm.Worker(ds)
        sess = nadmm.AdmmSession([nadmm.Dataset.dense(X[:300], y[:300], 4, ctx=ctx)],
                                 nadmm.AdmmConfig(n_workers=1, lam=1e-3))
        sess.step(1)
        # a reference cycle holding every handle, collected at exit in arbitrary finalizer order
        box = [ctx, ds, w, sess]
        box.append(box)
        ctx.close()
        print("ok")
        """
    )
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().endswith("ok")
