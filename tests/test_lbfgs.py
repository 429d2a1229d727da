"""L-BFGS inner solver on the device against the reference's own lbfgs_solve
(src/lbfgs.cpp:94-181, built in oracle/_ref).

L-BFGS has no per-iteration tolerance knob like CG: every trace decision (Wolfe acceptance, history
push, fallback) depends on FP64 scalars whose last bits differ with the reduction order. The
parity bar is therefore: identical iteration count and per-iteration fn_evals / fallback flags on
problems whose line searches are not decided within rounding, objectives <= 1e-9 relative, x <= 1e-7
relative, and the same convergence verdict. Config validation (src/lbfgs.cpp:9-15) runs before
any device work, so its error behaviour is checked on CPU too."""
import ctypes as C

import numpy as np
import pytest

import oracle
from util import random_csr, random_dense, rel

TOL_OBJ = 1e-9
TOL_X = 1e-7
CFG = (25, 1e-4, 0.9, 100, 20, 1e-8)


def _cmp(r, o, n_iters=None):
    tr, to = r.trace, o["trace"]
    n = len(to) if n_iters is None else n_iters
    assert len(tr) == len(to), (len(tr), len(to))
    for a, b in zip(tr[:n], to[:n]):
        assert a.iter == b["iter"]
        assert a.fn_evals == b["fn_evals"], (a, b)
        assert a.ls_fallback == bool(b["ls_fallback"]), (a, b)
        assert abs(a.step - b["step"]) <= 1e-9 * max(abs(b["step"]), 1e-300), (a, b)
        assert abs(a.objective - b["objective"]) <= TOL_OBJ * abs(b["objective"]), (a, b)
        assert abs(a.grad_norm - b["grad_norm"]) <= 1e-6 * max(b["grad_norm"], 1e-12), (a, b)
    assert r.converged == o["converged"]


def _cfg(nadmm, c):
    return nadmm.LbfgsConfig(*c)


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,C,lam,max_iters", [(300, 20, 4, 1e-2, 100), (500, 28, 2, 1e-3, 100),
                                                 (1003, 784, 10, 1e-2, 12), (101, 3072, 10, 1e-2, 8)])
def test_lbfgs_dense_matches_reference(nadmm, ref, n, p, C, lam, max_iters):
    rng = np.random.default_rng(n + p)
    X, y = random_dense(rng, n, p, C, scale=1.0 / np.sqrt(p))
    ds = nadmm.Dataset.dense(X, y, C)
    rd = ref.dataset(oracle.Shard(X, y, C))
    cfg = (25, 1e-4, 0.9, max_iters, 20, 1e-6)
    r = nadmm.lbfgs_solve(nadmm.make_softmax_objective(ds, lam), np.zeros(ds.weight_dim()), _cfg(nadmm, cfg))
    o = rd.lbfgs_solve(lam, np.zeros(ds.weight_dim()), cfg)
    _cmp(r, o)
    assert rel(r.x, o["x"]) <= TOL_X


@pytest.mark.gpu
def test_lbfgs_augmented_matches_reference(nadmm, ref):
    rng = np.random.default_rng(3)
    X, y = random_dense(rng, 400, 16, 5, scale=0.4)
    ds = nadmm.Dataset.dense(X, y, 5)
    rd = ref.dataset(oracle.Shard(X, y, 5))
    d = ds.weight_dim()
    z, yy, x0 = rng.normal(size=d) * 0.1, rng.normal(size=d) * 0.1, rng.normal(size=d) * 0.05
    cfg = (10, 1e-4, 0.9, 60, 20, 1e-5)  # stop before |g|^2 reaches the rounding of f (~600)
    obj = nadmm.make_augmented_objective(nadmm.make_softmax_objective(ds, 0.0), 1.5, z, yy)
    r = nadmm.lbfgs_solve(obj, x0, _cfg(nadmm, cfg))
    o = rd.lbfgs_solve(0.0, x0, cfg, rho=1.5, z=z, y=yy)
    _cmp(r, o)
    assert rel(r.x, o["x"]) <= TOL_X


@pytest.mark.gpu
def test_lbfgs_sparse_matches_reference(nadmm, ref):
    rng = np.random.default_rng(8)
    ip, ix, vv, y = random_csr(rng, 300, 400, 6, 0.03)
    ds = nadmm.Dataset.sparse(ip, ix, vv, y, 6, 400)
    rd = ref.dataset(oracle.Shard(labels=y, C_=6, csr=(ip, ix, vv), p=400))
    cfg = (25, 1e-4, 0.9, 40, 20, 1e-6)
    r = nadmm.lbfgs_solve(nadmm.make_softmax_objective(ds, 1e-2), np.zeros(ds.weight_dim()), _cfg(nadmm, cfg))
    o = rd.lbfgs_solve(1e-2, np.zeros(ds.weight_dim()), cfg)
    _cmp(r, o)
    assert rel(r.x, o["x"]) <= TOL_X


@pytest.mark.gpu
def test_lbfgs_short_history_and_fallback(nadmm, ref):
    """history = 2 (ring reuse) and ls_max_iters = 1 (Wolfe failures -> the -1e-3 g fallback)."""
    rng = np.random.default_rng(21)
    X, y = random_dense(rng, 250, 12, 3, scale=1.0)
    ds = nadmm.Dataset.dense(X, y, 3)
    rd = ref.dataset(oracle.Shard(X, y, 3))
    for cfg in [(2, 1e-4, 0.9, 30, 20, 1e-6), (3, 1e-4, 0.9, 12, 1, 1e-6)]:
        r = nadmm.lbfgs_solve(nadmm.make_softmax_objective(ds, 1e-2), np.zeros(ds.weight_dim()), _cfg(nadmm, cfg))
        o = rd.lbfgs_solve(1e-2, np.zeros(ds.weight_dim()), cfg)
        _cmp(r, o)
        assert rel(r.x, o["x"]) <= TOL_X
    assert any(t.ls_fallback for t in r.trace)


@pytest.mark.gpu
def test_lbfgs_zero_iters_and_converged_start(nadmm, ref):
    rng = np.random.default_rng(2)
    X, y = random_dense(rng, 100, 6, 3, scale=1.0)
    ds = nadmm.Dataset.dense(X, y, 3)
    obj = nadmm.make_softmax_objective(ds, 1e-3)
    r = nadmm.lbfgs_solve(obj, np.zeros(ds.weight_dim()), nadmm.LbfgsConfig(max_iters=0))
    assert r.trace == [] and not r.converged
    assert r.final_grad_norm == pytest.approx(np.linalg.norm(nadmm.gradient(ds, np.zeros(ds.weight_dim()), 1e-3)),
                                              rel=1e-12)
    r = nadmm.lbfgs_solve(obj, np.zeros(ds.weight_dim()), nadmm.LbfgsConfig(grad_tol=1e9))
    assert r.trace == [] and r.converged


BAD_CFGS = [((0, 1e-4, 0.9, 100, 20, 1e-8), "lbfgs history must be >= 1"),
            ((25, 0.9, 0.5, 100, 20, 1e-8), "wolfe constants must satisfy 0 < c1 < c2 < 1"),
            ((25, 0.0, 0.9, 100, 20, 1e-8), "wolfe constants must satisfy 0 < c1 < c2 < 1"),
            ((25, 1e-4, 1.0, 100, 20, 1e-8), "wolfe constants must satisfy 0 < c1 < c2 < 1"),
            ((25, 1e-4, 0.9, -1, 20, 1e-8), "lbfgs max_iters must be >= 0"),
            ((25, 1e-4, 0.9, 100, 0, 1e-8), "lbfgs ls_max_iters must be >= 1")]


@pytest.mark.parametrize("cfg,msg", BAD_CFGS)
def test_lbfgs_config_errors(ref, cfg, msg):
    """Validation precedes any device work: same ConfigError without a GPU, same text as the reference."""
    from paper_1807_07132_b200 import _lib as L

    lib = L.lib()
    c = L.LbfgsCfg(*cfg)
    x = np.zeros(4)
    rc = lib.nadmm_lbfgs_solve(None, C.byref(c), 0.0, 0, 0.0, None, None, x.ctypes.data_as(L.D), None, 0, None)
    assert rc == 2 and lib.nadmm_last_error().decode() == msg
    X, y = np.eye(3), np.array([1, 2, 1], dtype=np.int32)
    with pytest.raises(oracle.OracleError, match=msg):
        ref.dataset(oracle.Shard(X, y, 2)).lbfgs_solve(0.0, np.zeros(3), cfg)


def test_lbfgs_default_config():
    from paper_1807_07132_b200 import _lib as L
    import paper_1807_07132_b200 as nadmm

    c = L.LbfgsCfg()
    L.lib().nadmm_lbfgs_cfg_default(C.byref(c))
    d = nadmm.LbfgsConfig()
    assert (c.history, c.wolfe_c1, c.wolfe_c2, c.max_iters, c.ls_max_iters, c.grad_tol) == \
        (d.history, d.wolfe_c1, d.wolfe_c2, d.max_iters, d.ls_max_iters, d.grad_tol) == CFG
