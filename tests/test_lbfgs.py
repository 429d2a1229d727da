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


@pytest.mark.gpu
def test_worker_lbfgs_rounds_match_reference(nadmm, ref):
    """run_worker's L-BFGS branch (src/worker.cpp:183-195): warm-started rounds, InnerStats packing."""
    rng = np.random.default_rng(12)
    X, y = random_dense(rng, 300, 14, 4, scale=0.5)
    ds = nadmm.Dataset.dense(X, y, 4)
    rd = ref.dataset(oracle.Shard(X, y, 4))
    w = nadmm.Worker(ds)
    d = ds.weight_dim()
    x_ref = np.zeros(d)
    cfg = nadmm.LbfgsConfig(grad_tol=1e-6)
    for k in range(4):
        z, yy = rng.normal(size=d) * 0.1, rng.normal(size=d) * 0.1
        rho, inner = [1.0, 2.0, 0.5, 1.0][k], [3, 5, 2, 8][k]
        xg, st = w.solve_lbfgs(rho, z, yy, cfg, inner_iters=inner)
        o = rd.lbfgs_solve(0.0, x_ref, (25, 1e-4, 0.9, inner, 20, 1e-6), rho=rho, z=z, y=yy)
        x_ref = o["x"]
        assert rel(xg, x_ref) <= TOL_X
        assert st.inner_iters == len(o["trace"])
        assert st.fn_evals == sum(int(t["fn_evals"]) for t in o["trace"])
        assert st.flags == (1 if any(t["ls_fallback"] for t in o["trace"]) else 0)
        assert st.cg_iters == 0
        assert st.grad_norm == pytest.approx(o["final_grad_norm"], rel=1e-6)


@pytest.mark.gpu
def test_admm_lbfgs_inner_solver_matches_composed_reference(nadmm, port, ref):
    """run_admm with inner_solver = lbfgs against the reference's lbfgs_solve per worker composed with
    the SPEC z / y updates (fixed penalty), outer iteration by outer iteration."""
    N, C_, p, K, inner = 3, 4, 10, 5, 4
    Xtr, ytr, _, _ = port.generate_synthetic(900, p, C_, separation=3.0, noise=1.0, seed=2)
    owner = port.partition_owner(len(ytr), N)
    parts = [(Xtr[owner == i], ytr[owner == i]) for i in range(N)]
    lam = 1e-3
    cfg = nadmm.AdmmConfig(n_workers=N, lam=lam, stopping=nadmm.StoppingConfig(max_outer_iters=K),
                           inner_iters=inner, inner_solver="lbfgs", lbfgs=nadmm.LbfgsConfig(grad_tol=1e-6))
    rg = nadmm.run_admm([nadmm.Dataset.dense(X, y, C_) for X, y in parts], cfg,
                        nadmm.EvalContext(eval_objective=False, ignore_convergence=True))
    assert rg.iterations == K
    rds = [ref.dataset(oracle.Shard(X, y, C_)) for X, y in parts]
    d = (C_ - 1) * p
    x, yv, z = np.zeros((N, d)), np.zeros((N, d)), np.zeros(d)
    rho = np.ones(N)
    for k in range(K):
        fe = 0
        for i in range(N):
            o = rds[i].lbfgs_solve(0.0, x[i], (25, 1e-4, 0.9, inner, 20, 1e-6), rho=1.0, z=z, y=yv[i])
            x[i] = o["x"]
            fe += sum(int(t["fn_evals"]) for t in o["trace"])
        z = port.z_update(x, yv, rho, lam)
        yv = port.y_update(yv, x, z, rho)
        assert rg.metrics[k]["fn_evals"] == fe
        assert rg.metrics[k]["cg_iters"] == 0
    assert rel(rg.z, z) <= TOL_X
