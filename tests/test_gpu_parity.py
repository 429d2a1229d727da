"""GPU parity: the CUDA product (through the C ABI) against the CPU oracle on the same inputs.

Tiers: (i) kernel outputs at identical inputs <= 1e-12 relative; (ii) one Newton
solve: identical cg_iters / step / flags per iteration, x and objective <= 1e-10; (iii) full ADMM
run: identical iteration count and predictions, F(z) and z <= 1e-9 relative.
"""
import numpy as np
import pytest

import oracle
from util import random_csr, random_dense, rel

pytestmark = pytest.mark.gpu

TOL_KERNEL = 1e-12
TOL_NEWTON = 1e-10
TOL_ADMM = 1e-9

DENSE_SHAPES = [(50, 7, 4), (200, 33, 10), (129, 5, 2), (300, 28, 2), (1000, 784, 10), (96, 3072, 10), (77, 65, 21),
                (64, 31, 3), (100, 60, 2), (3000, 28, 2),
                (1003, 784, 10), (101, 3072, 10),  # DMMA shapes with a partial last row tile
                # two-GEMM DMMA path (K != 9, even p): partial row / feature tiles, 1..13 class frags
                (300, 34, 5), (129, 66, 2), (257, 200, 21), (130, 200, 100), (500, 96, 3), (389, 2048, 100)]


def shards(nadmm, X, y, C):
    return nadmm.Dataset.dense(X, y, C), oracle.Shard(X, y, C)


@pytest.mark.parametrize("n,p,C", DENSE_SHAPES)
@pytest.mark.parametrize("lam", [0.0, 1e-3])
def test_dense_model_ops(nadmm, port, n, p, C, lam):
    rng = np.random.default_rng(n * 1000 + p + C)
    X, y = random_dense(rng, n, p, C, scale=1.0 / np.sqrt(p))
    ds, sh = shards(nadmm, X, y, C)
    d = sh.d
    w = rng.normal(size=d)
    v = rng.normal(size=d)
    lg, rm, al, pr = port.cache(sh, w)
    c = nadmm.stable_exp_cache(ds, w)
    assert rel(c.logits, lg) <= TOL_KERNEL
    assert rel(c.row_max, rm) <= TOL_KERNEL
    assert rel(c.alpha, al) <= TOL_KERNEL
    assert rel(c.probs, pr) <= TOL_KERNEL
    assert abs(nadmm.loss(ds, w, lam) - port.loss(sh, w, lam)) <= TOL_KERNEL * abs(port.loss(sh, w, lam))
    assert rel(nadmm.gradient(ds, w, lam), port.gradient(sh, w, lam)) <= TOL_KERNEL
    assert rel(nadmm.hessian_vec(ds, w, v, lam), port.hessian_vec(sh, w, v, lam)) <= TOL_KERNEL
    np.testing.assert_array_equal(nadmm.predict(ds, w), port.predict(sh, w))


@pytest.mark.parametrize("n,p,C,dens", [(100, 50, 5, 0.2), (300, 2000, 20, 0.01), (64, 9, 2, 0.5)])
def test_sparse_model_ops(nadmm, port, n, p, C, dens):
    rng = np.random.default_rng(7 + n)
    ip, ix, vv, y = random_csr(rng, n, p, C, dens)
    ds = nadmm.Dataset.sparse(ip, ix, vv, y, C, p)
    sh = oracle.Shard(labels=y, C_=C, csr=(ip, ix, vv), p=p)
    w = rng.normal(size=sh.d) * 0.5
    v = rng.normal(size=sh.d)
    assert abs(nadmm.loss(ds, w, 1e-3) - port.loss(sh, w, 1e-3)) <= TOL_KERNEL * abs(port.loss(sh, w, 1e-3))
    assert rel(nadmm.gradient(ds, w, 0.0), port.gradient(sh, w, 0.0)) <= TOL_KERNEL
    assert rel(nadmm.hessian_vec(ds, w, v, 1e-3), port.hessian_vec(sh, w, v, 1e-3)) <= TOL_KERNEL
    np.testing.assert_array_equal(nadmm.predict(ds, w), port.predict(sh, w))
    # sparse / dense agreement (SPEC.md model-softmax invariants)
    dd = nadmm.Dataset.dense(sh.dense(), y, C)
    assert rel(nadmm.hessian_vec(dd, w, v, 0.0), nadmm.hessian_vec(ds, w, v, 0.0)) <= TOL_KERNEL


@pytest.mark.parametrize("n,p,C,sparse", [(50_000, 3072, 10, False), (60_000, 784, 10, False), (40_000, 2048, 100, False),
                                          (300_000, 28, 2, False), (20_000, 200_000, 20, True)])
def test_products_bitwise_repeatable(nadmm, n, p, C, sparse):
    """Race detector (compute-sanitizer is closed on this pool): every pass implementation --
    clustered DMMA (K = 9), two-GEMM DMMA with >= 3 tiles per CTA (C = 100), small-p ring, CSR
    gathers -- returns bit-identical gradients and products on repeated calls (fixed-order
    reductions, no atomics), so any data race in the mbarrier / DSMEM pipelines shows up here."""
    rng = np.random.default_rng(n + p)
    if sparse:
        ip, ix, vv, y = nadmm.generate_sparse(n, p, C, 100, 3)
        ds = nadmm.Dataset.sparse(ip, ix, vv, y, C, p)
    else:
        X = rng.normal(size=(n, p)) / np.sqrt(p)
        ds = nadmm.Dataset.dense(X, (np.arange(n) % C + 1).astype(np.int32), C)
    d = ds.weight_dim()
    w, v = rng.normal(size=d) * 0.1, rng.normal(size=d)
    g0 = nadmm.gradient(ds, w, 1e-3)
    h0 = nadmm.hessian_vec(ds, w, v, 1e-3)
    for _ in range(3):
        np.testing.assert_array_equal(nadmm.hessian_vec(ds, w, v, 1e-3), h0)
        ds2w = w * (1.0 + 1e-9)  # a new point forces a fresh cache pass, then back
        nadmm.gradient(ds, ds2w, 1e-3)
        np.testing.assert_array_equal(nadmm.gradient(ds, w, 1e-3), g0)


def test_spec_known_answers(nadmm):
    # loss, any data, w = 0, lambda = 0 -> n log C
    X = np.arange(12.0).reshape(4, 3)
    ds = nadmm.Dataset.dense(X, [1, 2, 3, 1], 3)
    assert abs(nadmm.loss(ds, np.zeros(6)) - 4 * np.log(3)) < 1e-12
    one = nadmm.Dataset.dense([[2.0]], [1], 2)
    assert abs(nadmm.loss(one, [0.0]) - np.log(2)) < 1e-15
    np.testing.assert_allclose(nadmm.gradient(one, [0.0]), [-1.0], rtol=0, atol=1e-15)
    np.testing.assert_allclose(nadmm.hessian_vec(one, [0.0], [3.0]), [3.0], rtol=0, atol=1e-15)
    np.testing.assert_array_equal(nadmm.hessian_vec(ds, np.ones(6), np.zeros(6)), np.zeros(6))
    big = nadmm.Dataset.dense([[1000.0]], [2], 2)
    assert nadmm.loss(big, [1.0]) == 1000.0  # src/softmax.cpp:69-77 (SPEC.md:57 typo; b=2 -> 1000)
    big1 = nadmm.Dataset.dense([[1000.0]], [1], 2)
    assert nadmm.loss(big1, [1.0]) == 0.0
    # predict: C=2, <a, x1> = 1 -> class 1; w = 0 -> class 1 (tie rule); C=3 logits (-5,-7) -> class 3
    assert nadmm.predict(nadmm.Dataset.dense([[1.0]], [1], 2), [1.0])[0] == 1
    assert nadmm.predict(ds, np.zeros(6)).tolist() == [1, 1, 1, 1]
    p3 = nadmm.Dataset.dense([[1.0]], [1], 3)
    assert nadmm.predict(p3, [-5.0, -7.0])[0] == 3


def test_stability_large_features(nadmm, port):
    rng = np.random.default_rng(3)
    X, y = random_dense(rng, 40, 6, 4)
    X *= 1e3
    ds, sh = shards(nadmm, X, y, 4)
    w = rng.normal(size=sh.d) * 1e2
    v = rng.normal(size=sh.d)
    assert np.isfinite(nadmm.loss(ds, w))
    assert np.all(np.isfinite(nadmm.gradient(ds, w)))
    assert np.all(np.isfinite(nadmm.hessian_vec(ds, w, v)))
    assert rel(nadmm.hessian_vec(ds, w, v), port.hessian_vec(sh, w, v)) <= TOL_KERNEL


def test_errors(nadmm):
    with pytest.raises(nadmm.DataError):
        nadmm.Dataset.dense([[1.0], [2.0]], [1, 3], 2)
    with pytest.raises(nadmm.ConfigError):
        nadmm.Dataset.dense([[1.0]], [1], 1)
    with pytest.raises(nadmm.DataError):
        nadmm.Dataset.dense([[np.nan]], [1], 2)
    ds = nadmm.Dataset.dense([[1.0, 2.0]], [1], 2)
    with pytest.raises(nadmm.ConfigError):
        nadmm.loss(ds, [1.0])
    with pytest.raises(nadmm.ConfigError):
        nadmm.make_augmented_objective(nadmm.make_softmax_objective(ds, 0.0), 0.0, [0, 0], [0, 0])
    with pytest.raises(nadmm.ConfigError):
        nadmm.newton_solve(nadmm.make_softmax_objective(ds, 0.0), [0.0, 0.0], nadmm.NewtonConfig(cg_tol=2.0))


def _cmp_trace(a, b):
    assert len(a) == len(b)
    for ra, rb in zip(a, b):
        assert ra.cg_iters == rb["cg_iters"]
        assert ra.fn_evals == rb["fn_evals"]
        assert ra.step == rb["step"]
        assert bool(ra.ls_capped) == bool(rb["ls_capped"])
        assert bool(ra.cg_fallback) == bool(rb["cg_fallback"])
        assert abs(ra.objective - rb["objective"]) <= TOL_NEWTON * abs(rb["objective"])
        assert abs(ra.grad_norm - rb["grad_norm"]) <= 1e-8 * max(rb["grad_norm"], 1e-12)


@pytest.mark.parametrize("n,p,C,lam", [(400, 20, 4, 1e-3), (2000, 784, 10, 1e-3), (300, 28, 2, 1e-3),
                                        (1235, 784, 10, 1e-3)])
def test_newton_single_node(nadmm, port, n, p, C, lam):
    Xtr, ytr, _, _ = port.generate_synthetic(n + n // 9 + 2, p, C, separation=3.0, noise=1.0, seed=1)
    ds, sh = shards(nadmm, Xtr, ytr, C)
    cfg = nadmm.NewtonConfig(newton_max_iters=4)
    r = nadmm.newton_solve(nadmm.make_softmax_objective(ds, lam), np.zeros(sh.d), cfg)
    o = port.newton_solve(sh, lam, np.zeros(sh.d), cfg=list(cfg.__dict__.values()))
    _cmp_trace(r.trace, o["trace"])
    assert rel(r.x, o["x"]) <= TOL_NEWTON
    assert abs(r.final_grad_norm - o["final_grad_norm"]) <= 1e-7 * max(o["final_grad_norm"], 1e-12)


def test_newton_augmented(nadmm, port):
    rng = np.random.default_rng(11)
    X, y = random_dense(rng, 500, 30, 5, scale=0.3)
    ds, sh = shards(nadmm, X, y, 5)
    z, yy, x0 = rng.normal(size=sh.d) * 0.1, rng.normal(size=sh.d) * 0.1, rng.normal(size=sh.d) * 0.05
    cfg = nadmm.NewtonConfig(newton_max_iters=3)
    base = nadmm.make_softmax_objective(ds, 0.0)
    r = nadmm.newton_solve(nadmm.make_augmented_objective(base, 2.5, z, yy), x0, cfg)
    o = port.newton_solve(sh, 0.0, x0, cfg=list(cfg.__dict__.values()), rho=2.5, z=z, y=yy)
    _cmp_trace(r.trace, o["trace"])
    assert rel(r.x, o["x"]) <= TOL_NEWTON


def test_worker_sequence_matches_reference(nadmm, ref):
    rng = np.random.default_rng(5)
    X, y = random_dense(rng, 300, 12, 3, scale=0.5)
    ds = nadmm.Dataset.dense(X, y, 3)
    rw = ref.dataset(oracle.Shard(X, y, 3)).worker()
    w = nadmm.Worker(ds)
    d = ds.weight_dim()
    for k in range(4):
        z, yy = rng.normal(size=d) * 0.1, rng.normal(size=d) * 0.1
        rho = [1.0, 1.0, 0.5, 3.0][k]
        if k % 2:
            xg, sg = w.solve(rho, z, yy)
        else:  # caller-provided output buffer
            buf = np.full(d, np.nan)
            xo, sg = w.solve(rho, z, yy, out=buf)
            assert xo is buf
            xg = buf
        xr, sr = rw.solve(rho, z, yy)
        assert rel(xg, xr) <= TOL_NEWTON
        assert sg.cg_iters == sr["cg_iters"] and sg.fn_evals == sr["fn_evals"] and sg.flags == sr["flags"]
        assert sg.inner_iters == sr["inner_iters"]


@pytest.mark.parametrize("penalty", ["fixed", "spectral", "tree"])
def test_admm_run_matches_oracle(nadmm, port, penalty):
    N, C, p = 4, 4, 10
    Xtr, ytr, _, _ = port.generate_synthetic(1200, p, C, separation=3.0, noise=1.0, seed=0)
    owner = port.partition_owner(len(ytr), N)
    parts_o = [oracle.Shard(Xtr[owner == i], ytr[owner == i], C) for i in range(N)]
    parts_g = [nadmm.Dataset.dense(Xtr[owner == i], ytr[owner == i], C) for i in range(N)]
    tree = penalty == "tree"  # bitwise-deterministic consensus mode: the oracle's pairwise z tree
    penalty = "spectral" if tree else penalty
    cfg_o = oracle.admm_cfg(n_workers=N, lam=1e-5, penalty=penalty, max_outer_iters=40)
    ro = port.admm_run(parts_o, cfg_o)
    cfg = nadmm.AdmmConfig(n_workers=N, lam=1e-5, penalty=nadmm.PenaltyPolicy(kind=penalty),
                           stopping=nadmm.StoppingConfig(max_outer_iters=40), consensus_tree=tree)
    rg = nadmm.run_admm(parts_g, cfg, nadmm.EvalContext(eval_objective=True))
    assert rg.iterations == ro["iterations"]
    assert rg.converged == ro["converged"]
    assert rel(rg.z, ro["z"]) <= TOL_ADMM
    for mg, mo in zip(rg.metrics, ro["metrics"]):
        assert abs(mg["train_objective"] - mo["train_objective"]) <= TOL_ADMM * abs(mo["train_objective"])
        assert mg["cg_iters"] == mo["cg_iters"] and mg["fn_evals"] == mo["fn_evals"]
    np.testing.assert_allclose(rg.rho, ro["rho"], rtol=1e-9)
    Xall = np.concatenate([s.X for s in parts_o])
    yall = np.concatenate([s.labels for s in parts_o])
    full_g = nadmm.Dataset.dense(Xall, yall, C)
    np.testing.assert_array_equal(nadmm.predict(full_g, rg.z), port.predict(oracle.Shard(Xall, yall, C), ro["z"]))


def test_shard_binding(nadmm):
    """A shard's solver state (x_local, z, y) belongs to one live Worker or ADMM session at a time
    (the reference's workers own their x_local, src/worker.cpp:135): other solver-level calls on it
    raise ConfigError instead of clobbering it; model-level calls stay allowed."""
    rng = np.random.default_rng(8)
    X, y = random_dense(rng, 120, 10, 3, scale=0.5)
    ds = nadmm.Dataset.dense(X, y, 3)
    d = ds.weight_dim()
    w = nadmm.Worker(ds)
    with pytest.raises(nadmm.ConfigError):
        nadmm.Worker(ds)
    with pytest.raises(nadmm.ConfigError):
        nadmm.newton_solve(nadmm.make_softmax_objective(ds, 1e-3), np.zeros(d))
    with pytest.raises(nadmm.ConfigError):
        nadmm.run_admm([ds], nadmm.AdmmConfig(n_workers=1, lam=1e-3))
    x1, _ = w.solve(1.0, np.zeros(d), np.zeros(d))
    assert np.isfinite(nadmm.loss(ds, x1, 1e-3))  # model level: fine
    x2, _ = w.solve(1.0, np.zeros(d), np.zeros(d))  # warm start survived the model-level call
    w.close()
    nadmm.newton_solve(nadmm.make_softmax_objective(ds, 1e-3), np.zeros(d))
    sess = nadmm.AdmmSession([ds], nadmm.AdmmConfig(n_workers=1, lam=1e-3))
    with pytest.raises(nadmm.ConfigError):
        nadmm.Worker(ds)
    sess.close()
    nadmm.Worker(ds).close()


def test_workers_round_matches_reference(nadmm, ref):
    """nadmm_workers_solve (the WorkerPool round, workers concurrent on the GPU) against the
    reference's run_worker ADMM branch, worker by worker, over several warm-started rounds."""
    rng = np.random.default_rng(15)
    parts = [random_dense(rng, 300 + 50 * i, 3072, 10, scale=0.02) for i in range(4)]  # DMMA shards
    dss = [nadmm.Dataset.dense(X, y, 10) for X, y in parts]
    rws = [ref.dataset(oracle.Shard(X, y, 10)).worker() for X, y in parts]
    ws = [nadmm.Worker(ds) for ds in dss]
    d = dss[0].weight_dim()
    for k in range(3):
        z = rng.normal(size=d) * 0.01
        ys = [rng.normal(size=d) * 0.01 for _ in ws]
        rho = [1.0, 0.5, 2.0, 1.5]
        xs, sts = nadmm.workers_solve(ws, rho, z, ys)
        for i in range(len(ws)):
            xr, sr = rws[i].solve(rho[i], z, ys[i])
            assert rel(xs[i], xr) <= TOL_NEWTON
            assert (sts[i].inner_iters, sts[i].cg_iters, sts[i].fn_evals, sts[i].flags) == \
                (sr["inner_iters"], sr["cg_iters"], sr["fn_evals"], sr["flags"])
    # inner_iters > 1 needs a host decision per Newton iteration: the round runs the workers in turn
    z = rng.normal(size=d) * 0.01
    ys = [rng.normal(size=d) * 0.01 for _ in ws]
    xs, sts = nadmm.workers_solve(ws, 1.0, z, ys, inner_iters=2)
    for i in range(len(ws)):
        xr, sr = rws[i].solve(1.0, z, ys[i], inner_iters=2)
        assert rel(xs[i], xr) <= TOL_NEWTON
        assert sts[i].inner_iters == sr["inner_iters"] and sts[i].cg_iters == sr["cg_iters"]


def test_admm_concurrent_dmma_nodes_match_oracle(nadmm, port):
    """run_admm over DMMA shards (C - 1 = 9): the nodes' solves run on the context's node streams
    with quarter-GPU layouts; the loop must still match the oracle's sequential one."""
    N, C, p = 4, 10, 784
    Xtr, ytr, _, _ = port.generate_synthetic(2400, p, C, separation=3.0, noise=1.0, seed=4)
    owner = port.partition_owner(len(ytr), N)
    parts_o = [oracle.Shard(Xtr[owner == i], ytr[owner == i], C) for i in range(N)]
    parts_g = [nadmm.Dataset.dense(Xtr[owner == i], ytr[owner == i], C) for i in range(N)]
    assert parts_g[0].ctx.node_streams() >= 2
    cfg_o = oracle.admm_cfg(n_workers=N, lam=1e-3, penalty="spectral", max_outer_iters=6)
    ro = port.admm_run(parts_o, cfg_o)
    cfg = nadmm.AdmmConfig(n_workers=N, lam=1e-3, penalty=nadmm.PenaltyPolicy(kind="spectral"),
                           stopping=nadmm.StoppingConfig(max_outer_iters=6))
    rg = nadmm.run_admm(parts_g, cfg, nadmm.EvalContext(eval_objective=True))
    assert rg.iterations == ro["iterations"]
    assert rel(rg.z, ro["z"]) <= TOL_ADMM
    for mg, mo in zip(rg.metrics, ro["metrics"]):
        assert abs(mg["train_objective"] - mo["train_objective"]) <= TOL_ADMM * abs(mo["train_objective"])
        assert mg["cg_iters"] == mo["cg_iters"] and mg["fn_evals"] == mo["fn_evals"]


@pytest.mark.parametrize("block_kb", [64, 16])
def test_sparse_column_blocked_rows_pass(nadmm, port, monkeypatch, block_kb):
    """Shards whose transposed weights exceed the L2 budget run the CSR rows pass once per column
    block (running logits between blocks); forced here with a small budget: same results."""
    monkeypatch.setenv("NADMM_SPARSE_BLOCK_KB", str(block_kb))
    rng = np.random.default_rng(31)
    n, p, C = 257, 3000, 12  # weights 3000 x 11 doubles = 258 KB -> 5 / 17 column blocks
    ip, ix, vv, y = random_csr(rng, n, p, C, 0.02)
    ds = nadmm.Dataset.sparse(ip, ix, vv, y, C, p)
    sh = oracle.Shard(labels=y, C_=C, csr=(ip, ix, vv), p=p)
    w = rng.normal(size=sh.d) * 0.5
    v = rng.normal(size=sh.d)
    assert abs(nadmm.loss(ds, w, 1e-3) - port.loss(sh, w, 1e-3)) <= TOL_KERNEL * abs(port.loss(sh, w, 1e-3))
    assert rel(nadmm.gradient(ds, w, 0.0), port.gradient(sh, w, 0.0)) <= TOL_KERNEL
    assert rel(nadmm.hessian_vec(ds, w, v, 1e-3), port.hessian_vec(sh, w, v, 1e-3)) <= TOL_KERNEL
    np.testing.assert_array_equal(nadmm.predict(ds, w), port.predict(sh, w))
    r = nadmm.newton_solve(nadmm.make_softmax_objective(ds, 1e-3), np.zeros(sh.d), nadmm.NewtonConfig(newton_max_iters=3))
    o = port.newton_solve(sh, 1e-3, np.zeros(sh.d), cfg=list(nadmm.NewtonConfig(newton_max_iters=3).__dict__.values()))
    _cmp_trace(r.trace, o["trace"])
    assert rel(r.x, o["x"]) <= TOL_NEWTON
