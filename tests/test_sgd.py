"""Synchronous mini-batch SGD: the worker's SGD branch (src/worker.cpp:197-218)
against the reference build's own Rng shuffle, Dataset::subset and gradient, and the coordinator of
SPEC.md:461-468 against a composition of those reference pieces."""
import numpy as np
import pytest

import oracle
from util import random_csr, random_dense, rel

TOL = 1e-12


@pytest.mark.parametrize("seed,epoch,n", [(0, 0, 1), (0, 0, 2), (7, 3, 1000), (2**63 + 5, 11, 777), (42, 0, 6250)])
def test_epoch_permutation_matches_reference(nadmm, ref, port, seed, epoch, n):
    ours = nadmm.sgd_permutation(seed, epoch, n)
    theirs = ref.shuffle(port.mix_seed(seed, epoch), n)
    np.testing.assert_array_equal(ours, theirs)


def _ref_batch_grad(ref_ds, perm, step, m, z):
    n = len(perm)
    rows = perm[(step * m + np.arange(m)) % n]
    return ref_ds.gradient_subset(rows, z, 0.0) / m


@pytest.mark.gpu
@pytest.mark.parametrize("sparse", [False, True])
def test_worker_sgd_grad_matches_reference(nadmm, ref, port, sparse):
    rng = np.random.default_rng(4)
    C_ = 5
    if sparse:
        ip, ix, vv, y = random_csr(rng, 230, 300, C_, 0.05)
        ds = nadmm.Dataset.sparse(ip, ix, vv, y, C_, 300)
        rd = ref.dataset(oracle.Shard(labels=y, C_=C_, csr=(ip, ix, vv), p=300))
    else:
        X, y = random_dense(rng, 230, 40, C_, scale=0.5)
        ds = nadmm.Dataset.dense(X, y, C_)
        rd = ref.dataset(oracle.Shard(X, y, C_))
    w = nadmm.Worker(ds)
    cfg = nadmm.SgdConfig(batch=32, steps_per_epoch=8, seed=9)  # 8 * 32 > 230: batches wrap around
    d = ds.weight_dim()
    for it in range(20):
        z = rng.normal(size=d) * 0.3
        g, st = w.sgd_grad(cfg, it, z)
        epoch, step = it // cfg.steps_per_epoch, it % cfg.steps_per_epoch
        perm = ref.shuffle(port.mix_seed(cfg.seed, epoch), ds.n())
        assert rel(g, _ref_batch_grad(rd, perm, step, cfg.batch, z)) <= TOL
        assert (st.inner_iters, st.fn_evals, st.cg_iters) == (1, 1, 0)


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [0, 231])
def test_worker_sgd_batch_errors(nadmm, batch):
    rng = np.random.default_rng(1)
    X, y = random_dense(rng, 230, 5, 3)
    w = nadmm.Worker(nadmm.Dataset.dense(X, y, 3))
    with pytest.raises(nadmm.ConfigError, match=r"sgd batch size must lie in \[1, local n\]"):
        w.sgd_grad(nadmm.SgdConfig(batch=batch, steps_per_epoch=1), 0, np.zeros(10))


@pytest.mark.gpu
def test_sync_sgd_matches_composed_reference(nadmm, ref, port):
    N, C_, p, lam = 3, 4, 12, 1e-3
    Xtr, ytr, _, _ = port.generate_synthetic(800, p, C_, separation=3.0, noise=1.0, seed=5)
    owner = port.partition_owner(len(ytr), N)
    parts = [(Xtr[owner == i], ytr[owner == i]) for i in range(N)]
    cfg = nadmm.SgdConfig(eta=0.5, batch=20, epochs=3, seed=3)
    res = nadmm.sync_sgd([nadmm.Dataset.dense(X, y, C_) for X, y in parts], cfg, lam)
    assert res.epochs == 3
    rds = [ref.dataset(oracle.Shard(X, y, C_)) for X, y in parts]
    spe = int(np.ceil(len(ytr) / (cfg.batch * N)))
    d = (C_ - 1) * p
    x = np.zeros(d)
    for e in range(cfg.epochs):
        for t in range(spe):
            it = e * spe + t
            gs = []
            for i in range(N):
                perm = ref.shuffle(port.mix_seed(cfg.seed, it // spe), len(parts[i][1]))
                gs.append(_ref_batch_grad(rds[i], perm, it % spe, cfg.batch, x))
            gsum = gs[0]
            for g in gs[1:]:
                gsum = gsum + g
            x = x - cfg.eta * (gsum / N)
        F = sum(rd.loss(x, 0.0) for rd in rds) + 0.5 * lam * float(x @ x)
        row = res.metrics[e]
        assert row["iteration"] == e and row["inner_iterations"] == spe
        assert row["messages"] == 2 * N * spe * (e + 1)  # cumulative (inc/metrics.hpp:23)
        assert abs(row["train_objective"] - F) <= 1e-10 * abs(F)
    assert rel(res.x, x) <= 1e-10


@pytest.mark.gpu
def test_sync_sgd_identical_workers_equal_one_worker(nadmm):
    """two workers holding identical shards follow one worker's trajectory."""
    rng = np.random.default_rng(6)
    X, y = random_dense(rng, 300, 10, 3, scale=0.5)
    cfg = nadmm.SgdConfig(eta=1.0, batch=25, epochs=2, seed=1)
    one = nadmm.sync_sgd([nadmm.Dataset.dense(X, y, 3)], cfg, 1e-3)
    two = nadmm.sync_sgd([nadmm.Dataset.dense(X, y, 3), nadmm.Dataset.dense(X, y, 3)], cfg, 1e-3)
    np.testing.assert_array_equal(one.x, two.x)


@pytest.mark.gpu
def test_sync_sgd_divergence_aborts(nadmm):
    rng = np.random.default_rng(2)
    X, y = random_dense(rng, 200, 10, 3, scale=3.0)
    with pytest.raises(nadmm.SolverError, match="sync_sgd: objective diverged"):
        nadmm.sync_sgd([nadmm.Dataset.dense(X, y, 3)], nadmm.SgdConfig(eta=1e6, batch=50, epochs=3), 0.0)
