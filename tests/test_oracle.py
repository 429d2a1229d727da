"""CPU tests of the oracle itself (no GPU): the SPEC known answers, the port pinned
against the reference's own sources (oracle/_ref), and the golden fixtures in tests/golden/."""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle
from util import random_csr, random_dense, rel

GOLDEN = Path(__file__).parent / "golden"


def checkers(port, ref):
    return [("port", port), ("ref", ref)] if ref is not None else [("port", port)]


@pytest.fixture(scope="module")
def both(port):
    r = oracle.ref()
    return checkers(port, r)


def _loss(chk, sh, w, lam=0.0):
    name, c = chk
    return c.loss(sh, w, lam) if name == "port" else c.dataset(sh).loss(w, lam)


def _grad(chk, sh, w, lam=0.0):
    name, c = chk
    return c.gradient(sh, w, lam) if name == "port" else c.dataset(sh).gradient(w, lam)


def _hv(chk, sh, w, v, lam=0.0):
    name, c = chk
    return c.hessian_vec(sh, w, v, lam) if name == "port" else c.dataset(sh).hessian_vec(w, v, lam)


def _pred(chk, sh, w):
    name, c = chk
    return c.predict(sh, w) if name == "port" else c.dataset(sh).predict(w)


# ---- SPEC.md known answers ------------------------------------------------------------------------
def test_spec_loss_known_answers(both):
    X = np.arange(12.0).reshape(4, 3)
    sh = oracle.Shard(X, [1, 2, 3, 1], 3)
    one = oracle.Shard([[2.0]], [1], 2)
    for chk in both:
        assert abs(_loss(chk, sh, np.zeros(6)) - 4 * np.log(3)) < 1e-12
        assert abs(_loss(chk, one, [0.0]) - 0.6931471805599453) < 1e-15
        assert _loss(chk, oracle.Shard([[1000.0]], [2], 2), [1.0]) == 1000.0  # src/softmax.cpp:69-77
        assert _loss(chk, oracle.Shard([[1000.0]], [1], 2), [1.0]) == 0.0


def test_spec_gradient_hessian_known_answers(both):
    one = oracle.Shard([[2.0]], [1], 2)
    rng = np.random.default_rng(0)
    X, y = random_dense(rng, 20, 5, 4)
    sh = oracle.Shard(X, y, 4)
    for chk in both:
        np.testing.assert_allclose(_grad(chk, one, [0.0]), [-1.0], atol=1e-15)
        g0 = _grad(chk, sh, np.zeros(sh.d))  # block c = sum_i (1/C - 1[b_i = c]) a_i
        want = np.concatenate([((1 / 4) - (y == c + 1)) @ X for c in range(3)])
        np.testing.assert_allclose(g0, want, atol=1e-12)
        np.testing.assert_allclose(_hv(chk, one, [0.0], [3.0]), [3.0], atol=1e-15)
        assert np.all(_hv(chk, sh, rng.normal(size=sh.d), np.zeros(sh.d)) == 0.0)


def test_spec_predict_known_answers(both):
    for chk in both:
        assert _pred(chk, oracle.Shard([[1.0]], [1], 2), [1.0])[0] == 1
        X = np.arange(12.0).reshape(4, 3)
        assert _pred(chk, oracle.Shard(X, [1, 2, 3, 1], 3), np.zeros(6)).tolist() == [1, 1, 1, 1]
        assert _pred(chk, oracle.Shard([[1.0]], [1], 3), [-5.0, -7.0])[0] == 3


def test_spec_cg_line_search_newton(port):
    refc = oracle.ref()
    for c in [port] + ([refc] if refc else []):
        r = c.cg_solve(lambda v: v, [1.0, 2.0], 1e-4, 10)
        np.testing.assert_allclose(r["p"], [-1, -2])
        assert r["iters"] == 1
        r = c.cg_solve(lambda v: np.array([1.0, 4.0]) * v, [1.0, 4.0], 1e-10, 10)
        np.testing.assert_allclose(r["p"], [-1, -1], atol=1e-12)
        assert r["iters"] <= 2
        cfg = [1e-4, 10, 0.5, 0.5, 10, 1e-8, 100]
        ls = c.line_search(lambda x: float(x[0] ** 2), [1.0], [-4.0], [2.0], 1.0, cfg)
        assert ls["alpha"] == 0.25 and ls["evals"] == 3 and not ls["capped"]
        cfg0 = [1e-4, 10, 0.5, 0.5, 0, 1e-8, 100]
        ls = c.line_search(lambda x: float(x[0] ** 2), [1.0], [-4.0], [2.0], 1.0, cfg0)
        assert ls["alpha"] == 1.0 and ls["capped"]
        H = np.array([1.0, 4.0])
        r = c.newton_solve_cb(lambda x: 0.5 * float(np.dot(H * x, x)), lambda x: H * x, lambda x, v: H * v, [1.0, 1.0],
                              [1e-10, 10, 1e-4, 0.5, 10, 1e-8, 100])
        np.testing.assert_allclose(r["x"], [0, 0], atol=1e-12)
        assert len(r["trace"]) == 1 and r["converged"]


def test_spec_newton_exactness_ill_conditioned(port):
    """ACCEPTANCE 4: one Newton iteration with theta = 1e-10 on SPD quadratics up to kappa 1e6."""
    rng = np.random.default_rng(1)
    for kappa in (1e2, 1e4, 1e6):
        d = 8
        Q, _ = np.linalg.qr(rng.normal(size=(d, d)))
        H = Q @ np.diag(np.logspace(0, np.log10(kappa), d)) @ Q.T
        x0 = rng.normal(size=d)
        g0 = np.linalg.norm(H @ x0)
        r = port.newton_solve_cb(lambda x: 0.5 * float(x @ H @ x), lambda x: H @ x, lambda x, v: H @ v, x0,
                                 [1e-10, 200, 1e-4, 0.5, 10, 0.0, 1])
        assert np.linalg.norm(H @ r["x"]) < 1e-8 * g0


def test_spec_admm_known_answers(port):
    np.testing.assert_allclose(port.z_update([[1.0], [3.0]], np.zeros((2, 1)), [1, 1], 0.0), [2.0])
    np.testing.assert_allclose(port.z_update([[1.0], [3.0]], np.zeros((2, 1)), [1, 1], 2.0), [1.0])
    np.testing.assert_allclose(port.z_update([[3.0]], [[1.0]], [2.0], 0.0), [2.5])
    np.testing.assert_allclose(port.y_update([[0.0]], [[1.0]], [2.0], [1.0]), [[1.0]])
    np.testing.assert_allclose(port.y_update([[1.0]], [[3.0]], [0.0], [2.0]), [[-5.0]])
    pr, du, _, _ = port.residuals([[1.0, 2.0]], [1.0, 2.0], [1.0, -2.0], [3.0])
    assert pr[0] == 0.0 and du[0] == 12.0
    ep, ed = port.tolerances(np.zeros((4, 10)), np.zeros((4, 10)), np.zeros(10), 1e-3, 1e-3)
    assert abs(ep - 2e-3) < 1e-15 and abs(ed - np.sqrt(10) * 1e-3) < 1e-15
    ep, _ = port.tolerances([[3.0, 4.0]], [[0.0, 0.0]], [0.0, 0.0], 0.0, 0.1)
    assert abs(ep - 2.5) < 1e-15
    v = np.array([1.0, 2.0, -1.0])
    rho, xo, zo = port.spectral_rho(v, v, v, -v, 3.0)  # unit curvature both sides -> rho = 1
    assert xo and zo and abs(rho - 1.0) < 1e-15
    rho, xo, zo = port.spectral_rho(v, -v, v, v, 3.0)  # both correlations fail -> unchanged
    assert not xo and not zo and rho == 3.0
    rho, _, _ = port.spectral_rho(v * 1e-9, v, v, -v * 1e9, 3.0)  # clamped into [1e-6, 1e6]
    assert 1e-6 <= rho <= 1e6


def test_partition_known_answers(port, ref):
    assert np.bincount(port.partition_owner(10, 3)).tolist() == [4, 4, 2]
    assert port.partition_owner(10, 2).tolist() == [0] * 5 + [1] * 5
    assert port.partition_owner(4, 2, strided=True).tolist() == [0, 1, 0, 1]
    for n, N in [(10, 3), (37, 5), (100, 8)]:
        np.testing.assert_array_equal(port.partition_owner(n, N), ref.partition_owner(n, N))
        np.testing.assert_array_equal(port.partition_owner(n, N, True), ref.partition_owner(n, N, True))
    with pytest.raises(oracle.OracleError):
        port.partition_owner(3, 4)


# ---- port vs the reference's own sources ----------------------------------------------------------
@pytest.mark.parametrize("n,p,C", [(50, 7, 4), (200, 33, 10), (129, 5, 2), (77, 65, 21)])
def test_port_matches_reference_dense(port, ref, n, p, C):
    rng = np.random.default_rng(n + p)
    X, y = random_dense(rng, n, p, C, scale=0.5)
    sh = oracle.Shard(X, y, C)
    rd = ref.dataset(sh)
    w, v = rng.normal(size=sh.d), rng.normal(size=sh.d)
    for a, b in zip(port.cache(sh, w), rd.cache(w)):
        assert rel(a, b) <= 1e-14
    assert port.loss(sh, w, 1e-3) == rd.loss(w, 1e-3)
    assert rel(port.gradient(sh, w, 1e-3), rd.gradient(w, 1e-3)) <= 1e-14
    assert rel(port.hessian_vec(sh, w, v, 1e-3), rd.hessian_vec(w, v, 1e-3)) <= 1e-14
    np.testing.assert_array_equal(port.predict(sh, w), rd.predict(w))


def test_port_matches_reference_sparse(port, ref):
    rng = np.random.default_rng(4)
    ip, ix, vv, y = random_csr(rng, 80, 40, 5, 0.2)
    sh = oracle.Shard(labels=y, C_=5, csr=(ip, ix, vv), p=40)
    rd = ref.dataset(sh)
    w, v = rng.normal(size=sh.d), rng.normal(size=sh.d)
    assert abs(port.loss(sh, w) - rd.loss(w)) <= 1e-13 * abs(rd.loss(w))
    assert rel(port.gradient(sh, w), rd.gradient(w)) <= 1e-14
    assert rel(port.hessian_vec(sh, w, v), rd.hessian_vec(w, v)) <= 1e-14


@pytest.mark.parametrize("lam,aug", [(1e-3, False), (0.0, True)])
def test_port_newton_matches_reference(port, ref, lam, aug):
    Xtr, ytr, _, _ = port.generate_synthetic(500, 12, 4, separation=3.0, noise=1.0, seed=3)
    sh = oracle.Shard(Xtr, ytr, 4)
    rng = np.random.default_rng(0)
    kw = dict(rho=1.5, z=rng.normal(size=sh.d) * 0.1, y=rng.normal(size=sh.d) * 0.1) if aug else {}
    cfg = [1e-4, 10, 1e-4, 0.5, 10, 1e-8, 6]
    a = port.newton_solve(sh, lam, np.zeros(sh.d), cfg=cfg, **kw)
    b = ref.dataset(sh).newton_solve(lam, np.zeros(sh.d), cfg=cfg, **kw)
    assert len(a["trace"]) == len(b["trace"])
    for ra, rb in zip(a["trace"], b["trace"]):
        assert ra["cg_iters"] == rb["cg_iters"] and ra["step"] == rb["step"] and ra["fn_evals"] == rb["fn_evals"]
        assert abs(ra["objective"] - rb["objective"]) <= 1e-12 * abs(rb["objective"])
    assert rel(a["x"], b["x"]) <= 1e-12


def test_rng_and_generator_match_reference(port, ref):
    for seed in (0, 1, 12345):
        for kind, bound in ((0, 0), (1, 0), (2, 7), (2, 1000003)):
            np.testing.assert_array_equal(port.rng_stream(seed, kind, 500, bound), ref.rng_stream(seed, kind, 500, bound))
    for args in ((100, 5, 3, 10.0, 0.1, 0), (333, 17, 7, 3.0, 1.0, 9)):
        for a, b in zip(port.generate_synthetic(*args), ref.generate_synthetic(*args)):
            np.testing.assert_array_equal(a, b)


# ---- mathematical invariants (SPEC.md model-softmax) ----------------------------------------------
def test_gradient_and_hessian_finite_differences(port):
    rng = np.random.default_rng(2)
    for _ in range(5):
        n, p, C = 20, 5, 4
        X, y = random_dense(rng, n, p, C)
        sh = oracle.Shard(X, y, C)
        w = rng.normal(size=sh.d) * 0.3
        g = port.gradient(sh, w, 1e-5)
        h = 1e-6
        fd = np.array([(port.loss(sh, w + h * e, 1e-5) - port.loss(sh, w - h * e, 1e-5)) / (2 * h)
                       for e in np.eye(sh.d)])
        assert np.linalg.norm(g - fd) / max(1, np.linalg.norm(g)) < 1e-5
        v = rng.normal(size=sh.d)
        hv = port.hessian_vec(sh, w, v)
        fdh = (port.gradient(sh, w + h * v) - port.gradient(sh, w - h * v)) / (2 * h)
        assert np.linalg.norm(hv - fdh) / max(1, np.linalg.norm(hv)) < 1e-4
        u = rng.normal(size=sh.d)
        assert abs(u @ port.hessian_vec(sh, w, v) - v @ port.hessian_vec(sh, w, u)) <= 1e-10 * abs(u @ hv + 1)
        assert v @ hv >= -1e-10


def test_decomposition_identity(port):
    """ACCEPTANCE 6: sum_i loss(D_i) == loss(D) (and gradient, Hv) for lambda = 0."""
    rng = np.random.default_rng(8)
    X, y = random_dense(rng, 90, 6, 3)
    sh = oracle.Shard(X, y, 3)
    w, v = rng.normal(size=sh.d), rng.normal(size=sh.d)
    owner = port.partition_owner(90, 4)
    parts = [oracle.Shard(X[owner == i], y[owner == i], 3) for i in range(4)]
    assert abs(sum(port.loss(s, w) for s in parts) - port.loss(sh, w)) <= 1e-12 * abs(port.loss(sh, w))
    assert rel(sum(port.gradient(s, w) for s in parts), port.gradient(sh, w)) <= 1e-12
    assert rel(sum(port.hessian_vec(s, w, v) for s in parts), port.hessian_vec(sh, w, v)) <= 1e-12


def test_exp_probe_never_positive(ref):
    rng = np.random.default_rng(6)
    X, y = random_dense(rng, 30, 4, 3)
    rd = ref.dataset(oracle.Shard(X * 1e3, y, 3))
    assert rd.exp_probe(rng.normal(size=8) * 1e2, rng.normal(size=8)) <= 0.0


def test_admm_port_converges(port):
    """ACCEPTANCE 5 analogue: N = 4, fixed rho = 1, lambda = 1e-5 reaches theta <= 0.05 (non-separable
    fixture: on separable data F* -> 0 and theta is degenerate)."""
    Xtr, ytr, _, _ = port.generate_synthetic(1000, 10, 4, separation=3.0, noise=1.0, seed=0)
    sh = oracle.Shard(Xtr, ytr, 4)
    ref_solve = port.newton_solve(sh, 1e-5, np.zeros(sh.d), cfg=[1e-10, 200, 1e-4, 0.5, 10, 1e-10, 100])
    fstar = port.loss(sh, ref_solve["x"], 1e-5)
    owner = port.partition_owner(len(ytr), 4)
    parts = [oracle.Shard(Xtr[owner == i], ytr[owner == i], 4) for i in range(4)]
    out = port.admm_run(parts, oracle.admm_cfg(n_workers=4, lam=1e-5, max_outer_iters=300))
    theta = [(m["train_objective"] - fstar) / fstar for m in out["metrics"]]
    assert min(theta) <= 0.05


@pytest.mark.parametrize("penalty,parallel", [("spectral", True), ("fixed", False)])
def test_ref_admm_matches_port_coordinator(port, ref, penalty, parallel):
    """The reference arm's consensus loop (reference worker solves + the port coordinator, stepped
    from Python, workers on a thread pool) reproduces the port's nor_admm_run: identical iteration
    trace (cg_iters / fn_evals / flags per outer iteration), z and F(z^k) to 1e-12."""
    Xtr, ytr, _, _ = port.generate_synthetic(1200, 12, 4, separation=3.0, noise=1.0, seed=0)
    owner = port.partition_owner(len(ytr), 4)
    parts = [oracle.Shard(Xtr[owner == i], ytr[owner == i], 4) for i in range(4)]
    cfg = oracle.admm_cfg(n_workers=4, lam=1e-3, penalty=penalty, max_outer_iters=25)
    want = port.admm_run(parts, cfg)
    run = oracle.RefAdmm(ref, parts, cfg, workers_parallel=parallel, threads_per_worker=1, eval_objective=True)
    try:
        for _ in range(want["iterations"]):
            run.step()
            if run.converged:
                break
    finally:
        run.close()
    assert run.k == want["iterations"] and run.converged == want["converged"]
    for a, b in zip(run.metrics, want["metrics"]):
        assert (a["cg_iters"], a["fn_evals"], a["flags"]) == (b["cg_iters"], b["fn_evals"], b["flags"])
        assert abs(a["train_objective"] - b["train_objective"]) <= 1e-12 * abs(b["train_objective"])
        assert abs(a["rho_mean"] - b["rho_mean"]) <= 1e-12 * abs(b["rho_mean"])
    assert rel(run.z, want["z"]) <= 1e-12


# ---- golden fixtures ------------------------------------------------------------------------------
def test_golden_fixtures(port):
    files = sorted(GOLDEN.glob("*.npz"))
    assert files, "tests/golden fixtures missing (tests/golden/make_golden.py)"
    for f in files:
        g = np.load(f)
        meta = json.loads(str(g["meta"]))
        if meta["kind"] == "model":
            sh = oracle.Shard(g["X"], g["y"], int(meta["C"]))
            assert abs(port.loss(sh, g["w"], meta["lam"]) - float(g["loss"])) <= 1e-13 * abs(float(g["loss"]))
            assert rel(port.gradient(sh, g["w"], meta["lam"]), g["grad"]) <= 1e-13
            assert rel(port.hessian_vec(sh, g["w"], g["v"], meta["lam"]), g["hv"]) <= 1e-13
            np.testing.assert_array_equal(port.predict(sh, g["w"]), g["pred"])
        elif meta["kind"] == "newton":
            sh = oracle.Shard(g["X"], g["y"], int(meta["C"]))
            r = port.newton_solve(sh, meta["lam"], np.zeros(sh.d), cfg=meta["cfg"])
            assert [t["cg_iters"] for t in r["trace"]] == g["cg_iters"].tolist()
            assert rel(r["x"], g["x"]) <= 1e-11
        elif meta["kind"] == "synthetic":
            Xtr, ytr, Xte, yte = port.generate_synthetic(*meta["args"])
            np.testing.assert_array_equal(Xtr, g["Xtr"])
            np.testing.assert_array_equal(yte, g["yte"])
