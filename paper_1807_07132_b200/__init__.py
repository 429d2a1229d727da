"""B200-native Newton-ADMM hot path (arxiv 1807.07132), host-side mirror of the reference API.

The names, argument meanings, defaults and error behaviour follow the reference C++ API under
/root/reference/proj (inc/dataset.hpp, inc/softmax.hpp, inc/objective.hpp, inc/newton.hpp,
inc/admm.hpp, inc/worker.hpp), so parity tests read like the reference's own. Every compute call
goes through the C ABI of include/nadmm_cuda.h into lib/libnadmm_cuda.so (hand-written sm_100a
kernels); nothing here computes on the CPU.

    ds   = Dataset.dense(X, labels, num_classes)             # Dataset::dense   (inc/dataset.hpp:22)
    obj  = make_softmax_objective(ds, lam)                   # src/objective.cpp:24-39
    aug  = make_augmented_objective(obj, rho, z, y)          # src/objective.cpp:41-56
    res  = newton_solve(aug, x0, NewtonConfig())             # src/newton.cpp:73-132
    run  = run_admm(parts, AdmmConfig(n_workers=len(parts))) # inc/admm.hpp:139-140
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib as L

__all__ = [
    "ConfigError", "DataError", "SolverError", "TransportError", "ProtocolError", "Context", "Dataset",
    "StableExpCache", "stable_exp_cache", "loss", "gradient", "hessian_vec", "predict", "accuracy",
    "weight_blocks", "Objective", "make_softmax_objective", "make_augmented_objective", "NewtonConfig",
    "NewtonIterRecord", "NewtonResult", "newton_solve", "InnerStats", "Worker", "PenaltyPolicy", "StoppingConfig",
    "AdmmConfig", "EvalContext", "AdmmRunResult", "run_admm", "Communicator", "generate_synthetic",
    "generate_sparse", "partition_owner", "partition", "mix_seed", "default_context", "LoadedData", "read_libsvm",
    "read_idx", "load_libsvm", "load_idx", "LbfgsConfig", "LbfgsIterRecord", "LbfgsResult", "lbfgs_solve",
    "SgdConfig", "SgdResult", "sgd_permutation", "sync_sgd", "workers_solve",
]


# ---- error taxonomy (inc/common.hpp:17-44) ------------------------------------------------------
class NadmmError(RuntimeError):
    code = 0


class ConfigError(NadmmError):
    code = 2


class SolverError(NadmmError):
    code = 3


class TransportError(NadmmError):
    code = 4


class DataError(NadmmError):
    code = 12


class ProtocolError(NadmmError):
    code = 14


class CudaError(NadmmError):
    code = 20


_ERRORS = {2: ConfigError, 3: SolverError, 4: TransportError, 12: DataError, 14: ProtocolError, 20: CudaError,
           21: TransportError}


def _check(rc: int, data: bool = False) -> None:
    if rc:
        msg = (L.lib().nadmm_data_last_error() if data else L.lib().nadmm_last_error()) or b""
        raise _ERRORS.get(rc, NadmmError)(msg.decode())


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(L.D)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(L.I32)


def _lp(a: np.ndarray):
    return a.ctypes.data_as(L.I64)


# ---- context -------------------------------------------------------------------------------------
class Context:
    """One CUDA device + stream (nadmm_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(L.lib().nadmm_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    def close(self) -> None:
        if getattr(self, "handle", None):
            L.lib().nadmm_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def node_streams(self) -> int:
        """Concurrent ADMM nodes per GPU (nadmm_ctx_node_streams)."""
        return int(L.lib().nadmm_ctx_node_streams(self.handle))

    def synchronize(self) -> None:
        _check(L.lib().nadmm_ctx_synchronize(self.handle))

    @property
    def stream(self) -> int:
        return L.lib().nadmm_ctx_stream(self.handle) or 0

    def stats(self) -> dict:
        s = L.Stats()
        _check(L.lib().nadmm_ctx_stats(self.handle, C.byref(s)))
        return {f: getattr(s, f) for f, _ in L.Stats._fields_}

    def reset_stats(self) -> None:
        _check(L.lib().nadmm_ctx_reset_stats(self.handle))

    def set_timing(self, enable: bool) -> None:
        _check(L.lib().nadmm_ctx_set_timing(self.handle, int(enable)))


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ---- data (inc/dataset.hpp) ----------------------------------------------------------------------
class Dataset:
    """Device-resident labelled design matrix (Dataset, inc/dataset.hpp:18-65)."""

    def __init__(self, handle, ctx: Context, n: int, p: int, C_: int, sparse: bool, labels: np.ndarray):
        self.handle, self.ctx = handle, ctx
        self._n, self._p, self._C, self._sparse = n, p, C_, sparse
        self._labels = labels
        self._label_values = np.zeros(0)

    @staticmethod
    def dense(features, labels, num_classes: int, ctx: Optional[Context] = None) -> "Dataset":
        ctx = ctx or default_context()
        X = _f64(features)
        if X.ndim != 2:
            raise ConfigError("features must be a 2-D n x p matrix")
        y = np.ascontiguousarray(labels, dtype=np.int32)
        n, p = X.shape
        if y.shape[0] != n:
            raise ConfigError(f"label count {y.shape[0]} does not match row count {n}")
        h = C.c_void_p()
        _check(L.lib().nadmm_shard_dense(ctx.handle, _dp(X), n, p, _ip(y), int(num_classes), C.byref(h)))
        return Dataset(h, ctx, n, p, int(num_classes), False, y)

    @staticmethod
    def sparse(indptr, indices, values, labels, num_classes: int, p: int,
               ctx: Optional[Context] = None) -> "Dataset":
        ctx = ctx or default_context()
        ip = np.ascontiguousarray(indptr, dtype=np.int64)
        ix = np.ascontiguousarray(indices, dtype=np.int32)
        vv = _f64(values)
        y = np.ascontiguousarray(labels, dtype=np.int32)
        n = len(ip) - 1
        if y.shape[0] != n:
            raise ConfigError(f"label count {y.shape[0]} does not match row count {n}")
        h = C.c_void_p()
        _check(L.lib().nadmm_shard_csr(ctx.handle, _lp(ip), _ip(ix), _dp(vv), n, int(p), _ip(y), int(num_classes),
                                       C.byref(h)))
        return Dataset(h, ctx, n, int(p), int(num_classes), True, y)

    def n(self) -> int:
        return self._n

    def p(self) -> int:
        return self._p

    def num_classes(self) -> int:
        return self._C

    def weight_dim(self) -> int:
        return (self._C - 1) * self._p

    def is_sparse(self) -> bool:
        return self._sparse

    def labels(self) -> np.ndarray:
        return self._labels

    def label_values(self) -> np.ndarray:
        """Original label values in class order: label_values()[c-1] is class c's (inc/dataset.hpp:46-50);
        empty unless the dataset came from a reader."""
        return self._label_values

    def set_label_values(self, values) -> None:
        self._label_values = np.asarray(values, dtype=np.float64).copy()

    def device_bytes(self) -> int:
        return int(L.lib().nadmm_shard_device_bytes(self.handle))

    def close(self) -> None:
        if getattr(self, "handle", None):
            L.lib().nadmm_shard_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _wvec(data: Dataset, w, what: str = "weight vector") -> np.ndarray:
    w = _f64(w)
    if w.shape != (data.weight_dim(),):
        raise ConfigError(f"{what} has {w.size} entries, expected (C-1)*p = {data.weight_dim()}")
    return w


# ---- model (inc/softmax.hpp) ----------------------------------------------------------------------
@dataclass
class StableExpCache:  # inc/softmax.hpp:28-33
    logits: np.ndarray
    row_max: np.ndarray
    alpha: np.ndarray
    probs: np.ndarray


def weight_blocks(w, p: int, num_classes: int) -> np.ndarray:
    """p x (C-1) view whose column c-1 is the class-c block (src/softmax.cpp:47-49)."""
    return np.asarray(w).reshape(num_classes - 1, p).T


def stable_exp_cache(data: Dataset, w) -> StableExpCache:
    w = _wvec(data, w)
    n, k = data.n(), data.num_classes() - 1
    lg, pr = np.zeros(n * k), np.zeros(n * k)
    rm, al = np.zeros(n), np.zeros(n)
    _check(L.lib().nadmm_cache(data.handle, _dp(w), _dp(lg), _dp(rm), _dp(al), _dp(pr)))
    return StableExpCache(lg.reshape(k, n).T, rm, al, pr.reshape(k, n).T)


def loss(data: Dataset, w, lam: float = 0.0) -> float:
    w = _wvec(data, w)
    out = C.c_double()
    _check(L.lib().nadmm_loss(data.handle, _dp(w), float(lam), C.byref(out)))
    return out.value


def gradient(data: Dataset, w, lam: float = 0.0) -> np.ndarray:
    w = _wvec(data, w)
    g = np.zeros(data.weight_dim())
    _check(L.lib().nadmm_gradient(data.handle, _dp(w), float(lam), _dp(g)))
    return g


def hessian_vec(data: Dataset, w, v, lam: float = 0.0) -> np.ndarray:
    w = _wvec(data, w)
    v = _wvec(data, v, "hessian_vec: direction")
    hv = np.zeros(data.weight_dim())
    _check(L.lib().nadmm_hessian_vec(data.handle, _dp(w), _dp(v), float(lam), _dp(hv)))
    return hv


def predict(data: Dataset, w) -> np.ndarray:
    w = _wvec(data, w)
    out = np.zeros(data.n(), dtype=np.int32)
    _check(L.lib().nadmm_predict(data.handle, _dp(w), _ip(out)))
    return out


def accuracy(predicted, truth) -> float:
    """Fraction of exact matches (src/softmax.cpp:141-153); host-side like the reference."""
    predicted, truth = np.asarray(predicted), np.asarray(truth)
    if predicted.shape != truth.shape:
        raise ConfigError(f"accuracy: length mismatch {predicted.size} vs {truth.size}")
    if predicted.size == 0:
        return 0.0
    return float(np.count_nonzero(predicted == truth)) / predicted.size


# ---- objective (inc/objective.hpp) ----------------------------------------------------------------
class Objective:
    """value / grad / hvp triple (inc/objective.hpp:12-16) backed by a device shard."""

    def __init__(self, data: Dataset, lam: float, rho: Optional[float] = None, z=None, y=None):
        self.data, self.lam = data, float(lam)
        self.rho = rho
        self.z = None if z is None else _wvec(data, z, "z")
        self.y = None if y is None else _wvec(data, y, "y")

    @property
    def augmented(self) -> bool:
        return self.rho is not None

    def _t(self, x):
        return (self.z - x) + self.y / self.rho

    def value(self, x) -> float:
        f = loss(self.data, x, self.lam)
        if self.augmented:
            t = self._t(_f64(x))
            f = f + 0.5 * self.rho * float(np.dot(t, t))
        return f

    def grad(self, x) -> np.ndarray:
        g = gradient(self.data, x, self.lam)
        if self.augmented:
            g = g - self.rho * self._t(_f64(x))
        return g

    def hvp(self, x, v) -> np.ndarray:
        hv = hessian_vec(self.data, x, v, self.lam)
        if self.augmented:
            hv = hv + self.rho * _f64(v)
        return hv


def make_softmax_objective(data: Dataset, lam: float) -> Objective:
    return Objective(data, lam)


def make_augmented_objective(base: Objective, rho: float, z, y) -> Objective:
    if not (rho > 0.0):
        raise ConfigError("augmented objective requires rho > 0")
    if base.augmented:
        raise ConfigError("base objective is already augmented")
    return Objective(base.data, base.lam, float(rho), z, y)


# ---- Newton-CG (inc/newton.hpp) -------------------------------------------------------------------
@dataclass
class NewtonConfig:  # inc/newton.hpp:9-17
    cg_tol: float = 1e-4
    cg_max_iters: int = 10
    armijo_beta: float = 1e-4
    backtrack_gamma: float = 0.5
    ls_max_iters: int = 10
    grad_tol: float = 1e-8
    newton_max_iters: int = 100

    def to_c(self) -> L.NewtonCfg:
        return L.NewtonCfg(self.cg_tol, self.cg_max_iters, self.armijo_beta, self.backtrack_gamma, self.ls_max_iters,
                           self.grad_tol, self.newton_max_iters)


@dataclass
class NewtonIterRecord:  # inc/newton.hpp:47-57
    iter: int = 0
    grad_norm: float = 0.0
    step: float = 0.0
    cg_iters: int = 0
    cg_residual: float = 0.0
    objective: float = 0.0
    ls_capped: bool = False
    cg_fallback: bool = False
    fn_evals: int = 0


@dataclass
class NewtonResult:  # inc/newton.hpp:59-64
    x: np.ndarray
    trace: list = field(default_factory=list)
    converged: bool = False
    final_grad_norm: float = 0.0


def newton_solve(obj: Objective, x0, cfg: Optional[NewtonConfig] = None) -> NewtonResult:
    """Inexact Newton-CG (src/newton.cpp:73-132), entirely on the device."""
    cfg = cfg or NewtonConfig()
    if not isinstance(obj, Objective):
        raise ConfigError("the device newton_solve takes a softmax Objective (make_softmax_objective)")
    data = obj.data
    x = _wvec(data, x0, "x0").copy()
    cap = max(1, min(cfg.newton_max_iters, 4096))
    tr = (L.NewtonIter * cap)()
    summ = L.NewtonSummary()
    c = cfg.to_c()
    z = obj.z if obj.augmented else np.zeros(0)
    y = obj.y if obj.augmented else np.zeros(0)
    _check(L.lib().nadmm_newton_solve(data.handle, C.byref(c), obj.lam, int(obj.augmented),
                                      float(obj.rho or 0.0), _dp(z), _dp(y), _dp(x), tr, cap, C.byref(summ)))
    recs = [NewtonIterRecord(r.iter, r.grad_norm, r.step, r.cg_iters, r.cg_residual, r.objective, bool(r.ls_capped),
                             bool(r.cg_fallback), r.fn_evals) for r in tr[: min(summ.iterations, cap)]]
    return NewtonResult(x, recs, bool(summ.converged), summ.final_grad_norm)


# ---- L-BFGS (inc/lbfgs.hpp; src/lbfgs.cpp) ---------------------------------------------------------
@dataclass
class LbfgsConfig:  # inc/lbfgs.hpp:9-18
    history: int = 25
    wolfe_c1: float = 1e-4
    wolfe_c2: float = 0.9
    max_iters: int = 100
    ls_max_iters: int = 20
    grad_tol: float = 1e-8

    def to_c(self) -> L.LbfgsCfg:
        return L.LbfgsCfg(self.history, self.wolfe_c1, self.wolfe_c2, self.max_iters, self.ls_max_iters,
                          self.grad_tol)


@dataclass
class LbfgsIterRecord:  # inc/lbfgs.hpp:20-27
    iter: int = 0
    grad_norm: float = 0.0
    step: float = 0.0
    objective: float = 0.0
    fn_evals: int = 0
    ls_fallback: bool = False


@dataclass
class LbfgsResult:  # inc/lbfgs.hpp:29-34
    x: np.ndarray
    trace: list
    converged: bool = False
    final_grad_norm: float = 0.0


def lbfgs_solve(obj: Objective, x0, cfg: Optional[LbfgsConfig] = None) -> LbfgsResult:
    """Limited-memory BFGS with the strong-Wolfe search (src/lbfgs.cpp:94-181) on the device."""
    cfg = cfg or LbfgsConfig()
    if not isinstance(obj, Objective):
        raise ConfigError("the device lbfgs_solve takes a softmax Objective (make_softmax_objective)")
    data = obj.data
    x = _wvec(data, x0, "x0").copy()
    cap = max(1, min(cfg.max_iters, 1 << 16))
    tr = (L.LbfgsIter * cap)()
    summ = L.NewtonSummary()
    c = cfg.to_c()
    z = obj.z if obj.augmented else np.zeros(0)
    y = obj.y if obj.augmented else np.zeros(0)
    _check(L.lib().nadmm_lbfgs_solve(data.handle, C.byref(c), obj.lam, int(obj.augmented), float(obj.rho or 0.0),
                                     _dp(z), _dp(y), _dp(x), tr, cap, C.byref(summ)))
    recs = [LbfgsIterRecord(r.iter, r.grad_norm, r.step, r.objective, r.fn_evals, bool(r.ls_fallback))
            for r in tr[: min(summ.iterations, cap)]]
    return LbfgsResult(x, recs, bool(summ.converged), summ.final_grad_norm)


def workers_solve(workers: Sequence["Worker"], rho, z, ys, cfg: Optional[NewtonConfig] = None, inner_iters: int = 1,
                  outs=None):
    """One scatter -> gather round over several workers (the reference's WorkerPool): the workers
    run concurrently on the GPU; x_i land in `outs[i]` (e.g. pinned float64 buffers) if given."""
    cfg = cfg or NewtonConfig()
    n = len(workers)
    if n == 0:
        raise ConfigError("at least one worker required")
    rho = np.ascontiguousarray(np.broadcast_to(np.asarray(rho, dtype=np.float64), (n,)))
    z = _wvec(workers[0].shard, z, "z")
    ys = [_wvec(w.shard, y, "y") for w, y in zip(workers, ys)]
    xs = [w._out(None if outs is None else outs[i]) for i, w in enumerate(workers)]
    hs = (C.c_void_p * n)(*[w.handle for w in workers])
    yp = (L.D * n)(*[_dp(y) for y in ys])
    xp = (L.D * n)(*[_dp(x) for x in xs])
    st = (L.InnerStats * n)()
    c = cfg.to_c()
    _check(L.lib().nadmm_workers_solve(hs, n, _dp(rho), _dp(z), yp, C.byref(c), int(inner_iters), xp, st))
    return xs, [InnerStats(s.grad_norm, s.inner_iters, s.cg_iters, s.fn_evals, s.flags) for s in st]


# ---- synchronous SGD (src/worker.cpp:197-218) -----------------------------------
@dataclass
class SgdConfig:  # SgdConfig + WorkerSessionConfig sgd_batch / steps_per_epoch / seed
    eta: float = 1.0
    batch: int = 100
    epochs: int = 1
    steps_per_epoch: int = 0  # worker: >= 1; sync_sgd: 0 -> ceil(n / (batch N))
    seed: int = 0

    def to_c(self) -> L.SgdCfg:
        return L.SgdCfg(self.eta, self.batch, self.epochs, self.steps_per_epoch, self.seed)


@dataclass
class SgdResult:
    x: np.ndarray
    metrics: list
    epochs: int


def sgd_permutation(seed: int, epoch: int, n: int) -> np.ndarray:
    """The SGD worker's epoch permutation Rng(mix_seed(seed, epoch)).shuffle(0..n-1)."""
    out = np.empty(n, dtype=np.int32)
    _check(L.lib().nadmm_sgd_permutation(seed, epoch, n, _ip(out)))
    return out


def sync_sgd(parts: Sequence[Dataset], cfg: SgdConfig, lam: float = 0.0, x0=None,
             comm: Optional[Communicator] = None) -> SgdResult:
    """Synchronous mini-batch SGD over device shards: one metrics row per epoch."""
    if not parts:
        raise ConfigError("sync_sgd needs at least one shard")
    d = parts[0].weight_dim()
    x = np.zeros(d) if x0 is None else _wvec(parts[0], x0, "x0").copy()
    hs = (C.c_void_p * len(parts))(*[p.handle for p in parts])
    cap = max(1, cfg.epochs)
    rows = (L.MetricsRow * cap)()
    done = C.c_int32()
    c = cfg.to_c()
    _check(L.lib().nadmm_sgd_run(hs, len(parts), comm.handle if comm else None, C.byref(c), float(lam), _dp(x), rows,
                                 cap, C.byref(done)))
    metrics = [{f: getattr(r, f) for f, _ in L.MetricsRow._fields_} for r in rows[: min(done.value, cap)]]
    return SgdResult(x, metrics, done.value)


# ---- worker (inc/worker.hpp; src/worker.cpp:127-196) ----------------------------------------------
@dataclass
class InnerStats:  # inc/comm.hpp:67-73
    grad_norm: float = 0.0
    inner_iters: int = 0
    cg_iters: int = 0
    fn_evals: int = 0
    flags: int = 0


class Worker:
    """The ADMM branch of run_worker: persistent base objective (lambda = 0) and warm start x_local."""

    def __init__(self, shard: Dataset):
        h = C.c_void_p()
        _check(L.lib().nadmm_worker_create(shard.handle, C.byref(h)))
        self.handle, self.shard = h, shard

    def solve(self, rho: float, z, y, cfg: Optional[NewtonConfig] = None, inner_iters: int = 1, out=None):
        """One scatter -> gather round; `out` (optional, e.g. a pinned float64 buffer of length d)
        receives x directly."""
        cfg = cfg or NewtonConfig()
        z = _wvec(self.shard, z, "z")
        y = _wvec(self.shard, y, "y")
        x = self._out(out)
        st = L.InnerStats()
        c = cfg.to_c()
        _check(L.lib().nadmm_worker_solve(self.handle, float(rho), _dp(z), _dp(y), C.byref(c), int(inner_iters),
                                          _dp(x), C.byref(st)))
        return x, InnerStats(st.grad_norm, st.inner_iters, st.cg_iters, st.fn_evals, st.flags)

    def solve_lbfgs(self, rho: float, z, y, cfg: Optional[LbfgsConfig] = None, inner_iters: int = 1, out=None):
        """The same round with the L-BFGS inner solver (src/worker.cpp:183-195)."""
        cfg = cfg or LbfgsConfig()
        z = _wvec(self.shard, z, "z")
        y = _wvec(self.shard, y, "y")
        x = self._out(out)
        st = L.InnerStats()
        c = cfg.to_c()
        _check(L.lib().nadmm_worker_solve_lbfgs(self.handle, float(rho), _dp(z), _dp(y), C.byref(c),
                                                int(inner_iters), _dp(x), C.byref(st)))
        return x, InnerStats(st.grad_norm, st.inner_iters, st.cg_iters, st.fn_evals, st.flags)

    def sgd_grad(self, cfg: SgdConfig, iteration: int, z):
        """The SGD branch of run_worker for scatter `iteration`: the mini-batch gradient at z / batch."""
        z = _wvec(self.shard, z, "z")
        g = np.zeros(self.shard.weight_dim())
        st = L.InnerStats()
        c = cfg.to_c()
        _check(L.lib().nadmm_worker_sgd_grad(self.handle, C.byref(c), int(iteration), _dp(z), _dp(g), C.byref(st)))
        return g, InnerStats(st.grad_norm, st.inner_iters, st.cg_iters, st.fn_evals, st.flags)

    def _out(self, out):
        d = self.shard.weight_dim()
        if out is None:
            return np.zeros(d)
        if not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.shape == (d,)
                and out.flags.c_contiguous):
            raise ConfigError(f"out must be a contiguous float64 array of length {d}")
        return out

    def close(self) -> None:
        """Release the worker (and its binding of the shard's solver state)."""
        if getattr(self, "handle", None):
            L.lib().nadmm_worker_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- consensus (inc/admm.hpp) ---------------------------------------------------------------------
@dataclass
class PenaltyPolicy:  # inc/admm.hpp:37-47
    kind: str = "fixed"  # "fixed" | "spectral"
    rho0: float = 1.0
    update_period: int = 2
    eps_cor: float = 0.2
    rho_min: float = 1e-6
    rho_max: float = 1e6


@dataclass
class StoppingConfig:  # inc/admm.hpp:49-56
    eps_abs: float = 1e-3
    eps_rel: float = 1e-3
    max_outer_iters: int = 300
    standard_norms: bool = False


@dataclass
class AdmmConfig:  # inc/admm.hpp:107-117
    n_workers: int = 4
    lam: float = 1e-5
    penalty: PenaltyPolicy = field(default_factory=PenaltyPolicy)
    stopping: StoppingConfig = field(default_factory=StoppingConfig)
    newton: NewtonConfig = field(default_factory=NewtonConfig)
    inner_iters: int = 1
    inner_solver: str = "newton"  # InnerSolverKind (inc/admm.hpp:105-114): "newton" | "lbfgs"
    lbfgs: LbfgsConfig = field(default_factory=LbfgsConfig)
    # bitwise-deterministic consensus: all-gather of the per-worker terms and the
    # oracle's ascending-id pairwise tree for z, identical for any number of ranks
    consensus_tree: bool = False

    def to_c(self) -> L.AdmmCfg:
        c = L.AdmmCfg()
        L.lib().nadmm_admm_cfg_default(C.byref(c))
        c.lam = self.lam
        c.penalty_kind = 1 if self.penalty.kind == "spectral" else 0
        c.rho0, c.update_period, c.eps_cor = self.penalty.rho0, self.penalty.update_period, self.penalty.eps_cor
        c.rho_min, c.rho_max = self.penalty.rho_min, self.penalty.rho_max
        c.eps_abs, c.eps_rel = self.stopping.eps_abs, self.stopping.eps_rel
        c.max_outer_iters, c.standard_norms = self.stopping.max_outer_iters, int(self.stopping.standard_norms)
        c.inner_iters = self.inner_iters
        c.newton = self.newton.to_c()
        if self.inner_solver not in ("newton", "lbfgs"):
            raise ConfigError(f"unknown inner solver {self.inner_solver!r}")
        c.inner_solver = 1 if self.inner_solver == "lbfgs" else 0
        c.lbfgs = self.lbfgs.to_c()
        c.consensus_tree = int(self.consensus_tree)
        return c


@dataclass
class EvalContext:  # inc/admm.hpp:132-136
    eval_objective: bool = True
    f_star: Optional[float] = None
    theta_stop: float = 0.0
    ignore_convergence: bool = False  # throughput runs: keep iterating past has_converged


@dataclass
class AdmmRunResult:  # inc/admm.hpp:119-126
    z: np.ndarray
    metrics: list
    converged: bool
    iterations: int
    rho: np.ndarray


class Communicator:
    """NCCL communicator of one rank (nadmm_comm)."""

    def __init__(self, ctx: Context, uid: bytes, nranks: int, rank: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(L.lib().nadmm_comm_create(ctx.handle, buf, nranks, rank, C.byref(h)))
        self.handle, self.nranks, self.rank = h, nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(L.lib().nadmm_comm_unique_id(buf))
        return bytes(buf)

    def close(self) -> None:
        if getattr(self, "handle", None):
            L.lib().nadmm_comm_destroy(self.handle)
            self.handle = None


def run_admm(parts: Sequence[Dataset], cfg: AdmmConfig, eval: Optional[EvalContext] = None,
             comm: Optional[Communicator] = None) -> AdmmRunResult:
    """Consensus loop over device shards (inc/admm.hpp:139-140). `parts` are this rank's workers."""
    if not parts:
        raise ConfigError("run_admm needs at least one shard")
    if comm is None and cfg.n_workers != len(parts):
        raise ConfigError(f"n_workers={cfg.n_workers} but {len(parts)} shards given")
    ev = eval or EvalContext(eval_objective=False)
    c = cfg.to_c()
    c.eval_objective = int(ev.eval_objective)
    c.f_star = float(ev.f_star or 0.0)
    c.theta_stop = float(ev.theta_stop)
    hs = (C.c_void_p * len(parts))(*[p.handle for p in parts])
    d = parts[0].weight_dim()
    z = np.zeros(d)
    rho = np.zeros(len(parts))
    cap = max(1, c.max_outer_iters)
    rows = (L.MetricsRow * cap)()
    it, conv = C.c_int32(), C.c_int32()
    _check(L.lib().nadmm_admm_run(hs, len(parts), comm.handle if comm else None, C.byref(c), _dp(z), _dp(rho), rows,
                                  cap, C.byref(it), C.byref(conv)))
    metrics = [{f: getattr(r, f) for f, _ in L.MetricsRow._fields_} for r in rows[: min(it.value, cap)]]
    return AdmmRunResult(z, metrics, bool(conv.value), it.value, rho)


class AdmmSession:
    """Stepping form of run_admm: AdmmState::initial, then `step(n)` outer iterations at a time."""

    def __init__(self, parts: Sequence[Dataset], cfg: AdmmConfig, eval: Optional[EvalContext] = None,
                 comm: Optional[Communicator] = None):
        if not parts:
            raise ConfigError("AdmmSession needs at least one shard")
        ev = eval or EvalContext(eval_objective=False)
        c = cfg.to_c()
        c.eval_objective = int(ev.eval_objective)
        c.f_star = float(ev.f_star or 0.0)
        c.theta_stop = float(ev.theta_stop)
        c.ignore_convergence = int(ev.ignore_convergence)
        self._hs = (C.c_void_p * len(parts))(*[p.handle for p in parts])
        self.parts, self.cfg = list(parts), cfg
        h = C.c_void_p()
        _check(L.lib().nadmm_admm_create(self._hs, len(parts), comm.handle if comm else None, C.byref(c), C.byref(h)))
        self.handle = h
        self.metrics: list = []
        self.finished = False

    def step(self, n: int) -> int:
        rows = (L.MetricsRow * max(1, n))()
        done, fin = C.c_int32(), C.c_int32()
        _check(L.lib().nadmm_admm_step(self.handle, int(n), rows, max(1, n), C.byref(done), C.byref(fin)))
        self.metrics += [{f: getattr(r, f) for f, _ in L.MetricsRow._fields_} for r in rows[: done.value]]
        self.finished = bool(fin.value)
        return done.value

    def result(self) -> AdmmRunResult:
        d = self.parts[0].weight_dim()
        z, rho = np.zeros(d), np.zeros(len(self.parts))
        it, conv = C.c_int32(), C.c_int32()
        _check(L.lib().nadmm_admm_result(self.handle, _dp(z), _dp(rho), C.byref(it), C.byref(conv)))
        return AdmmRunResult(z, self.metrics, bool(conv.value), it.value, rho)

    def close(self) -> None:
        if getattr(self, "handle", None):
            L.lib().nadmm_admm_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- data fixtures (src/data_io.cpp) --------------------------------------------------------------
def mix_seed(seed: int, salt: int) -> int:
    return int(L.lib().nadmm_mix_seed(seed, salt))


def generate_synthetic(n: int, p: int, num_classes: int, separation: float = 10.0, noise: float = 0.1,
                       seed: int = 0):
    """Gaussian class clusters, 90/10 split (src/data_io.cpp:330-370) -> (Xtr, ytr, Xte, yte)."""
    nt = (n * 9) // 10
    Xtr, ytr = np.empty((nt, p)), np.empty(nt, dtype=np.int32)
    Xte, yte = np.empty((n - nt, p)), np.empty(n - nt, dtype=np.int32)
    _check(L.lib().nadmm_generate_synthetic(n, p, num_classes, separation, noise, seed, _dp(Xtr), _ip(ytr), _dp(Xte),
                                            _ip(yte)), data=True)
    return Xtr, ytr, Xte, yte


def generate_sparse(n: int, p: int, num_classes: int, nnz_per_row: int, seed: int = 0):
    indptr = np.empty(n + 1, dtype=np.int64)
    indices = np.empty(n * nnz_per_row, dtype=np.int32)
    vals = np.empty(n * nnz_per_row)
    labels = np.empty(n, dtype=np.int32)
    _check(L.lib().nadmm_generate_sparse(n, p, num_classes, nnz_per_row, seed, _lp(indptr), _ip(indices), _dp(vals),
                                         _ip(labels)), data=True)
    return indptr, indices, vals, labels


# ---- real-data readers (src/data_io.cpp:85-137, 220-271) -----------------------------------------
@dataclass
class LoadedData:
    """A file read into host arrays, before it becomes a device shard. Sparse files fill the CSR
    triple (canonical rows: columns ascending, duplicates summed); dense files fill X (n x p)."""
    n: int
    p: int
    num_classes: int
    labels: np.ndarray
    label_values: np.ndarray
    indptr: Optional[np.ndarray] = None
    indices: Optional[np.ndarray] = None
    vals: Optional[np.ndarray] = None
    X: Optional[np.ndarray] = None

    @property
    def sparse(self) -> bool:
        return self.X is None

    def to_device(self, ctx: Optional[Context] = None) -> "Dataset":
        if self.sparse:
            ds = Dataset.sparse(self.indptr, self.indices, self.vals, self.labels, self.num_classes, self.p, ctx=ctx)
        else:
            ds = Dataset.dense(self.X, self.labels, self.num_classes, ctx=ctx)
        ds.set_label_values(self.label_values)
        return ds


def read_libsvm(path) -> LoadedData:
    """LIBSVM text ("label idx:val ...", 1-based) -> host CSR, labels remapped to 1..C ascending.
    Same errors as the reference's load_libsvm: ConfigError (cannot open, < 2 classes, p = 0),
    DataError (non-integer label, malformed token, 0-based index, no rows, non-finite value)."""
    lib = L.lib()
    h = C.c_void_p()
    n, p, nnz, c = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
    _check(lib.nadmm_libsvm_parse(str(path).encode(), C.byref(h), C.byref(n), C.byref(p), C.byref(nnz), C.byref(c)),
           data=True)
    try:
        out = LoadedData(n.value, p.value, c.value, np.empty(n.value, dtype=np.int32), np.empty(c.value),
                         indptr=np.empty(n.value + 1, dtype=np.int64), indices=np.empty(nnz.value, dtype=np.int32),
                         vals=np.empty(nnz.value))
        _check(lib.nadmm_libsvm_fetch(h, _lp(out.indptr), _ip(out.indices), _dp(out.vals), _ip(out.labels),
                                      _dp(out.label_values)), data=True)
        return out
    finally:
        lib.nadmm_libsvm_free(h)


def read_idx(images, labels) -> LoadedData:
    """IDX image (0x803) + label (0x801) files -> host dense X in [0, 1], labels digit + 1."""
    lib = L.lib()
    n, p = C.c_int64(), C.c_int64()
    ib, lb = str(images).encode(), str(labels).encode()
    _check(lib.nadmm_idx_info(ib, lb, C.byref(n), C.byref(p)), data=True)
    X = np.empty((n.value, p.value))
    y = np.empty(n.value, dtype=np.int32)
    lv = np.empty(256)
    c = C.c_int32()
    _check(lib.nadmm_idx_load(ib, lb, _dp(X), _ip(y), C.byref(c), _dp(lv)), data=True)
    return LoadedData(n.value, p.value, c.value, y, lv[:c.value].copy(), X=X)


def load_libsvm(path, ctx: Optional[Context] = None) -> "Dataset":
    """load_libsvm (inc/nadmm/data_io.hpp:52-57): the file as a device-resident sparse Dataset."""
    return read_libsvm(path).to_device(ctx)


def load_idx(images, labels, ctx: Optional[Context] = None) -> "Dataset":
    """load_idx (inc/nadmm/data_io.hpp:63-65): MNIST-style IDX files as a device-resident dense Dataset."""
    return read_idx(images, labels).to_device(ctx)


def partition_owner(n: int, n_workers: int, strided: bool = False) -> np.ndarray:
    out = np.empty(n, dtype=np.int32)
    _check(L.lib().nadmm_partition(n, n_workers, int(strided), _ip(out)), data=True)
    return out


def partition(X, labels, n_workers: int, strided: bool = False):
    """Row subsets per worker (src/data_io.cpp:300-328) as host (X_i, y_i) pairs."""
    owner = partition_owner(len(labels), n_workers, strided)
    X, labels = np.asarray(X), np.asarray(labels)
    return [(X[owner == i], labels[owner == i]) for i in range(n_workers)]
