"""CPU oracle for the Newton-ADMM hot path -- TEST INFRASTRUCTURE ONLY.

Two checkers, both plain CPU code:

* ``Port`` -- ``oracle/port/nadmm_oracle.c``: a C restatement of the reference hot path
  (src/dataset.cpp:28-85, src/softmax.cpp:47-153, src/objective.cpp:9-56, src/newton.cpp:8-132,
  src/worker.cpp:127-196, src/data_io.cpp:16-43/300-370) plus the ADMM coordinator the reference
  only declares (inc/admm.hpp:17-140; SPEC.md:196-304 -> "parity unpinned" for that part).
* ``Ref`` -- ``oracle/_ref/libnadmm_ref.so``: the REFERENCE's own sources compiled in place from
  /root/reference/proj/src against ``oracle/eigen_shim`` (Eigen is absent from the image).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm may
import this package. The product (``paper_1807_07132_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "build" / "libnadmm_oracle.so"
REF_SO = HERE / "_ref" / "libnadmm_ref.so"

D = C.POINTER(C.c_double)
I32 = C.POINTER(C.c_int32)
I64 = C.POINTER(C.c_int64)
VP = C.c_void_p

VALUE_FN = C.CFUNCTYPE(C.c_double, D, C.c_int64, VP)
GRAD_FN = C.CFUNCTYPE(None, D, D, C.c_int64, VP)
HVP_FN = C.CFUNCTYPE(None, D, D, D, C.c_int64, VP)
APPLY_FN = C.CFUNCTYPE(None, D, D, C.c_int64, VP)

DEFAULT_NEWTON = (1e-4, 10, 1e-4, 0.5, 10, 1e-8, 100)  # inc/newton.hpp:9-17
TRACE_FIELDS = ("iter", "grad_norm", "step", "cg_iters", "cg_residual", "objective", "ls_capped", "cg_fallback",
                "fn_evals")


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build(ref: bool = True) -> None:
    """Compile the port (always) and the reference build (when /root/reference is present)."""
    targets = ["port"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(D)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(I32)


def _lp(a: np.ndarray):
    return a.ctypes.data_as(I64)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _cfg(cfg) -> np.ndarray:
    return _f64(DEFAULT_NEWTON if cfg is None else cfg)


def _put(ptr, n: int, values) -> None:
    """Write a length-n vector into a ctypes double* (callback output)."""
    np.ctypeslib.as_array(ptr, (n,))[:] = np.asarray(values, dtype=np.float64)


def _get(ptr, n: int) -> np.ndarray:
    return np.ctypeslib.as_array(ptr, (n,)).copy()


def _trace_rows(buf: np.ndarray, n: int):
    return [dict(zip(TRACE_FIELDS, row.tolist())) for row in buf[: min(n, len(buf))]]


class _NorData(C.Structure):
    _fields_ = [("n", C.c_int64), ("p", C.c_int64), ("C", C.c_int32), ("sparse", C.c_int32), ("X", D),
                ("indptr", I64), ("indices", I32), ("vals", D), ("labels", I32)]


class NorAdmmCfg(C.Structure):
    _fields_ = [("n_workers", C.c_int32), ("lam", C.c_double), ("penalty_kind", C.c_int32), ("rho0", C.c_double),
                ("update_period", C.c_int32), ("eps_cor", C.c_double), ("rho_min", C.c_double),
                ("rho_max", C.c_double), ("eps_abs", C.c_double), ("eps_rel", C.c_double),
                ("max_outer_iters", C.c_int32), ("standard_norms", C.c_int32), ("inner_iters", C.c_int32),
                ("newton", C.c_double * 7)]


class NorMetricsRow(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("train_objective", C.c_double), ("primal_norm", C.c_double),
                ("dual_norm", C.c_double), ("eps_pri", C.c_double), ("eps_dual", C.c_double),
                ("inner_iterations", C.c_int32), ("cg_iters", C.c_int32), ("fn_evals", C.c_int32),
                ("flags", C.c_int32), ("rho_mean", C.c_double)]


def admm_cfg(n_workers=4, lam=1e-5, penalty="fixed", rho0=1.0, update_period=2, eps_cor=0.2, rho_min=1e-6,
             rho_max=1e6, eps_abs=1e-3, eps_rel=1e-3, max_outer_iters=300, standard_norms=False, inner_iters=1,
             newton=None) -> NorAdmmCfg:
    """AdmmConfig defaults (inc/admm.hpp:37-56, 107-117)."""
    c = NorAdmmCfg()
    c.n_workers, c.lam, c.rho0 = n_workers, lam, rho0
    c.penalty_kind = 1 if penalty == "spectral" else 0
    c.update_period, c.eps_cor, c.rho_min, c.rho_max = update_period, eps_cor, rho_min, rho_max
    c.eps_abs, c.eps_rel, c.max_outer_iters = eps_abs, eps_rel, max_outer_iters
    c.standard_norms, c.inner_iters = int(standard_norms), inner_iters
    for i, v in enumerate(DEFAULT_NEWTON if newton is None else newton):
        c.newton[i] = v
    return c


class Shard:
    """Host shard in reference layout; keeps the numpy buffers alive for the C structs."""

    def __init__(self, X=None, labels=None, C_: int = 2, csr=None, p: int | None = None):
        self.labels = _i32(labels)
        self.C = int(C_)
        if csr is not None:
            indptr, indices, vals = csr
            self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
            self.indices = _i32(indices)
            self.vals = _f64(vals)
            self.n, self.p, self.sparse, self.X = len(self.labels), int(p), 1, None
        else:
            self.X = _f64(X)
            self.n, self.p = self.X.shape
            self.sparse = 0
            self.indptr = self.indices = self.vals = None

    @property
    def d(self) -> int:
        return (self.C - 1) * self.p

    def dense(self) -> np.ndarray:
        if not self.sparse:
            return self.X
        out = np.zeros((self.n, self.p))
        for i in range(self.n):
            s, e = self.indptr[i], self.indptr[i + 1]
            out[i, self.indices[s:e]] += self.vals[s:e]
        return out

    def nor(self) -> _NorData:
        s = _NorData()
        s.n, s.p, s.C, s.sparse = self.n, self.p, self.C, self.sparse
        s.labels = _ip(self.labels)
        if self.sparse:
            s.indptr, s.indices, s.vals = _lp(self.indptr), _ip(self.indices), _dp(self.vals)
        else:
            s.X = _dp(self.X)
        return s


class Port:
    """ctypes view of oracle/build/libnadmm_oracle.so."""

    def __init__(self, path: Path = PORT_SO):
        if not path.exists():
            build(ref=False)
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.nor_last_error.restype = C.c_char_p
        L.nor_newton_solve.argtypes = None
        L.nor_spectral_rho.restype = C.c_double
        L.nor_mix_seed.restype = C.c_uint64
        L.nor_mix_seed.argtypes = [C.c_uint64, C.c_uint64]

    def _chk(self, rc: int):
        if rc:
            raise OracleError(rc, self.lib.nor_last_error().decode())

    # ---- model (src/softmax.cpp) ----
    def cache(self, sh: Shard, w):
        k = sh.C - 1
        lg, pr = np.zeros(sh.n * k), np.zeros(sh.n * k)
        rm, al = np.zeros(sh.n), np.zeros(sh.n)
        nd = sh.nor()
        self._chk(self.lib.nor_cache_at(C.byref(nd), _dp(_f64(w)), _dp(lg), _dp(rm), _dp(al), _dp(pr)))
        return lg.reshape(k, sh.n).T, rm, al, pr.reshape(k, sh.n).T

    def loss(self, sh: Shard, w, lam: float = 0.0) -> float:
        out = C.c_double()
        nd = sh.nor()
        self._chk(self.lib.nor_loss_at(C.byref(nd), _dp(_f64(w)), C.c_double(lam), C.byref(out)))
        return out.value

    def gradient(self, sh: Shard, w, lam: float = 0.0) -> np.ndarray:
        g = np.zeros(sh.d)
        nd = sh.nor()
        self._chk(self.lib.nor_gradient_at(C.byref(nd), _dp(_f64(w)), C.c_double(lam), _dp(g)))
        return g

    def hessian_vec(self, sh: Shard, w, v, lam: float = 0.0) -> np.ndarray:
        hv = np.zeros(sh.d)
        nd = sh.nor()
        self._chk(self.lib.nor_hessian_vec_at(C.byref(nd), _dp(_f64(w)), _dp(_f64(v)), C.c_double(lam), _dp(hv)))
        return hv

    def predict(self, sh: Shard, w) -> np.ndarray:
        out = np.zeros(sh.n, dtype=np.int32)
        nd = sh.nor()
        self._chk(self.lib.nor_predict(C.byref(nd), _dp(_f64(w)), _ip(out)))
        return out

    def validate(self, sh: Shard) -> None:
        nd = sh.nor()
        self._chk(self.lib.nor_validate(C.byref(nd)))

    # ---- solver (src/newton.cpp) ----
    def newton_solve(self, sh: Shard, lam: float, x0, cfg=None, rho: float | None = None, z=None, y=None,
                     trace_cap: int = 256):
        x = np.zeros(sh.d)
        tr = np.zeros((trace_cap, 9))
        nt, conv, gn = C.c_int(), C.c_int(), C.c_double()
        aug = rho is not None
        zz = _f64(z if aug else np.zeros(sh.d))
        yy = _f64(y if aug else np.zeros(sh.d))
        nd = sh.nor()
        self._chk(self.lib.nor_newton_solve_softmax(
            C.byref(nd), C.c_double(lam), C.c_int(int(aug)), C.c_double(rho or 0.0), _dp(zz), _dp(yy),
            _dp(_f64(x0)), _dp(_cfg(cfg)), _dp(x), _dp(tr), C.c_int(trace_cap), C.byref(nt), C.byref(conv),
            C.byref(gn)))
        return dict(x=x, trace=_trace_rows(tr, nt.value), converged=bool(conv.value), final_grad_norm=gn.value)

    def cg_solve(self, apply, g, theta: float, max_iters: int):
        g = _f64(g)
        d = len(g)
        cb = APPLY_FN(lambda i, o, n, u: _put(o, n, apply(_get(i, n))))
        p = np.zeros(d)
        it, ach, neg = C.c_int(), C.c_double(), C.c_int()
        self._chk(self.lib.nor_cg_solve(cb, None, _dp(g), C.c_int64(d), C.c_double(theta), C.c_int(max_iters),
                                        _dp(p), C.byref(it), C.byref(ach), C.byref(neg)))
        return dict(p=p, iters=it.value, achieved_residual=ach.value, negative_curvature=bool(neg.value))

    def _iface(self, value, grad=None, hvp=None, d=0):
        class Obj(C.Structure):
            _fields_ = [("value", VALUE_FN), ("grad", GRAD_FN), ("hvp", HVP_FN), ("user", VP), ("d", C.c_int64)]

        keep = [VALUE_FN(lambda x, n, u: float(value(np.ctypeslib.as_array(x, (n,)).copy())))]
        keep.append(GRAD_FN(lambda x, g, n, u: _put(g, n, grad(_get(x, n)))) if grad else GRAD_FN())
        keep.append(HVP_FN(lambda x, v, o, n, u: _put(o, n, hvp(_get(x, n), _get(v, n)))) if hvp else HVP_FN())
        o = Obj(keep[0], keep[1], keep[2], None, d)
        return o, keep

    def line_search(self, value, x, p, g, f_x: float, cfg=None):
        x, p, g = _f64(x), _f64(p), _f64(g)
        o, keep = self._iface(value, d=len(x))
        a, ev, cap = C.c_double(), C.c_int(), C.c_int()
        self._chk(self.lib.nor_line_search(C.byref(o), _dp(x), _dp(p), _dp(g), C.c_double(f_x), _dp(_cfg(cfg)),
                                           C.byref(a), C.byref(ev), C.byref(cap)))
        return dict(alpha=a.value, evals=ev.value, capped=bool(cap.value))

    def newton_solve_cb(self, value, grad, hvp, x0, cfg=None, trace_cap=64):
        x0 = _f64(x0)
        o, keep = self._iface(value, grad, hvp, d=len(x0))
        x = np.zeros(len(x0))
        tr = np.zeros((trace_cap, 9))
        nt, conv, gn = C.c_int(), C.c_int(), C.c_double()
        self._chk(self.lib.nor_newton_solve(C.byref(o), _dp(x0), _dp(_cfg(cfg)), _dp(x), _dp(tr), C.c_int(trace_cap),
                                            C.byref(nt), C.byref(conv), C.byref(gn)))
        return dict(x=x, trace=_trace_rows(tr, nt.value), converged=bool(conv.value), final_grad_norm=gn.value)

    # ---- ADMM (inc/admm.hpp) ----
    def z_update(self, x, y, rho, lam):
        x, y, rho = _f64(x), _f64(y), _f64(rho)
        N, d = x.shape
        z = np.zeros(d)
        self._chk(self.lib.nor_z_update(_dp(x), _dp(y), _dp(rho), C.c_int(N), C.c_int64(d), C.c_double(lam), _dp(z)))
        return z

    def y_update(self, y, x, z, rho):
        x, y, z, rho = _f64(x), _f64(y), _f64(z), _f64(rho)
        N, d = x.shape
        out = np.zeros((N, d))
        self.lib.nor_y_update(_dp(y), _dp(x), _dp(z), _dp(rho), C.c_int(N), C.c_int64(d), _dp(out))
        return out

    def residuals(self, x, z, prev_z, rho):
        x, z, pz, rho = _f64(x), _f64(z), _f64(prev_z), _f64(rho)
        N, d = x.shape
        pr, du = np.zeros(N), np.zeros(N)
        pt, dt = C.c_double(), C.c_double()
        self.lib.nor_residuals(_dp(x), _dp(z), _dp(pz), _dp(rho), C.c_int(N), C.c_int64(d), _dp(pr), _dp(du),
                               C.byref(pt), C.byref(dt))
        return pr, du, pt.value, dt.value

    def tolerances(self, x, y, z, eps_abs, eps_rel, standard_norms=False):
        x, y, z = _f64(x), _f64(y), _f64(z)
        N, d = x.shape
        ep, ed = C.c_double(), C.c_double()
        self.lib.nor_tolerances(_dp(x), _dp(y), _dp(z), C.c_int(N), C.c_int64(d), C.c_double(eps_abs),
                                C.c_double(eps_rel), C.c_int(int(standard_norms)), C.byref(ep), C.byref(ed))
        return ep.value, ed.value

    def spectral_rho(self, dx, dyhat, dz, dy, rho, eps_cor=0.2, rho_min=1e-6, rho_max=1e6):
        dx, dyhat, dz, dy = _f64(dx), _f64(dyhat), _f64(dz), _f64(dy)
        xo, zo = C.c_int(), C.c_int()
        self.lib.nor_spectral_rho.argtypes = [D, D, D, D, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_double,
                                              C.POINTER(C.c_int), C.POINTER(C.c_int)]
        r = self.lib.nor_spectral_rho(_dp(dx), _dp(dyhat), _dp(dz), _dp(dy), len(dx), rho, eps_cor, rho_min, rho_max,
                                      C.byref(xo), C.byref(zo))
        return r, bool(xo.value), bool(zo.value)

    def admm_run(self, shards, cfg: NorAdmmCfg, eval_objective=True, row_cap=None):
        N = cfg.n_workers
        arr = (_NorData * N)(*[s.nor() for s in shards])
        d = shards[0].d
        z, rho = np.zeros(d), np.zeros(N)
        cap = row_cap or cfg.max_outer_iters
        rows = (NorMetricsRow * cap)()
        it, conv = C.c_int(), C.c_int()
        self._chk(self.lib.nor_admm_run(arr, C.byref(cfg), C.c_int(int(eval_objective)), _dp(z), _dp(rho), rows,
                                        C.c_int(cap), C.byref(it), C.byref(conv)))
        out = [{f: getattr(r, f) for f, _ in NorMetricsRow._fields_} for r in rows[: min(it.value, cap)]]
        return dict(z=z, rho=rho, iterations=it.value, converged=bool(conv.value), metrics=out)

    # ---- fixtures (src/data_io.cpp) ----
    def rng_stream(self, seed: int, kind: int, count: int, bound: int = 0) -> np.ndarray:
        out = np.zeros(count)
        self._chk(self.lib.nor_rng_stream(C.c_uint64(seed), C.c_int(kind), C.c_uint64(bound), C.c_int64(count),
                                          _dp(out)))
        return out

    def mix_seed(self, seed: int, salt: int) -> int:
        return int(self.lib.nor_mix_seed(seed, salt))

    def generate_synthetic(self, n, p, C_, separation=10.0, noise=0.1, seed=0):
        nt = (n * 9) // 10
        Xtr, ytr = np.zeros((nt, p)), np.zeros(nt, dtype=np.int32)
        Xte, yte = np.zeros((n - nt, p)), np.zeros(n - nt, dtype=np.int32)
        self._chk(self.lib.nor_generate_synthetic(
            C.c_int64(n), C.c_int64(p), C.c_int32(C_), C.c_double(separation), C.c_double(noise), C.c_uint64(seed),
            _dp(Xtr), _ip(ytr), _dp(Xte), _ip(yte)))
        return Xtr, ytr, Xte, yte

    def generate_sparse(self, n, p, C_, nnz_per_row, seed=0):
        indptr = np.zeros(n + 1, dtype=np.int64)
        indices = np.zeros(n * nnz_per_row, dtype=np.int32)
        vals = np.zeros(n * nnz_per_row)
        labels = np.zeros(n, dtype=np.int32)
        self._chk(self.lib.nor_generate_sparse(C.c_int64(n), C.c_int64(p), C.c_int32(C_), C.c_int32(nnz_per_row),
                                               C.c_uint64(seed), _lp(indptr), _ip(indices), _dp(vals), _ip(labels)))
        return indptr, indices, vals, labels

    def partition_owner(self, n, n_workers, strided=False) -> np.ndarray:
        out = np.zeros(n, dtype=np.int32)
        self._chk(self.lib.nor_partition_owner(C.c_int64(n), C.c_int(n_workers), C.c_int(int(strided)), _ip(out)))
        return out


class Ref:
    """ctypes view of oracle/_ref/libnadmm_ref.so: the reference's own code (see module doc)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (needs /root/reference; run oracle.build())")
        self.lib = C.CDLL(str(path))
        self.lib.nadmm_ref_last_error.restype = C.c_char_p
        self.lib.nadmm_ref_dataset_free.argtypes = [VP]
        self.lib.nadmm_ref_worker_free.argtypes = [VP]

    @staticmethod
    def available() -> bool:
        return REF_SO.exists()

    def _chk(self, rc: int):
        if rc:
            raise OracleError(rc, self.lib.nadmm_ref_last_error().decode())

    def dataset(self, sh: Shard) -> "RefDataset":
        h = VP()
        if sh.sparse:
            self._chk(self.lib.nadmm_ref_dataset_csr(_lp(sh.indptr), _ip(sh.indices), _dp(sh.vals), C.c_int64(sh.n),
                                                     C.c_int64(sh.p), _ip(sh.labels), C.c_int(sh.C), C.byref(h)))
        else:
            self._chk(self.lib.nadmm_ref_dataset_dense(_dp(sh.X), C.c_int64(sh.n), C.c_int64(sh.p), _ip(sh.labels),
                                                       C.c_int(sh.C), C.byref(h)))
        return RefDataset(self, h, sh)

    def cg_solve(self, apply, g, theta, max_iters):
        g = _f64(g)
        d = len(g)
        cb = APPLY_FN(lambda i, o, n, u: _put(o, n, apply(_get(i, n))))
        p = np.zeros(d)
        it, ach, neg = C.c_int(), C.c_double(), C.c_int()
        self._chk(self.lib.nadmm_ref_cg_solve(cb, None, _dp(g), C.c_int64(d), C.c_double(theta), C.c_int(max_iters),
                                              _dp(p), C.byref(it), C.byref(ach), C.byref(neg)))
        return dict(p=p, iters=it.value, achieved_residual=ach.value, negative_curvature=bool(neg.value))

    def line_search(self, value, x, p, g, f_x, cfg=None):
        x, p, g = _f64(x), _f64(p), _f64(g)
        cb = VALUE_FN(lambda xx, n, u: float(value(np.ctypeslib.as_array(xx, (n,)).copy())))
        a, ev, cap = C.c_double(), C.c_int(), C.c_int()
        self._chk(self.lib.nadmm_ref_line_search(cb, None, _dp(x), _dp(p), _dp(g), C.c_int64(len(x)),
                                                 C.c_double(f_x), _dp(_cfg(cfg)), C.byref(a), C.byref(ev),
                                                 C.byref(cap)))
        return dict(alpha=a.value, evals=ev.value, capped=bool(cap.value))

    def newton_solve_cb(self, value, grad, hvp, x0, cfg=None, trace_cap=64):
        x0 = _f64(x0)
        d = len(x0)
        v = VALUE_FN(lambda x, n, u: float(value(np.ctypeslib.as_array(x, (n,)).copy())))
        gr = GRAD_FN(lambda x, g, n, u: _put(g, n, grad(_get(x, n))))
        hv = HVP_FN(lambda x, vv, o, n, u: _put(o, n, hvp(_get(x, n), _get(vv, n))))
        x = np.zeros(d)
        tr = np.zeros((trace_cap, 9))
        nt, conv, gn = C.c_int(), C.c_int(), C.c_double()
        self._chk(self.lib.nadmm_ref_newton_solve_cb(v, gr, hv, None, _dp(x0), C.c_int64(d), _dp(_cfg(cfg)), _dp(x),
                                                     _dp(tr), C.c_int(trace_cap), C.byref(nt), C.byref(conv),
                                                     C.byref(gn)))
        return dict(x=x, trace=_trace_rows(tr, nt.value), converged=bool(conv.value), final_grad_norm=gn.value)

    def set_threads(self, n: int) -> int:
        """OpenMP threads of the calling host thread (nadmm_ref_set_threads)."""
        return int(self.lib.nadmm_ref_set_threads(C.c_int(int(n))))

    def rng_stream(self, seed, kind, count, bound=0):
        out = np.zeros(count)
        self._chk(self.lib.nadmm_ref_rng_stream(C.c_uint64(seed), C.c_int(kind), C.c_uint64(bound),
                                                C.c_int64(count), _dp(out)))
        return out

    def generate_synthetic(self, n, p, C_, separation=10.0, noise=0.1, seed=0):
        nt = (n * 9) // 10
        Xtr, ytr = np.zeros((nt, p)), np.zeros(nt, dtype=np.int32)
        Xte, yte = np.zeros((n - nt, p)), np.zeros(n - nt, dtype=np.int32)
        self._chk(self.lib.nadmm_ref_generate_synthetic(
            C.c_int64(n), C.c_int64(p), C.c_int(C_), C.c_double(separation), C.c_double(noise), C.c_uint64(seed),
            _dp(Xtr), _ip(ytr), _dp(Xte), _ip(yte)))
        return Xtr, ytr, Xte, yte

    def _loaded(self, h) -> dict:
        """Copy a Dataset returned by the reference's readers out of the heap handle."""
        try:
            n, p, nnz = C.c_int64(), C.c_int64(), C.c_int64()
            c, sp = C.c_int(), C.c_int()
            self._chk(self.lib.nadmm_ref_dataset_info(h, C.byref(n), C.byref(p), C.byref(nnz), C.byref(c), C.byref(sp)))
            out = dict(n=n.value, p=p.value, C=c.value, labels=np.zeros(n.value, dtype=np.int32),
                       label_values=np.zeros(c.value))
            if sp.value:
                out.update(indptr=np.zeros(n.value + 1, dtype=np.int64), indices=np.zeros(nnz.value, dtype=np.int32),
                           vals=np.zeros(nnz.value))
                self._chk(self.lib.nadmm_ref_dataset_fetch(h, _lp(out["indptr"]), _ip(out["indices"]),
                                                           _dp(out["vals"]), _ip(out["labels"]),
                                                           _dp(out["label_values"])))
            else:
                out["X"] = np.zeros((n.value, p.value))
                self._chk(self.lib.nadmm_ref_dataset_fetch(h, None, None, _dp(out["X"]), _ip(out["labels"]),
                                                           _dp(out["label_values"])))
            return out
        finally:
            self.lib.nadmm_ref_dataset_free(h)

    def shuffle(self, seed, n):
        out = np.zeros(n, dtype=np.int64)
        self._chk(self.lib.nadmm_ref_shuffle(C.c_uint64(seed), C.c_int64(n), _lp(out)))
        return out

    def load_libsvm(self, path) -> dict:
        h = VP()
        self._chk(self.lib.nadmm_ref_load_libsvm(str(path).encode(), C.byref(h)))
        return self._loaded(h)

    def load_idx(self, images, labels) -> dict:
        h = VP()
        self._chk(self.lib.nadmm_ref_load_idx(str(images).encode(), str(labels).encode(), C.byref(h)))
        return self._loaded(h)

    def partition_owner(self, n, n_workers, strided=False):
        out = np.zeros(n, dtype=np.int32)
        self._chk(self.lib.nadmm_ref_partition(C.c_int64(n), C.c_int(n_workers), C.c_int(int(strided)), _ip(out)))
        return out


class RefDataset:
    def __init__(self, ref: Ref, handle: VP, sh: Shard):
        self.ref, self.h, self.sh = ref, handle, sh

    def __del__(self):
        try:
            self.ref.lib.nadmm_ref_dataset_free(self.h)
        except Exception:
            pass

    def cache(self, w):
        sh, k = self.sh, self.sh.C - 1
        lg, pr = np.zeros(sh.n * k), np.zeros(sh.n * k)
        rm, al = np.zeros(sh.n), np.zeros(sh.n)
        self.ref._chk(self.ref.lib.nadmm_ref_cache(self.h, _dp(_f64(w)), _dp(lg), _dp(rm), _dp(al), _dp(pr)))
        return lg.reshape(k, sh.n).T, rm, al, pr.reshape(k, sh.n).T

    def loss(self, w, lam=0.0):
        out = C.c_double()
        self.ref._chk(self.ref.lib.nadmm_ref_loss(self.h, _dp(_f64(w)), C.c_double(lam), C.byref(out)))
        return out.value

    def gradient(self, w, lam=0.0):
        g = np.zeros(self.sh.d)
        self.ref._chk(self.ref.lib.nadmm_ref_gradient(self.h, _dp(_f64(w)), C.c_double(lam), _dp(g)))
        return g

    def hessian_vec(self, w, v, lam=0.0):
        hv = np.zeros(self.sh.d)
        self.ref._chk(self.ref.lib.nadmm_ref_hessian_vec(self.h, _dp(_f64(w)), _dp(_f64(v)), C.c_double(lam), _dp(hv)))
        return hv

    def hessian_vec_repeat(self, w, v, lam, reps):
        hv = np.zeros(self.sh.d)
        self.ref._chk(self.ref.lib.nadmm_ref_hessian_vec_repeat(self.h, _dp(_f64(w)), _dp(_f64(v)), C.c_double(lam),
                                                                C.c_int(reps), _dp(hv)))
        return hv

    def predict(self, w):
        out = np.zeros(self.sh.n, dtype=np.int32)
        self.ref._chk(self.ref.lib.nadmm_ref_predict(self.h, _dp(_f64(w)), _ip(out)))
        return out

    def exp_probe(self, w, v):
        out = C.c_double()
        self.ref._chk(self.ref.lib.nadmm_ref_exp_probe(self.h, _dp(_f64(w)), _dp(_f64(v)), C.byref(out)))
        return out.value

    def newton_solve(self, lam, x0, cfg=None, rho=None, z=None, y=None, trace_cap=256):
        d = self.sh.d
        x = np.zeros(d)
        tr = np.zeros((trace_cap, 9))
        nt, conv, gn = C.c_int(), C.c_int(), C.c_double()
        aug = rho is not None
        zz = _f64(z if aug else np.zeros(d))
        yy = _f64(y if aug else np.zeros(d))
        self.ref._chk(self.ref.lib.nadmm_ref_newton_solve(
            self.h, C.c_double(lam), C.c_int(int(aug)), C.c_double(rho or 0.0), _dp(zz), _dp(yy), _dp(_f64(x0)),
            _dp(_cfg(cfg)), _dp(x), _dp(tr), C.c_int(trace_cap), C.byref(nt), C.byref(conv), C.byref(gn)))
        return dict(x=x, trace=_trace_rows(tr, nt.value), converged=bool(conv.value), final_grad_norm=gn.value)

    def lbfgs_solve(self, lam, x0, cfg=(25, 1e-4, 0.9, 100, 20, 1e-8), rho=None, z=None, y=None, trace_cap=1024):
        """The reference's lbfgs_solve (src/lbfgs.cpp:94-181); cfg = (history, c1, c2, max_iters,
        ls_max_iters, grad_tol)."""
        d = self.sh.d
        x = np.zeros(d)
        tr = np.zeros((trace_cap, 6))
        nt, conv, gn = C.c_int(), C.c_int(), C.c_double()
        aug = rho is not None
        zz = _f64(z if aug else np.zeros(d))
        yy = _f64(y if aug else np.zeros(d))
        self.ref._chk(self.ref.lib.nadmm_ref_lbfgs_solve(
            self.h, C.c_double(lam), C.c_int(int(aug)), C.c_double(rho or 0.0), _dp(zz), _dp(yy), _dp(_f64(x0)),
            _dp(_f64(cfg)), _dp(x), _dp(tr), C.c_int(trace_cap), C.byref(nt), C.byref(conv), C.byref(gn)))
        keys = ("iter", "grad_norm", "step", "objective", "fn_evals", "ls_fallback")
        rows = [dict(zip(keys, r.tolist())) for r in tr[: min(nt.value, trace_cap)]]
        return dict(x=x, trace=rows, converged=bool(conv.value), final_grad_norm=gn.value)

    def gradient_subset(self, rows, w, lam=0.0):
        """gradient(data.subset(rows), w, lam) (src/softmax.cpp:80-95; src/dataset.cpp:87-115)."""
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        h = VP()
        self.ref._chk(self.ref.lib.nadmm_ref_subset(self.h, _lp(rows), C.c_int64(len(rows)), C.byref(h)))
        try:
            g = np.zeros(self.sh.d)
            self.ref._chk(self.ref.lib.nadmm_ref_gradient(h, _dp(_f64(w)), C.c_double(lam), _dp(g)))
            return g
        finally:
            self.ref.lib.nadmm_ref_dataset_free(h)

    def worker(self) -> "RefWorker":
        h = VP()
        self.ref._chk(self.ref.lib.nadmm_ref_worker_create(self.h, C.byref(h)))
        return RefWorker(self, h)


class RefWorker:
    """run_worker ADMM branch state (src/worker.cpp:127-196)."""

    def __init__(self, ds: RefDataset, h: VP):
        self.ds, self.h = ds, h

    def __del__(self):
        try:
            self.ds.ref.lib.nadmm_ref_worker_free(self.h)
        except Exception:
            pass

    def solve(self, rho, z, y, cfg=None, inner_iters=1):
        x = np.zeros(self.ds.sh.d)
        st = np.zeros(5)
        self.ds.ref._chk(self.ds.ref.lib.nadmm_ref_worker_solve(self.h, C.c_double(rho), _dp(_f64(z)), _dp(_f64(y)),
                                                                 _dp(_cfg(cfg)), C.c_int(inner_iters), _dp(x), _dp(st)))
        return x, dict(zip(("grad_norm", "inner_iters", "cg_iters", "fn_evals", "flags"), st.tolist()))


class RefAdmm:
    """Newton-ADMM with the REFERENCE's own worker solves (run_worker ADMM branch through
    ``RefWorker``) and the port's coordinator (the reference declares the coordinator in
    inc/admm.hpp:58-140 but ships no implementation, restated in
    nor_admm_run_cb). One ``step()`` = one outer iteration in SPEC order: scatter ->
    solves -> z-update -> y-hat / y-update -> residuals / tolerances -> spectral penalty -> metrics.

    ``workers_parallel``: the workers' solves run on one host thread each, like the reference's
    WorkerPool (src/worker.cpp:225-242); ``threads_per_worker`` OpenMP threads each (the Eigen
    stand-in's GEMM loops). ctypes releases the GIL during the calls.
    """

    def __init__(self, ref: "Ref", shards, cfg: NorAdmmCfg, workers_parallel: bool = True,
                 threads_per_worker: int | None = None, eval_objective: bool = False):
        import concurrent.futures as cf

        self.ref, self.cfg, self.port = ref, cfg, Port()
        self.N = cfg.n_workers
        assert len(shards) == self.N
        self.shards = shards
        self.ds = [ref.dataset(s) for s in shards]
        self.workers = [ds.worker() for ds in self.ds]
        self.d = shards[0].d
        N, d = self.N, self.d
        self.x, self.y, self.yh = np.zeros((N, d)), np.zeros((N, d)), np.zeros((N, d))
        self.z, self.rho = np.zeros(d), np.full(N, cfg.rho0)
        self.xs, self.ys, self.yhs, self.zs = np.zeros((N, d)), np.zeros((N, d)), np.zeros((N, d)), np.zeros(d)
        self.k, self.snap_it, self.converged = 0, 0, False
        self.newton = list(cfg.newton)
        self.eval_objective = eval_objective
        self.metrics = []
        self.hv = 0  # Hessian-vector products applied (CG + certificate), as the GPU counts them
        self.solve_seconds = 0.0  # wall time inside the workers' solves
        cores = os.cpu_count() or 1
        self.tpw = threads_per_worker or (max(1, cores // N) if workers_parallel else cores)
        self.pool = cf.ThreadPoolExecutor(N) if workers_parallel else None
        if not workers_parallel:
            ref.set_threads(self.tpw)

    def _solve(self, i):
        if self.pool is not None:
            self.ref.set_threads(self.tpw)
        return self.workers[i].solve(self.rho[i], self.z, self.y[i], cfg=self.newton,
                                     inner_iters=self.cfg.inner_iters)

    def objective(self, z) -> float:
        """F(z) = sum_i loss(D_i, z) + (lambda/2)|z|^2 (port_fval: global objective of Eq. (5))."""
        return sum(ds.loss(z, 0.0) for ds in self.ds) + 0.5 * self.cfg.lam * float(np.dot(z, z))

    def step(self) -> dict:
        import time

        cfg, P, N, d = self.cfg, self.port, self.N, self.d
        t0 = time.perf_counter()
        if self.pool is not None:
            res = list(self.pool.map(self._solve, range(N)))
        else:
            res = [self._solve(i) for i in range(N)]
        self.solve_seconds += time.perf_counter() - t0
        inner = cg = fe = flags = 0
        for i, (xi, st) in enumerate(res):
            self.x[i] = xi
            inner += int(st["inner_iters"])
            cg += int(st["cg_iters"])
            fe += int(st["fn_evals"])
            flags |= int(st["flags"])
        self.hv += cg + inner
        pz = self.z.copy()
        self.z = P.z_update(self.x, self.y, self.rho, cfg.lam)
        self.yh = self.y + self.rho[:, None] * (pz[None, :] - self.x)
        self.y = P.y_update(self.y, self.x, self.z, self.rho)
        self.k += 1
        pr, du, pt, dt = P.residuals(self.x, self.z, pz, self.rho)
        ep, ed = P.tolerances(self.x, self.y, self.z, cfg.eps_abs, cfg.eps_rel, bool(cfg.standard_norms))
        self.converged = bool(np.all(pr <= ep) and np.all(du <= ed))
        if cfg.penalty_kind == 1 and self.k - self.snap_it >= cfg.update_period:
            for i in range(N):
                self.rho[i] = P.spectral_rho(self.x[i] - self.xs[i], self.yh[i] - self.yhs[i], self.z - self.zs,
                                             self.y[i] - self.ys[i], self.rho[i], cfg.eps_cor, cfg.rho_min,
                                             cfg.rho_max)[0]
            self.xs, self.ys, self.yhs, self.zs = self.x.copy(), self.y.copy(), self.yh.copy(), self.z.copy()
            self.snap_it = self.k
        row = dict(iteration=self.k, train_objective=self.objective(self.z) if self.eval_objective else float("nan"),
                   primal_norm=pt, dual_norm=dt, eps_pri=ep, eps_dual=ed, inner_iterations=inner, cg_iters=cg,
                   fn_evals=fe, flags=flags, rho_mean=float(np.mean(self.rho)))
        self.metrics.append(row)
        return row

    def close(self):
        if self.pool is not None:
            self.pool.shutdown()


def port() -> Port:
    return Port()


def ref() -> Ref | None:
    return Ref() if Ref.available() else None
