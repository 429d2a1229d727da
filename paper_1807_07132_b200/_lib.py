"""ctypes binding of include/nadmm_cuda.h (the C ABI of lib/libnadmm_cuda.so).

The shared library is the product: every compute call below runs sm_100a kernels. There is no CPU
fallback -- a missing library or a missing GPU raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("NADMM_LIB", PKG / "lib" / "libnadmm_cuda.so"))

D = C.POINTER(C.c_double)
I32 = C.POINTER(C.c_int32)
I64 = C.POINTER(C.c_int64)
VP = C.c_void_p


class NewtonCfg(C.Structure):  # nadmm_newton_cfg == NewtonConfig (inc/newton.hpp:9-17)
    _fields_ = [("cg_tol", C.c_double), ("cg_max_iters", C.c_int32), ("armijo_beta", C.c_double),
                ("backtrack_gamma", C.c_double), ("ls_max_iters", C.c_int32), ("grad_tol", C.c_double),
                ("newton_max_iters", C.c_int32)]


class NewtonIter(C.Structure):  # NewtonIterRecord (inc/newton.hpp:47-57)
    _fields_ = [("iter", C.c_int32), ("grad_norm", C.c_double), ("step", C.c_double), ("cg_iters", C.c_int32),
                ("cg_residual", C.c_double), ("objective", C.c_double), ("ls_capped", C.c_int32),
                ("cg_fallback", C.c_int32), ("fn_evals", C.c_int32)]


class NewtonSummary(C.Structure):
    _fields_ = [("converged", C.c_int32), ("final_grad_norm", C.c_double), ("iterations", C.c_int32)]


class LbfgsCfg(C.Structure):  # nadmm_lbfgs_cfg == LbfgsConfig (inc/lbfgs.hpp:9-18)
    _fields_ = [("history", C.c_int32), ("wolfe_c1", C.c_double), ("wolfe_c2", C.c_double),
                ("max_iters", C.c_int32), ("ls_max_iters", C.c_int32), ("grad_tol", C.c_double)]


class LbfgsIter(C.Structure):  # LbfgsIterRecord (inc/lbfgs.hpp:20-27)
    _fields_ = [("iter", C.c_int32), ("grad_norm", C.c_double), ("step", C.c_double), ("objective", C.c_double),
                ("fn_evals", C.c_int32), ("ls_fallback", C.c_int32)]


class SgdCfg(C.Structure):  # nadmm_sgd_cfg: SgdConfig + the worker session's SGD keys
    _fields_ = [("eta", C.c_double), ("batch", C.c_int32), ("epochs", C.c_int32), ("steps_per_epoch", C.c_int32),
                ("seed", C.c_uint64)]


class InnerStats(C.Structure):  # InnerStats (inc/comm.hpp:67-73)
    _fields_ = [("grad_norm", C.c_double), ("inner_iters", C.c_uint32), ("cg_iters", C.c_uint32),
                ("fn_evals", C.c_uint32), ("flags", C.c_uint32)]


class Stats(C.Structure):
    _fields_ = [("kernel_launches", C.c_int64), ("hv_products", C.c_int64), ("data_passes", C.c_int64),
                ("hv_kernel_ms", C.c_double), ("hv_kernel_samples", C.c_int64), ("hv_kernel_shards", C.c_int64)]


class AdmmCfg(C.Structure):  # AdmmConfig + PenaltyPolicy + StoppingConfig (inc/admm.hpp:37-117)
    _fields_ = [("lam", C.c_double), ("penalty_kind", C.c_int32), ("rho0", C.c_double), ("update_period", C.c_int32),
                ("eps_cor", C.c_double), ("rho_min", C.c_double), ("rho_max", C.c_double),
                ("eps_abs", C.c_double), ("eps_rel", C.c_double), ("max_outer_iters", C.c_int32),
                ("standard_norms", C.c_int32), ("inner_iters", C.c_int32), ("newton", NewtonCfg),
                ("eval_objective", C.c_int32), ("f_star", C.c_double), ("theta_stop", C.c_double),
                ("ignore_convergence", C.c_int32), ("inner_solver", C.c_int32), ("lbfgs", LbfgsCfg),
                ("consensus_tree", C.c_int32)]


class MetricsRow(C.Structure):  # MetricsRow (inc/metrics.hpp:15-27)
    _fields_ = [("iteration", C.c_int32), ("wall_seconds", C.c_double), ("train_objective", C.c_double),
                ("theta", C.c_double), ("primal_norm", C.c_double), ("dual_norm", C.c_double),
                ("eps_pri", C.c_double), ("eps_dual", C.c_double), ("inner_iterations", C.c_int32),
                ("cg_iters", C.c_int32), ("fn_evals", C.c_int32), ("flags", C.c_int32), ("rho_mean", C.c_double),
                ("messages", C.c_int64)]


# Every symbol include/nadmm_cuda.h declares, with (restype, argtypes).
S = C.c_int  # nadmm_status
SIGNATURES = {
    "nadmm_last_error": (C.c_char_p, []),
    "nadmm_abi_version": (C.c_int32, []),
    "nadmm_ctx_create": (S, [C.c_int32, C.POINTER(VP)]),
    "nadmm_ctx_destroy": (S, [VP]),
    "nadmm_ctx_synchronize": (S, [VP]),
    "nadmm_ctx_stream": (VP, [VP]),
    "nadmm_ctx_stats": (S, [VP, C.POINTER(Stats)]),
    "nadmm_ctx_reset_stats": (S, [VP]),
    "nadmm_ctx_set_timing": (S, [VP, C.c_int32]),
    "nadmm_shard_dense": (S, [VP, D, C.c_int64, C.c_int64, I32, C.c_int32, C.POINTER(VP)]),
    "nadmm_shard_csr": (S, [VP, I64, I32, D, C.c_int64, C.c_int64, I32, C.c_int32, C.POINTER(VP)]),
    "nadmm_shard_free": (S, [VP]),
    "nadmm_shard_info": (S, [VP, I64, I64, I32, I32]),
    "nadmm_shard_device_bytes": (C.c_int64, [VP]),
    "nadmm_cache": (S, [VP, D, D, D, D, D]),
    "nadmm_loss": (S, [VP, D, C.c_double, D]),
    "nadmm_gradient": (S, [VP, D, C.c_double, D]),
    "nadmm_hessian_vec": (S, [VP, D, D, C.c_double, D]),
    "nadmm_predict": (S, [VP, D, I32]),
    "nadmm_accuracy": (S, [VP, D, D]),
    "nadmm_set_point_dev": (S, [VP, VP]),
    "nadmm_hessian_vec_dev": (S, [VP, VP, C.c_double, VP]),
    "nadmm_newton_cfg_default": (None, [C.POINTER(NewtonCfg)]),
    "nadmm_lbfgs_cfg_default": (None, [C.POINTER(LbfgsCfg)]),
    "nadmm_lbfgs_solve": (S, [VP, C.POINTER(LbfgsCfg), C.c_double, C.c_int32, C.c_double, D, D, D,
                              C.POINTER(LbfgsIter), C.c_int32, C.POINTER(NewtonSummary)]),
    "nadmm_newton_solve": (S, [VP, C.POINTER(NewtonCfg), C.c_double, C.c_int32, C.c_double, D, D, D,
                               C.POINTER(NewtonIter), C.c_int32, C.POINTER(NewtonSummary)]),
    "nadmm_ctx_node_streams": (C.c_int32, [VP]),
    "nadmm_worker_create": (S, [VP, C.POINTER(VP)]),
    "nadmm_workers_solve": (S, [C.POINTER(VP), C.c_int32, D, D, C.POINTER(D), C.POINTER(NewtonCfg), C.c_int32,
                                C.POINTER(D), C.POINTER(InnerStats)]),
    "nadmm_worker_sgd_grad": (S, [VP, C.POINTER(SgdCfg), C.c_uint32, D, D, C.POINTER(InnerStats)]),
    "nadmm_sgd_permutation": (S, [C.c_uint64, C.c_uint32, C.c_int64, I32]),
    "nadmm_sgd_run": (S, [C.POINTER(VP), C.c_int32, VP, C.POINTER(SgdCfg), C.c_double, D, C.POINTER(MetricsRow),
                          C.c_int32, C.POINTER(C.c_int32)]),
    "nadmm_worker_solve_lbfgs": (S, [VP, C.c_double, D, D, C.POINTER(LbfgsCfg), C.c_int32, D,
                                     C.POINTER(InnerStats)]),
    "nadmm_worker_free": (S, [VP]),
    "nadmm_worker_solve": (S, [VP, C.c_double, D, D, C.POINTER(NewtonCfg), C.c_int32, D, C.POINTER(InnerStats)]),
    "nadmm_comm_unique_id": (S, [C.POINTER(C.c_uint8)]),
    "nadmm_comm_create": (S, [VP, C.POINTER(C.c_uint8), C.c_int32, C.c_int32, C.POINTER(VP)]),
    "nadmm_comm_destroy": (S, [VP]),
    "nadmm_admm_cfg_default": (None, [C.POINTER(AdmmCfg)]),
    "nadmm_admm_run": (S, [C.POINTER(VP), C.c_int32, VP, C.POINTER(AdmmCfg), D, D, C.POINTER(MetricsRow),
                           C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "nadmm_admm_create": (S, [C.POINTER(VP), C.c_int32, VP, C.POINTER(AdmmCfg), C.POINTER(VP)]),
    "nadmm_admm_step": (S, [VP, C.c_int32, C.POINTER(MetricsRow), C.c_int32, C.POINTER(C.c_int32),
                            C.POINTER(C.c_int32)]),
    "nadmm_admm_result": (S, [VP, D, D, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "nadmm_admm_free": (S, [VP]),
    "nadmm_data_last_error": (C.c_char_p, []),
    "nadmm_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "nadmm_generate_synthetic": (S, [C.c_int64, C.c_int64, C.c_int32, C.c_double, C.c_double, C.c_uint64, D, I32,
                                     D, I32]),
    "nadmm_generate_sparse": (S, [C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_uint64, I64, I32, D, I32]),
    "nadmm_partition": (S, [C.c_int64, C.c_int32, C.c_int32, I32]),
    "nadmm_libsvm_parse": (S, [C.c_char_p, C.POINTER(VP), I64, I64, I64, I32]),
    "nadmm_libsvm_fetch": (S, [VP, I64, I32, D, I32, D]),
    "nadmm_libsvm_free": (None, [VP]),
    "nadmm_idx_info": (S, [C.c_char_p, C.c_char_p, I64, I64]),
    "nadmm_idx_load": (S, [C.c_char_p, C.c_char_p, D, I32, I32, D]),
    "nadmm_hcoord_create": (S, [C.c_int64, C.c_int32, C.c_double, C.c_int32, C.c_double, C.c_int32, C.c_double,
                                C.c_double, C.c_double, C.c_int32, C.POINTER(VP)]),
    "nadmm_hcoord_sum": (S, [VP, C.POINTER(D), C.POINTER(D), D]),
    "nadmm_hcoord_update": (S, [VP, C.POINTER(D), C.POINTER(D), D, D, D]),
    "nadmm_hcoord_free": (S, [VP]),
    "nadmm_hcoord_last_error": (C.c_char_p, []),
}

_lib = None


def _preload_nccl() -> None:
    """Bind libnccl.so.2 to the newest NCCL in the environment before our library resolves it.

    The library links against the libnccl.so.2 soname. When PyTorch is in the process it needs its
    own (newer) NCCL; loading the system copy first would break a later `import torch`. Preloading the
    wheel's NCCL (RTLD_GLOBAL) makes both resolve to one, ABI-compatible, copy."""
    import importlib.util

    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    if not spec or not spec.submodule_search_locations:
        return
    for loc in spec.submodule_search_locations:
        cand = Path(loc) / "lib" / "libnccl.so.2"
        if cand.exists():
            try:
                C.CDLL(str(cand), mode=C.RTLD_GLOBAL)
            except OSError:
                pass
            return


def lib() -> C.CDLL:
    """Load the CUDA library (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        _preload_nccl()
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} missing: build it with paper_1807_07132_b200/build.sh "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
