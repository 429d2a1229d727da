"""CPU tests of the product boundary (no GPU): the C-ABI library loads, exports every symbol the
headers in include/ declare, refuses to compute without a GPU (no CPU fallback), and its host-only
data fixtures reproduce the reference generator byte for byte."""
import re
from pathlib import Path

import numpy as np
import pytest

import oracle

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        for m in re.finditer(r"^\s*(?:const\s+)?[\w\s\*]+?\b(nadmm_\w+)\s*\(", h.read_text(), re.M):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol(nadmm):
    lib = nadmm._lib.lib()
    declared = declared_symbols()
    assert len(declared) >= 40
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, f"missing exports: {missing}"
    assert set(nadmm._lib.SIGNATURES) == declared, "ctypes signature table out of sync with include/nadmm_cuda.h"


def test_abi_version(nadmm):
    assert nadmm._lib.lib().nadmm_abi_version() == 1


def test_no_cpu_fallback_without_gpu(nadmm):
    from conftest import gpu_available

    if gpu_available():
        pytest.skip("GPU present")
    with pytest.raises(nadmm.CudaError):
        nadmm.Context(0)


def test_data_fixtures_match_reference_generator(nadmm, port):
    for args in ((100, 5, 3, 10.0, 0.1, 0), (555, 31, 10, 3.0, 1.0, 7)):
        for a, b in zip(nadmm.generate_synthetic(*args), port.generate_synthetic(*args)):
            np.testing.assert_array_equal(a, b)
    r = oracle.ref()
    if r is not None:
        for a, b in zip(nadmm.generate_synthetic(120, 4, 3, 3.0, 1.0, 5), r.generate_synthetic(120, 4, 3, 3.0, 1.0, 5)):
            np.testing.assert_array_equal(a, b)
    for a, b in zip(nadmm.generate_sparse(40, 300, 20, 15, 3), port.generate_sparse(40, 300, 20, 15, 3)):
        np.testing.assert_array_equal(a, b)
    ip, ix, vv, y = nadmm.generate_sparse(40, 300, 20, 15, 3)
    assert np.all(np.diff(ip) == 15) and np.all(y == np.arange(40) % 20 + 1)
    for i in range(40):
        cols = ix[ip[i]:ip[i + 1]]
        assert np.all(np.diff(cols) > 0)
        assert abs(np.linalg.norm(vv[ip[i]:ip[i + 1]]) - 1.0) < 1e-12
    assert nadmm.mix_seed(0, 3) == port.mix_seed(0, 3)


def test_partition_matches(nadmm, port):
    for n, N, s in ((10, 3, False), (101, 8, False), (17, 4, True)):
        np.testing.assert_array_equal(nadmm.partition_owner(n, N, s), port.partition_owner(n, N, s))
    with pytest.raises(nadmm.ConfigError):
        nadmm.partition_owner(3, 4)


def test_config_defaults_mirror_reference(nadmm):
    c = nadmm.NewtonConfig()  # inc/newton.hpp:9-17
    assert (c.cg_tol, c.cg_max_iters, c.armijo_beta, c.backtrack_gamma, c.ls_max_iters, c.grad_tol,
            c.newton_max_iters) == (1e-4, 10, 1e-4, 0.5, 10, 1e-8, 100)
    a = nadmm.AdmmConfig()  # inc/admm.hpp:37-56, 107-117
    assert (a.n_workers, a.lam, a.inner_iters) == (4, 1e-5, 1)
    assert (a.penalty.rho0, a.penalty.update_period, a.penalty.eps_cor, a.penalty.rho_min, a.penalty.rho_max) == (
        1.0, 2, 0.2, 1e-6, 1e6)
    assert (a.stopping.eps_abs, a.stopping.eps_rel, a.stopping.max_outer_iters) == (1e-3, 1e-3, 300)
    cc = a.to_c()
    assert cc.newton.cg_max_iters == 10 and cc.max_outer_iters == 300
