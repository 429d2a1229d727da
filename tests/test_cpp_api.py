"""The C++ host side: include/nadmm_cuda.hpp (the reference-shaped API over the C ABI) compiles and
links with g++ against the library; without a GPU the program gets the library's CudaError (no CPU
fallback); on a GPU its results equal the Python API's on the same inputs."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_1807_07132_b200" / "lib"


def _build(tmp_path):
    exe = tmp_path / "abi_example"
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Werror", f"-I{ROOT / 'include'}",
                    str(ROOT / "tests" / "cpp" / "abi_example.cpp"), f"-L{LIBDIR}", "-lnadmm_cuda",
                    f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    return exe


def _run(exe):
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    return r.returncode, json.loads(line)


def test_cpp_wrapper_builds_and_reports_no_gpu(tmp_path):
    from conftest import gpu_available

    exe = _build(tmp_path)
    if gpu_available():
        pytest.skip("GPU present: covered by test_cpp_matches_python")
    rc, out = _run(exe)
    assert rc == 3 and out["error"] == "CudaError"


@pytest.mark.gpu
def test_cpp_matches_python(tmp_path, nadmm):
    rc, out = _run(_build(tmp_path))
    assert rc == 0, out
    Xtr, ytr, _, _ = nadmm.generate_synthetic(1111, 30, 4, 2.0, 1.0, 7)
    ds = nadmm.Dataset.dense(Xtr, ytr, 4)
    d = ds.weight_dim()
    j = np.arange(d)
    w = 0.01 * ((j * 37) % 11 - 5).astype(float)
    v = ((j * 13) % 7 - 3).astype(float)
    assert out["loss"] == nadmm.loss(ds, w, 1e-3)
    assert out["hv_sum"] == pytest.approx(float(np.sum(nadmm.hessian_vec(ds, w, v, 1e-3))), rel=1e-12)
    res = nadmm.newton_solve(nadmm.make_softmax_objective(ds, 1e-3), np.zeros(d), nadmm.NewtonConfig(newton_max_iters=3))
    assert out["newton_iters"] == len(res.trace)
    assert out["newton_x_sum"] == pytest.approx(float(np.sum(res.x)), rel=1e-12)
    half = len(ytr) // 2
    parts = [nadmm.Dataset.dense(Xtr[:half], ytr[:half], 4), nadmm.Dataset.dense(Xtr[half:], ytr[half:], 4)]
    ar = nadmm.run_admm(parts, nadmm.AdmmConfig(n_workers=2, lam=1e-3,
                                                stopping=nadmm.StoppingConfig(max_outer_iters=8)))
    assert out["admm_iters"] == ar.iterations
    assert out["admm_z_sum"] == pytest.approx(float(np.sum(ar.z)), rel=1e-12)
    assert out["accuracy"] == nadmm.accuracy(nadmm.predict(parts[0], ar.z), ytr[:half])
