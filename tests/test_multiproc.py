"""N > 1 host logic on CPU: world_size-2 gloo process groups (127.0.0.1) drive the rank plumbing of
the multi-GPU consensus loop (paper_1807_07132_b200/dist.py) and the library's host coordinator
(nadmm_hcoord_*, the bench's e2e coordinator), which must reproduce the single-process run, the
oracle's z/y updates and the torch restatement in tests/coord_ref.py."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1807_07132_b200 import dist as nd

import coord_ref

NODES, D, LAM, STEPS = 4, 37, 1e-3, 5


def _x(i, step):
    return np.random.default_rng(100 * i + step).normal(size=D) * (1.0 + 0.1 * step)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fixture(seed=0):
    rng = np.random.default_rng(seed)
    xs = [rng.normal(size=D) for _ in range(NODES)]
    ys = [rng.normal(size=D) * 0.1 for _ in range(NODES)]
    rhos = [1.0, 0.5, 2.0, 1.5]
    return xs, ys, rhos


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = nd.node_range(NODES, world, rank)
        uid = nd.share_unique_id(dist, rank, lambda: bytes(range(128)))
        xs, ys, rhos = _fixture()
        co = nd.NativeHostCoordinator(D, LAM, len(mine), penalty="spectral", allreduce=nd.torch_allreduce(dist),
                                      threads=2)
        co.y[:] = [ys[i] for i in mine]
        zs = []
        for step in range(STEPS):  # consensus rounds on a fixed x trajectory (z / y / rho evolve)
            zs.append(co.step(np.stack([_x(i, step) for i in mine])).copy())
        out[rank] = {"nodes": list(mine), "uid": uid, "z": zs, "y": co.y.copy(), "rho": co.rho.copy()}
        co.close()
    finally:
        dist.destroy_process_group()


def test_node_range():
    assert list(nd.node_range(8, 2, 1)) == [4, 5, 6, 7]
    assert list(nd.node_range(8, 8, 3)) == [3]
    with pytest.raises(ValueError):
        nd.node_range(8, 3, 0)


def _single(xs_rows, ys):
    co = nd.NativeHostCoordinator(D, LAM, NODES, penalty="spectral", threads=2)
    co.y[:] = ys
    zs = [co.step(np.stack([_x(i, s) for i in range(NODES)])).copy() for s in range(STEPS)]
    return co, zs


def test_world2_coordinator_matches_single_process(port):
    world = 2
    out = mp.Manager().dict()
    p = _free_port()
    mp.start_processes(_worker, args=(world, p, out), nprocs=world, join=True, start_method="spawn")
    xs, ys, rhos = _fixture()
    co, zs1 = _single(xs, ys)
    assert out[0]["uid"] == out[1]["uid"] == bytes(range(128))
    assert out[0]["nodes"] + out[1]["nodes"] == list(range(NODES))
    for r in range(world):
        for za, zb in zip(out[r]["z"], zs1):
            np.testing.assert_allclose(za, zb, rtol=1e-14, atol=1e-15)
    y2 = np.concatenate([out[0]["y"], out[1]["y"]])
    np.testing.assert_allclose(y2, co.y, rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(np.concatenate([out[0]["rho"], out[1]["rho"]]), co.rho, rtol=1e-14)


def test_host_coordinator_matches_oracle_coordinator(port):
    """The library's host coordinator's z / y-hat / y / spectral-penalty sequence against the oracle's
    coordinator pieces (nor_z_update pairwise tree, nor_y_update, nor_spectral_rho)."""
    xs, ys, rhos = _fixture()
    co, zs1 = _single(xs, ys)
    z, y, rho = np.zeros(D), np.array(ys), np.ones(NODES)
    snap = None
    for s in range(STEPS):
        X = np.stack([_x(i, s) for i in range(NODES)])
        pz = z
        z = port.z_update(X, y, rho, LAM)
        yh = y + rho[:, None] * (pz[None, :] - X)
        y = port.y_update(y, X, z, rho)
        k = s + 1
        if snap is None:
            snap = (np.zeros((NODES, D)), np.zeros((NODES, D)), np.zeros((NODES, D)), np.zeros(D), 0)
        xs_, ys_, yhs_, zs_, it = snap
        if k - it >= 2:
            rho = np.array([port.spectral_rho(X[i] - xs_[i], yh[i] - yhs_[i], z - zs_, y[i] - ys_[i], rho[i])[0]
                            for i in range(NODES)])
            snap = (X.copy(), y.copy(), yh.copy(), z.copy(), k)
        np.testing.assert_allclose(zs1[s], z, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(co.y, y, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(co.rho, rho, rtol=1e-12)
    assert not np.allclose(rho, 1.0)  # the spectral update actually fired


@pytest.mark.parametrize("penalty", ["fixed", "spectral"])
def test_native_host_coordinator_matches(penalty, port):
    """nadmm_hcoord_* (the library's fused host coordinator) against the torch restatement
    (tests/coord_ref.py): z, y and rho over several rounds (sums in different orders: 1e-12)."""
    xs, ys, rhos = _fixture()
    a = coord_ref.HostCoordinator(D, LAM, NODES, penalty=penalty)
    b = nd.NativeHostCoordinator(D, LAM, NODES, penalty=penalty, threads=3)
    a.y[:] = ys
    b.y[:] = ys
    for s in range(STEPS + 2):
        X = np.stack([_x(i, s) for i in range(NODES)])
        za = a.step(X).copy()
        zb = b.step(X).copy()
        np.testing.assert_allclose(zb, za, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(b.y, a.y, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(b.rho, a.rho, rtol=1e-12)
    if penalty == "spectral":
        assert not np.allclose(b.rho, 1.0)
    b.close()


def test_spectral_rho_matches_oracle(port):
    rng = np.random.default_rng(5)
    for trial in range(40):
        a, b, c, d = (rng.normal(size=D) for _ in range(4))
        if trial % 3 == 0:
            b = a * 2.0 + 0.1 * b  # correlated x-side
        if trial % 4 == 0:
            d = -c * 0.5 + 0.05 * d  # correlated z-side
        want = port.spectral_rho(a, b, c, d, 1.3)[0]
        assert abs(coord_ref.spectral_rho(a, b, c, d, 1.3) - want) <= 1e-12 * abs(want)
