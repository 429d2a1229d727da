"""N > 1 host logic on CPU: world_size-2 gloo process groups (127.0.0.1) drive the rank plumbing of
the multi-GPU consensus loop (paper_1807_07132_b200/dist.py) and must reproduce the single-process
coordinator and the oracle's z/y updates."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1807_07132_b200 import dist as nd

NODES, D, LAM = 4, 37, 1e-3


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
        co = nd.HostCoordinator(D, LAM, nd.torch_allreduce(dist))
        my_y = [ys[i].copy() for i in mine]
        zs = []
        for step in range(3):  # three consensus rounds with fixed x (only z/y evolve)
            zs.append(co.step([xs[i] for i in mine], my_y, [rhos[i] for i in mine]).copy())
        out[rank] = {"nodes": list(mine), "uid": uid, "z": zs, "y": my_y}
    finally:
        dist.destroy_process_group()


def test_node_range():
    assert list(nd.node_range(8, 2, 1)) == [4, 5, 6, 7]
    assert list(nd.node_range(8, 8, 3)) == [3]
    with pytest.raises(ValueError):
        nd.node_range(8, 3, 0)


def test_world2_coordinator_matches_single_process(port):
    world = 2
    out = mp.Manager().dict()
    p = _free_port()
    mp.start_processes(_worker, args=(world, p, out), nprocs=world, join=True, start_method="spawn")
    xs, ys, rhos = _fixture()
    co = nd.HostCoordinator(D, LAM)
    y1 = [y.copy() for y in ys]
    zs1 = [co.step(xs, y1, rhos).copy() for _ in range(3)]
    assert out[0]["uid"] == out[1]["uid"] == bytes(range(128))
    assert out[0]["nodes"] + out[1]["nodes"] == list(range(NODES))
    for r in range(world):
        for za, zb in zip(out[r]["z"], zs1):
            np.testing.assert_allclose(za, zb, rtol=1e-14, atol=1e-15)
    y2 = list(out[0]["y"]) + list(out[1]["y"])
    for a, b in zip(y2, y1):
        np.testing.assert_allclose(a, b, rtol=1e-14, atol=1e-15)
    # the oracle's z_update / y_update (ascending-id pairwise tree) on the first round
    y0 = [y.copy() for y in ys]
    z_or = port.z_update(xs, y0, rhos, LAM)
    np.testing.assert_allclose(zs1[0], z_or, rtol=1e-13, atol=1e-15)
