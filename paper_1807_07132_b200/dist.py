"""Multi-process plumbing of the N-GPU consensus loop (one process per GPU) and the
host-side consensus coordinator of the worker-transport deployment.

The device-resident loop (`run_admm` / `AdmmSession` with a `Communicator`) does its exchange with
one NCCL allreduce inside the library. This module holds the host-side pieces around it:

* `node_range` — which ADMM nodes (contiguous row shards, src/data_io.cpp:300-328) a rank owns.
* `share_unique_id` — ship rank 0's NCCL id to every rank over an existing torch.distributed group.
* `NativeHostCoordinator` — the reference's coordinator over HOST buffers (the library's
  `nadmm_hcoord_*`), for callers that drive the workers through `workers_solve` / `Worker.solve`
  (nadmm_worker_solve) themselves, as the reference's coordinator drives its workers through frames
  (inc/admm.hpp:58-140): z = (Σ_i ρ_i x_i − y_i) / (λ + Σ_i ρ_i),
  ŷ_i = y_i + ρ_i (z_prev − x_i), y_i += ρ_i (z − x_i), and spectral penalty selection every T_f
  iterations. With several processes the local sums are combined by one allreduce
  of [Σ(ρx−y) | Σρ] (`allreduce` callback, e.g. `torch_allreduce` over gloo or an NCCL staging
  copy); SPS needs nothing global beyond z.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np


def node_range(n_nodes: int, world: int, rank: int) -> range:
    """Contiguous block of ADMM node ids owned by `rank` (n_nodes must be a multiple of world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if n_nodes % world:
        raise ValueError(f"{n_nodes} ADMM nodes do not split over {world} ranks")
    per = n_nodes // world
    return range(rank * per, (rank + 1) * per)


def share_unique_id(dist, rank: int, make_id: Callable[[], bytes]) -> bytes:
    """Rank 0 creates the communicator id; every rank returns the same bytes."""
    box = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    return box[0]


class NativeHostCoordinator:
    """Consensus coordinator for this rank's `n_local` nodes, run by the library's host code
    (nadmm_hcoord_*: two fused OpenMP sweeps per round over caller-owned buffers, no GPU needed).
    State (AdmmState::initial): z = 0, y_i = 0, rho_i = rho0. `X` and `y` are
    (n_local, d) float64 arrays (e.g. pinned); `y` is updated in place; `allreduce(buf)` sums the
    (d + 1)-long consensus buffer over processes when there are several."""

    def __init__(self, d: int, lam: float, n_local: int = 1, penalty: str = "fixed", rho0: float = 1.0,
                 update_period: int = 2, eps_cor: float = 0.2, rho_min: float = 1e-6, rho_max: float = 1e6,
                 allreduce: Optional[Callable[[np.ndarray], None]] = None, y: Optional[np.ndarray] = None,
                 threads: int = 8):
        import ctypes as C

        from . import _lib as L

        if penalty not in ("fixed", "spectral"):
            raise ValueError(f"unknown penalty {penalty!r}")
        self._C, self._L = C, L
        self.d, self.n, self.allreduce = d, n_local, allreduce
        self.y = y if y is not None else np.zeros((n_local, d))
        self.y[:] = 0.0
        self.z = np.zeros(d)
        self.rho = np.full(n_local, float(rho0))
        self._S = np.zeros(d + 1)
        h = C.c_void_p()
        rc = L.lib().nadmm_hcoord_create(d, n_local, lam, 1 if penalty == "spectral" else 0, rho0, update_period,
                                         eps_cor, rho_min, rho_max, threads, C.byref(h))
        if rc:
            raise ValueError(L.lib().nadmm_hcoord_last_error().decode())
        self._h = h
        D = L.D
        self._yp = (D * n_local)(*[row.ctypes.data_as(D) for row in self.y])

    def _ptrs(self, X):
        D = self._L.D
        return (D * self.n)(*[row.ctypes.data_as(D) for row in X])

    def step(self, X: np.ndarray) -> np.ndarray:
        L, D = self._L, self._L.D
        xp = self._ptrs(X)
        rc = L.lib().nadmm_hcoord_sum(self._h, xp, self._yp, self._S.ctypes.data_as(D))
        if rc:
            raise ValueError(L.lib().nadmm_hcoord_last_error().decode())
        if self.allreduce is not None:
            self.allreduce(self._S)
        rc = L.lib().nadmm_hcoord_update(self._h, xp, self._yp, self._S.ctypes.data_as(D), self.z.ctypes.data_as(D),
                                         self.rho.ctypes.data_as(D))
        if rc:
            raise ValueError(L.lib().nadmm_hcoord_last_error().decode())
        return self.z

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.lib().nadmm_hcoord_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def torch_allreduce(dist, group=None) -> Callable[[np.ndarray], None]:
    """allreduce callback over a torch.distributed group (gloo on CPU tensors)."""
    import torch

    def f(buf: np.ndarray) -> None:
        t = torch.from_numpy(buf)
        dist.all_reduce(t, group=group)

    return f
