"""Multi-process plumbing of the N-GPU consensus loop (one process per GPU).

The device-resident loop (`run_admm` / `AdmmSession` with a `Communicator`) does its exchange with
one NCCL allreduce inside the library. This module holds the host-side pieces around it:

* `node_range` — which ADMM nodes (contiguous row shards, src/data_io.cpp:300-328) a rank owns.
* `share_unique_id` — ship rank 0's NCCL id to every rank over an existing torch.distributed group.
* `HostCoordinator` — the reference-facing consensus step over HOST buffers, for callers that drive
  `Worker.solve` (nadmm_worker_solve) themselves, as the reference's coordinator drives its workers
  through frames: z = (Σ_i ρ_i x_i − y_i) / (λ + Σ_i ρ_i), then y_i += ρ_i (z − x_i).
  With a process group the local sums are combined by one allreduce of [Σ(ρx−y) | Σρ].
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

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


class HostCoordinator:
    """Consensus z/y update over host vectors (one per local node), optionally across ranks.

    `allreduce(buf)` sums a float64 numpy buffer over all ranks in place (None: single process)."""

    def __init__(self, d: int, lam: float, allreduce: Optional[Callable[[np.ndarray], None]] = None):
        self.d, self.lam, self.allreduce = d, lam, allreduce
        self.z = np.zeros(d)
        self._buf = np.zeros(d + 1)

    def step(self, xs: Sequence[np.ndarray], ys: Sequence[np.ndarray], rhos: Sequence[float]) -> np.ndarray:
        S = self._buf
        S[:] = 0.0
        for x, y, r in zip(xs, ys, rhos):  # ascending local node order
            S[: self.d] += r * x - y
            S[self.d] += r
        if self.allreduce is not None:
            self.allreduce(S)
        den = self.lam + S[self.d]
        if den == 0.0:
            raise ValueError("z_update: lambda + sum(rho) == 0")  # ConfigError in the reference coordinator
        self.z[:] = S[: self.d] / den
        for x, y, r in zip(xs, ys, rhos):
            y += r * (self.z - x)
        return self.z


def torch_allreduce(dist) -> Callable[[np.ndarray], None]:
    """allreduce callback over a torch.distributed group (gloo on CPU tensors)."""
    import torch

    def f(buf: np.ndarray) -> None:
        t = torch.from_numpy(buf)
        dist.all_reduce(t)

    return f
