"""Multi-process plumbing of the N-GPU consensus loop (one process per GPU) and the
host-side consensus coordinator of the worker-transport deployment.

The device-resident loop (`run_admm` / `AdmmSession` with a `Communicator`) does its exchange with
one NCCL allreduce inside the library. This module holds the host-side pieces around it:

* `node_range` — which ADMM nodes (contiguous row shards, src/data_io.cpp:300-328) a rank owns.
* `share_unique_id` — ship rank 0's NCCL id to every rank over an existing torch.distributed group.
* `HostCoordinator` — the reference's coordinator over HOST buffers, for callers that drive the
  workers through `workers_solve` / `Worker.solve` (nadmm_worker_solve) themselves, as the
  reference's coordinator drives its workers through frames (inc/admm.hpp:58-140):
  z = (Σ_i ρ_i x_i − y_i) / (λ + Σ_i ρ_i), ŷ_i = y_i + ρ_i (z_prev − x_i), y_i += ρ_i (z − x_i), and
  spectral penalty selection every T_f iterations. With several processes the
  local sums are combined by one allreduce of [Σ(ρx−y) | Σρ]; SPS needs nothing global beyond z.
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


def _spectral_est(ab: float, aa: float, bb: float, eps_cor: float):
    """Hybrid spectral estimate of one side from its secant inner products <a,b>, |a|^2, |b|^2, with
    the correlation safeguard: alpha_SD = |b|^2/<a,b>, alpha_MG = <a,b>/|a|^2;
    None when the safeguard fails (or a zero-norm secant)."""
    if not (aa > 0.0 and bb > 0.0 and ab > 0.0):
        return None
    if not ab / (np.sqrt(aa) * np.sqrt(bb)) > eps_cor:
        return None
    sd, mg = bb / ab, ab / aa
    return mg if 2.0 * mg > sd else sd - mg / 2.0


def _spectral_combine(a, b, rho, rho_min, rho_max) -> float:
    """sqrt(a b) if both sides pass, sqrt of the passing one otherwise, clamped."""
    r = rho
    if a is not None and b is not None:
        r = np.sqrt(a * b)
    elif a is not None:
        r = np.sqrt(a)
    elif b is not None:
        r = np.sqrt(b)
    return float(min(max(r, rho_min), rho_max))


def spectral_rho(dx, dyhat, dz, dy, rho, eps_cor=0.2, rho_min=1e-6, rho_max=1e6) -> float:
    """Spectral penalty of one worker (inc/admm.hpp:26-47): x-side pairs (Δx, Δŷ), z-side pairs
    (Δz, −Δy)."""
    a = _spectral_est(float(np.dot(dx, dyhat)), float(np.dot(dx, dx)), float(np.dot(dyhat, dyhat)), eps_cor)
    b = _spectral_est(-float(np.dot(dz, dy)), float(np.dot(dz, dz)), float(np.dot(dy, dy)), eps_cor)
    return _spectral_combine(a, b, rho, rho_min, rho_max)


class HostCoordinator:
    """Consensus coordinator over host vectors for this rank's `n_local` nodes, optionally across
    ranks (`allreduce(buf)` sums a float64 numpy buffer over all ranks in place; None: one process).

    State (AdmmState::initial): z = 0, y_i = 0, rho_i = rho0. `y` is an (n_local, d)
    array the caller scatters to its workers; `step(X)` takes the gathered x_i rows."""

    def __init__(self, d: int, lam: float, n_local: int = 1, penalty: str = "fixed", rho0: float = 1.0,
                 update_period: int = 2, eps_cor: float = 0.2, rho_min: float = 1e-6, rho_max: float = 1e6,
                 allreduce: Optional[Callable[[np.ndarray], None]] = None, y: Optional[np.ndarray] = None):
        if penalty not in ("fixed", "spectral"):
            raise ValueError(f"unknown penalty {penalty!r}")
        self.d, self.lam, self.allreduce = d, lam, allreduce
        self.penalty, self.T, self.eps_cor, self.rho_min, self.rho_max = penalty, update_period, eps_cor, rho_min, rho_max
        self.z = np.zeros(d)
        self.prev_z = np.zeros(d)
        self.y = y if y is not None else np.zeros((n_local, d))  # may be caller memory (e.g. pinned)
        self.y[:] = 0.0
        self.yh = np.zeros((n_local, d))
        self.rho = np.full(n_local, float(rho0))
        self.k, self.snap_it = 0, 0
        if penalty == "spectral":
            self.xs, self.ys, self.yhs, self.zs = (np.zeros((n_local, d)), np.zeros((n_local, d)),
                                                   np.zeros((n_local, d)), np.zeros(d))
        self._buf = np.zeros(d + 1)
        self._t = np.zeros((n_local, d))

    def step(self, X: np.ndarray) -> np.ndarray:
        """One coordinator round on the gathered iterates X (n_local x d): z-update, ŷ / y-update,
        spectral penalty (SPEC.md:274 order). Returns z (also self.z)."""
        X = np.asarray(X)
        S, T, rho = self._buf, self._t, self.rho
        np.multiply(X, rho[:, None], out=T)
        T -= self.y
        np.sum(T, axis=0, out=S[: self.d])  # ascending local node order
        S[self.d] = rho.sum()
        if self.allreduce is not None:
            self.allreduce(S)
        den = self.lam + S[self.d]
        if den == 0.0:
            raise ValueError("z_update: lambda + sum(rho) == 0")  # ConfigError in the reference coordinator
        self.prev_z[:] = self.z
        np.divide(S[: self.d], den, out=self.z)
        # y_hat^k = y^{k-1} + rho^{k-1} (z^{k-1} - x^k); y^k = y^{k-1} + rho (z^k - x^k)
        np.subtract(self.prev_z[None, :], X, out=T)
        T *= rho[:, None]
        np.add(self.y, T, out=self.yh)
        np.subtract(self.z[None, :], X, out=T)
        T *= rho[:, None]
        self.y += T
        self.k += 1
        if self.penalty == "spectral" and self.k - self.snap_it >= self.T:
            # the secant pairs of every local worker at once: x-side (Δx, Δŷ), z-side (Δz, −Δy)
            DX = X - self.xs
            DH = self.yh - self.yhs
            DY = self.y - self.ys
            dz = self.z - self.zs
            ab_x, aa_x, bb_x = (np.einsum("ij,ij->i", DX, DH), np.einsum("ij,ij->i", DX, DX),
                                np.einsum("ij,ij->i", DH, DH))
            ab_z, aa_z, bb_z = -(DY @ dz), float(np.dot(dz, dz)), np.einsum("ij,ij->i", DY, DY)
            for i in range(len(rho)):
                rho[i] = _spectral_combine(_spectral_est(ab_x[i], aa_x[i], bb_x[i], self.eps_cor),
                                           _spectral_est(ab_z[i], aa_z, bb_z[i], self.eps_cor), rho[i],
                                           self.rho_min, self.rho_max)
            self.xs[:] = X
            self.ys[:] = self.y
            self.yhs[:] = self.yh
            self.zs[:] = self.z
            self.snap_it = self.k
        return self.z


def torch_allreduce(dist, group=None) -> Callable[[np.ndarray], None]:
    """allreduce callback over a torch.distributed group (gloo on CPU tensors)."""
    import torch

    def f(buf: np.ndarray) -> None:
        t = torch.from_numpy(buf)
        dist.all_reduce(t, group=group)

    return f
