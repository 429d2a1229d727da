"""Test restatement of the host consensus coordinator on torch CPU kernels (inc/admm.hpp:58-140,
SPEC.md:196-304, spectral penalty SPEC.md:262-270): the cross-check for the library's fused
`nadmm_hcoord_*` (paper_1807_07132_b200.dist.NativeHostCoordinator). Test infrastructure only."""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np


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
    array the caller scatters to its workers; `step(X)` takes the gathered x_i rows. The vector work
    runs as torch CPU kernels on zero-copy views of the numpy buffers (intra-op threads: the
    coordinator is memory bound -- ~20 passes over n_local x d doubles per round)."""

    def __init__(self, d: int, lam: float, n_local: int = 1, penalty: str = "fixed", rho0: float = 1.0,
                 update_period: int = 2, eps_cor: float = 0.2, rho_min: float = 1e-6, rho_max: float = 1e6,
                 allreduce: Optional[Callable[[np.ndarray], None]] = None, y: Optional[np.ndarray] = None):
        import torch

        if penalty not in ("fixed", "spectral"):
            raise ValueError(f"unknown penalty {penalty!r}")
        self.d, self.lam, self.allreduce = d, lam, allreduce
        self.penalty, self.T, self.eps_cor, self.rho_min, self.rho_max = penalty, update_period, eps_cor, rho_min, rho_max
        t = lambda *shape: torch.zeros(*shape, dtype=torch.float64)
        self._z, self._pz = t(d), t(d)
        self.z = self._z.numpy()
        self.y = y if y is not None else np.zeros((n_local, d))  # may be caller memory (e.g. pinned)
        self.y[:] = 0.0
        self._y = torch.from_numpy(self.y)
        self._yh = t(n_local, d)
        self.yh = self._yh.numpy()
        self.rho = np.full(n_local, float(rho0))
        self.k, self.snap_it = 0, 0
        if penalty == "spectral":
            self._xs, self._ys, self._yhs, self._zs = t(n_local, d), t(n_local, d), t(n_local, d), t(d)
        self._buf = t(d + 1)
        self._T, self._T2 = t(n_local, d), t(n_local, d)

    def step(self, X: np.ndarray) -> np.ndarray:
        """One coordinator round on the gathered iterates X (n_local x d): z-update, ŷ / y-update,
        spectral penalty (SPEC.md:274 order). Returns z (also self.z)."""
        import torch

        Xt = torch.from_numpy(np.ascontiguousarray(X))
        rho = torch.from_numpy(self.rho)[:, None]
        S, T, T2 = self._buf, self._T, self._T2
        torch.mul(Xt, rho, out=T)
        T.sub_(self._y)
        torch.sum(T, 0, out=S[: self.d])  # ascending local node order
        S[self.d] = float(self.rho.sum())
        if self.allreduce is not None:
            self.allreduce(S.numpy())
        den = self.lam + float(S[self.d])
        if den == 0.0:
            raise ValueError("z_update: lambda + sum(rho) == 0")  # ConfigError in the reference coordinator
        self._pz.copy_(self._z)
        torch.div(S[: self.d], den, out=self._z)
        # y_hat^k = y^{k-1} + rho^{k-1} (z^{k-1} - x^k); y^k = y^{k-1} + rho (z^k - x^k)
        torch.sub(self._pz, Xt, out=T)
        T.mul_(rho)
        torch.add(self._y, T, out=self._yh)
        torch.sub(self._z, Xt, out=T)
        T.mul_(rho)
        self._y.add_(T)
        self.k += 1
        if self.penalty == "spectral" and self.k - self.snap_it >= self.T:
            # the secant pairs of every local worker at once: x-side (Δx, Δŷ), z-side (Δz, −Δy)
            torch.sub(Xt, self._xs, out=T)  # Δx
            torch.sub(self._yh, self._yhs, out=T2)  # Δŷ
            ab_x, aa_x, bb_x = (T * T2).sum(1), (T * T).sum(1), (T2 * T2).sum(1)
            torch.sub(self._y, self._ys, out=T)  # Δy
            dz = self._z - self._zs
            ab_z, aa_z, bb_z = -(T @ dz), float(dz @ dz), (T * T).sum(1)
            for i in range(len(self.rho)):
                self.rho[i] = _spectral_combine(_spectral_est(float(ab_x[i]), float(aa_x[i]), float(bb_x[i]), self.eps_cor),
                                                _spectral_est(float(ab_z[i]), aa_z, float(bb_z[i]), self.eps_cor),
                                                self.rho[i], self.rho_min, self.rho_max)
            self._xs.copy_(Xt)
            self._ys.copy_(self._y)
            self._yhs.copy_(self._yh)
            self._zs.copy_(self._z)
            self.snap_it = self.k
        return self.z
