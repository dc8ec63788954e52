"""The reference CLI's model problems, emitted in ``BlockTridiagSystem`` form.

``acr solve/verify/sweep/export --problem poisson|helmholtz|convdiff``
(reference ``cli.py:153-158``) builds its systems with the reference's
generators (``problems.py:32-224``).  They are restated here so that the
device CLI (``paper_1604_00617_b200.cli``) accepts the
same command lines and produces bit-identical inputs -- pinned against the
reference's own arrays in ``tests/golden/small_systems.npz`` (``poisson16``,
``checker16``, ``helm16_k*``, ``conv16_a100``).  Host-side input
construction only; nothing here is on the factor/solve path.

* ``Grid2D`` (``problems.py:32-52``): n interior points per dimension,
  h = 1/(n+1), node (i, j) at ((i+1)h, (j+1)h).
* ``poisson2d`` (``:146-178``): conservative -div(kappa grad u), kappa
  sampled once per edge midpoint (so A is exactly symmetric).
* ``helmholtz2d`` (``:181-199``): lap u + k^2 u (the reference's sign).
* ``convdiff2d`` (``:202-224``): -lap u + alpha b.grad u, centred
  differences, b = (cos 8 pi x, sin 8 pi y).
* ``assemble_full`` (``:227-255``): the sparse operator (nonzeros only).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from .system import BlockTridiagSystem

__all__ = ["Grid2D", "CoefficientField", "constant_kappa", "checkerboard_kappa",
           "gaussian_rhs", "poisson2d", "helmholtz2d", "convdiff2d",
           "assemble_full"]


@dataclass(frozen=True)
class Grid2D:
    n: int

    def __post_init__(self):
        if self.n < 2:
            raise ValueError(f"grid needs n >= 2 interior points, got {self.n}")

    @property
    def h(self) -> float:
        return 1.0 / (self.n + 1)

    @property
    def n_unknowns(self) -> int:
        return self.n * self.n

    def interior_coords(self) -> np.ndarray:
        return (np.arange(self.n) + 1) * self.h


class CoefficientField:
    """kappa(x, y) > 0, evaluated at edge midpoints during assembly."""

    def __init__(self, fn: Callable[[np.ndarray, np.ndarray], np.ndarray],
                 name: str = "kappa"):
        self.fn = fn
        self.name = name

    def __call__(self, x, y) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        y = np.asarray(y, dtype=np.float64)
        shape = np.broadcast_shapes(x.shape, y.shape)
        v = np.asarray(self.fn(x, y), dtype=np.float64)
        return np.array(np.broadcast_to(v, shape))


def constant_kappa(value: float = 1.0) -> CoefficientField:
    v = float(value)
    return CoefficientField(lambda x, y: np.full_like(x, v), name=f"const:{value}")


def checkerboard_kappa(contrast: float = 1e3, cells: int = 4) -> CoefficientField:
    """kappa = contrast on the cells x cells tiles with even (ix + iy), else 1."""
    hi = float(contrast)

    def fn(x, y):
        parity = (np.floor(x * cells).astype(int) + np.floor(y * cells).astype(int)) % 2
        return np.where(parity == 0, hi, 1.0)

    return CoefficientField(fn, name=f"checkerboard:{contrast}:{cells}")


def gaussian_rhs(grid: Grid2D) -> np.ndarray:
    """100 exp(-100 |x - (1/2, 1/2)|^2) at the interior nodes, y-line blocks."""
    c = grid.interior_coords()
    X, Y = np.meshgrid(c, c, indexing="xy")
    return (100.0 * np.exp(-100.0 * ((X - 0.5) ** 2 + (Y - 0.5) ** 2))).ravel()


def poisson2d(grid: Grid2D, kappa: Optional[CoefficientField] = None,
              rhs: Optional[np.ndarray] = None) -> BlockTridiagSystem:
    n, h = grid.n, grid.h
    kappa = kappa or constant_kappa(1.0)
    node = grid.interior_coords()
    edge = (np.arange(n + 1) + 0.5) * h
    kx = kappa(edge[None, :], node[:, None])     # [line j, vertical edge i]
    ky = kappa(node[None, :], edge[:, None])     # [horizontal edge k, column i]
    if (kx <= 0).any() or (ky <= 0).any():
        raise ValueError("kappa must be positive at every sampled midpoint")
    h2 = h * h
    diag = (kx[:, :-1] + kx[:, 1:] + ky[:-1, :] + ky[1:, :]) / h2
    sup = -kx[:, 1:-1] / h2
    cpl = -ky[1:-1, :] / h2
    f = gaussian_rhs(grid) if rhs is None else rhs
    return BlockTridiagSystem(n, n, sup.copy(), diag, sup, cpl.copy(), cpl, f,
                              name=f"poisson[{kappa.name}]")


def helmholtz2d(grid: Grid2D, k: float,
                rhs: Optional[np.ndarray] = None) -> BlockTridiagSystem:
    if k < 0:
        raise ValueError(f"wavenumber must be >= 0, got {k}")
    n, h = grid.n, grid.h
    h2 = h * h
    off = 1.0 / h2
    f = gaussian_rhs(grid) if rhs is None else rhs
    return BlockTridiagSystem(
        n, n, np.full((n, n - 1), off), np.full((n, n), -4.0 / h2 + k * k),
        np.full((n, n - 1), off), np.full((n - 1, n), off),
        np.full((n - 1, n), off), f, name=f"helmholtz[k={k}]")


def convdiff2d(grid: Grid2D, alpha: float,
               rhs: Optional[np.ndarray] = None) -> BlockTridiagSystem:
    if alpha < 0:
        raise ValueError(f"convection strength must be >= 0, got {alpha}")
    n, h = grid.n, grid.h
    h2 = h * h
    c = grid.interior_coords()
    bx = np.cos(8.0 * np.pi * c)
    by = np.sin(8.0 * np.pi * c)
    lap = -1.0 / h2
    sup = np.tile(lap + alpha * bx[:-1] / (2.0 * h), (n, 1))
    sub = np.tile(lap - alpha * bx[1:] / (2.0 * h), (n, 1))
    F = np.tile(lap, (n - 1, n)) + alpha * by[:-1, None] / (2.0 * h)
    E = np.tile(lap, (n - 1, n)) - alpha * by[1:, None] / (2.0 * h)
    f = gaussian_rhs(grid) if rhs is None else rhs
    return BlockTridiagSystem(n, n, sub, np.full((n, n), 4.0 / h2), sup, E, F, f,
                              name=f"convdiff[alpha={alpha}]")


def assemble_full(sys: BlockTridiagSystem):
    """Sparse A (scipy COO) with the nonzero band entries only."""
    import scipy.sparse as sp
    m, n = sys.n_blocks, sys.block_dim
    i = np.arange(n)
    parts = []
    for b in range(m):
        o = b * n
        parts += [(o + i, o + i, sys.D_diag[b]), (o + i[:-1], o + i[1:], sys.D_sup[b]),
                  (o + i[1:], o + i[:-1], sys.D_sub[b])]
        if b < m - 1:
            parts += [(o + n + i, o + i, sys.E[b]), (o + i, o + n + i, sys.F[b])]
    r = np.concatenate([p[0] for p in parts])
    c = np.concatenate([p[1] for p in parts])
    v = np.concatenate([p[2] for p in parts])
    nz = v != 0.0
    N = m * n
    return sp.coo_matrix((v[nz], (r[nz], c[nz])), shape=(N, N))
