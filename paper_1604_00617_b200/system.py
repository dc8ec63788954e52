"""Input format and H-matrix parameters of the ACR hot path.

These mirror the reference's public types so a caller can switch packages
without touching its own code:

* ``BlockTridiagSystem`` -- reference ``problems.py:88-133``: block
  tridiagonal ``tridiag(E_i, D_i, F_i) u = f`` with tridiagonal ``D_i``
  stored as three bands and diagonal couplings.  ``E[i]`` couples block
  ``i+1`` back to block ``i``; ``F[i]`` couples block ``i`` to ``i+1``.
  ``rhs`` is block-row-major (x fastest), shape ``(m*n,)``; this package
  also accepts ``(m*n, k)`` for ``k`` right-hand sides (the reference
  rejects 2-D input, ``algebra.py:78-83``).
* ``Tolerance`` -- reference ``hodlr.py:29-44``.
* ``SingularBlockError`` -- reference ``algebra.py:32-40``.
* ``RankProfile`` / ``SolveReport`` -- reference ``algebra.py:256-269`` and
  ``reduction.py:124-153``.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

__all__ = ["Tolerance", "BlockTridiagSystem", "SingularBlockError",
           "RankProfile", "SolveReport"]


@dataclass(frozen=True)
class Tolerance:
    """Relative truncation threshold (singular values below ``eps * s_1``
    are dropped) and optional hard rank cap (reference ``hodlr.py:29-44``)."""

    eps: float
    max_rank_cap: Optional[int] = None

    def __post_init__(self):
        if self.eps <= 0:
            raise ValueError(f"eps must be > 0, got {self.eps}")
        if self.max_rank_cap is not None and self.max_rank_cap < 1:
            raise ValueError("max_rank_cap must be positive")


@dataclass
class BlockTridiagSystem:
    """Block tridiagonal system in band storage (reference
    ``problems.py:88-133``).  Arrays are coerced to float64 C-contiguous."""

    n_blocks: int
    block_dim: int
    D_sub: np.ndarray    # (m, n-1)  row i+1, column i of D_b
    D_diag: np.ndarray   # (m, n)
    D_sup: np.ndarray    # (m, n-1)  row i, column i+1 of D_b
    E: np.ndarray        # (m-1, n)  block b+1 -> block b coupling (diagonal)
    F: np.ndarray        # (m-1, n)  block b -> block b+1 coupling (diagonal)
    rhs: np.ndarray      # (m*n,) or (m*n, k)
    name: str = "custom"

    def __post_init__(self):
        m, n = self.n_blocks, self.block_dim
        expect = {"D_sub": (m, n - 1), "D_diag": (m, n), "D_sup": (m, n - 1),
                  "E": (m - 1, n), "F": (m - 1, n)}
        for attr, shape in expect.items():
            a = np.ascontiguousarray(getattr(self, attr), dtype=np.float64)
            if a.shape != shape:
                raise ValueError(f"{attr} has shape {a.shape}, expected {shape}")
            setattr(self, attr, a)
        r = np.ascontiguousarray(self.rhs, dtype=np.float64)
        if r.ndim not in (1, 2) or r.shape[0] != m * n:
            raise ValueError(f"rhs has shape {r.shape}, expected ({m * n},) "
                             f"or ({m * n}, k)")
        self.rhs = r

    @property
    def n_unknowns(self) -> int:
        return self.n_blocks * self.block_dim

    @property
    def n_rhs(self) -> int:
        return 1 if self.rhs.ndim == 1 else self.rhs.shape[1]

    def rhs_segment(self, i: int) -> np.ndarray:
        n = self.block_dim
        return self.rhs[i * n:(i + 1) * n]

    def dense_block_d(self, i: int) -> np.ndarray:
        n = self.block_dim
        blk = np.diag(self.D_diag[i])
        k = np.arange(n - 1)
        blk[k, k + 1] = self.D_sup[i]
        blk[k + 1, k] = self.D_sub[i]
        return blk

    def matvec(self, u: np.ndarray) -> np.ndarray:
        """A @ u straight from the bands (CPU; used by tests and generators)."""
        m, n = self.n_blocks, self.block_dim
        U = np.asarray(u, dtype=np.float64).reshape((m, n) + u.shape[1:])
        y = self.D_diag.reshape((m, n) + (1,) * (U.ndim - 2)) * U
        y[:, :-1] += self.D_sup.reshape((m, n - 1) + (1,) * (U.ndim - 2)) * U[:, 1:]
        y[:, 1:] += self.D_sub.reshape((m, n - 1) + (1,) * (U.ndim - 2)) * U[:, :-1]
        if m > 1:
            ex = (1,) * (U.ndim - 2)
            y[1:] += self.E.reshape((m - 1, n) + ex) * U[:-1]
            y[:-1] += self.F.reshape((m - 1, n) + ex) * U[1:]
        return y.reshape(u.shape)


class SingularBlockError(np.linalg.LinAlgError):
    """A dense leaf pivot could not be factorized (reference
    ``algebra.py:32-40``).  The message format is identical:
    ``singular dense leaf on index range [lo,hi): level L, pivot block i``."""

    def __init__(self, lo: int, hi: int, detail: str = ""):
        self.lo, self.hi = lo, hi
        msg = f"singular dense leaf on index range [{lo},{hi})"
        if detail:
            msg += f": {detail}"
        super().__init__(msg)


@dataclass
class RankProfile:
    """Per-tree-depth max / mean off-diagonal rank (reference
    ``algebra.py:256-269``)."""

    max_by_depth: List[int] = field(default_factory=list)
    mean_by_depth: List[float] = field(default_factory=list)

    @property
    def max_rank(self) -> int:
        return max(self.max_by_depth, default=0)

    def to_dict(self):
        return {"max_by_depth": list(self.max_by_depth),
                "mean_by_depth": [round(m, 3) for m in self.mean_by_depth]}


@dataclass
class SolveReport:
    """Diagnostics of one solve (reference ``reduction.py:124-153``).

    ``reduce_ms`` here is the GPU factor phase (lift + every reduction level
    + the cutoff LU factorisation, no right-hand side); ``backsub_ms`` is the
    solve phase (forward RHS sweep + cutoff solve + back-substitution).  The
    reference folds its single-column RHS sweep into ``reduce_ms`` and its
    cutoff LU into ``backsub_ms`` (``reduction.py:289-312``); both boundaries
    are stated in DESIGN.md.
    """

    residual: float
    levels: int
    cutoff_blocks: int
    cutoff_dim: int
    per_level_ranks: List[RankProfile]
    max_rank: int
    storage_bytes: int
    reduce_ms: float
    backsub_ms: float
    total_ms: float
    threads: int = 1

    def to_dict(self):
        return {
            "residual": self.residual,
            "levels": self.levels,
            "cutoff_blocks": self.cutoff_blocks,
            "cutoff_dim": self.cutoff_dim,
            "per_level_ranks": [p.to_dict() for p in self.per_level_ranks],
            "max_rank": self.max_rank,
            "storage_bytes": self.storage_bytes,
            "reduce_ms": round(self.reduce_ms, 3),
            "backsub_ms": round(self.backsub_ms, 3),
            "total_ms": round(self.total_ms, 3),
            "threads": self.threads,
        }
