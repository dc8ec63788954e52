"""Host HODLR objects rebuilt from device storage.

The GPU keeps every block in the level-ordered layout of DESIGN.md ("HBM
layout"): one dense leaf panel, per-depth U / V column panels addressed by
global row range, and a rank table.  ``export_block`` copies one block out
through the C ABI (``acr_block_export`` / ``acr_step_export``) and rebuilds
the reference's recursive objects:

* ``LowRankFactor(U, V)`` -- reference ``hodlr.py:47-99`` (U (m, r), V (k, r),
  C-contiguous float64; ``rank``, ``shape``, ``to_dense``, ``apply``,
  ``apply_t``);
* ``HodlrMatrix`` -- reference ``hodlr.py:102-173`` (``n``, ``shape``,
  ``is_leaf``, ``dense`` / ``a11``, ``off12``, ``off21``, ``a22``,
  ``to_dense``, ``storage_bytes``, ``max_rank``).

These are read-only views for inspection and tests (``to_dense`` of a
level, ``max_rank`` of a block): the arithmetic never runs on them.
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from .tree import NodeTable, build_node_table

__all__ = ["LowRankFactor", "HodlrMatrix", "export_block", "hodlr_from_storage"]


class LowRankFactor:
    """U V^T with U (m, r) and V (k, r)."""

    def __init__(self, U: np.ndarray, V: np.ndarray):
        self.U = np.ascontiguousarray(U, dtype=np.float64)
        self.V = np.ascontiguousarray(V, dtype=np.float64)
        if self.U.ndim != 2 or self.V.ndim != 2 or self.U.shape[1] != self.V.shape[1]:
            raise ValueError(f"factor shapes {self.U.shape} / {self.V.shape} do not match")

    @classmethod
    def zero(cls, m: int, k: int) -> "LowRankFactor":
        return cls(np.zeros((m, 0)), np.zeros((k, 0)))

    @property
    def rank(self) -> int:
        return self.U.shape[1]

    @property
    def shape(self):
        return (self.U.shape[0], self.V.shape[0])

    def to_dense(self) -> np.ndarray:
        return self.U @ self.V.T

    def apply(self, x: np.ndarray) -> np.ndarray:
        return self.U @ (self.V.T @ x)

    def apply_t(self, x: np.ndarray) -> np.ndarray:
        return self.V @ (self.U.T @ x)


class HodlrMatrix:
    """A leaf (``dense``) or a 2 x 2 split with HODLR diagonal children and
    low-rank off-diagonal blocks."""

    def __init__(self, n: int, dense: Optional[np.ndarray] = None, a11=None, a22=None,
                 off12: Optional[LowRankFactor] = None, off21: Optional[LowRankFactor] = None):
        self._n = int(n)
        self.dense = dense
        self.a11, self.a22, self.off12, self.off21 = a11, a22, off12, off21

    @property
    def n(self) -> int:
        return self._n

    @property
    def shape(self):
        return (self._n, self._n)

    @property
    def is_leaf(self) -> bool:
        return self.dense is not None

    def to_dense(self) -> np.ndarray:
        if self.is_leaf:
            return self.dense.copy()
        n1 = self.a11.n
        out = np.empty((self._n, self._n))
        out[:n1, :n1] = self.a11.to_dense()
        out[n1:, n1:] = self.a22.to_dense()
        out[:n1, n1:] = self.off12.to_dense()
        out[n1:, :n1] = self.off21.to_dense()
        return out

    def storage_bytes(self) -> int:
        """8 bytes per stored scalar (reference hodlr.py:157-163)."""
        if self.is_leaf:
            return 8 * self.dense.size
        return (self.a11.storage_bytes() + self.a22.storage_bytes()
                + 8 * (self.off12.U.size + self.off12.V.size
                       + self.off21.U.size + self.off21.V.size))

    def max_rank(self) -> int:
        if self.is_leaf:
            return 0
        return max(self.off12.rank, self.off21.rank, self.a11.max_rank(), self.a22.max_rank())


def hodlr_from_storage(t: NodeTable, leaf: np.ndarray, U: np.ndarray, V: np.ndarray,
                       ranks: np.ndarray, node: int = 0) -> HodlrMatrix:
    """Recursive object of node ``node`` from one block's raw storage:
    leaf (n, bw), U / V (nd, R, n), ranks (nnodes, 2)."""
    lo, hi = int(t.lo[node]), int(t.hi[node])
    if t.is_leaf[node]:
        return HodlrMatrix(hi - lo, dense=np.ascontiguousarray(leaf[lo:hi, :hi - lo]))
    mid = (lo + hi) // 2
    d = int(t.depth[node])
    r12, r21 = int(ranks[node, 0]), int(ranks[node, 1])
    c0, c1 = int(t.child[node, 0]), int(t.child[node, 1])
    off12 = LowRankFactor(U[d, :r12, lo:mid].T, V[d, :r12, mid:hi].T)
    off21 = LowRankFactor(U[d, :r21, mid:hi].T, V[d, :r21, lo:mid].T)
    return HodlrMatrix(hi - lo, a11=hodlr_from_storage(t, leaf, U, V, ranks, c0),
                       a22=hodlr_from_storage(t, leaf, U, V, ranks, c1),
                       off12=off12, off21=off21)


def export_block(lib, plan, n: int, leaf_size: int, R: int, call, stream) -> HodlrMatrix:
    """Copy one block out of the device (``call(leaf, U, V, ranks)`` issues the
    ABI export into the given device buffers) and rebuild it."""
    import torch
    t = build_node_table(n, leaf_size)
    nd = max(t.n_depths, 1)
    bw = (t.max_leaf + 1) & ~1          # the engine's leaf panel width (even)
    f64 = dict(dtype=torch.float64, device="cuda")
    leaf = torch.empty((n, bw), **f64)
    U = torch.empty((nd, max(R, 1), n), **f64)
    V = torch.empty((nd, max(R, 1), n), **f64)
    rk = torch.empty((t.nnodes, 2), dtype=torch.int32, device="cuda")
    ptr = lambda x: C.c_void_p(x.data_ptr())   # noqa: E731
    call(ptr(leaf), ptr(U), ptr(V), ptr(rk))
    return hodlr_from_storage(t, leaf.cpu().numpy(), U.cpu().numpy(), V.cpu().numpy(),
                              rk.cpu().numpy())
