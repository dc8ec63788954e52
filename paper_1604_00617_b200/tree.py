"""Cluster tree of one HODLR block, flattened into a level-ordered node table.

The partition is the reference's balanced midpoint bisection
(``cluster.py:54-71``): node ``[lo, hi)`` is a leaf iff ``hi - lo <= leaf``,
otherwise it splits at ``(lo + hi) // 2``.  One tree serves every block of
every reduction level (reference ``reduction.py:159``).

The GPU engine never walks pointers: it receives this table as flat int32
arrays (breadth-first order, so every depth is a contiguous index range)
and addresses every factor by *global row range*.  See DESIGN.md "HBM
layout".
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np

__all__ = ["NodeTable", "build_node_table"]


@dataclass
class NodeTable:
    n: int
    leaf_size: int
    lo: np.ndarray        # int32 [nnodes]
    hi: np.ndarray
    depth: np.ndarray
    parent: np.ndarray    # -1 at the root
    child: np.ndarray     # int32 [nnodes, 2], -1 for leaves
    is_leaf: np.ndarray   # bool

    @property
    def nnodes(self) -> int:
        return int(self.lo.shape[0])

    @property
    def mid(self) -> np.ndarray:
        return (self.lo + self.hi) // 2

    @property
    def n_depths(self) -> int:
        """Number of depths that hold branch nodes (0 for a single leaf)."""
        br = ~self.is_leaf
        return int(self.depth[br].max()) + 1 if br.any() else 0

    @property
    def max_leaf(self) -> int:
        sz = (self.hi - self.lo)[self.is_leaf]
        return int(sz.max())

    def branches(self) -> List[int]:
        return [int(i) for i in np.nonzero(~self.is_leaf)[0]]

    def leaves(self) -> List[int]:
        """Leaf node ids in left-to-right (row) order."""
        ids = [int(i) for i in np.nonzero(self.is_leaf)[0]]
        return sorted(ids, key=lambda i: int(self.lo[i]))

    def as_int32_arrays(self):
        """(lo, hi, depth, parent, child0, child1, is_leaf) as int32."""
        return [np.ascontiguousarray(a, dtype=np.int32) for a in
                (self.lo, self.hi, self.depth, self.parent,
                 self.child[:, 0], self.child[:, 1],
                 self.is_leaf.astype(np.int32))]


def build_node_table(n: int, leaf_size: int) -> NodeTable:
    """Breadth-first node table of the midpoint bisection of ``[0, n)``.

    Same partition as reference ``cluster.py:54-71`` (same errors too)."""
    if n < 1:
        raise ValueError(f"dimension must be >= 1, got {n}")
    if leaf_size < 1:
        raise ValueError(f"leaf_size must be >= 1, got {leaf_size}")
    lo, hi, depth, parent = [0], [n], [0], [-1]
    child = []
    i = 0
    while i < len(lo):
        a, b = lo[i], hi[i]
        if b - a <= leaf_size:
            child.append((-1, -1))
        else:
            m = (a + b) // 2
            c0 = len(lo)
            lo += [a, m]
            hi += [m, b]
            depth += [depth[i] + 1] * 2
            parent += [i, i]
            child.append((c0, c0 + 1))
        i += 1
    child = np.array(child, dtype=np.int32).reshape(-1, 2)
    return NodeTable(n=n, leaf_size=leaf_size,
                     lo=np.array(lo, np.int32), hi=np.array(hi, np.int32),
                     depth=np.array(depth, np.int32),
                     parent=np.array(parent, np.int32), child=child,
                     is_leaf=child[:, 0] < 0)
