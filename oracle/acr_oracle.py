"""CPU oracle for the ACR hot path -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline leg may import this module, and only as the checker / the timed
CPU baseline.  The product path (``paper_1604_00617_b200``) never imports
it and fails loudly when its CUDA library is missing.

What it is: a plain numpy/scipy restatement of the reference ``acrsolve``
algorithm (arXiv 1604.00617, reference tree at
``/root/reference/pkg/src/acrsolve``), written against this repo's node
table (``paper_1604_00617_b200/tree.py``) instead of the reference's
recursive objects.  It keeps the reference's *truncation schedule* exactly
(SURVEY.md Appendix A): the same recompression points, the same product
association, the same threshold rule and shortcuts, the same LAPACK calls
(``numpy.linalg.qr``/``svd``/``solve``, ``scipy.linalg.lu_factor``).

Pinning: ``tests/golden/make_golden.py`` runs the real reference (importable
only in the build container) and stores its outputs under ``tests/golden``;
``tests/test_oracle.py`` checks this restatement against those fixtures
(solutions, residuals, per-level rank profiles, storage bytes, kernel-level
truncation and leaf-inverse vectors).

Storage of one HODLR block (``Hb``): ``leaf[node]`` dense leaf blocks and
``fac[(node, side)] = (U, V)``; side 0 is the reference's ``off12``
(U on rows [lo, mid), V on rows [mid, hi)), side 1 is ``off21`` (U on
[mid, hi), V on [lo, mid)).
"""

from __future__ import annotations

import time
from typing import Dict, List, Optional, Tuple

import numpy as np
import scipy.linalg

from paper_1604_00617_b200.system import (BlockTridiagSystem, RankProfile,
                                          SingularBlockError, SolveReport,
                                          Tolerance)
from paper_1604_00617_b200.tree import NodeTable, build_node_table

_EPS64 = np.finfo(np.float64).eps

Factor = Tuple[np.ndarray, np.ndarray]


class Hb:
    """One HODLR block (or a subtree of one) in node-keyed storage."""

    __slots__ = ("leaf", "fac")

    def __init__(self, leaf=None, fac=None):
        self.leaf: Dict[int, np.ndarray] = {} if leaf is None else leaf
        self.fac: Dict[Tuple[int, int], Factor] = {} if fac is None else fac

    def merged(self, *others: "Hb") -> "Hb":
        out = Hb(dict(self.leaf), dict(self.fac))
        for o in others:
            out.leaf.update(o.leaf)
            out.fac.update(o.fac)
        return out

    def to_dense(self, t: NodeTable, node: int = 0) -> np.ndarray:
        if t.is_leaf[node]:
            return self.leaf[node].copy()
        c0, c1 = t.child[node]
        n1 = int(t.hi[c0] - t.lo[c0])
        sz = int(t.hi[node] - t.lo[node])
        out = np.empty((sz, sz))
        out[:n1, :n1] = self.to_dense(t, c0)
        out[n1:, n1:] = self.to_dense(t, c1)
        out[:n1, n1:] = _fdense(self.fac[(node, 0)])
        out[n1:, :n1] = _fdense(self.fac[(node, 1)])
        return out

    def storage_bytes(self) -> int:
        """reference hodlr.py:157-163 (8 bytes per stored scalar)."""
        s = sum(a.size for a in self.leaf.values())
        s += sum(U.size + V.size for U, V in self.fac.values())
        return 8 * s


def _rank(F: Factor) -> int:
    return F[0].shape[1]


def _zero(m: int, k: int) -> Factor:
    return np.zeros((m, 0)), np.zeros((k, 0))


def _fdense(F: Factor) -> np.ndarray:
    U, V = F
    if U.shape[1] == 0:
        return np.zeros((U.shape[0], V.shape[0]))
    return U @ V.T


def _sizes(t: NodeTable, node: int):
    c0, c1 = t.child[node]
    return int(c0), int(c1), int(t.hi[c0] - t.lo[c0]), int(t.hi[c1] - t.lo[c1])


# ---------------------------------------------------------------------------
# recompression -- reference hodlr.py:176-200
# ---------------------------------------------------------------------------

def truncate(F: Factor, tol: Tolerance) -> Factor:
    U, V = F
    R = U.shape[1]
    if R == 0:
        return F
    if R == 1:                                   # hodlr.py:181-185
        if np.any(U) and np.any(V):
            return F
        return _zero(U.shape[0], V.shape[0])
    Qu, Ru = np.linalg.qr(U)                     # hodlr.py:186-188
    Qv, Rv = np.linalg.qr(V)
    W, s, Zt = np.linalg.svd(Ru @ Rv.T)
    guard = R * _EPS64 * np.linalg.norm(Ru) * np.linalg.norm(Rv)
    if s.size == 0 or s[0] <= guard:             # hodlr.py:191-194
        return _zero(U.shape[0], V.shape[0])
    keep = int(np.count_nonzero(s >= tol.eps * s[0]))
    if tol.max_rank_cap is not None:
        keep = min(keep, tol.max_rank_cap)
    if keep == 0:
        return _zero(U.shape[0], V.shape[0])
    return (np.ascontiguousarray(Qu @ (W[:, :keep] * s[:keep])),
            np.ascontiguousarray(Qv @ Zt[:keep].T))


def combine(F: Factor, G: Factor, tol: Tolerance) -> Factor:
    """Truncated sum, rank-0 operands pass through (algebra.py:90-97)."""
    if _rank(F) == 0:
        return G
    if _rank(G) == 0:
        return F
    return truncate((np.hstack([F[0], G[0]]), np.hstack([F[1], G[1]])), tol)


# ---------------------------------------------------------------------------
# lift -- reference hodlr.py:242-314, reduction.py:156-166
# ---------------------------------------------------------------------------

def lift_tridiag(sub, diag, sup, t: NodeTable) -> Hb:
    H = Hb()
    for v in range(t.nnodes):
        lo, hi = int(t.lo[v]), int(t.hi[v])
        if t.is_leaf[v]:
            blk = np.diag(diag[lo:hi]).astype(np.float64)
            k = np.arange(hi - lo - 1)
            blk[k, k + 1] = sup[lo:hi - 1]
            blk[k + 1, k] = sub[lo:hi - 1]
            H.leaf[v] = blk
            continue
        mid = (lo + hi) // 2
        m1, m2 = mid - lo, hi - mid
        a = float(sup[mid - 1])          # entry (mid-1, mid): U e_last, V e_0
        if a == 0.0:
            H.fac[(v, 0)] = _zero(m1, m2)
        else:
            U = np.zeros((m1, 1)); U[m1 - 1, 0] = a
            V = np.zeros((m2, 1)); V[0, 0] = 1.0
            H.fac[(v, 0)] = (U, V)
        b = float(sub[mid - 1])          # entry (mid, mid-1): U e_0, V e_last
        if b == 0.0:
            H.fac[(v, 1)] = _zero(m2, m1)
        else:
            U = np.zeros((m2, 1)); U[0, 0] = b
            V = np.zeros((m1, 1)); V[m1 - 1, 0] = 1.0
            H.fac[(v, 1)] = (U, V)
    return H


def lift_diag(d, t: NodeTable) -> Hb:
    H = Hb()
    for v in range(t.nnodes):
        lo, hi = int(t.lo[v]), int(t.hi[v])
        if t.is_leaf[v]:
            H.leaf[v] = np.diag(d[lo:hi]).astype(np.float64)
        else:
            mid = (lo + hi) // 2
            H.fac[(v, 0)] = _zero(mid - lo, hi - mid)
            H.fac[(v, 1)] = _zero(hi - mid, mid - lo)
    return H


# ---------------------------------------------------------------------------
# products with panels -- reference algebra.py:52-83, hodlr.py:89-99
# ---------------------------------------------------------------------------

def hmat(H: Hb, t: NodeTable, v: int, X: np.ndarray, trans=False) -> np.ndarray:
    """H_v @ X (``trans``: H_v^T @ X) for the subtree rooted at v."""
    if t.is_leaf[v]:
        L = H.leaf[v]
        return (L.T if trans else L) @ X
    c0, c1, n1, _ = _sizes(t, v)
    X1, X2 = X[:n1], X[n1:]
    if not trans:
        top = hmat(H, t, c0, X1) + _apply(H.fac[(v, 0)], X2)
        bot = hmat(H, t, c1, X2) + _apply(H.fac[(v, 1)], X1)
    else:
        top = hmat(H, t, c0, X1, True) + _apply_t(H.fac[(v, 1)], X2)
        bot = hmat(H, t, c1, X2, True) + _apply_t(H.fac[(v, 0)], X1)
    return np.concatenate([top, bot])


def _apply(F: Factor, x):
    U, V = F
    if U.shape[1] == 0:
        return np.zeros((U.shape[0],) + x.shape[1:])
    return U @ (V.T @ x)


def _apply_t(F: Factor, x):
    U, V = F
    if U.shape[1] == 0:
        return np.zeros((V.shape[0],) + x.shape[1:])
    return V @ (U.T @ x)


# ---------------------------------------------------------------------------
# add / negate / low-rank update -- reference algebra.py:100-145
# ---------------------------------------------------------------------------

def _subtree(t: NodeTable, v: int) -> List[int]:
    out, stack = [], [v]
    while stack:
        u = stack.pop()
        out.append(u)
        if not t.is_leaf[u]:
            stack.extend(int(c) for c in t.child[u])
    return out


def add(A: Hb, B: Hb, t: NodeTable, tol: Tolerance, v: int = 0) -> Hb:
    out = Hb()
    for u in _subtree(t, v):
        if t.is_leaf[u]:
            out.leaf[u] = A.leaf[u] + B.leaf[u]
        else:
            for s in (0, 1):
                out.fac[(u, s)] = combine(A.fac[(u, s)], B.fac[(u, s)], tol)
    return out


def negate(H: Hb) -> Hb:
    """scale(H, -1), exact (algebra.py:115-125)."""
    return Hb({k: -1.0 * a for k, a in H.leaf.items()},
              {k: (-1.0 * U, V) for k, (U, V) in H.fac.items()})


def add_lowrank(H: Hb, t: NodeTable, v: int, F: Factor, tol: Tolerance) -> Hb:
    """H_v + U V^T split along the tree (algebra.py:128-145)."""
    if _rank(F) == 0:
        return Hb({u: H.leaf[u] for u in _subtree(t, v) if t.is_leaf[u]},
                  {k: f for k, f in H.fac.items() if k[0] in set(_subtree(t, v))})
    out = Hb()
    _add_lr(H, t, v, F[0], F[1], tol, out)
    return out


def _add_lr(H, t, v, U, V, tol, out):
    if t.is_leaf[v]:
        out.leaf[v] = H.leaf[v] + _fdense((U, V))
        return
    c0, c1, n1, _ = _sizes(t, v)
    Ut, Ub, Vt, Vb = U[:n1], U[n1:], V[:n1], V[n1:]
    _add_lr(H, t, c0, Ut, Vt, tol, out)
    _add_lr(H, t, c1, Ub, Vb, tol, out)
    out.fac[(v, 0)] = combine(H.fac[(v, 0)], (Ut, Vb), tol)
    out.fac[(v, 1)] = combine(H.fac[(v, 1)], (Ub, Vt), tol)


def _restrict(H: Hb, t: NodeTable, v: int) -> Hb:
    nodes = set(_subtree(t, v))
    return Hb({u: a for u, a in H.leaf.items() if u in nodes},
              {k: f for k, f in H.fac.items() if k[0] in nodes})


# ---------------------------------------------------------------------------
# multiply -- reference algebra.py:152-185
# ---------------------------------------------------------------------------

def _lr_lr(F: Factor, G: Factor) -> Factor:
    if _rank(F) == 0 or _rank(G) == 0:
        return _zero(F[0].shape[0], G[1].shape[0])
    return F[0] @ (F[1].T @ G[0]), G[1]


def multiply(A: Hb, B: Hb, t: NodeTable, tol: Tolerance, v: int = 0) -> Hb:
    if t.is_leaf[v]:
        return Hb({v: A.leaf[v] @ B.leaf[v]})
    c0, c1, n1, n2 = _sizes(t, v)
    a12, a21 = A.fac[(v, 0)], A.fac[(v, 1)]
    b12, b21 = B.fac[(v, 0)], B.fac[(v, 1)]
    c11 = add_lowrank(multiply(A, B, t, tol, c0), t, c0, _lr_lr(a12, b21), tol)
    c22 = add_lowrank(multiply(A, B, t, tol, c1), t, c1, _lr_lr(a21, b12), tol)
    f1 = (hmat(A, t, c0, b12[0]), b12[1]) if _rank(b12) else _zero(n1, n2)
    f2 = (a12[0], hmat(B, t, c1, a12[1], True)) if _rank(a12) else _zero(n1, n2)
    g1 = (a21[0], hmat(B, t, c0, a21[1], True)) if _rank(a21) else _zero(n2, n1)
    g2 = (hmat(A, t, c1, b21[0]), b21[1]) if _rank(b21) else _zero(n2, n1)
    out = c11.merged(c22)
    out.fac[(v, 0)] = combine(f1, f2, tol)
    out.fac[(v, 1)] = combine(g1, g2, tol)
    return out


# ---------------------------------------------------------------------------
# invert -- reference algebra.py:192-240
# ---------------------------------------------------------------------------

def invert(H: Hb, t: NodeTable, tol: Tolerance, v: int = 0) -> Hb:
    if t.is_leaf[v]:
        lo, hi = int(t.lo[v]), int(t.hi[v])
        try:
            inv = np.linalg.solve(H.leaf[v], np.eye(hi - lo))
        except np.linalg.LinAlgError as e:
            raise SingularBlockError(lo, hi, str(e)) from e
        if not np.all(np.isfinite(inv)):
            raise SingularBlockError(lo, hi, "non-finite inverse")
        return Hb({v: inv})
    c0, c1, n1, n2 = _sizes(t, v)
    u12, v12 = H.fac[(v, 0)]
    u21, v21 = H.fac[(v, 1)]
    r12, r21 = u12.shape[1], u21.shape[1]
    x11 = invert(H, t, tol, c0)
    if r21 and r12:
        core = v21.T @ hmat(x11, t, c0, u12)
        S = add_lowrank(H, t, c1, (-u21 @ core, v12), tol)
    else:
        S = _restrict(H, t, c1)
    sinv = invert(S, t, tol, c1)
    if r12 and r21:
        c = v12.T @ hmat(sinv, t, c1, u21)
        b11 = add_lowrank(x11, t, c0, (hmat(x11, t, c0, u12) @ c,
                                       hmat(x11, t, c0, v21, True)), tol)
    else:
        b11 = x11
    out = b11.merged(sinv)
    out.fac[(v, 0)] = truncate((-hmat(x11, t, c0, u12),
                                hmat(sinv, t, c1, v12, True)), tol) \
        if r12 else _zero(n1, n2)
    out.fac[(v, 1)] = truncate((-hmat(sinv, t, c1, u21),
                                hmat(x11, t, c0, v21, True)), tol) \
        if r21 else _zero(n2, n1)
    return out


# ---------------------------------------------------------------------------
# rank instrumentation -- reference algebra.py:272-291
# ---------------------------------------------------------------------------

def rank_profile(t: NodeTable, blocks: List[Hb]) -> RankProfile:
    buckets: Dict[int, List[int]] = {}
    for H in blocks:
        for (v, _s), F in H.fac.items():
            buckets.setdefault(int(t.depth[v]), []).append(_rank(F))
    prof = RankProfile()
    for d in sorted(buckets):
        prof.max_by_depth.append(max(buckets[d]))
        prof.mean_by_depth.append(float(np.mean(buckets[d])))
    return prof


# ---------------------------------------------------------------------------
# cyclic reduction driver -- reference reduction.py:156-326
# ---------------------------------------------------------------------------

class Level:
    """One level of the reduction (reference ``HBlockTridiag``)."""

    def __init__(self, level, D, E, F, f):
        self.level, self.D, self.E, self.F, self.f = level, D, E, F, f

    @property
    def m(self):
        return len(self.D)

    def blocks(self):
        return [b for seq in (self.D, self.E, self.F) for b in seq if b is not None]

    def storage_bytes(self):
        return sum(b.storage_bytes() for b in self.blocks()) + \
            sum(x.nbytes for x in self.f)

    def to_dense(self, t: NodeTable) -> np.ndarray:
        m, n = self.m, t.n
        A = np.zeros((m * n, m * n))
        for i in range(m):
            r = slice(i * n, (i + 1) * n)
            A[r, r] = self.D[i].to_dense(t)
            if self.E[i] is not None:
                A[r, (i - 1) * n:i * n] = self.E[i].to_dense(t)
            if self.F[i] is not None:
                A[r, (i + 1) * n:(i + 2) * n] = self.F[i].to_dense(t)
        return A


def lift(sys: BlockTridiagSystem, t: NodeTable) -> Level:
    m = sys.n_blocks
    D = [lift_tridiag(sys.D_sub[i], sys.D_diag[i], sys.D_sup[i], t)
         for i in range(m)]
    E = [None] + [lift_diag(sys.E[i], t) for i in range(m - 1)]
    F = [lift_diag(sys.F[i], t) for i in range(m - 1)] + [None]
    f = [sys.rhs_segment(i).copy() for i in range(m)]
    return Level(0, D, E, F, f)


def reduce_level(lv: Level, t: NodeTable, tol: Tolerance, order=None):
    """One even-elimination step (reference reduction.py:173-232)."""
    m = lv.m
    if m < 2:
        raise ValueError(f"need at least 2 blocks to reduce, got {m}")
    even = list(range(0, m, 2))
    odd = list(range(1, m, 2))
    order = list(range(len(even))) if order is None else list(order)
    if sorted(order) != list(range(len(even))):
        raise ValueError("inversion_order must permute the even-block indices")
    Dinv = {}
    for pos in order:
        i = even[pos]
        try:
            Dinv[i] = invert(lv.D[i], t, tol)
        except SingularBlockError as e:
            raise SingularBlockError(
                e.lo, e.hi, f"level {lv.level}, pivot block {i}") from e
    D2, E2, F2, f2 = [], [], [], []
    for j in odd:
        P = multiply(lv.E[j], Dinv[j - 1], t, tol)        # E_j Dinv_{j-1}
        Dp = add(lv.D[j], negate(multiply(P, lv.F[j - 1], t, tol)), t, tol)
        fp = lv.f[j] - hmat(lv.E[j], t, 0, hmat(Dinv[j - 1], t, 0, lv.f[j - 1]))
        Ep = negate(multiply(P, lv.E[j - 1], t, tol)) if j >= 2 else None
        Fp = None
        if j + 1 <= m - 1:
            Q = multiply(lv.F[j], Dinv[j + 1], t, tol)    # F_j Dinv_{j+1}
            Dp = add(Dp, negate(multiply(Q, lv.E[j + 1], t, tol)), t, tol)
            fp = fp - hmat(lv.F[j], t, 0, hmat(Dinv[j + 1], t, 0, lv.f[j + 1]))
            if j + 2 <= m - 1:
                Fp = negate(multiply(Q, lv.F[j + 1], t, tol))
        D2.append(Dp); E2.append(Ep); F2.append(Fp); f2.append(fp)
    rec = dict(m=m, even=even, odd=odd, Dinv=[Dinv[i] for i in even],
               E=[lv.E[i] for i in even], F=[lv.F[i] for i in even],
               f=[lv.f[i] for i in even])
    return Level(lv.level + 1, D2, E2, F2, f2), rec


def record_bytes(rec) -> int:
    s = sum(b.storage_bytes() for b in rec["Dinv"])
    s += sum(b.storage_bytes() for b in rec["E"] if b is not None)
    s += sum(b.storage_bytes() for b in rec["F"] if b is not None)
    return s + sum(x.nbytes for x in rec["f"])


def backsubstitute(records, t: NodeTable, u_final) -> np.ndarray:
    """reference reduction.py:235-256."""
    u = list(u_final)
    for rec in reversed(records):
        if len(u) != len(rec["odd"]):
            raise ValueError(f"solution has {len(u)} segments, record level "
                             f"expects {len(rec['odd'])}")
        full: List[Optional[np.ndarray]] = [None] * rec["m"]
        for k, j in enumerate(rec["odd"]):
            full[j] = u[k]
        for idx, i in enumerate(rec["even"]):
            r = rec["f"][idx].copy()
            if rec["E"][idx] is not None:
                r = r - hmat(rec["E"][idx], t, 0, full[i - 1])
            if rec["F"][idx] is not None:
                r = r - hmat(rec["F"][idx], t, 0, full[i + 1])
            full[i] = hmat(rec["Dinv"][idx], t, 0, r)
        u = full
    return np.concatenate(u)


def dense_lu_solve(A, f):
    """reference oracles.py:20-31."""
    lu, piv = scipy.linalg.lu_factor(A)
    if np.any(np.abs(np.diag(lu)) == 0.0):
        raise np.linalg.LinAlgError("matrix is singular to working precision")
    return scipy.linalg.lu_solve((lu, piv), f)


def expected_levels(m: int, cutoff: int) -> int:
    lv = 0
    while m > cutoff:
        m //= 2
        lv += 1
    return lv


def relative_residual(sys: BlockTridiagSystem, u: np.ndarray) -> float:
    """||A u - f|| / ||f|| (reference oracles.py:34-49); for k columns the
    largest per-column ratio."""
    r = sys.matvec(u) - sys.rhs
    if r.ndim == 1:
        fn = np.linalg.norm(sys.rhs)
        return float(np.linalg.norm(r) / fn) if fn else float(np.linalg.norm(r))
    fn = np.linalg.norm(sys.rhs, axis=0)
    rn = np.linalg.norm(r, axis=0)
    return float(np.max(np.where(fn > 0, rn / np.where(fn > 0, fn, 1), rn)))


def acr_solve(sys: BlockTridiagSystem, tol: Tolerance, cutoff_blocks: int = 1,
              leaf_size: int = 32, inversion_order: str = "forward",
              max_levels: Optional[int] = None):
    """Restatement of reference reduction.py:273-326.  Accepts a k-column
    RHS (SURVEY.md 8(c) option (ii): the matrix path is RHS-independent).
    ``max_levels`` stops the reduction early (bounded CPU-baseline samples:
    returns ``(None, partial_report)``)."""
    if cutoff_blocks < 1:
        raise ValueError(f"cutoff_blocks must be >= 1, got {cutoff_blocks}")
    if inversion_order not in ("forward", "reversed"):
        raise ValueError(f"unknown inversion_order {inversion_order!r}")
    t0 = time.perf_counter()
    t = build_node_table(sys.block_dim, leaf_size)
    lv = lift(sys, t)
    records = []
    profiles = [rank_profile(t, lv.blocks())]
    rbytes = 0
    while lv.m > cutoff_blocks:
        if max_levels is not None and len(records) >= max_levels:
            return None, dict(levels_done=len(records),
                              reduce_ms=(time.perf_counter() - t0) * 1e3)
        ne = len(range(0, lv.m, 2))
        order = list(range(ne))
        if inversion_order == "reversed":
            order = order[::-1]
        lv, rec = reduce_level(lv, t, tol, order)
        records.append(rec)
        profiles.append(rank_profile(t, lv.blocks()))
        rbytes += record_bytes(rec)
    t1 = time.perf_counter()
    A = lv.to_dense(t)
    fs = np.concatenate(lv.f)
    us = dense_lu_solve(A, fs)
    n = t.n
    u = backsubstitute(records, t, [us[i * n:(i + 1) * n] for i in range(lv.m)])
    t2 = time.perf_counter()
    rep = SolveReport(
        residual=relative_residual(sys, u), levels=len(records),
        cutoff_blocks=lv.m, cutoff_dim=A.shape[0], per_level_ranks=profiles,
        max_rank=max(p.max_rank for p in profiles),
        storage_bytes=rbytes + lv.storage_bytes(),
        reduce_ms=(t1 - t0) * 1e3, backsub_ms=(t2 - t1) * 1e3,
        total_ms=(t2 - t0) * 1e3)
    return u, rep
