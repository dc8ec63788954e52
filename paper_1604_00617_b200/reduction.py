"""The reference's lower-level reduction surface on the GPU (SURVEY.md 8(b)
"lower-level surface", 8(f) row 3).

``lift_system``, ``reduce_level``, ``backsubstitute``, ``expected_levels``,
``HBlockTridiag``, ``LevelRecord``, ``EliminationRecord`` with the
reference's signatures and behaviour (``reduction.py:42-270``), so that the
reference's own tests (``test_reduction.py:46-151``) run against this
package.  The blocks stay on the device: every level and record entry is a
handle of a plan of the C ABI's stepwise API (``acr_step_*``), whose kernels
are the factorisation's own (lift, one ``reduce`` level, the forward RHS
update and one back-substitution level of ``engine.cu``).  Block contents
reach the host only when inspected -- ``D[i]``, ``Dinv[i]``, ``to_dense()``
export reference-shaped ``HodlrMatrix`` objects (``hodlr.py``).  Levels are
immutable like the reference's (``reduce_level`` leaves its input intact).

The right-hand side segments ``f`` are host arrays, as in the reference;
``reduce_level`` updates them on the device (``acr_step_rhs``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi
from .hodlr import HodlrMatrix, export_block
from .solver import _raise, _stream, _torch, acr_solve, expected_levels
from .system import BlockTridiagSystem, RankProfile, Tolerance
from .tree import build_node_table

__all__ = ["HBlockTridiag", "LevelRecord", "EliminationRecord", "lift_system",
           "reduce_level", "backsubstitute", "expected_levels", "acr_solve"]


class _StepPlan:
    """One plan of the stepwise API (owns every handle made from it)."""

    def __init__(self, m: int, n: int, leaf_size: int):
        self.torch = _torch()
        self.lib = _capi.load()
        self.m, self.n, self.leaf = m, n, leaf_size
        h = C.c_void_p()
        rc = self.lib.acr_plan_create(m, n, int(leaf_size), 1e-8, 0, 1, C.byref(h))
        if rc != 0:
            _raise(None, rc)
        self.plan = h
        self.tree = build_node_table(n, leaf_size)

    def __del__(self):
        try:
            if getattr(self, "plan", None):
                self.lib.acr_plan_destroy(self.plan)
                self.plan = None
        except Exception:
            pass

    def check(self, rc):
        if rc != 0:
            _raise(self.plan, rc)

    def free(self, handle):
        if getattr(self, "plan", None):
            self.lib.acr_step_free(self.plan, handle)

    def info(self, handle, which):
        cnt, R, lv, ml = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        self.check(self.lib.acr_step_info(self.plan, handle, which, C.byref(cnt), C.byref(R),
                                          C.byref(lv), C.byref(ml)))
        return cnt.value, R.value, lv.value, ml.value

    def export(self, handle, which, block) -> HodlrMatrix:
        _, R, _, _ = self.info(handle, which)
        st = _stream(self.torch)

        def call(leaf, U, V, rk):
            self.check(self.lib.acr_step_export(self.plan, handle, which, block, leaf, U, V,
                                                rk, st))
        return export_block(self.lib, self.plan, self.n, self.leaf, R, call, st)

    def ranks(self, handle, which, block) -> np.ndarray:
        torch = self.torch
        rk = torch.empty((self.tree.nnodes, 2), dtype=torch.int32, device="cuda")
        self.check(self.lib.acr_step_export(self.plan, handle, which, block, None, None, None,
                                            C.c_void_p(rk.data_ptr()), _stream(torch)))
        return rk.cpu().numpy()

    def dev(self, a):
        return self.torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


class _Blocks(Sequence):
    """D, E or F of a level (or Dinv/E/F of a record): block i is exported to
    a host ``HodlrMatrix`` on first access; ``None`` where the reference has
    no coupling (E[0], F[-1])."""

    def __init__(self, owner, which: int, idx: List[Optional[int]]):
        self._owner, self._which, self._idx = owner, which, idx
        self._cache = {}

    def __len__(self):
        return len(self._idx)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        b = self._idx[i]
        if b is None:
            return None
        if i not in self._cache:
            self._cache[i] = self._owner._sp.export(self._owner._handle, self._which, b)
        return self._cache[i]

    def ranks(self, i):
        b = self._idx[i]
        return None if b is None else self._owner._sp.ranks(self._owner._handle, self._which, b)


class HBlockTridiag:
    """One level of the reduction (reference ``reduction.py:42-90``):
    ``E[i]`` couples block i to i-1 (``E[0]`` is None), ``F[i]`` couples block
    i to i+1 (``F[-1]`` is None); blocks on the device, ``f`` on the host."""

    def __init__(self, sp: _StepPlan, handle: int, f: List[np.ndarray]):
        self._sp, self._handle = sp, handle
        cnt, _, lv, m = sp.info(handle, 0)
        self.tree = sp.tree
        self.level = lv
        self.D = _Blocks(self, 0, list(range(m)))
        self.E = _Blocks(self, 1, [None] + list(range(1, m)))
        self.F = _Blocks(self, 2, list(range(m - 1)) + [None])
        self.f = f
        self._m = m

    def __del__(self):
        try:
            self._sp.free(self._handle)
        except Exception:
            pass

    @property
    def n_blocks(self) -> int:
        return len(self.D)

    @property
    def block_dim(self) -> int:
        return self._sp.n

    def to_dense(self) -> np.ndarray:
        m, n = self.n_blocks, self.block_dim
        A = np.zeros((m * n, m * n))
        for i in range(m):
            A[i * n:(i + 1) * n, i * n:(i + 1) * n] = self.D[i].to_dense()
            if self.E[i] is not None:
                A[i * n:(i + 1) * n, (i - 1) * n:i * n] = self.E[i].to_dense()
            if self.F[i] is not None:
                A[i * n:(i + 1) * n, (i + 1) * n:(i + 2) * n] = self.F[i].to_dense()
        return A

    def rhs_vector(self) -> np.ndarray:
        return np.concatenate(self.f)

    def storage_bytes(self) -> int:
        total = 0
        for blocks in (self.D, self.E, self.F):
            total += sum(b.storage_bytes() for b in blocks if b is not None)
        return total + sum(seg.nbytes for seg in self.f)

    def rank_profile(self) -> RankProfile:
        """Per-depth max / mean rank over D, E, F (reference algebra.py:272-291),
        from the device rank tables."""
        t = self.tree
        br = np.flatnonzero(~t.is_leaf)
        buckets = {}
        for blocks in (self.D, self.E, self.F):
            for i in range(len(blocks)):
                rk = blocks.ranks(i)
                if rk is None:
                    continue
                for v in br:
                    buckets.setdefault(int(t.depth[v]), []).extend(rk[v].tolist())
        prof = RankProfile([], [])
        for d in sorted(buckets):
            prof.max_by_depth.append(int(max(buckets[d])))
            prof.mean_by_depth.append(float(np.mean(buckets[d])))
        return prof


@dataclass
class LevelRecord:
    """What one level keeps for back-substitution (reference
    ``reduction.py:93-110``); blocks on the device."""

    m: int
    even: List[int]
    odd: List[int]
    Dinv: Sequence
    E: Sequence
    F: Sequence
    f: List[np.ndarray]
    _sp: object = None
    _handle: int = 0

    def __del__(self):
        try:
            if self._sp is not None:
                self._sp.free(self._handle)
        except Exception:
            pass

    def storage_bytes(self) -> int:
        total = sum(b.storage_bytes() for b in self.Dinv)
        total += sum(b.storage_bytes() for b in self.E if b is not None)
        total += sum(b.storage_bytes() for b in self.F if b is not None)
        return total + sum(seg.nbytes for seg in self.f)


@dataclass
class EliminationRecord:
    entries: List[LevelRecord] = field(default_factory=list)

    @property
    def levels(self) -> int:
        return len(self.entries)


class _RecView:
    def __init__(self, sp, handle):
        self._sp, self._handle = sp, handle


def lift_system(sys: BlockTridiagSystem, leaf_size: int = 32) -> HBlockTridiag:
    """Exact HODLR lift of the system on the device (reference
    ``reduction.py:156-166``)."""
    if leaf_size < 1:
        raise ValueError(f"leaf_size must be >= 1, got {leaf_size}")
    sp = _StepPlan(sys.n_blocks, sys.block_dim, leaf_size)
    bands = [sp.dev(a) for a in (sys.D_sub, sys.D_diag, sys.D_sup, sys.E, sys.F)]
    h = C.c_int()
    sp.check(sp.lib.acr_step_lift(sp.plan, *[C.c_void_p(t.data_ptr()) for t in bands],
                                  C.byref(h), _stream(sp.torch)))
    n = sys.block_dim
    f = [np.array(sys.rhs[i * n:(i + 1) * n], dtype=np.float64) for i in range(sys.n_blocks)]
    return HBlockTridiag(sp, h.value, f)


def reduce_level(level: HBlockTridiag, tol: Tolerance,
                 inversion_order: Optional[Sequence[int]] = None):
    """One even-block elimination step on the device (reference
    ``reduction.py:173-232``): returns ``(reduced, LevelRecord)``."""
    m = level.n_blocks
    if m < 2:
        raise ValueError(f"need at least 2 blocks to reduce, got {m}")
    if m != level._m or len(level.f) != m:
        raise ValueError("level blocks were edited on the host; device levels are immutable")
    sp = level._sp
    even = list(range(0, m, 2))
    odd = list(range(1, m, 2))
    order = list(inversion_order) if inversion_order is not None else list(range(len(even)))
    if sorted(order) != list(range(len(even))):
        raise ValueError("inversion_order must permute the even-block indices")
    perm = (C.c_int * len(order))(*order)
    nid, rid = C.c_int(), C.c_int()
    st = _stream(sp.torch)
    sp.check(sp.lib.acr_step_reduce(sp.plan, level._handle, float(tol.eps),
                                    int(tol.max_rank_cap or 0), perm, C.byref(nid),
                                    C.byref(rid), st))
    n = level.block_dim
    f = np.stack([np.asarray(s, dtype=np.float64) for s in level.f])   # (m, n[, k])
    k = 1 if f.ndim == 2 else f.shape[2]
    fd = sp.dev(f.reshape(m * n, k))
    fo = sp.torch.empty((len(odd) * n, k), dtype=sp.torch.float64, device="cuda")
    if odd:
        sp.check(sp.lib.acr_step_rhs(sp.plan, rid.value, C.c_void_p(fd.data_ptr()), k,
                                     C.c_void_p(fo.data_ptr()), st))
    fo = fo.cpu().numpy()
    shp = (n,) if f.ndim == 2 else (n, k)
    newf = [fo[i * n:(i + 1) * n].reshape(shp).copy() for i in range(len(odd))]
    reduced = HBlockTridiag(sp, nid.value, newf)
    rv = _RecView(sp, rid.value)
    entry = LevelRecord(
        m=m, even=even, odd=odd,
        Dinv=_Blocks(rv, 3, list(range(len(even)))),
        E=_Blocks(rv, 4, [i if i >= 1 else None for i in even]),
        F=_Blocks(rv, 5, [i if i <= m - 2 else None for i in even]),
        f=[level.f[i] for i in even], _sp=sp, _handle=rid.value)
    return reduced, entry


def backsubstitute(record: EliminationRecord, u_final: Sequence[np.ndarray]) -> np.ndarray:
    """Recover every block's solution from the deepest level's, walking the
    record in reverse on the device (reference ``reduction.py:235-256``)."""
    u = [np.asarray(s, dtype=np.float64) for s in u_final]
    for entry in reversed(record.entries):
        if len(u) != len(entry.odd):
            raise ValueError(f"solution has {len(u)} segments, record level expects "
                             f"{len(entry.odd)}")
        sp = entry._sp
        n = sp.n
        shp = u[0].shape if u else entry.f[0].shape
        k = 1 if len(shp) == 1 else shp[1]
        f = np.zeros((entry.m * n, k))
        for idx, i in enumerate(entry.even):
            f[i * n:(i + 1) * n] = np.asarray(entry.f[idx]).reshape(n, k)
        uo = np.concatenate([s.reshape(n, k) for s in u]) if u else np.zeros((0, k))
        fd, ud = sp.dev(f), sp.dev(uo)
        out = sp.torch.empty((entry.m * n, k), dtype=sp.torch.float64, device="cuda")
        sp.check(sp.lib.acr_step_backsub(sp.plan, entry._handle, C.c_void_p(fd.data_ptr()),
                                         C.c_void_p(ud.data_ptr()), k,
                                         C.c_void_p(out.data_ptr()), _stream(sp.torch)))
        full = out.cpu().numpy()
        u = [full[i * n:(i + 1) * n].reshape(shp).copy() for i in range(entry.m)]
    return np.concatenate(u)
