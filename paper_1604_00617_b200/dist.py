"""Sharded ACR over several GPUs.

Each rank owns a contiguous, even-aligned range of block rows.  Per
reduction level the only exchange is the right neighbour's first even
block ({Dinv, E, F}; one n x k vector per boundary in the solve), so each
level's odd-block Schur updates stay local.  When the windows would hold
fewer than two blocks (or alignment breaks) active ranks merge pairwise --
the upper levels consolidate onto P/2, P/4, ... GPUs as the block count
halves -- and rank 0 finishes the cutoff LU (the reference's algorithm is
unchanged: same blocks, same products, same truncations -> the sharded
result is the single-GPU one).

``block_partition`` is the pure host rule (tested on CPU); ``DistAcrSolver``
drives the C ABI with NCCL between one process per GPU (torch.distributed
supplies the rendezvous); ``loopback_solve`` runs the same sharded C++ path
with virtual ranks on one GPU.
"""

from __future__ import annotations

import ctypes as C
from typing import List

import numpy as np

from . import _capi
from .system import BlockTridiagSystem, Tolerance

__all__ = ["block_partition", "level_bounds", "distributed_levels", "schedule",
           "DistAcrSolver", "loopback_solve"]


def block_partition(m: int, P: int) -> List[int]:
    """Level-0 boundaries b[0..P] (b[0] = 0, b[P] = m), even starts,
    as equal as possible."""
    if P < 1 or m < P:
        raise ValueError(f"cannot split {m} block rows over {P} ranks")
    b = [2 * ((r * m) // (2 * P)) for r in range(P)] + [m]
    for r in range(P):
        if b[r + 1] - b[r] < 1:
            raise ValueError(f"rank {r} would own no block rows")
    return b


def level_bounds(b0: List[int], m: int, level: int) -> List[int]:
    """Boundaries of every rank's window at reduction level ``level``
    (mirrors Plan::bounds in csrc/engine.cu)."""
    mg = m
    for _ in range(level):
        mg //= 2
    return [x >> level for x in b0[:-1]] + [mg]


def distributed_ok(b0: List[int], m: int, level: int) -> bool:
    """Plan::dist_ok: every window starts even with >= 2 blocks, and all
    but the last have even length."""
    P = len(b0) - 1
    if P <= 1:
        return False
    b = level_bounds(b0, m, level)
    for r in range(P):
        c = b[r + 1] - b[r]
        if b[r] % 2 or c < 2 or (r < P - 1 and c % 2):
            return False
    return True


def distributed_levels(m: int, P: int, cutoff: int = 1) -> int:
    """Number of levels reduced with every rank active (before the first
    merge)."""
    b0 = block_partition(m, P)
    lv, mg = 0, m
    while mg > cutoff and distributed_ok(b0, m, lv):
        mg //= 2
        lv += 1
    return lv


def _active(b: List[int]) -> List[int]:
    return [r for r in range(len(b) - 1) if b[r + 1] > b[r]]


def windows_ok(b: List[int]) -> bool:
    """Active windows start even, hold >= 2 blocks, and all but the last
    have even length (Plan::win_ok)."""
    a = _active(b)
    for i, r in enumerate(a):
        c = b[r + 1] - b[r]
        if b[r] % 2 or c < 2 or (i + 1 < len(a) and c % 2):
            return False
    return True


def merge_pairs(b: List[int]) -> List[int]:
    """The (2i+1)-th active rank hands its window to the 2i-th
    (Plan::merge_pairs)."""
    a, nb = _active(b), list(b)
    for i in range(len(a) // 2):
        dst, src = a[2 * i], a[2 * i + 1]
        for x in range(dst + 1, src + 1):
            nb[x] = b[src + 1]
    return nb


def schedule(m: int, P: int, cutoff: int = 1):
    """Progressive consolidation schedule (Plan::schedule, csrc/engine.cu):
    returns (wins, steps, L) with wins[l] every rank's window boundaries at
    level l after that level's merges, steps = [(level, before, after)] the
    pairwise merges in order, L the cutoff level.  Upper levels move onto
    P/2, P/4, ... ranks as the block count halves; at the cutoff everything
    is on rank 0."""
    cur = block_partition(m, P) if P > 1 else [0, m]
    wins, steps = [], []
    mg, lv = m, 0
    while True:
        last = mg <= cutoff
        while len(_active(cur)) > 1 and (last or not windows_ok(cur)):
            nb = merge_pairs(cur)
            steps.append((lv, list(cur), nb))
            cur = nb
        wins.append(list(cur))
        if last:
            return wins, steps, lv
        mg //= 2
        lv += 1
        cur = [x >> 1 for x in cur[:-1]] + [mg]


def owner(b: List[int], pos: int) -> int:
    for r in range(len(b) - 1):
        if b[r] <= pos < b[r + 1]:
            return r
    return -1


def loopback_solve(sys: BlockTridiagSystem, tol: Tolerance, P: int,
                   cutoff_blocks: int = 1, leaf_size: int = 32):
    """Sharded factor + solve with P virtual ranks (threads) on the current
    GPU.  Returns (u, max-over-ranks factor ms)."""
    import torch
    from .solver import _ptr, _raise
    lib = _capi.load()
    m, n = sys.n_blocks, sys.block_dim
    bnd = (C.c_int * (P + 1))(*block_partition(m, P))
    dev = torch.device("cuda", torch.cuda.current_device())
    t = [torch.as_tensor(np.ascontiguousarray(a), device=dev) for a in
         (sys.D_sub, sys.D_diag, sys.D_sup, sys.E, sys.F, sys.rhs)]
    u = torch.zeros_like(t[-1])
    k = 1 if t[-1].dim() == 1 else t[-1].shape[1]
    torch.cuda.synchronize()
    ms = C.c_double()
    rc = lib.acr_loopback_solve(P, bnd, m, n, leaf_size, float(tol.eps),
                                int(tol.max_rank_cap or 0), cutoff_blocks,
                                *[_ptr(x) for x in t], k, _ptr(u), C.byref(ms))
    if rc:
        _raise(None, rc)
    return u.cpu().numpy(), ms.value


class DistAcrSolver:
    """One rank of a sharded factorisation (NCCL between processes)."""

    def __init__(self, m: int, n: int, tol: Tolerance, cutoff_blocks: int = 1,
                 leaf_size: int = 32):
        import torch
        import torch.distributed as dist
        from .solver import _raise
        self.torch, self.dist = torch, dist
        self.lib = _capi.load()
        self.rank, self.P = dist.get_rank(), dist.get_world_size()
        self.m, self.n = m, n
        self.bounds = block_partition(m, self.P)
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if self.rank == 0 and self.P > 1:
            host = (C.c_uint8 * 128)()
            if self.lib.acr_nccl_unique_id(host):
                _raise(None, 3)
            uid.copy_(torch.tensor(list(host), dtype=torch.uint8))
        if self.P > 1:
            dist.broadcast(uid, 0)
        uid_h = (C.c_uint8 * 128)(*uid.cpu().tolist())
        h = C.c_void_p()
        bnd = (C.c_int * (self.P + 1))(*self.bounds)
        rc = self.lib.acr_plan_create_dist(m, n, leaf_size, float(tol.eps),
                                           int(tol.max_rank_cap or 0), cutoff_blocks,
                                           self.rank, self.P, bnd, uid_h, C.byref(h))
        if rc:
            _raise(None, rc)
        self.plan = h

    def __del__(self):
        try:
            if getattr(self, "plan", None):
                self.lib.acr_plan_destroy(self.plan)
                self.plan = None
        except Exception:
            pass

    def factor(self, bands):
        from .solver import _ptr, _raise, _stream
        rc = self.lib.acr_factor(self.plan, *[_ptr(t) for t in bands], 0,
                                 _stream(self.torch))
        if rc:
            _raise(self.plan, rc)

    def solve(self, rhs, u=None):
        """rhs: global (N,[k]) CUDA tensor; returns u with this rank's rows set."""
        from .solver import _ptr, _raise, _stream
        if u is None:
            u = self.torch.zeros_like(rhs)
        k = 1 if rhs.dim() == 1 else rhs.shape[1]
        rc = self.lib.acr_solve(self.plan, _ptr(rhs), k, _ptr(u), _stream(self.torch))
        if rc:
            _raise(self.plan, rc)
        return u

    @property
    def factor_ms(self) -> float:
        return float(self.lib.acr_factor_ms(self.plan))

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.acr_kernel_launches(self.plan))
