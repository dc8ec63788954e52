"""Drop-in replacement for the reference solve entry point.

``acr_solve(sys, tol, cutoff_blocks=1, leaf_size=32, inversion_order="forward")``
has the reference's signature, argument checks, return value
``(u, SolveReport)`` and error behaviour (reference
``reduction.py:273-326``; errors ``ValueError`` / ``SingularBlockError`` /
``LinAlgError`` as at ``reduction.py:284-287``, ``algebra.py:32-40``,
``oracles.py:28-30``).  Underneath, ``AcrSolver`` drives the sm_100a
library through its C ABI (``include/acr_b200.h``) with torch tensors as
device storage for inputs and outputs.  There is no CPU path: without a
CUDA device these functions raise.
"""

from __future__ import annotations

import ctypes as C
import time
from typing import Optional

import numpy as np

from . import _capi
from .system import (BlockTridiagSystem, RankProfile, SingularBlockError,
                     SolveReport, Tolerance)

__all__ = ["AcrSolver", "acr_solve", "relative_residual_gpu", "expected_levels"]


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1604_00617_b200 needs a CUDA device "
                           "(B200, sm_100a); there is no CPU fallback")
    return torch


def expected_levels(n_blocks: int, cutoff_blocks: int) -> int:
    """reference reduction.py:259-270."""
    m, levels = n_blocks, 0
    while m > cutoff_blocks:
        m //= 2
        levels += 1
    return levels


def _raise(plan, code: int, lo_msg: str = ""):
    msg = _capi.last_error(plan)
    if code == _capi.ACR_EARG:
        raise ValueError(msg)
    if code == _capi.ACR_ESINGULAR:
        if msg.startswith("singular dense leaf on index range ["):
            rng, _, detail = msg[len("singular dense leaf on index range ["):].partition("): ")
            lo, hi = (int(x) for x in rng.split(","))
            raise SingularBlockError(lo, hi, detail)
        raise np.linalg.LinAlgError(msg)
    raise RuntimeError(f"ACR CUDA library error ({code}): {msg} {lo_msg}")


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def _stream(torch, stream=None) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class AcrSolver:
    """Plan + factorisation of one block tridiagonal operator.

    ``factor()`` runs lift + every reduction level + the cutoff LU on the
    GPU; ``solve(rhs)`` runs the forward sweep, cutoff solve and
    back-substitution for any number of right-hand-side columns.
    """

    def __init__(self, n_blocks: int, block_dim: int, tol: Tolerance,
                 cutoff_blocks: int = 1, leaf_size: int = 32,
                 keep_levels: bool = False):
        if cutoff_blocks < 1:
            raise ValueError(f"cutoff_blocks must be >= 1, got {cutoff_blocks}")
        if leaf_size < 1:
            raise ValueError(f"leaf_size must be >= 1, got {leaf_size}")
        self.torch = _torch()
        self.lib = _capi.load()
        self.m, self.n = int(n_blocks), int(block_dim)
        self.tol = tol
        self.cutoff_blocks = cutoff_blocks
        self.leaf_size = leaf_size
        h = C.c_void_p()
        rc = self.lib.acr_plan_create(self.m, self.n, int(leaf_size),
                                      float(tol.eps), int(tol.max_rank_cap or 0),
                                      int(cutoff_blocks), C.byref(h))
        if rc != 0:
            _raise(None, rc)
        self.plan = h
        if keep_levels:
            self.lib.acr_plan_set_option(self.plan, 1, 1)
        self._bands = None
        self.factored = False

    def __del__(self):
        try:
            if getattr(self, "plan", None):
                self.lib.acr_plan_destroy(self.plan)
                self.plan = None
        except Exception:
            pass

    # -- inputs -----------------------------------------------------------
    def device_bands(self, sys: BlockTridiagSystem):
        torch = self.torch
        dev = torch.device("cuda", torch.cuda.current_device())
        f = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64),
                                      device=dev)
        return [f(sys.D_sub), f(sys.D_diag), f(sys.D_sup), f(sys.E), f(sys.F)]

    def _as_rhs(self, rhs):
        torch = self.torch
        if not isinstance(rhs, torch.Tensor):
            rhs = torch.as_tensor(np.ascontiguousarray(rhs, dtype=np.float64), device="cuda")
        N = self.m * self.n
        if rhs.shape[0] != N or rhs.dim() not in (1, 2):
            raise ValueError(f"rhs has shape {tuple(rhs.shape)}, expected ({N},[k])")
        return rhs.to(torch.float64).contiguous()

    def factor(self, bands, inversion_order: str = "forward", stream=None, rhs=None):
        """``bands`` = [D_sub, D_diag, D_sup, E, F] CUDA float64 tensors or a
        ``BlockTridiagSystem``.  With ``rhs`` ((N,) or (N, k)), the forward
        sweep of that right-hand side runs inside the factorisation (each
        level's RHS update overlapping the next levels, as the reference
        fuses it, reduction.py:204-216); ``solve()`` without arguments then
        finishes it (cutoff solve + back-substitution)."""
        if inversion_order not in ("forward", "reversed"):
            raise ValueError(f"unknown inversion_order {inversion_order!r}")
        if isinstance(bands, BlockTridiagSystem):
            if (bands.n_blocks, bands.block_dim) != (self.m, self.n):
                raise ValueError("system shape does not match the plan")
            bands = self.device_bands(bands)
        m, n = self.m, self.n
        shapes = [(m, n - 1), (m, n), (m, n - 1), (m - 1, n), (m - 1, n)]
        for t, s in zip(bands, shapes):
            if tuple(t.shape) != s or t.dtype != self.torch.float64 or not t.is_cuda:
                raise ValueError(f"band has shape {tuple(t.shape)} / {t.dtype}, "
                                 f"expected {s} float64 on CUDA")
        bands = [t.contiguous() for t in bands]
        self._bands = bands
        cur = self.torch.cuda.current_stream()
        other = stream is not None and stream != cur
        if other:
            stream.wait_stream(cur)
        order = 1 if inversion_order == "reversed" else 0
        self._fused = None
        if rhs is not None:
            rhs = self._as_rhs(rhs)
            k = 1 if rhs.dim() == 1 else rhs.shape[1]
            rc = self.lib.acr_factor_rhs(self.plan, *[_ptr(t) for t in bands], order, _ptr(rhs),
                                         int(k), _stream(self.torch, stream))
            if rc == 0:
                self._fused = (tuple(rhs.shape), rhs.dtype)
        else:
            rc = self.lib.acr_factor(self.plan, *[_ptr(t) for t in bands], order,
                                     _stream(self.torch, stream))
        if other:
            for t in bands:
                t.record_stream(stream)
            if rhs is not None:
                rhs.record_stream(stream)
        if rc != 0:
            self.factored = False
            _raise(self.plan, rc)
        self.factored = True
        return self

    def solve(self, rhs=None, stream=None):
        """rhs: CUDA float64 tensor (N,) or (N, k); returns u of the same shape.
        Without rhs: finish the right-hand side given to ``factor(rhs=...)``
        (once per such factorisation)."""
        torch = self.torch
        if not self.factored:
            raise RuntimeError("factor() must succeed before solve()")
        cur = torch.cuda.current_stream()
        if rhs is None:
            if not getattr(self, "_fused", None):
                raise RuntimeError("solve() without a right-hand side needs factor(rhs=...)")
            shape, dtype = self._fused
            self._fused = None
            u = torch.empty(shape, dtype=dtype, device="cuda")
            if stream is not None and stream != cur:
                stream.wait_stream(cur)
            rc = self.lib.acr_solve_back(self.plan, _ptr(u), _stream(torch, stream))
            if rc != 0:
                _raise(self.plan, rc)
            if stream is not None and stream != cur:
                u.record_stream(stream)
            self._nrhs = 1 if len(shape) == 1 else shape[1]
            return u
        rhs = self._as_rhs(rhs)
        k = 1 if rhs.dim() == 1 else rhs.shape[1]
        u = torch.empty_like(rhs)
        if stream is not None and stream != cur:
            # rhs (possibly a converted temporary) and u were allocated on the
            # current stream; the solve runs asynchronously on `stream`
            stream.wait_stream(cur)
        rc = self.lib.acr_solve(self.plan, _ptr(rhs), int(k), _ptr(u),
                                _stream(torch, stream))
        if rc != 0:
            _raise(self.plan, rc)
        if stream is not None and stream != cur:
            rhs.record_stream(stream)
            u.record_stream(stream)
        self._nrhs = k
        return u

    # -- report -----------------------------------------------------------
    @property
    def levels(self) -> int:
        return self.lib.acr_levels(self.plan)

    @property
    def remaining_blocks(self) -> int:
        return self.lib.acr_cutoff_blocks(self.plan)

    def rank_profiles(self):
        nd = self.lib.acr_tree_depths(self.plan)
        out = []
        for lv in range(self.levels + 1):
            mx = (C.c_int * max(nd, 1))()
            mn = (C.c_double * max(nd, 1))()
            self.lib.acr_rank_profile(self.plan, lv, mx, mn)
            out.append(RankProfile(list(mx)[:nd], list(mn)[:nd]))
        return out

    def storage_bytes(self, nrhs: int = 1) -> int:
        return int(self.lib.acr_storage_bytes(self.plan, int(nrhs)))

    @property
    def factor_ms(self) -> float:
        return float(self.lib.acr_factor_ms(self.plan))

    @property
    def solve_ms(self) -> float:
        return float(self.lib.acr_solve_ms(self.plan))

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.acr_kernel_launches(self.plan))

    def export_hodlr(self, level: int, which: str, block: int):
        """One block of the factorisation as a reference-shaped host
        ``HodlrMatrix`` (``hodlr.py``; reference ``hodlr.py:102-173``):
        which in D, E, F (level system) or Dinv (elimination record)."""
        from .hodlr import export_block
        code = {"D": 0, "E": 1, "F": 2, "Dinv": 3}[which]
        R, cnt = C.c_int(), C.c_int()
        st = _stream(self.torch)
        rc = self.lib.acr_block_export(self.plan, level, code, block, None, None, None, None,
                                       C.byref(R), C.byref(cnt), st)
        if rc != 0:
            _raise(self.plan, rc)

        def call(leaf, U, V, rk):
            rc_ = self.lib.acr_block_export(self.plan, level, code, block, leaf, U, V, rk,
                                            None, None, st)
            if rc_ != 0:
                _raise(self.plan, rc_)
        return export_block(self.lib, self.plan, self.n, self.leaf_size, R.value, call, st)

    def block_dense(self, level: int, which: str, block: int):
        """Dense copy of one block (tests): which in D, E, F, Dinv."""
        code = {"D": 0, "E": 1, "F": 2, "Dinv": 3}[which]
        out = self.torch.empty((self.n, self.n), dtype=self.torch.float64,
                               device="cuda")
        rc = self.lib.acr_block_to_dense(self.plan, level, code, block, _ptr(out),
                                         _stream(self.torch))
        if rc != 0:
            _raise(self.plan, rc)
        return out


def relative_residual_gpu(bands, u, f, m: int, n: int):
    """||A u - f|| / ||f|| per column on the GPU (reference oracles.py:34-49);
    returns (max over columns, Frobenius ratio)."""
    torch = _torch()
    lib = _capi.load()
    k = 1 if u.dim() == 1 else u.shape[1]
    r = (C.c_double * k)()
    fn = (C.c_double * k)()
    rc = lib.acr_residual(m, n, k, *[_ptr(t) for t in bands], _ptr(u), _ptr(f),
                          r, fn, _stream(torch))
    if rc != 0:
        _raise(None, rc)
    rs, fs = np.array(list(r)), np.array(list(fn))
    per = np.where(fs > 0, rs / np.where(fs > 0, fs, 1.0), rs)
    fro = float(np.sqrt((rs ** 2).sum()) / np.sqrt((fs ** 2).sum())) \
        if (fs > 0).any() else float(np.sqrt((rs ** 2).sum()))
    return float(per.max()), fro


def acr_solve(sys: BlockTridiagSystem, tol: Tolerance, cutoff_blocks: int = 1,
              leaf_size: int = 32, inversion_order: str = "forward"):
    """Solve a block tridiagonal system by accelerated cyclic reduction on
    the GPU.  Same contract as reference ``reduction.py:273-326``; the RHS
    may also be ``(N, k)``."""
    if cutoff_blocks < 1:
        raise ValueError(f"cutoff_blocks must be >= 1, got {cutoff_blocks}")
    if inversion_order not in ("forward", "reversed"):
        raise ValueError(f"unknown inversion_order {inversion_order!r}")
    if leaf_size < 1:
        raise ValueError(f"leaf_size must be >= 1, got {leaf_size}")
    torch = _torch()
    t0 = time.perf_counter()
    solver = AcrSolver(sys.n_blocks, sys.block_dim, tol, cutoff_blocks, leaf_size)
    bands = solver.device_bands(sys)
    f = torch.as_tensor(sys.rhs, device="cuda")
    # the forward sweep rides with the factorisation (reduction.py:204-216);
    # the report's reduce_ms therefore includes it, like the reference's
    solver.factor(bands, inversion_order, rhs=f)
    u = solver.solve()
    u_host = u.cpu().numpy()
    t1 = time.perf_counter()
    res, _ = relative_residual_gpu(bands, u, f, sys.n_blocks, sys.block_dim)
    profiles = solver.rank_profiles()
    k = sys.n_rhs
    rep = SolveReport(
        residual=res, levels=solver.levels,
        cutoff_blocks=solver.remaining_blocks,
        cutoff_dim=solver.remaining_blocks * sys.block_dim,
        per_level_ranks=profiles,
        max_rank=max((p.max_rank for p in profiles), default=0),
        storage_bytes=solver.storage_bytes(k),
        reduce_ms=solver.factor_ms, backsub_ms=solver.solve_ms,
        total_ms=(t1 - t0) * 1e3)
    return u_host, rep
