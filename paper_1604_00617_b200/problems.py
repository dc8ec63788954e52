"""Seeded generators for the five BASELINE.json configurations.

The reference ships no generator for any of them (SURVEY.md section 0,
fact 5); these follow the formulas in SURVEY.md section 8(d) and emit the
reference's input format (``BlockTridiagSystem``, reference
``problems.py:88-133``).  Grid convention as in the reference
(``problems.py:32-52``): ``h = 1/(n+1)``, node ``(i, j)`` at
``((i+1)h, (j+1)h)``, block ``j`` = grid line ``y_j``, x fastest.

All inputs are synthetic (there is no public dataset for this path).
Right-hand sides are iid Uniform[-1, 1]; a ``k``-column RHS is drawn as a
``(k, N)`` sample transposed, so its column 0 equals the single-column draw.
"""

from __future__ import annotations

import numpy as np

from .system import BlockTridiagSystem

__all__ = ["CONFIGS", "make_config", "device_config", "DeviceSystem", "poisson_const",
           "varcoef_diffusion", "upwind_convdiff", "helmholtz_neg", "random_system",
           "uniform_rhs"]


def uniform_rhs(rng: np.random.Generator, N: int, k: int = 1) -> np.ndarray:
    f = rng.uniform(-1.0, 1.0, size=(k, N))
    return f[0].copy() if k == 1 else np.ascontiguousarray(f.T)


def _varcoef_params(rng: np.random.Generator):
    """Configs 2 and 5 field parameters in the draw order c, p, q, phi."""
    c = rng.normal(0.0, 0.5, 8)
    p = rng.integers(0, 5, 8)
    q = rng.integers(0, 5, 8)
    phi = rng.uniform(0.0, 2.0 * np.pi, 8)
    return c, p, q, phi


def _const_values(kind: str, n: int, beta: float = 1000.0, ppw: float = 10.0):
    """(sub, diag, sup, E, F) of the constant-coefficient configs."""
    h = 1.0 / (n + 1)
    h2 = h * h
    if kind == "poisson":
        return (-1.0, 4.0, -1.0, -1.0, -1.0)
    if kind == "upwind":
        b1 = b2 = 1.0 / np.sqrt(2.0)
        return (float(-1.0 / h2 - beta * b1 / h), float(4.0 / h2 + beta * (b1 + b2) / h),
                float(-1.0 / h2), float(-1.0 / h2 - beta * b2 / h), float(-1.0 / h2))
    if kind == "helmholtz":
        kap2 = (2.0 * np.pi / ppw) ** 2 / h2
        return (-1.0 / h2, float(4.0 / h2 - kap2), -1.0 / h2, -1.0 / h2, -1.0 / h2)
    raise ValueError(kind)


def _const_system(kind: str, n: int, seed: int, k: int, name: str, **kw):
    rng = np.random.default_rng(seed)
    m = n
    sub, diag, sup, e, f = _const_values(kind, n, **kw)
    return BlockTridiagSystem(
        m, n, np.full((m, n - 1), sub), np.full((m, n), diag),
        np.full((m, n - 1), sup), np.full((m - 1, n), e),
        np.full((m - 1, n), f), uniform_rhs(rng, m * n, k), name=name)


def poisson_const(n: int, seed: int = 0, k: int = 1) -> BlockTridiagSystem:
    """Config 1: unscaled 4 / -1 five-point stencil (no 1/h^2)."""
    return _const_system("poisson", n, seed, k, f"poisson-const[{n}]")


def varcoef_diffusion(n: int, seed: int = 0, k: int = 1) -> BlockTridiagSystem:
    """Configs 2 and 5: -div(a grad u) = f, finite volumes, harmonic-mean
    face coefficients, a = exp(sum_k c_k cos(2 pi (p_k x + q_k y) + phi_k)).

    Draw order: c (8 normals, sigma 0.5), p, q (8 integers in 0..4 each),
    phi (8 uniforms on [0, 2 pi)), then the right-hand side."""
    rng = np.random.default_rng(seed)
    c, p, q, phi = _varcoef_params(rng)
    h = 1.0 / (n + 1)
    # nodes including the boundary ring: index -1..n -> coordinate 0..1
    t = np.arange(n + 2) * h
    X, Y = np.meshgrid(t, t, indexing="xy")        # [y, x]
    expo = np.zeros_like(X)
    for ck, pk, qk, fk in zip(c, p, q, phi):
        expo += ck * np.cos(2.0 * np.pi * (pk * X + qk * Y) + fk)
    a = np.exp(expo)

    def hmean(P, Q):
        return 2.0 * P * Q / (P + Q)

    # horizontal faces between x-neighbours, for every interior line
    ax = hmean(a[1:-1, :-1], a[1:-1, 1:])          # [n, n+1]: face i-1/2+..
    # vertical faces between y-neighbours, for every interior column
    ay = hmean(a[:-1, 1:-1], a[1:, 1:-1])          # [n+1, n]
    aW, aE = ax[:, :-1], ax[:, 1:]                 # [n, n]
    aS, aN = ay[:-1, :], ay[1:, :]                 # [n, n]
    h2 = h * h
    D_diag = (aW + aE + aS + aN) / h2
    D_sup = -aE[:, :-1] / h2
    D_sub = -aW[:, 1:] / h2
    F = -aN[:-1, :] / h2
    E = -aS[1:, :] / h2
    return BlockTridiagSystem(n, n, D_sub, D_diag, D_sup, E, F,
                              uniform_rhs(rng, n * n, k),
                              name=f"varcoef[{n}]")


def upwind_convdiff(n: int, beta: float = 1000.0, seed: int = 0,
                    k: int = 1) -> BlockTridiagSystem:
    """Config 3: -lap u + beta (b . grad u) = f, b = (1,1)/sqrt 2,
    first-order upwind (backward differences for positive velocity)."""
    return _const_system("upwind", n, seed, k, f"upwind[{n},beta={beta}]", beta=beta)


def helmholtz_neg(n: int, ppw: float = 10.0, seed: int = 0,
                  k: int = 1) -> BlockTridiagSystem:
    """Config 4: -lap u - kappa^2 u = f with kappa h = 2 pi / ppw."""
    return _const_system("helmholtz", n, seed, k, f"helmholtz[{n},ppw={ppw}]", ppw=ppw)


def random_system(m: int, n: int, seed: int, shift: float = 6.0,
                  k: int = 1) -> BlockTridiagSystem:
    """Diagonally dominant random system, same recipe as the reference
    test helper ``test_reduction.py:17-28``."""
    rng = np.random.default_rng(seed)
    sub = rng.standard_normal((m, n - 1))
    diag = rng.standard_normal((m, n)) + shift
    sup = rng.standard_normal((m, n - 1))
    E = rng.standard_normal((m - 1, n))
    F = rng.standard_normal((m - 1, n))
    rhs = rng.standard_normal(m * n) if k == 1 else \
        rng.standard_normal((m * n, k))
    return BlockTridiagSystem(m, n, sub, diag, sup, E, F, rhs,
                              name=f"random[{m}x{n},{seed}]")


# name -> (builder, H parameters); sizes are BASELINE.json's
CONFIGS = {
    "cfg1": dict(build=lambda s=0, k=1: poisson_const(64, s, k),
                 n=64, leaf=16, eps=1e-8, nrhs=1, kind="poisson"),
    "cfg2": dict(build=lambda s=0, k=1: varcoef_diffusion(256, s, k),
                 n=256, leaf=32, eps=1e-6, nrhs=1, kind="varcoef"),
    "cfg3": dict(build=lambda s=0, k=1: upwind_convdiff(512, 1000.0, s, k),
                 n=512, leaf=32, eps=1e-6, nrhs=1, kind="upwind"),
    "cfg4": dict(build=lambda s=0, k=1: helmholtz_neg(1024, 10.0, s, k),
                 n=1024, leaf=32, eps=1e-6, nrhs=1, kind="helmholtz"),
    "cfg5": dict(build=lambda s=0, k=16: varcoef_diffusion(2048, s, k),
                 n=2048, leaf=64, eps=1e-6, nrhs=16, kind="varcoef"),
}


def make_config(name: str, seed: int = 0, nrhs=None) -> BlockTridiagSystem:
    c = CONFIGS[name]
    return c["build"](seed, c["nrhs"] if nrhs is None else nrhs)


class DeviceSystem:
    """A BASELINE configuration generated on the GPU: ``bands`` = (D_sub,
    D_diag, D_sup, E, F) and ``rhs`` ((N,) or (N, k)) as CUDA tensors, in the
    layout ``AcrSolver.factor`` / ``solve`` take."""

    def __init__(self, name, m, n, bands, rhs):
        self.name, self.n_blocks, self.block_dim = name, m, n
        self.bands, self.rhs = bands, rhs


def device_config(name: str, seed: int = 0, nrhs=None) -> DeviceSystem:
    """``make_config`` on the device: the few field
    parameters are drawn on the host in numpy's order, the bands are computed
    by ``acr_gen_constant`` / ``acr_gen_varcoef`` and the right-hand side by
    ``acr_gen_uniform`` continuing numpy's PCG64 stream, so the RHS is bitwise
    ``make_config``'s and the bands agree to a few ulp (CUDA cos/exp).
    Needs the CUDA library and a GPU (raises otherwise)."""
    import ctypes as C

    import torch

    from . import _capi
    from .solver import _raise, _stream
    lib = _capi.load()
    c = CONFIGS[name]
    n = m = c["n"]
    k = c["nrhs"] if nrhs is None else nrhs
    dev = torch.device("cuda", torch.cuda.current_device())
    f64 = dict(dtype=torch.float64, device=dev)
    bands = (torch.empty((m, n - 1), **f64), torch.empty((m, n), **f64),
             torch.empty((m, n - 1), **f64), torch.empty((m - 1, n), **f64),
             torch.empty((m - 1, n), **f64))
    ptr = [C.c_void_p(t.data_ptr()) for t in bands]
    st = _stream(torch)
    rng = np.random.default_rng(seed)
    if c["kind"] == "varcoef":
        cc, p, q, phi = _varcoef_params(rng)
        work = torch.empty((n + 2) * (n + 2), **f64)
        arr = lambda t, v: (t * 8)(*[t(x) for x in v])   # noqa: E731
        rc = lib.acr_gen_varcoef(n, arr(C.c_double, cc), arr(C.c_longlong, p),
                                 arr(C.c_longlong, q), arr(C.c_double, phi),
                                 C.c_void_p(work.data_ptr()), *ptr, st)
    else:
        vals = (C.c_double * 5)(*_const_values(c["kind"], n))
        rc = lib.acr_gen_constant(m, n, vals, *ptr, st)
    if rc:
        _raise(None, rc)
    state = rng.bit_generator.state["state"]
    M64 = (1 << 64) - 1
    s4 = (C.c_ulonglong * 4)(state["state"] >> 64, state["state"] & M64,
                             state["inc"] >> 64, state["inc"] & M64)
    N = m * n
    rhs = torch.empty((N,) if k == 1 else (N, k), **f64)
    rc = lib.acr_gen_uniform(s4, N, k, -1.0, 1.0, C.c_void_p(rhs.data_ptr()), st)
    if rc:
        _raise(None, rc)
    return DeviceSystem(name, m, n, bands, rhs)
