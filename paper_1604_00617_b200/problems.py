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

__all__ = ["CONFIGS", "make_config", "poisson_const", "varcoef_diffusion",
           "upwind_convdiff", "helmholtz_neg", "random_system", "uniform_rhs"]


def uniform_rhs(rng: np.random.Generator, N: int, k: int = 1) -> np.ndarray:
    f = rng.uniform(-1.0, 1.0, size=(k, N))
    return f[0].copy() if k == 1 else np.ascontiguousarray(f.T)


def poisson_const(n: int, seed: int = 0, k: int = 1) -> BlockTridiagSystem:
    """Config 1: unscaled 4 / -1 five-point stencil (no 1/h^2)."""
    rng = np.random.default_rng(seed)
    m = n
    return BlockTridiagSystem(
        m, n, np.full((m, n - 1), -1.0), np.full((m, n), 4.0),
        np.full((m, n - 1), -1.0), np.full((m - 1, n), -1.0),
        np.full((m - 1, n), -1.0), uniform_rhs(rng, m * n, k),
        name=f"poisson-const[{n}]")


def varcoef_diffusion(n: int, seed: int = 0, k: int = 1) -> BlockTridiagSystem:
    """Configs 2 and 5: -div(a grad u) = f, finite volumes, harmonic-mean
    face coefficients, a = exp(sum_k c_k cos(2 pi (p_k x + q_k y) + phi_k)).

    Draw order: c (8 normals, sigma 0.5), p, q (8 integers in 0..4 each),
    phi (8 uniforms on [0, 2 pi)), then the right-hand side."""
    rng = np.random.default_rng(seed)
    c = rng.normal(0.0, 0.5, 8)
    p = rng.integers(0, 5, 8)
    q = rng.integers(0, 5, 8)
    phi = rng.uniform(0.0, 2.0 * np.pi, 8)
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
    rng = np.random.default_rng(seed)
    h = 1.0 / (n + 1)
    h2 = h * h
    b1 = b2 = 1.0 / np.sqrt(2.0)
    m = n
    return BlockTridiagSystem(
        m, n,
        np.full((m, n - 1), -1.0 / h2 - beta * b1 / h),
        np.full((m, n), 4.0 / h2 + beta * (b1 + b2) / h),
        np.full((m, n - 1), -1.0 / h2),
        np.full((m - 1, n), -1.0 / h2 - beta * b2 / h),
        np.full((m - 1, n), -1.0 / h2),
        uniform_rhs(rng, m * n, k), name=f"upwind[{n},beta={beta}]")


def helmholtz_neg(n: int, ppw: float = 10.0, seed: int = 0,
                  k: int = 1) -> BlockTridiagSystem:
    """Config 4: -lap u - kappa^2 u = f with kappa h = 2 pi / ppw."""
    rng = np.random.default_rng(seed)
    h = 1.0 / (n + 1)
    h2 = h * h
    kap2 = (2.0 * np.pi / ppw) ** 2 / h2
    m = n
    return BlockTridiagSystem(
        m, n, np.full((m, n - 1), -1.0 / h2),
        np.full((m, n), 4.0 / h2 - kap2), np.full((m, n - 1), -1.0 / h2),
        np.full((m - 1, n), -1.0 / h2), np.full((m - 1, n), -1.0 / h2),
        uniform_rhs(rng, m * n, k), name=f"helmholtz[{n},ppw={ppw}]")


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
                 n=64, leaf=16, eps=1e-8, nrhs=1),
    "cfg2": dict(build=lambda s=0, k=1: varcoef_diffusion(256, s, k),
                 n=256, leaf=32, eps=1e-6, nrhs=1),
    "cfg3": dict(build=lambda s=0, k=1: upwind_convdiff(512, 1000.0, s, k),
                 n=512, leaf=32, eps=1e-6, nrhs=1),
    "cfg4": dict(build=lambda s=0, k=1: helmholtz_neg(1024, 10.0, s, k),
                 n=1024, leaf=32, eps=1e-6, nrhs=1),
    "cfg5": dict(build=lambda s=0, k=16: varcoef_diffusion(2048, s, k),
                 n=2048, leaf=64, eps=1e-6, nrhs=16),
}


def make_config(name: str, seed: int = 0, nrhs=None) -> BlockTridiagSystem:
    c = CONFIGS[name]
    return c["build"](seed, c["nrhs"] if nrhs is None else nrhs)
