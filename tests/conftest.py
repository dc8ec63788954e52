"""pytest plumbing: the ``gpu`` marker and shared fixtures.

``-m "not gpu"`` runs the oracle-vs-golden checks, host logic and the ABI
symbol checks (no GPU needed); ``-m gpu`` runs the parity tests proper
through the C ABI on a B200.
"""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def load_npz(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def golden_case(z, name):
    from paper_1604_00617_b200.system import BlockTridiagSystem, Tolerance
    g = lambda k: z[f"{name}/{k}"]
    m = g("D_diag").shape[0]
    n = g("D_diag").shape[1]
    sys_ = BlockTridiagSystem(m, n, g("D_sub"), g("D_diag"), g("D_sup"),
                              g("E"), g("F"), g("rhs"), name=name)
    leaf, eps, cut = g("params")
    cap = int(z[f"{name}/cap"]) if f"{name}/cap" in z.files else None
    return sys_, Tolerance(float(eps), cap), int(leaf), int(cut)


def golden_profiles(z, prefix):
    mx = z[prefix + "rank_max"]
    mn = z[prefix + "rank_mean"]
    out = []
    for i in range(mx.shape[0]):
        k = mx[i] >= 0
        out.append((list(map(int, mx[i][k])), list(map(float, mn[i][k]))))
    return out


@pytest.fixture(scope="session")
def small_golden():
    return load_npz("small_systems.npz")


def projections(u, nproj=8, seed=1234, chunk=1 << 20):
    """G @ u for the seeded Gaussian G of tests/golden/make_golden.py
    ``projections`` (same numpy stream): compares every entry of a solution
    whose fixture keeps only a subsample."""
    rng = np.random.default_rng(seed)
    N = u.shape[0]
    acc = np.zeros((nproj,) + u.shape[1:])
    for c0 in range(0, N, chunk):
        c1 = min(N, c0 + chunk)
        acc += rng.standard_normal((nproj, c1 - c0)) @ u[c0:c1]
    return acc
