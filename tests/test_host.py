"""Host-side logic that needs no GPU: node table, generators, ABI symbols."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO
from paper_1604_00617_b200 import problems as P
from paper_1604_00617_b200.system import BlockTridiagSystem, Tolerance
from paper_1604_00617_b200.tree import build_node_table


def ref_tree(n, leaf, lo=0):
    """midpoint bisection as in reference cluster.py:54-71"""
    hi = lo + n
    if n <= leaf:
        return (lo, hi, None)
    mid = (lo + hi) // 2
    return (lo, hi, (ref_tree(mid - lo, leaf, lo), ref_tree(hi - mid, leaf, mid)))


@pytest.mark.parametrize("n,leaf", [(64, 16), (256, 32), (2048, 64), (13, 4),
                                    (63, 16), (6, 2), (1, 4), (1000, 37)])
def test_node_table_matches_bisection(n, leaf):
    t = build_node_table(n, leaf)
    ids = {}
    def walk(node, v):
        lo, hi, ch = node
        assert (t.lo[v], t.hi[v]) == (lo, hi)
        assert bool(t.is_leaf[v]) == (ch is None)
        if ch:
            assert t.parent[t.child[v, 0]] == v
            walk(ch[0], t.child[v, 0]); walk(ch[1], t.child[v, 1])
    walk(ref_tree(n, leaf), 0)
    assert np.all(np.diff(t.depth) >= 0)          # breadth-first ids


def test_node_table_errors():
    with pytest.raises(ValueError):
        build_node_table(0, 4)
    with pytest.raises(ValueError):
        build_node_table(8, 0)


def test_generators_shapes_and_symmetry():
    s = P.varcoef_diffusion(32, seed=0)
    assert s.D_diag.shape == (32, 32)
    np.testing.assert_array_equal(s.D_sub, s.D_sup)
    np.testing.assert_array_equal(s.E, s.F)
    assert np.all(s.D_diag > 0)
    c = P.upwind_convdiff(16)
    assert not np.array_equal(c.D_sub, c.D_sup)       # nonsymmetric
    h = P.helmholtz_neg(64)
    assert (h.D_diag < 4.0 / (1 / 65) ** 2).all()
    m = P.make_config("cfg1", nrhs=4)
    m1 = P.make_config("cfg1")
    np.testing.assert_array_equal(m.rhs[:, 0], m1.rhs)


def test_matvec_bands_against_dense():
    s = P.random_system(5, 6, seed=2, k=2)
    N = 30
    A = np.zeros((N, N))
    for i in range(5):
        A[i*6:(i+1)*6, i*6:(i+1)*6] = s.dense_block_d(i)
        if i < 4:
            A[(i+1)*6:(i+2)*6, i*6:(i+1)*6] = np.diag(s.E[i])
            A[i*6:(i+1)*6, (i+1)*6:(i+2)*6] = np.diag(s.F[i])
    u = np.random.default_rng(0).standard_normal((N, 2))
    np.testing.assert_allclose(s.matvec(u), A @ u, atol=1e-12)


def test_system_validation():
    with pytest.raises(ValueError):
        BlockTridiagSystem(2, 3, np.zeros((2, 2)), np.zeros((2, 3)), np.zeros((2, 1)),
                           np.zeros((1, 3)), np.zeros((1, 3)), np.zeros(6))
    with pytest.raises(ValueError):
        Tolerance(0.0)
    with pytest.raises(ValueError):
        Tolerance(1e-6, max_rank_cap=0)


def _header_symbols():
    h = open(os.path.join(REPO, "include", "acr_b200.h")).read()
    return sorted(set(re.findall(r"\b(acr_[a-z_0-9]+)\s*\(", h)))


def test_library_exports_every_header_symbol():
    from paper_1604_00617_b200 import _capi
    path = _capi.lib_path()
    if not os.path.exists(path):
        from paper_1604_00617_b200 import build
        build.build()
    lib = ctypes.CDLL(path)
    syms = _header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_capi.EXPORTED)


def test_product_path_has_no_oracle_import():
    pkg = os.path.join(REPO, "paper_1604_00617_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(root, f)).read()
                assert "oracle" not in re.sub(r'""".*?"""|#.*', "", src, flags=re.S), f


def test_block_partition_rules():
    from paper_1604_00617_b200.dist import (block_partition, distributed_levels,
                                            distributed_ok, level_bounds)
    assert block_partition(2048, 8) == [256 * r for r in range(8)] + [2048]
    for m, Pn in [(2048, 2), (2048, 4), (2048, 8), (13, 3), (256, 8), (100, 7)]:
        b = block_partition(m, Pn)
        assert b[0] == 0 and b[-1] == m
        assert all(x % 2 == 0 for x in b[:-1])
        assert all(b[r + 1] > b[r] for r in range(Pn))
    # cfg5 on 8 GPUs: 8 sharded levels (2048 -> 8 blocks), then rank 0
    assert distributed_levels(2048, 8) == 8
    assert distributed_levels(2048, 2) == 10
    assert level_bounds(block_partition(2048, 8), 2048, 3) == [32 * r for r in range(8)] + [256]
    assert not distributed_ok(block_partition(2048, 8), 2048, 8)


def _pcg64_uniform(state, inc, count, low=-1.0, high=1.0):
    """Pure-Python PCG64 (XSL-RR 128/64) + next_double, the algorithm the
    device generator acr_gen_uniform implements."""
    M = 0x2360ED051FC65DA44385DF649FCCF645
    MASK = (1 << 128) - 1
    out = []
    for _ in range(count):
        state = (state * M + inc) & MASK
        x = ((state >> 64) ^ state) & 0xFFFFFFFFFFFFFFFF
        r = state >> 122
        x = ((x >> r) | (x << (64 - r))) & 0xFFFFFFFFFFFFFFFF
        out.append(low + (high - low) * ((x >> 11) * (1.0 / 9007199254740992.0)))
    return out


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_device_generator_rng_handoff(name):
    """The host draws of device_config leave numpy's PCG64 at the state whose
    continuation is make_config's right-hand side (pins the hand-off and the
    generator algorithm against numpy itself)."""
    import numpy as np
    from paper_1604_00617_b200 import problems as PR
    rng = np.random.default_rng(0)
    if PR.CONFIGS[name]["kind"] == "varcoef":
        PR._varcoef_params(rng)
    st = rng.bit_generator.state["state"]
    got = _pcg64_uniform(st["state"], st["inc"], 64)
    ref = PR.make_config(name).rhs[:64]
    assert np.array_equal(np.array(got), ref)
