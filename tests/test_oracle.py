"""The CPU oracle (oracle/acr_oracle.py) against the reference's own
outputs stored in tests/golden (made by tests/golden/make_golden.py from the
real reference).  CPU only."""

import numpy as np
import pytest

from conftest import golden_case, golden_profiles, load_npz
from oracle import acr_oracle as O
from paper_1604_00617_b200 import problems as P
from paper_1604_00617_b200.system import SingularBlockError, Tolerance
from paper_1604_00617_b200.tree import build_node_table


def _names(z):
    return [str(x) for x in z["names"]]


@pytest.mark.parametrize("idx", range(21))
def test_small_systems_match_reference(small_golden, idx):
    z = small_golden
    names = _names(z)
    if idx >= len(names):
        pytest.skip("no case")
    name = names[idx]
    if name in ("poisson128_e6",):
        pytest.skip("covered by the GPU parity suite (slow on CPU)")
    sys_, tol, leaf, cut = golden_case(z, name)
    u, rep = O.acr_solve(sys_, tol, cutoff_blocks=cut, leaf_size=leaf)
    uref = z[f"{name}/u"]
    # the restatement performs the reference's LAPACK calls in the same order
    assert np.linalg.norm(u - uref) <= 1e-12 * np.linalg.norm(uref)
    assert rep.levels == int(z[f"{name}/levels"])
    assert rep.storage_bytes == int(z[f"{name}/storage_bytes"])
    prof = golden_profiles(z, f"{name}/")
    assert [p.max_by_depth for p in rep.per_level_ranks] == [p[0] for p in prof]
    np.testing.assert_allclose([x for p in rep.per_level_ranks for x in p.mean_by_depth],
                               [x for p in prof for x in p[1]], rtol=0, atol=1e-12)
    assert rep.residual == pytest.approx(float(z[f"{name}/residual"]), rel=1e-3, abs=1e-15)


def test_config1_matches_reference():
    z = load_npz("cfg1.npz")
    c = P.CONFIGS["cfg1"]
    u, rep = O.acr_solve(P.make_config("cfg1"), Tolerance(c["eps"]), leaf_size=c["leaf"])
    assert np.array_equal(u, z["u"])          # bitwise: same LAPACK call sequence
    assert rep.storage_bytes == int(z["storage_bytes"])
    assert [p.max_by_depth for p in rep.per_level_ranks] == \
        [p[0] for p in golden_profiles(z, "")]


def test_truncate_vectors():
    z = load_npz("kernels_cfg1.npz")
    for i in range(int(z["n_trunc"])):
        U, V = z[f"t{i}/U"], z[f"t{i}/V"]
        G = O.truncate((U, V), Tolerance(float(z[f"t{i}/eps"])))
        assert G[0].shape[1] == int(z[f"t{i}/rank"])
        ref = z[f"t{i}/dense"]
        d = O._fdense(G)
        assert np.linalg.norm(d - ref) <= 1e-13 * max(np.linalg.norm(ref), 1e-300)


def test_leaf_inverse_vectors():
    z = load_npz("kernels_cfg1.npz")
    t = build_node_table(16, 16)
    for i in range(int(z["n_inv"])):
        A, X = z[f"i{i}/A"], z[f"i{i}/X"]
        H = O.Hb({0: A})
        inv = O.invert(H, t, Tolerance(1e-8))
        assert np.array_equal(inv.leaf[0], X)


def test_truncate_edge_cases():
    tol = Tolerance(1e-8)
    z = (np.zeros((5, 0)), np.zeros((7, 0)))
    assert O.truncate(z, tol)[0].shape[1] == 0
    u = np.zeros((5, 1)); v = np.ones((7, 1))
    assert O.truncate((u, v), tol)[0].shape[1] == 0        # rank-1 zero
    u[2] = 1.0
    out = O.truncate((u, v), tol)
    assert out[0] is u                                      # rank-1 passthrough
    rng = np.random.default_rng(5)
    a, b = rng.standard_normal((10, 1)), rng.standard_normal((10, 1))
    G = O.truncate((np.hstack([a, a]), np.hstack([b, b])), Tolerance(1e-10))
    assert G[0].shape[1] == 1
    # cancellation guard: u v^T - u v^T
    G = O.truncate((np.hstack([a, -a]), np.hstack([b, b])), tol)
    assert G[0].shape[1] == 0


def test_singular_pivot_message():
    s = P.random_system(4, 4, seed=6)
    s.D_diag[2] = 0.0
    s.D_sub[2] = 0.0
    s.D_sup[2] = 0.0
    with pytest.raises(SingularBlockError, match="pivot block 2"):
        O.acr_solve(s, Tolerance(1e-12), leaf_size=2)


def test_invalid_arguments():
    s = P.random_system(4, 4, seed=1)
    with pytest.raises(ValueError):
        O.acr_solve(s, Tolerance(1e-12), cutoff_blocks=0)
    with pytest.raises(ValueError):
        O.acr_solve(s, Tolerance(1e-12), inversion_order="random")


def test_multi_rhs_equals_columns():
    s1 = P.random_system(6, 8, seed=3, k=3)
    u, _ = O.acr_solve(s1, Tolerance(1e-12), leaf_size=4)
    for c in range(3):
        sc = P.BlockTridiagSystem(6, 8, s1.D_sub, s1.D_diag, s1.D_sup, s1.E, s1.F,
                                  s1.rhs[:, c].copy())
        uc, _ = O.acr_solve(sc, Tolerance(1e-12), leaf_size=4)
        assert np.linalg.norm(u[:, c] - uc) <= 1e-14 * np.linalg.norm(uc)
