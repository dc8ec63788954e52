"""The reference's lower-level reduction tests (test_reduction.py:46-151)
against the GPU stepwise API (``paper_1604_00617_b200.reduction``).

Same assertions and tolerances as the reference's ``TestLift``,
``TestReduceLevel`` and ``TestBacksubstitute``: the lifted level
reassembles the sparse operator, one reduction level equals the Schur
complement of the even blocks (an independent dense oracle built here from
the assembled matrix), the record's Dinv equals the dense inverses,
inversion order does not change the result (bitwise), a singular pivot
names its block, and one back-substitution level recovers the dense LU
solution.  Plus: the stepwise levels equal the full factorisation's
blocks and the exported HODLR objects' ranks / storage bytes equal the
rank tables behind the SolveReport."""

import numpy as np
import pytest

from paper_1604_00617_b200 import problems as P
from paper_1604_00617_b200 import stencils as S
from paper_1604_00617_b200.system import SingularBlockError, Tolerance

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
TOL = Tolerance(1e-12)


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1604_00617_b200 import reduction
    return reduction


def schur_of_even(sys_):
    """Dense Schur complement of the even blocks and the reduced RHS."""
    A = S.assemble_full(sys_).toarray()
    n, m = sys_.block_dim, sys_.n_blocks
    ev = np.concatenate([np.arange(i * n, (i + 1) * n) for i in range(0, m, 2)])
    od = np.concatenate([np.arange(i * n, (i + 1) * n) for i in range(1, m, 2)])
    Ainv = np.linalg.inv(A[np.ix_(ev, ev)])
    S_ = A[np.ix_(od, od)] - A[np.ix_(od, ev)] @ Ainv @ A[np.ix_(ev, od)]
    g = sys_.rhs[od] - A[np.ix_(od, ev)] @ (Ainv @ sys_.rhs[ev])
    return S_, g


def test_lift_reconstructs_full_matrix(R):
    s = P.random_system(5, 8, seed=1)
    lv = R.lift_system(s, leaf_size=4)
    np.testing.assert_allclose(lv.to_dense(), S.assemble_full(s).toarray(), atol=1e-14)
    np.testing.assert_array_equal(lv.rhs_vector(), s.rhs)
    assert lv.level == 0


def test_lift_block_ranks(R):
    lv = R.lift_system(S.poisson2d(S.Grid2D(8)), leaf_size=4)
    assert all(d.max_rank() <= 1 for d in lv.D)
    assert all(e.max_rank() == 0 for e in lv.E if e is not None)
    assert all(f.max_rank() == 0 for f in lv.F if f is not None)
    assert lv.E[0] is None and lv.F[-1] is None


@pytest.mark.parametrize("m", [4, 5, 6, 7])
def test_reduce_level_matches_schur(R, m):
    s = P.random_system(m, 8, seed=m)
    red, _ = R.reduce_level(R.lift_system(s, leaf_size=4), TOL)
    S_, g = schur_of_even(s)
    assert red.n_blocks == m // 2 and red.level == 1
    assert np.linalg.norm(red.to_dense() - S_) <= 1e-10 * np.linalg.norm(S_)
    np.testing.assert_allclose(red.rhs_vector(), g, atol=1e-10)


def test_poisson_schur(R):
    s = S.poisson2d(S.Grid2D(8))
    red, _ = R.reduce_level(R.lift_system(s, leaf_size=4), TOL)
    S_, _ = schur_of_even(s)
    assert np.linalg.norm(red.to_dense() - S_) <= 1e-10 * np.linalg.norm(S_)


def test_record_holds_even_data(R):
    s = P.random_system(6, 4, seed=9)
    _, e = R.reduce_level(R.lift_system(s, leaf_size=4), TOL)
    assert e.even == [0, 2, 4] and e.odd == [1, 3, 5] and len(e.Dinv) == 3
    for idx, i in enumerate(e.even):
        ref = np.linalg.inv(s.dense_block_d(i))
        assert np.linalg.norm(e.Dinv[idx].to_dense() - ref) <= 1e-10 * np.linalg.norm(ref)
    assert e.E[0] is None and e.F[2] is not None


def test_single_block_rejected(R):
    lv = R.lift_system(P.random_system(4, 4, seed=3), leaf_size=4)
    lv.D, lv.E, lv.F, lv.f = lv.D[:1], lv.E[:1], lv.F[:1], lv.f[:1]
    with pytest.raises(ValueError):
        R.reduce_level(lv, TOL)


def test_inversion_order_validated_and_irrelevant(R):
    with pytest.raises(ValueError):
        R.reduce_level(R.lift_system(P.random_system(6, 4, seed=4), leaf_size=4), TOL,
                       inversion_order=[0, 0, 1])
    s = P.random_system(7, 8, seed=5)
    a, _ = R.reduce_level(R.lift_system(s, leaf_size=4), TOL)
    b, _ = R.reduce_level(R.lift_system(s, leaf_size=4), TOL, inversion_order=[3, 1, 0, 2])
    np.testing.assert_array_equal(a.to_dense(), b.to_dense())
    np.testing.assert_array_equal(a.rhs_vector(), b.rhs_vector())


def test_singular_pivot_identifies_block(R):
    s = P.random_system(4, 4, seed=6)
    s.D_diag[2] = 0.0
    s.D_sub[2] = 0.0
    s.D_sup[2] = 0.0
    with pytest.raises(SingularBlockError, match="pivot block 2"):
        R.reduce_level(R.lift_system(s, leaf_size=2), TOL)


def test_input_level_unchanged(R):
    s = P.random_system(6, 8, seed=12)
    lv = R.lift_system(s, leaf_size=4)
    before = lv.to_dense()
    R.reduce_level(lv, TOL)
    lv2 = R.lift_system(s, leaf_size=4)
    R.reduce_level(lv, TOL)
    np.testing.assert_array_equal(lv2.to_dense(), before)


def test_backsubstitute_empty_record_passthrough(R):
    segs = [np.arange(4.0), np.arange(4.0, 8.0)]
    np.testing.assert_array_equal(R.backsubstitute(R.EliminationRecord(), segs), np.arange(8.0))


def test_one_level_recovers_dense_solution(R):
    import scipy.linalg
    s = P.random_system(6, 6, seed=7)
    A = S.assemble_full(s).toarray()
    u_ref = np.linalg.solve(A, s.rhs)
    red, e = R.reduce_level(R.lift_system(s, leaf_size=3), TOL)
    u_odd = scipy.linalg.solve(red.to_dense(), red.rhs_vector())
    n = s.block_dim
    u = R.backsubstitute(R.EliminationRecord(entries=[e]),
                         [u_odd[i * n:(i + 1) * n] for i in range(red.n_blocks)])
    assert np.linalg.norm(u - u_ref) <= 1e-9 * np.linalg.norm(u_ref)


def test_segment_count_mismatch(R):
    _, e = R.reduce_level(R.lift_system(P.random_system(6, 4, seed=8), leaf_size=4), TOL)
    with pytest.raises(ValueError):
        R.backsubstitute(R.EliminationRecord(entries=[e]), [np.zeros(4)] * 2)


def test_expected_levels(R):
    assert [R.expected_levels(*a) for a in ((64, 1), (65, 1), (128, 1), (64, 4), (13, 1))] == \
        [6, 6, 7, 4, 3]


def test_stepwise_chain_equals_factorisation(R):
    """Every level of a stepwise chain down to one block, then dense solve
    and back-substitution, equals acr_solve bitwise (same kernels, same
    schedule); level blocks and record Dinv equal the factorisation's
    exported blocks; report rank profiles / storage bytes agree."""
    import scipy.linalg
    from paper_1604_00617_b200.solver import AcrSolver, acr_solve
    s = P.varcoef_diffusion(32, seed=3)
    tol = Tolerance(1e-8)
    u_ref, rep = acr_solve(s, tol, leaf_size=8)
    sol = AcrSolver(32, 32, tol, 1, 8, keep_levels=True)
    sol.factor(s)
    lv = R.lift_system(s, leaf_size=8)
    rec = R.EliminationRecord()
    profs = [lv.rank_profile()]
    while lv.n_blocks > 1:
        nxt, e = R.reduce_level(lv, tol)
        got = nxt.D[nxt.n_blocks - 1].to_dense()
        ref = sol.block_dense(nxt.level, "D", nxt.n_blocks - 1).cpu().numpy()
        np.testing.assert_array_equal(got, ref)
        np.testing.assert_array_equal(e.Dinv[0].to_dense(),
                                      sol.block_dense(lv.level, "Dinv", 0).cpu().numpy())
        rec.entries.append(e)
        lv = nxt
        profs.append(lv.rank_profile())
    assert [p.max_by_depth for p in profs] == [p.max_by_depth for p in rep.per_level_ranks]
    for p, q in zip(profs, rep.per_level_ranks):
        assert p.mean_by_depth == pytest.approx(q.mean_by_depth, rel=1e-12)
    assert sum(e.storage_bytes() for e in rec.entries) + lv.storage_bytes() == rep.storage_bytes
    u_small = scipy.linalg.lu_solve(scipy.linalg.lu_factor(lv.to_dense()), lv.rhs_vector())
    u = R.backsubstitute(rec, [u_small])
    assert np.linalg.norm(u - u_ref) <= 1e-12 * np.linalg.norm(u_ref)


def test_factor_export_objects(R):
    """acr_block_export of the factorisation: exported objects reassemble to
    acr_block_to_dense's dense block and carry the report's ranks."""
    from paper_1604_00617_b200.solver import AcrSolver
    c = P.CONFIGS["cfg1"]
    s = P.make_config("cfg1")
    sol = AcrSolver(s.n_blocks, s.block_dim, Tolerance(c["eps"]), 1, c["leaf"], keep_levels=True)
    sol.factor(s)
    for lv, which, b in ((0, "Dinv", 3), (2, "D", 1), (3, "E", 2), (sol.levels, "D", 0)):
        H = sol.export_hodlr(lv, which, b)
        np.testing.assert_array_equal(H.to_dense(), sol.block_dense(lv, which, b).cpu().numpy())
    prof = sol.rank_profiles()
    top = sol.export_hodlr(sol.levels, "D", 0)
    assert top.max_rank() <= max(prof[-1].max_by_depth)
