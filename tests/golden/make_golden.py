"""Generate golden fixtures by running the REAL reference (acrsolve).

Run in the build container only (the reference tree does not exist on the
GPU box):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py [small|cfg1|cfg2|cfg3|cfg4|cfg5|kernels]

Inputs come from this repo's seeded generators
(``paper_1604_00617_b200/problems.py``) or, for the reference's own test
problems, from the reference generators -- whose arrays are stored in the
fixture so the GPU box never needs the reference.  Outputs: the
reference's ``acr_solve`` solution, residual, per-level rank profiles,
storage bytes, level count; kernel-level vectors for ``truncate_factor``
and the leaf inverse captured from a config-1 run.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import acrsolve as R                                    # noqa: E402
import acrsolve.algebra as RA                           # noqa: E402
import acrsolve.hodlr as RH                             # noqa: E402
from paper_1604_00617_b200 import problems as P         # noqa: E402


def to_ref(s):
    return R.BlockTridiagSystem(s.n_blocks, s.block_dim, s.D_sub, s.D_diag,
                                s.D_sup, s.E, s.F, s.rhs)


def sys_arrays(prefix, s):
    return {f"{prefix}D_sub": s.D_sub, f"{prefix}D_diag": s.D_diag,
            f"{prefix}D_sup": s.D_sup, f"{prefix}E": s.E, f"{prefix}F": s.F,
            f"{prefix}rhs": s.rhs}


def report_arrays(prefix, rep):
    L = len(rep.per_level_ranks)
    D = max((len(p.max_by_depth) for p in rep.per_level_ranks), default=0)
    mx = np.full((L, D), -1, np.int64)
    mn = np.full((L, D), -1.0)
    for i, p in enumerate(rep.per_level_ranks):
        mx[i, :len(p.max_by_depth)] = p.max_by_depth
        mn[i, :len(p.mean_by_depth)] = p.mean_by_depth
    return {f"{prefix}residual": rep.residual, f"{prefix}levels": rep.levels,
            f"{prefix}cutoff_blocks": rep.cutoff_blocks,
            f"{prefix}cutoff_dim": rep.cutoff_dim,
            f"{prefix}rank_max": mx, f"{prefix}rank_mean": mn,
            f"{prefix}storage_bytes": rep.storage_bytes,
            f"{prefix}reduce_ms": rep.reduce_ms}


def small():
    """Reference test problems at small n (test_reduction.py, test_acceptance.py)."""
    G = R.Grid2D
    cases = []

    def rnd(m, n, seed):
        s = P.random_system(m, n, seed)
        return s

    for m in (4, 5, 6, 7):
        cases.append((f"rand_m{m}", rnd(m, 8, m), 4, 1e-12, 1))
    cases.append(("rand_13x13", rnd(13, 13, 3), 4, 1e-12, 1))
    cases.append(("rand_16x6_c4", rnd(16, 6, 44), 2, 1e-12, 4))
    cases.append(("rand_20x4_c4", rnd(20, 4, 24), 4, 1e-12, 4))
    cases.append(("rand_7x4_c2", rnd(7, 4, 9), 4, 1e-12, 2))
    ref_builders = [
        ("poisson16", lambda: R.poisson2d(G(16)), 8, 1e-12),
        ("checker16", lambda: R.poisson2d(G(16), R.checkerboard_kappa()), 8, 1e-12),
        ("helm16_k1", lambda: R.helmholtz2d(G(16), 1.0), 8, 1e-12),
        ("conv16_a100", lambda: R.convdiff2d(G(16), 100.0), 8, 1e-12),
        ("helm16_k2", lambda: R.helmholtz2d(G(16), 2.0), 8, 1e-12),
        ("poisson32_e8", lambda: R.poisson2d(G(32)), 8, 1e-8),
        ("conv32_a100_e8", lambda: R.convdiff2d(G(32), 100.0), 8, 1e-8),
        ("poisson32_e2", lambda: R.poisson2d(G(32)), 8, 1e-2),
        ("poisson32_e6", lambda: R.poisson2d(G(32)), 8, 1e-6),
        ("helm63_k6pi", lambda: R.helmholtz2d(G(63), 6.0 * np.pi), 16, 1e-10),
        ("conv63_a1e4", lambda: R.convdiff2d(G(63), 1e4), 16, 1e-8),
        ("poisson128_e6", lambda: R.poisson2d(G(128)), 16, 1e-6),
    ]
    out = {}
    names = []
    for name, s, leaf, eps, cut in cases:
        u, rep = R.acr_solve(to_ref(s), R.Tolerance(eps), cutoff_blocks=cut,
                             leaf_size=leaf)
        out.update(sys_arrays(name + "/", s))
        out.update(report_arrays(name + "/", rep))
        out[name + "/u"] = u
        out[name + "/params"] = np.array([leaf, eps, cut])
        names.append(name)
    for name, build, leaf, eps in ref_builders:
        rs = build()
        u, rep = R.acr_solve(rs, R.Tolerance(eps), leaf_size=leaf)
        out.update(sys_arrays(name + "/", rs))
        out.update(report_arrays(name + "/", rep))
        out[name + "/u"] = u
        out[name + "/params"] = np.array([leaf, eps, 1])
        names.append(name)
    # capped tolerance
    s = P.random_system(8, 16, 77)
    u, rep = R.acr_solve(to_ref(s), R.Tolerance(1e-12, max_rank_cap=2),
                         leaf_size=4)
    out.update(sys_arrays("rand_cap2/", s))
    out.update(report_arrays("rand_cap2/", rep))
    out["rand_cap2/u"] = u
    out["rand_cap2/params"] = np.array([4, 1e-12, 1])
    out["rand_cap2/cap"] = 2
    names.append("rand_cap2")
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "small_systems.npz"), **out)
    print("small:", len(names), "cases")


def config(name, stride=1, nrhs=1):
    c = P.CONFIGS[name]
    s = P.make_config(name, nrhs=nrhs)
    t0 = time.perf_counter()
    u, rep = R.acr_solve(to_ref(s), R.Tolerance(c["eps"]), leaf_size=c["leaf"])
    wall = time.perf_counter() - t0
    out = report_arrays("", rep)
    out["u_stride"] = stride
    out["u"] = u[::stride]
    out["u_norm"] = np.linalg.norm(u)
    out["u_proj"] = projections(u)
    out["wall_s"] = wall
    out["backsub_ms"] = rep.backsub_ms
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "residual", rep.residual, "max_rank", rep.max_rank,
          "storage", rep.storage_bytes, "reduce_ms", rep.reduce_ms, "wall", wall)


def projections(u, nproj=8, seed=1234, chunk=1 << 20):
    """G @ u for a seeded Gaussian G (nproj x N): a size-independent
    fingerprint of EVERY entry of the solution (the committed fixtures keep
    only a subsample).  tests/ regenerate G with the same numpy stream."""
    rng = np.random.default_rng(seed)
    N = u.shape[0]
    acc = np.zeros((nproj,) + u.shape[1:])
    for c0 in range(0, N, chunk):
        c1 = min(N, c0 + chunk)
        G = rng.standard_normal((nproj, c1 - c0))
        acc += G @ u[c0:c1]
    return acc


def multi_rhs(name, nrhs=16, stride=512, check_col0=True):
    """k-column reference solution by the SURVEY.md 8(c) shim: replay
    ``acr_solve``'s body (reduction.py:273-326) with the reference's own
    functions, the level RHS replaced by (n, k) segments and
    ``acrsolve.reduction.matvec`` rebound to ``acrsolve.algebra.matmat``
    (2-D capable, algebra.py:52-62) for the forward sweep (:204-216) and
    back-substitution (:235-256).  The factorisation never reads f, so it is
    the single-column run's; each column differs from a per-column
    ``acr_solve`` only by GEMM-vs-GEMV roundoff (checked on column 0 against
    ``{name}.npz`` when ``check_col0``)."""
    import scipy.linalg
    import acrsolve.reduction as RR
    from acrsolve.problems import assemble_full
    c = P.CONFIGS[name]
    s = P.make_config(name, nrhs=nrhs)
    m, n = s.n_blocks, s.block_dim
    F = s.rhs.reshape(m * n, nrhs)
    rs = R.BlockTridiagSystem(m, n, s.D_sub, s.D_diag, s.D_sup, s.E, s.F,
                              np.ascontiguousarray(F[:, 0]))
    tol = R.Tolerance(c["eps"])
    orig = RR.matvec
    RR.matvec = RA.matmat
    try:
        t0 = time.perf_counter()
        level = RR.lift_system(rs, c["leaf"])
        level.f = [np.ascontiguousarray(F[i * n:(i + 1) * n]) for i in range(m)]
        record = RR.EliminationRecord()
        while level.n_blocks > 1:
            level, entry = RR.reduce_level(level, tol)
            record.entries.append(entry)
        t_red = time.perf_counter()
        A_small = level.to_dense()
        f_small = np.concatenate(level.f)
        lu, piv = scipy.linalg.lu_factor(A_small)
        u_small = scipy.linalg.lu_solve((lu, piv), f_small)
        segs = [u_small[i * n:(i + 1) * n] for i in range(level.n_blocks)]
        u = RR.backsubstitute(record, segs)
        t_end = time.perf_counter()
    finally:
        RR.matvec = orig
    A = assemble_full(rs).tocsr()
    res = np.linalg.norm(A @ u - F, axis=0) / np.linalg.norm(F, axis=0)
    out = {"u_stride": stride, "u": u[::stride], "u_norm": np.linalg.norm(u, axis=0),
           "u_sum": u.sum(axis=0), "residual": res, "nrhs": nrhs,
           "u_proj": projections(u),
           "reduce_ms": (t_red - t0) * 1e3, "backsub_ms": (t_end - t_red) * 1e3}
    if check_col0:
        z = np.load(os.path.join(HERE, f"{name}.npz"))
        st = int(z["u_stride"])
        d = np.linalg.norm(u[::st, 0] - z["u"]) / np.linalg.norm(z["u"])
        out["col0_vs_single"] = d
        out["col0_residual_single"] = float(z["residual"])
        print(name, "column 0 vs single-column acr_solve (rel, subsampled):", d)
    np.savez_compressed(os.path.join(HERE, f"{name}x{nrhs}.npz"), **out)
    print(name, f"x{nrhs}", "residual per column", res, "reduce_ms", out["reduce_ms"])


def mmio_files():
    """Reference ``acr export`` output (cli.py:288-309 via mmio.py:19-62) for
    two small problems: the byte-for-byte target of this package's writer."""
    from acrsolve import cli as RC
    for argv, stem in ((["--problem", "poisson", "--n", "6", "--kappa",
                         "checkerboard:100:2"], "mmio_poisson6"),
                       (["--problem", "convdiff", "--n", "5", "--alpha", "30"],
                        "mmio_convdiff5")):
        rc = RC.main(["export", *argv, "--out", os.path.join(HERE, stem)])
        assert rc == 0
        print("mmio:", stem)


def kernels():
    """truncate_factor and leaf-inverse vectors captured from a config-1
    solve (both module bindings patched)."""
    trunc_calls, inv_calls = [], []
    orig_t = RH.truncate_factor

    def wrap_t(F, tol):
        G = orig_t(F, tol)
        trunc_calls.append((F.U.copy(), F.V.copy(), tol.eps, G.rank,
                            G.to_dense()))
        return G

    orig_solve = np.linalg.solve

    def wrap_solve(a, b):
        x = orig_solve(a, b)
        if a.ndim == 2 and b.ndim == 2 and b.shape == a.shape and \
                np.array_equal(b, np.eye(a.shape[0])):
            inv_calls.append((a.copy(), x.copy()))
        return x

    RH.truncate_factor = wrap_t
    RA.truncate_factor = wrap_t
    RA.np.linalg.solve = wrap_solve
    try:
        s = P.make_config("cfg1")
        R.acr_solve(to_ref(s), R.Tolerance(1e-8), leaf_size=16)
    finally:
        RH.truncate_factor = orig_t
        RA.truncate_factor = orig_t
        RA.np.linalg.solve = orig_solve
    rng = np.random.default_rng(0)
    # keep a diverse sample: every shape class, capped count per class
    by_shape = {}
    for c in trunc_calls:
        key = (c[0].shape, c[1].shape, c[3])
        by_shape.setdefault(key, []).append(c)
    pick = []
    for key in sorted(by_shape):
        lst = by_shape[key]
        idx = rng.choice(len(lst), size=min(2, len(lst)), replace=False)
        pick += [lst[i] for i in sorted(idx)]
    out = {"n_trunc": len(pick)}
    for i, (U, V, eps, r, dense) in enumerate(pick):
        out[f"t{i}/U"] = U
        out[f"t{i}/V"] = V
        out[f"t{i}/eps"] = eps
        out[f"t{i}/rank"] = r
        out[f"t{i}/dense"] = dense
    idx = rng.choice(len(inv_calls), size=min(16, len(inv_calls)), replace=False)
    out["n_inv"] = len(idx)
    for k, i in enumerate(sorted(idx)):
        out[f"i{k}/A"], out[f"i{k}/X"] = inv_calls[i]
    np.savez_compressed(os.path.join(HERE, "kernels_cfg1.npz"), **out)
    print("kernels:", len(trunc_calls), "truncations,", len(pick), "kept;",
          len(inv_calls), "leaf inverses,", len(idx), "kept")


if __name__ == "__main__":
    what = sys.argv[1:] or ["small", "cfg1", "kernels"]
    for w in what:
        if w == "small":
            small()
        elif w == "kernels":
            kernels()
        elif w in ("cfg1", "cfg2"):
            config(w)
        elif w == "cfg3":
            config(w, stride=1)
        elif w in ("cfg4", "cfg5"):
            config(w, stride=64)
        elif w == "mmio":
            mmio_files()
        elif w == "cfg1x16":
            multi_rhs("cfg1", stride=1)
        elif w == "cfg2x16":
            multi_rhs("cfg2", stride=16)
        elif w == "cfg5x16":
            multi_rhs("cfg5", stride=512)
        else:
            raise SystemExit(f"unknown target {w}")
