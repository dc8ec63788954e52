"""Matrix Market / right-hand-side text I/O (reference ``mmio.py:19-62``).

Same file format byte for byte: ``coordinate real general``, 1-based
indices, triplets in row-major order, values as ``%.17g`` (exact round
trip of doubles), one vector entry per line.  The writers format whole
arrays at once (numpy ``savetxt``) instead of a Python loop per entry, so a
config-5 export (21 M nonzeros) takes seconds, not minutes.  Used by
``acr export``; not on the solve path.
"""

from __future__ import annotations

import numpy as np

__all__ = ["write_matrix_market", "read_matrix_market", "write_vector",
           "read_vector", "system_to_coo", "coo_to_system"]

_HEADER = "%%MatrixMarket matrix coordinate real general"


def write_matrix_market(path, A, comment: str = ""):
    import scipy.sparse as sp
    A = sp.coo_matrix(A)
    order = np.lexsort((A.col, A.row))
    tab = np.empty(len(order), dtype=[("r", np.int64), ("c", np.int64), ("v", np.float64)])
    tab["r"] = A.row[order] + 1
    tab["c"] = A.col[order] + 1
    tab["v"] = A.data[order]
    with open(path, "w") as fh:
        fh.write(_HEADER + "\n")
        for line in comment.splitlines() if comment else []:
            fh.write(f"% {line}\n")
        fh.write(f"{A.shape[0]} {A.shape[1]} {len(order)}\n")
        np.savetxt(fh, tab, fmt="%d %d %.17g")


def read_matrix_market(path):
    import scipy.sparse as sp
    with open(path) as fh:
        header = fh.readline().strip()
        if header != _HEADER:
            raise ValueError(f"unsupported Matrix Market header: {header!r}")
        line = fh.readline()
        while line.startswith("%"):
            line = fh.readline()
        m, n, nnz = (int(t) for t in line.split())
        data = np.loadtxt(fh, dtype=np.float64, ndmin=2) if nnz else np.zeros((0, 3))
    if data.shape[0] != nnz:
        raise ValueError(f"expected {nnz} entries, found {data.shape[0]}")
    rows = data[:, 0].astype(np.int64) - 1
    cols = data[:, 1].astype(np.int64) - 1
    return sp.coo_matrix((data[:, 2], (rows, cols)), shape=(m, n))


def write_vector(path, v):
    v = np.asarray(v, dtype=np.float64).reshape(-1)
    with open(path, "w") as fh:
        np.savetxt(fh, v, fmt="%.17g")


def read_vector(path) -> np.ndarray:
    return np.atleast_1d(np.loadtxt(path, dtype=np.float64))


def system_to_coo(sys):
    """The assembled operator of a ``BlockTridiagSystem`` (reference
    ``problems.assemble_full``, ``problems.py:227-255``)."""
    from .stencils import assemble_full
    return assemble_full(sys)


def coo_to_system(A, block_dim: int, rhs, name: str = "mtx"):
    """Band storage of a block tridiagonal matrix read from Matrix Market:
    D_i tridiagonal, E_i / F_i diagonal.  Entries outside that pattern raise
    ``ValueError`` (the solver has no representation for them)."""
    import scipy.sparse as sp
    from .system import BlockTridiagSystem
    A = sp.coo_matrix(A)
    N = A.shape[0]
    n = int(block_dim)
    if A.shape[0] != A.shape[1] or n < 2 or N % n:
        raise ValueError(f"matrix {A.shape} is not square with blocks of {n}")
    m = N // n
    r, c, v = A.row.astype(np.int64), A.col.astype(np.int64), A.data
    br, bc, ir, ic = r // n, c // n, r % n, c % n
    D_sub, D_diag, D_sup = np.zeros((m, n - 1)), np.zeros((m, n)), np.zeros((m, n - 1))
    E, F = np.zeros((max(m - 1, 0), n)), np.zeros((max(m - 1, 0), n))
    used = np.zeros(len(v), dtype=bool)
    same = br == bc
    for mask, tgt, bi, ii in (
            (same & (ic == ir), D_diag, br, ir),
            (same & (ic == ir + 1), D_sup, br, ir),
            (same & (ic + 1 == ir), D_sub, br, ic),
            ((br == bc + 1) & (ir == ic), E, bc, ic),
            ((bc == br + 1) & (ir == ic), F, br, ir)):
        np.add.at(tgt, (bi[mask], ii[mask]), v[mask])
        used |= mask
    if not used.all():
        k = int(np.flatnonzero(~used)[0])
        raise ValueError(f"entry ({r[k] + 1}, {c[k] + 1}) is outside the block "
                         f"tridiagonal pattern for block size {n}")
    return BlockTridiagSystem(m, n, D_sub, D_diag, D_sup, E, F,
                              np.asarray(rhs, dtype=np.float64), name=name)
