"""N>1 host logic on CPU (gloo, world size 2 and 3).

An emulation of the sharded schedule of csrc/engine.cu (Plan::reduce halo,
Plan::consolidate, Plan::solve halo vectors) written with the CPU oracle's
HODLR operations and torch.distributed point-to-point messages.  The same
partition rules (paper_1604_00617_b200.dist) decide windows and the
consolidation level.  Because each block's arithmetic is unchanged by the
sharding, the result must equal the single-process oracle bitwise -- this
checks that the halo data (right neighbour's first even block: Dinv, E, F;
one vector per boundary in the solve) is sufficient and correctly placed.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import acr_oracle as O
from paper_1604_00617_b200 import problems as P
from paper_1604_00617_b200.dist import block_partition, distributed_ok, level_bounds
from paper_1604_00617_b200.system import Tolerance


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _send(obj, dst):
    dist.send_object_list([obj], dst=dst)


def _recv(src):
    box = [None]
    dist.recv_object_list(box, src=src)
    return box[0]


def sharded_solve(sys_, tol, leaf, cutoff=1):
    """Rank-local part of the sharded factor + solve (oracle arithmetic)."""
    rank, Pn = dist.get_rank(), dist.get_world_size()
    m = sys_.n_blocks
    t = O.build_node_table(sys_.block_dim, leaf)
    b0 = block_partition(m, Pn)
    full = O.lift(sys_, t)
    lo, hi = b0[rank], b0[rank + 1]
    # window of level 0; E/F None outside the global system
    D, E, F = full.D[lo:hi], full.E[lo:hi], full.F[lo:hi]
    f = [x.copy() for x in full.f[lo:hi]]
    first, mg = lo, m
    records = []
    lvl = 0
    while mg > cutoff and distributed_ok(b0, m, lvl):
        mm = len(D)
        right = first + mm < mg
        even = list(range(0, mm, 2))
        Dinv = {i: O.invert(D[i], t, tol) for i in even}
        # halo: our first even block to the left, the right neighbour's to us
        if first > 0:
            _send((Dinv[0], E[0], F[0]), rank - 1)
        if right:
            hD, hE, hF = _recv(rank + 1)
            Dinv[mm], Eh, Fh = hD, hE, hF
        get_E = lambda i: E[i] if i < mm else Eh
        get_F = lambda i: F[i] if i < mm else Fh
        D2, E2, F2 = [], [], []
        for j in range(1, mm, 2):
            jg = first + j
            Pj = O.multiply(E[j], Dinv[j - 1], t, tol)
            Dp = O.add(D[j], O.negate(O.multiply(Pj, F[j - 1], t, tol)), t, tol)
            Ep = O.negate(O.multiply(Pj, E[j - 1], t, tol)) if jg >= 2 else None
            Fp = None
            if jg + 1 <= mg - 1:
                Qj = O.multiply(F[j], Dinv[j + 1], t, tol)
                Dp = O.add(Dp, O.negate(O.multiply(Qj, get_E(j + 1), t, tol)), t, tol)
                if jg + 2 <= mg - 1:
                    Fp = O.negate(O.multiply(Qj, get_F(j + 1), t, tol))
            D2.append(Dp); E2.append(Ep); F2.append(Fp)
        records.append(dict(m=mm, first=first, mg=mg, right=right,
                            Dinv=[Dinv[i] for i in even], E=E, F=F))
        D, E, F = D2, E2, F2
        first, mg = first // 2, mg // 2
        lvl += 1
    Ld = lvl
    # consolidation of level Ld on rank 0
    gathered = [None] * Pn if rank == 0 else None
    dist.gather_object((D, E, F), gathered, dst=0)
    # ---- solve: forward sweep over the sharded levels ----
    for rec in records:
        mm, fr, mgl = rec["m"], rec["first"], rec["mg"]
        z = {i: O.hmat(rec["Dinv"][i // 2], t, 0, f[i]) for i in range(0, mm, 2)}
        if fr > 0:
            _send(z[0], rank - 1)
        if rec["right"]:
            z[mm] = _recv(rank + 1)
        f2 = []
        for j in range(1, mm, 2):
            fp = f[j] - O.hmat(rec["E"][j], t, 0, z[j - 1])
            if fr + j + 1 <= mgl - 1:
                fp = fp - O.hmat(rec["F"][j], t, 0, z[j + 1])
            f2.append(fp)
        rec["f"] = f
        f = f2
    fg = [None] * Pn if rank == 0 else None
    dist.gather_object(f, fg, dst=0)
    if rank == 0:
        D = [b for part in gathered for b in part[0]]
        E = [b for part in gathered for b in part[1]]
        F = [b for part in gathered for b in part[2]]
        ff = [x for part in fg for x in part]
        lv = O.Level(Ld, D, E, F, ff)
        top = []
        while lv.m > cutoff:
            lv, rec = O.reduce_level(lv, t, tol)
            top.append(rec)
        us = O.dense_lu_solve(lv.to_dense(t), np.concatenate(lv.f))
        n = t.n
        u_top = O.backsubstitute(top, t, [us[i * n:(i + 1) * n] for i in range(lv.m)])
        bnd = level_bounds(b0, m, Ld)
        segs = [u_top[i * n:(i + 1) * n] for i in range(bnd[-1])]
        parts = [segs[bnd[r]:bnd[r + 1]] for r in range(Pn)]
    else:
        parts = None
    box = [None]
    dist.scatter_object_list(box, parts, src=0)
    u = box[0]
    # ---- back-substitution over the sharded levels ----
    for rec in reversed(records):
        mm, fr, mgl = rec["m"], rec["first"], rec["mg"]
        full_u = [None] * mm
        for k, j in enumerate(range(1, mm, 2)):
            full_u[j] = u[k]
        if rec["right"]:
            _send(full_u[mm - 1], rank + 1)
        uleft = _recv(rank - 1) if fr > 0 else None
        for i in range(0, mm, 2):
            r = rec["f"][i].copy()
            if fr + i >= 1:
                r = r - O.hmat(rec["E"][i], t, 0, full_u[i - 1] if i > 0 else uleft)
            if fr + i <= mgl - 2:
                r = r - O.hmat(rec["F"][i], t, 0, full_u[i + 1])
            full_u[i] = O.hmat(rec["Dinv"][i // 2], t, 0, r)
        u = full_u
    out = [None] * Pn if rank == 0 else None
    dist.gather_object(u, out, dst=0)
    return np.concatenate([x for part in out for x in part]) if rank == 0 else None


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s, tol, leaf, cutoff = case
        u = sharded_solve(s, tol, leaf, cutoff)
        if rank == 0:
            q.put(u)
    finally:
        dist.destroy_process_group()


CASES = {
    "rand16": (P.random_system(16, 16, seed=31), Tolerance(1e-10), 4, 1),
    "rand13_c2": (P.random_system(13, 8, seed=2), Tolerance(1e-10), 4, 2),
    "poisson32": (P.poisson_const(32, seed=1), Tolerance(1e-8), 8, 1),
}


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", sorted(CASES))
def test_sharded_schedule_matches_single_process(world, name):
    s, tol, leaf, cutoff = CASES[name]
    if s.n_blocks < 2 * world:
        pytest.skip("too few blocks")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES[name], q))
             for r in range(world)]
    for p in procs:
        p.start()
    u = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref, _ = O.acr_solve(s, tol, cutoff_blocks=cutoff, leaf_size=leaf)
    np.testing.assert_array_equal(u, ref)
