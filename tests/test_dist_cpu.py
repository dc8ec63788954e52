"""N>1 host logic on CPU (gloo, world sizes 2, 3, 4).

An emulation of the sharded schedule of csrc/engine.cu (Plan::reduce halo,
Plan::apply_merges progressive consolidation, Plan::solve halo vectors and
merge replay) written with the CPU oracle's
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
from paper_1604_00617_b200.dist import block_partition, owner, schedule
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
    """Rank-local part of the sharded factor + solve (oracle arithmetic),
    following the engine's schedule: halo of the right active neighbour's
    first even block per level, pairwise merges (progressive consolidation)
    before a level whose windows break the alignment rules, everything on
    rank 0 at the cutoff; the solve replays the merges forward and undoes
    them backward."""
    rank, Pn = dist.get_rank(), dist.get_world_size()
    m = sys_.n_blocks
    t = O.build_node_table(sys_.block_dim, leaf)
    wins, steps, Lt = schedule(m, Pn, cutoff)
    b0 = block_partition(m, Pn)
    full = O.lift(sys_, t)
    lo, hi = b0[rank], b0[rank + 1]
    D, E, F = full.D[lo:hi], full.E[lo:hi], full.F[lo:hi]
    f = [x.copy() for x in full.f[lo:hi]]
    cnt = lambda b: b[rank + 1] - b[rank]                       # noqa: E731
    act = lambda b, r: b[r + 1] > b[r]                          # noqa: E731
    first, mg = lo, m
    records = []
    lret = Lt
    for lvl in range(Lt + 1):
        out = False
        for (sl, before, after) in steps:
            if sl != lvl or cnt(before) <= 0:
                continue
            if cnt(after) <= 0:
                _send((D, E, F, f), owner(after, before[rank]))
                out = True
                break
            if after[rank + 1] == before[rank + 1]:
                continue
            for q in range(rank + 1, Pn):
                if before[q + 1] - before[q] <= 0:
                    continue
                if before[q] >= after[rank + 1]:
                    break
                d2, e2, f2_, ff = _recv(q)
                D, E, F, f = D + d2, E + e2, F + f2_, f + ff
        if out:
            lret = lvl
            break
        if lvl == Lt:
            break
        w = wins[lvl]
        left = next((r for r in range(rank - 1, -1, -1) if act(w, r)), -1)
        rightnb = next((r for r in range(rank + 1, Pn) if act(w, r)), -1)
        mm = len(D)
        right = first + mm < mg
        even = list(range(0, mm, 2))
        Dinv = {i: O.invert(D[i], t, tol) for i in even}
        if first > 0:
            _send((Dinv[0], E[0], F[0], f[0]), left)
        if right:
            hD, Eh, Fh, fh = _recv(rightnb)
            Dinv[mm] = hD
        get_E = lambda i: E[i] if i < mm else Eh               # noqa: E731
        get_F = lambda i: F[i] if i < mm else Fh               # noqa: E731
        get_f = lambda i: f[i] if i < mm else fh               # noqa: E731
        D2, E2, F2, f2 = [], [], [], []
        for j in range(1, mm, 2):
            jg = first + j
            Pj = O.multiply(E[j], Dinv[j - 1], t, tol)
            Dp = O.add(D[j], O.negate(O.multiply(Pj, F[j - 1], t, tol)), t, tol)
            fp = f[j] - O.hmat(E[j], t, 0, O.hmat(Dinv[j - 1], t, 0, f[j - 1]))
            Ep = O.negate(O.multiply(Pj, E[j - 1], t, tol)) if jg >= 2 else None
            Fp = None
            if jg + 1 <= mg - 1:
                Qj = O.multiply(F[j], Dinv[j + 1], t, tol)
                Dp = O.add(Dp, O.negate(O.multiply(Qj, get_E(j + 1), t, tol)), t, tol)
                fp = fp - O.hmat(F[j], t, 0, O.hmat(Dinv[j + 1], t, 0, get_f(j + 1)))
                if jg + 2 <= mg - 1:
                    Fp = O.negate(O.multiply(Qj, get_F(j + 1), t, tol))
            D2.append(Dp); E2.append(Ep); F2.append(Fp); f2.append(fp)
        records.append(dict(m=mm, first=first, mg=mg, right=right, left=left,
                            rightnb=rightnb, Dinv=[Dinv[i] for i in even], E=E, F=F, f=f))
        D, E, F, f = D2, E2, F2, f2
        first, mg = first // 2, mg // 2
    u = None
    if rank == 0:
        lv = O.Level(Lt, D, E, F, f)
        us = O.dense_lu_solve(lv.to_dense(t), np.concatenate(lv.f))
        n = t.n
        u = [us[i * n:(i + 1) * n] for i in range(lv.m)]
    for lvl in range(lret, -1, -1):
        for (sl, before, after) in reversed(steps):
            if sl != lvl or cnt(before) <= 0:
                continue
            if cnt(after) <= 0:
                u = _recv(owner(after, before[rank]))
                continue
            if after[rank + 1] == before[rank + 1]:
                continue
            for q in range(rank + 1, Pn):
                c = before[q + 1] - before[q]
                if c <= 0:
                    continue
                if before[q] >= after[rank + 1]:
                    break
                off = before[q] - after[rank]
                _send(u[off:off + c], q)
            u = u[:cnt(before)]
        if lvl == 0:
            break
        rec = records[lvl - 1]
        mm, fr, mgl = rec["m"], rec["first"], rec["mg"]
        full_u = [None] * mm
        for k, j in enumerate(range(1, mm, 2)):
            full_u[j] = u[k]
        if rec["right"]:
            _send(full_u[mm - 1], rec["rightnb"])
        uleft = _recv(rec["left"]) if fr > 0 else None
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
    "rand32_c3": (P.random_system(32, 8, seed=5), Tolerance(1e-10), 4, 3),
}


@pytest.mark.parametrize("world", [2, 3, 4])
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
