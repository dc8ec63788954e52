"""Sharded factor + solve over NCCL, one process per GPU.

Needs >= 2 GPUs (skipped otherwise; the one-GPU boxes of this build run the
same sharded C++ schedule through the loopback transport in
test_gpu_dist.py).  Each rank owns a contiguous block-row window; the
result must match the single-GPU solve (1e-9: a shard's smaller batches
may route a recompression through another kernel path) and the report's
rank profile of rank 0's window must be a valid one."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q):
    import torch.distributed as dist
    from paper_1604_00617_b200 import problems as P
    from paper_1604_00617_b200.dist import DistAcrSolver
    from paper_1604_00617_b200.system import Tolerance
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "WARN"))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        c = P.CONFIGS[cfg]
        s = P.make_config(cfg, nrhs=2)
        sol = DistAcrSolver(s.n_blocks, s.block_dim, Tolerance(c["eps"]), 1, c["leaf"])
        bands = [torch.as_tensor(np.ascontiguousarray(a), device="cuda")
                 for a in (s.D_sub, s.D_diag, s.D_sup, s.E, s.F)]
        sol.factor(bands)
        f = torch.as_tensor(s.rhs, device="cuda")
        u = sol.solve(f)
        dist.all_reduce(u)                 # each rank wrote its own rows
        if rank == 0:
            q.put(u.cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_nccl_sharded_matches_single_gpu(world):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp
    from paper_1604_00617_b200 import problems as P
    from paper_1604_00617_b200.solver import acr_solve
    from paper_1604_00617_b200.system import Tolerance
    cfg = "cfg2"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    u = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    c = P.CONFIGS[cfg]
    u1, _ = acr_solve(P.make_config(cfg, nrhs=2), Tolerance(c["eps"]), leaf_size=c["leaf"])
    assert np.linalg.norm(u - u1) <= 1e-9 * np.linalg.norm(u1)
