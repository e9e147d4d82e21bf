"""Multi-worker (N > 1) path on CPU: the plane-partitioned cyclic reduction
(paper_1701_00182_b200/partition.py, the orchestration of the reference's
execute_parallel_factor, parallel.cpp:96-297) over torch.distributed gloo with
world_size 2 and 4.  Checks (test_parallel.cpp:66-123): bitwise-identical solution to
the single-worker run, neighbour-only messages, the message count the schedule implies."""
import os
import socket

import numpy as np
import pytest

from paper_1701_00182_b200 import problems as P
from partition_ref import partitioned_solve, Transport
from paper_1701_00182_b200.plan import plan_schedule, messages


def dense_blocks(sysm):
    d = sysm.dim
    D, E, F = [], [], []
    for j in range(sysm.n):
        M = np.zeros((d, d)); r, c, v = sysm.D(j); np.add.at(M, (r, c), v); D.append(M)
        if j > 0:
            M = np.zeros((d, d)); r, c, v = sysm.E(j); np.add.at(M, (r, c), v); E.append(M)
        else:
            E.append(None)
        if j < sysm.n - 1:
            M = np.zeros((d, d)); r, c, v = sysm.F(j); np.add.at(M, (r, c), v); F.append(M)
        else:
            F.append(None)
    return D, E, F, [sysm.rhs[0][j] for j in range(sysm.n)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sysm = P.config_system(2, n=n)
    D, E, F, f = dense_blocks(sysm)
    plan = plan_schedule(n, world)
    u, ledger = partitioned_solve(D, E, F, f, plan, rank, Transport(rank, world, dist))
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, {j: v.tolist() for j, v in u.items()}, ledger))


@pytest.mark.parametrize("world", [2, 4])
def test_partitioned_gloo_bitwise(world):
    import torch.multiprocessing as mp
    n = 8
    sysm = P.config_system(2, n=n)
    D, E, F, f = dense_blocks(sysm)
    u1, led1 = partitioned_solve(D, E, F, f, plan_schedule(n, 1), 0)
    assert led1 == []
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    u = {}
    ledger = []
    for rank, uu, led in res:
        u.update({j: np.array(v) for j, v in uu.items()})
        ledger += led
    assert sorted(u) == list(range(n))
    for j in range(n):
        assert np.array_equal(u[j], u1[j]), j
    # correct solution of the system
    uu = np.stack([u[j] for j in range(n)])
    assert sysm.relative_residual(uu) <= 1e-9
    # neighbour-only traffic, matching the schedule's message sets
    for (lvl, a, b, nbytes, solve) in ledger:
        assert abs(a - b) == 1 and nbytes > 0
    exp = messages(plan_schedule(n, world))
    n_fac = sum(len(fm) for fm, sm in exp)
    n_sol = sum(len(sm) for fm, sm in exp)
    assert sum(1 for r in ledger if not r[4]) == n_fac
    assert sum(1 for r in ledger if r[4]) == n_sol
