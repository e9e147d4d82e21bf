"""The plane partition across REAL processes (execute_parallel_factor, parallel.cpp:96-297),
through libacrgpu.so: two processes share the one GPU of the test box, each with its own
CUDA context, and the wire images travel over the host-staged communicator
(acrgpu_comm_create_host) driven by torch.distributed isend/irecv on gloo.  Everything the
NCCL path runs on each rank -- lifting its own planes, pack_store / adopt_image of
{Dinv, E, F}, the (peer, key) message ordering, the per-level exchange, the partitioned
solve -- runs here across address spaces; only the final byte transfer differs.

Contract (test_parallel.cpp:75-101): the gathered solution is bitwise equal to the
single-GPU factor/solve, the per-rank message ledger equals the in-process partition's, and
every stored inverse a rank owns has the single-GPU leaf ranks."""
import json
import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = {
    "c2n16_p2": dict(config=2, n=16, p=2, eps=1e-6),
    "c3n16_p2": dict(config=3, n=16, p=2, eps=1e-6),
    "poisson16_p4": dict(config=1, n=16, p=4, eps=1e-3),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _system(case):
    from paper_1701_00182_b200 import problems as P
    c = CASES[case]
    return P.config_system(c["config"], n=c["n"], nrhs=2)


def _worker(rank, world, port, case, outdir):
    # several contexts share one GPU: small arenas
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), ACRGPU_PERSIST_FRAC="0.08",
                      ACRGPU_TRANS_FRAC="0.05")
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1701_00182_b200 import acr
    sysm = _system(case)
    cfg = acr.AcrConfig(eps=CASES[case]["eps"])
    ctx = acr.Context(0)
    comm = acr.Comm.host(acr.torch_exchange(), world, rank)
    f = acr.acr_factor_partitioned(sysm, comm, cfg, ctx=ctx)
    u = f.solve(sysm.rhs)                      # this rank's planes; zero elsewhere
    ut = torch.from_numpy(np.ascontiguousarray(u))
    dist.all_reduce(ut)                        # x + 0 is exact: the gathered u is bitwise
    dinv = {}
    for li, lv in enumerate(f.level_info()[:-1]):
        for j in range(lv.plane_count):
            r = f.dinv_ranks(li, j)
            if r is not None:
                dinv[f"{li}:{j}"] = [int(x) for x in r]
    st = f.inverse_rank_stats()
    out = dict(rank=rank, dinv=dinv, largest=st.largest_rank, lowrank=st.lowrank_leaf_count,
               rank_sum=st.average_rank * st.lowrank_leaf_count, bytes=f.factor_bytes(),
               messages=[(m.level, m.from_plane, m.to_plane, m.bytes) for m in f.messages()])
    np.save(os.path.join(outdir, f"u{rank}.npy"), ut.numpy())
    with open(os.path.join(outdir, f"r{rank}.json"), "w") as fh:
        json.dump(out, fh)
    del f
    comm.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", list(CASES))
def test_multiprocess_partition_bitwise(case):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    from paper_1701_00182_b200 import acr
    p = CASES[case]["p"]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(p, _free_port(), case, d), nprocs=p, join=True)
        us = [np.load(os.path.join(d, f"u{r}.npy")) for r in range(p)]
        rs = [json.load(open(os.path.join(d, f"r{r}.json"))) for r in range(p)]
    sysm = _system(case)
    cfg = acr.AcrConfig(eps=CASES[case]["eps"])
    f1 = acr.acr_factor(sysm, cfg)
    u1 = f1.solve(sysm.rhs)
    for u in us:
        assert np.array_equal(u, u1)
    # ledger: each process records its own sends; together they are the in-process ledger
    fl = acr.acr_factor_partitioned(sysm, acr.Comm.local_ranks(p), cfg)
    local = sorted((m.level, m.from_plane, m.to_plane, m.bytes) for m in fl.messages())
    multi = sorted(tuple(m) for r in rs for m in r["messages"])
    assert multi == local and len(local) > 0
    # stored inverses: every rank's own planes have the single-GPU leaf ranks
    seen = set()
    for r in rs:
        for key, ranks in r["dinv"].items():
            li, j = map(int, key.split(":"))
            assert np.array_equal(np.asarray(ranks), f1.dinv_ranks(li, j)), key
            seen.add(key)
    m0 = f1.level_info()[0].plane_count
    assert {f"0:{j}" for j in range(0, m0, 2)} <= seen
    s1 = f1.inverse_rank_stats()
    assert max(r["largest"] for r in rs) == s1.largest_rank
    assert sum(r["lowrank"] for r in rs) == s1.lowrank_leaf_count
    assert abs(sum(r["rank_sum"] for r in rs) - s1.average_rank * s1.lowrank_leaf_count) <= 1e-6
