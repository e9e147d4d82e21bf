"""Multi-GPU plane partition (execute_parallel_factor, parallel.cpp:96-297) through
the C-ABI, checked on one GPU with in-process ranks (acrgpu_comm_create_local): the
partitioned factor/solve must be bitwise identical to the single-rank path for
every rank count (the reference's contract, test_parallel.cpp:75-89), with the same
stored-inverse statistics, and must reject what plan_schedule rejects
(parallel.cpp:383-405).  The NCCL transport moves the same wire images between
processes; its host schedule is the one exercised here."""
import numpy as np
import pytest

from paper_1701_00182_b200 import problems as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def acr():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1701_00182_b200 import acr as A
    A.lib()
    return A


def _levels(f):
    return [(l.plane_count, l.eliminated, l.largest_rank, round(l.average_rank, 9), l.bytes) for l in f.level_info()]


@pytest.mark.parametrize("name,p", [("poisson16", 2), ("poisson16", 4), ("poisson16", 8), ("poisson16", 16),
                                    ("c2n16", 4), ("c3n16", 2)])
def test_partitioned_bitwise(acr, name, p):                                     # test_parallel.cpp:75-89
    sysm = {"poisson16": lambda: P.poisson(16), "c2n16": lambda: P.config_system(2, n=16),
            "c3n16": lambda: P.config_system(3, n=16)}[name]()
    eps = 1e-3 if name == "poisson16" else 1e-6
    cfg = acr.AcrConfig(eps=eps)
    f1 = acr.acr_factor(sysm, cfg)
    u1 = f1.solve(sysm.rhs)
    comm = acr.Comm.local_ranks(p)
    fp = acr.acr_factor_partitioned(sysm, comm, cfg)
    up = fp.solve(sysm.rhs)
    assert np.array_equal(u1, up)
    s1, sp = f1.inverse_rank_stats(), fp.inverse_rank_stats()
    assert (s1.average_rank, s1.largest_rank, s1.bytes) == (sp.average_rank, sp.largest_rank, sp.bytes)
    assert f1.factor_bytes() == fp.factor_bytes()
    assert _levels(f1) == _levels(fp)
    for lvl in range(len(f1.level_info()) - 1):
        m = f1.level_info()[lvl].plane_count
        for j in range(0, m, 2):
            a, b = f1.dinv_ranks(lvl, j), fp.dinv_ranks(lvl, j)
            if a is not None or b is not None:
                assert np.array_equal(a, b), (lvl, j)


def test_partitioned_config1_multi_rhs(acr):
    sysm = P.config_system(1, nrhs=3)
    cfg = acr.AcrConfig(eps=1e-6)
    u1 = acr.acr_factor(sysm, cfg).solve(sysm.rhs)
    fp = acr.acr_factor_partitioned(sysm, acr.Comm.local_ranks(8), cfg)
    up = fp.solve(sysm.rhs)
    assert np.array_equal(u1, up)
    assert sysm.relative_residual(up) < 1e-5


def test_partition_schedule_errors(acr):                                        # parallel.cpp:383-405
    with pytest.raises(acr.UsageError):
        acr.acr_factor_partitioned(P.poisson(12), acr.Comm.local_ranks(2), acr.AcrConfig(eps=1e-3))
    with pytest.raises(acr.UsageError):
        acr.acr_factor_partitioned(P.poisson(8), acr.Comm.local_ranks(3), acr.AcrConfig(eps=1e-3))
    with pytest.raises(acr.UsageError):
        acr.acr_factor_partitioned(P.poisson(4), acr.Comm.local_ranks(8), acr.AcrConfig(eps=1e-3))
    with pytest.raises(acr.UsageError):
        acr.acr_factor_partitioned(P.poisson(8), acr.Comm.local_ranks(2), acr.AcrConfig(eps=1e-3, stop_planes=2))


def test_partitioned_singular_location(acr):                                    # parallel.cpp:353-354
    n, d = 4, 16
    I = (np.arange(d, dtype=np.int32), np.arange(d, dtype=np.int32), np.ones(d))
    Z = (np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0))
    sysm = P._assemble(n, d, P.plane_coords(4), [I, I, Z, I] + [Z] * 6, np.ones((1, n, d)))
    with pytest.raises(acr.SingularBlockError) as ei:
        acr.acr_factor_partitioned(sysm, acr.Comm.local_ranks(2), acr.AcrConfig(eps=1e-6, leaf_size=8))
    assert ei.value.level == 0 and ei.value.plane == 2


def test_nccl_transport_single_rank(acr):
    """NCCL communicator through the library (dlopen'ed libnccl): a one-rank partition runs
    the same exchange code with empty message lists and matches the single-rank path."""
    sysm = P.poisson(8)
    cfg = acr.AcrConfig(eps=1e-3)
    u1 = acr.acr_factor(sysm, cfg).solve(sysm.rhs)
    uid = acr.Comm.unique_id()
    assert len(uid) == acr.COMM_ID_BYTES
    comm = acr.Comm.nccl(uid, 1, 0)
    f = acr.acr_factor_partitioned(sysm, comm, cfg)
    assert np.array_equal(f.solve(sysm.rhs), u1)
    del f
    comm.close()
