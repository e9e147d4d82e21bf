"""Pins the CPU oracle's H-matrix arithmetic to the reference's own tests
(proj/tests/test_hmatrix.cpp, test_cluster.cpp).  The reference ships no
golden vectors; each test below restates one reference TEST_CASE with its
tolerance (cited file:line)."""
import numpy as np
import pytest

from paper_1701_00182_b200 import problems as P


def grid(side):
    return np.array([[x, y] for y in range(side) for x in range(side)], float)


def ident_coords(dim):
    side = int(round(np.sqrt(dim)))
    return np.stack([np.arange(dim) % side, np.arange(dim) // side], 1).astype(float)


def random_matrix(r, c, seed):
    return P.uniform_pm1(seed, 7, r * c).reshape(c, r).T.copy()


def fixture(oracle, side, leaf, eta=2.0, weak=False):
    r, c, v, coords = P.poisson2d_block(side)
    return oracle.Structure(coords, leaf, eta, weak), (r, c, v)


# ---- cluster tree pins (test_cluster.cpp)
def test_cluster_shapes(oracle):
    assert oracle.Structure(np.array([[0.5, 0.5]]), 32).cluster_info() == (1, 0)      # :31-36
    assert oracle.Structure(grid(4), 4).cluster_info() == (4, 2)                       # :38-45
    s = oracle.Structure(grid(64), 32)                                                  # :48-55
    assert s.cluster_info()[0] == 128
    p = oracle.Structure(grid(8), 4).perm()                                             # :61-86
    assert sorted(p.tolist()) == list(range(64))


def test_admissibility_pair(oracle):                                                    # :104-114
    s = oracle.Structure(np.array([[0, 0], [0, 1], [3, 0], [3, 1]], float), 2)
    kinds = s.leaves()[:, 4]
    assert (kinds == 1).sum() >= 2


def test_dense_leaves_only_where_inadmissible(oracle):                                  # :116-137
    s, _ = fixture(oracle, 32, 32)
    lv = s.leaves()
    assert (lv[:, 4] == 1).sum() > 0 and (lv[:, 4] == 0).sum() > 0
    area = ((lv[:, 1] - lv[:, 0]) * (lv[:, 3] - lv[:, 2])).sum()
    assert area == 1024 * 1024


def test_weak_coarser(oracle):                                                          # :139-165
    w = oracle.Structure(grid(16), 8, 2.0, True).leaves()
    s = oracle.Structure(grid(16), 8, 2.0, False).leaves()
    for rb, re, cb, ce, k in w:
        if re <= cb or ce <= rb:
            assert k == 1
    assert len(w) <= len(s)


# ---- H-matrix pins (test_hmatrix.cpp)
def test_zero_and_identity(oracle):                                                     # :63-80
    s = oracle.Structure(ident_coords(256), 8)
    z = oracle.HMatrix.compress_sparse(s, [], [], [], 1e-6)
    st = z.rank_stats()
    assert st["largest_rank"] == 0 and st["average_rank"] == 0.0
    assert np.linalg.norm(z.to_dense()) == 0.0
    i = np.arange(256)
    I = oracle.HMatrix.compress_sparse(s, i, i, np.ones(256), 1e-6)
    assert I.rank_stats()["largest_rank"] == 0
    assert np.linalg.norm(I.to_dense() - np.eye(256)) <= 1e-14
    x = P.uniform_pm1(1, 3, 256)
    assert np.linalg.norm(I.apply(x) - x) <= 1e-12 * np.linalg.norm(x)


def test_poisson_plane_matvec_bound(oracle):                                            # :88-99
    eps = 1e-4
    s, (r, c, v) = fixture(oracle, 32, 32)
    H = oracle.HMatrix.compress_sparse(s, r, c, v, eps)
    A = np.zeros((1024, 1024))
    np.add.at(A, (r, c), v)
    anorm = np.linalg.norm(A)
    for t in range(20):
        x = P.uniform_pm1(100 + t, 3, 1024)
        assert np.linalg.norm(H.apply(x) - A @ x) <= 10 * eps * anorm * np.linalg.norm(x)


def test_random_dense_matvec(oracle):                                                   # :101-110
    s = oracle.Structure(ident_coords(64), 8)
    A = random_matrix(64, 64, 5)
    H = oracle.HMatrix.compress_dense(s, A, 1e-8)
    x = P.uniform_pm1(6, 3, 64)
    assert np.linalg.norm(H.apply(x) - A @ x) <= 1e-6 * np.linalg.norm(A @ x)


def test_matvec_dimension_error(oracle):                                                # :112-116
    s, (r, c, v) = fixture(oracle, 16, 8)
    H = oracle.HMatrix.compress_sparse(s, r, c, v, 1e-6)
    with pytest.raises(oracle.OracleError):
        H.apply(np.zeros(100))


def test_add_sub_identities(oracle):                                                    # :118-128
    s, (r, c, v) = fixture(oracle, 16, 8)
    eps = 1e-8
    A = oracle.HMatrix.compress_sparse(s, r, c, v, eps)
    Z = oracle.HMatrix.compress_sparse(s, [], [], [], eps)
    assert np.linalg.norm(A.add(Z, 1.0, eps).to_dense() - A.to_dense()) <= 1e-12
    D = A.add(A, -1.0, eps)
    assert np.linalg.norm(D.to_dense()) <= 1e-12
    assert D.rank_stats()["largest_rank"] == 0


def test_lowrank_addition(oracle):                                                      # :130-145
    s = oracle.Structure(ident_coords(64), 16, 2.0, True)
    A = random_matrix(64, 3, 8) @ random_matrix(3, 64, 9)
    B = random_matrix(64, 4, 10) @ random_matrix(4, 64, 11)
    eps = 1e-10
    Hs = oracle.HMatrix.compress_dense(s, A, eps).add(oracle.HMatrix.compress_dense(s, B, eps), 1.0, eps)
    assert Hs.rank_stats()["largest_rank"] <= 7
    assert np.linalg.norm(Hs.to_dense() - (A + B)) <= 100 * eps * np.linalg.norm(A + B)


def test_truncate_lowrank(oracle):                                                      # :147-157
    U = random_matrix(32, 6, 21)
    V = random_matrix(32, 6, 22)
    M = U @ V.T
    U2, V2 = oracle.truncate(U, V, 1e-12)
    assert U2.shape[1] <= 6
    assert np.linalg.norm(U2 @ V2.T - M) <= 1e-10 * np.linalg.norm(M)
    U3, V3 = oracle.truncate(U2, V2, 0.999)
    assert U3.shape[1] == 1


def test_svd_values_match_numpy(oracle):
    for shape in ((5, 5), (32, 32), (40, 17), (17, 40)):
        A = random_matrix(*shape, 3)
        np.testing.assert_allclose(oracle.svd_values(A), np.linalg.svd(A, compute_uv=False), rtol=1e-12, atol=1e-13)


def test_lu_inverse(oracle):
    A = random_matrix(32, 32, 4) + 8 * np.eye(32)
    inv, rc = oracle.lu_inverse(A)
    assert np.linalg.norm(inv @ A - np.eye(32)) <= 1e-12
    rc_np = 1.0 / (np.linalg.norm(A, 1) * np.linalg.norm(np.linalg.inv(A), 1))
    assert rc_np / 3 <= rc <= rc_np * 1.0000001 * 3
    _, rc0 = oracle.lu_inverse(np.zeros((8, 8)))
    assert rc0 == 0.0


def test_hmultiply_identities(oracle):                                                  # :159-168
    s, (r, c, v) = fixture(oracle, 16, 8)
    eps = 1e-8
    A = oracle.HMatrix.compress_sparse(s, r, c, v, eps)
    i = np.arange(256)
    I = oracle.HMatrix.compress_sparse(s, i, i, np.ones(256), eps)
    Z = oracle.HMatrix.compress_sparse(s, [], [], [], eps)
    Ad = A.to_dense()
    assert np.linalg.norm(A.multiply(I, eps).to_dense() - Ad) <= 100 * eps * np.linalg.norm(Ad)
    assert np.linalg.norm(A.multiply(Z, eps).to_dense()) <= 1e-12


def test_hmultiply_random(oracle):                                                      # :170-181
    s = oracle.Structure(ident_coords(64), 8)
    A = random_matrix(64, 64, 31)
    B = random_matrix(64, 64, 32)
    eps = 1e-8
    Pm = oracle.HMatrix.compress_dense(s, A, eps).multiply(oracle.HMatrix.compress_dense(s, B, eps), eps).to_dense()
    assert np.linalg.norm(Pm - A @ B) <= 1e-6 * np.linalg.norm(A @ B)


def test_hinvert_identities(oracle):                                                    # :183-195
    s, _ = fixture(oracle, 16, 8)
    eps = 1e-8
    i = np.arange(256)
    I = oracle.HMatrix.compress_sparse(s, i, i, np.ones(256), eps)
    assert np.linalg.norm(I.invert(eps).to_dense() - np.eye(256)) <= 1e-10
    D = oracle.HMatrix.compress_sparse(s, i, i, 2.0 * (i + 1), eps)
    np.testing.assert_allclose(np.diag(D.invert(eps).to_dense()), 1.0 / (2.0 * (i + 1)), rtol=1e-12)


def test_hinvert_poisson_bound(oracle):                                                 # :197-208
    eps = 1e-4
    s, (r, c, v) = fixture(oracle, 32, 32)
    H = oracle.HMatrix.compress_sparse(s, r, c, v, eps)
    Hinv = H.invert(eps)
    Pm = H.multiply(Hinv, eps).to_dense()
    assert np.linalg.norm(Pm - np.eye(1024)) / np.sqrt(1024) <= 100 * eps


def test_singular_pivot(oracle):                                                        # :210-214
    s, _ = fixture(oracle, 16, 8)
    Z = oracle.HMatrix.compress_sparse(s, [], [], [], 1e-8)
    with pytest.raises(oracle.OracleError) as ei:
        Z.invert(1e-8)
    assert ei.value.code == 2


def test_rank_stats_accounting(oracle):                                                 # :216-226
    s, _ = fixture(oracle, 16, 8)
    i = np.arange(256)
    I = oracle.HMatrix.compress_sparse(s, i, i, np.ones(256), 1e-8)
    st = I.rank_stats()
    assert st["largest_rank"] == 0 and st["bytes"] > 0


def test_leafwise_reconstruction(oracle):                                               # :240-258 (via dense)
    eps = 1e-3
    s, (r, c, v) = fixture(oracle, 32, 32)
    H = oracle.HMatrix.compress_sparse(s, r, c, v, eps)
    A = np.zeros((1024, 1024))
    np.add.at(A, (r, c), v)
    assert np.linalg.norm(H.to_dense() - A) <= eps * np.linalg.norm(A) * 1.0001


def test_bytes_monotone_in_eps(oracle):                                                 # :260-270
    s, (r, c, v) = fixture(oracle, 32, 32)
    prev = 0
    for eps in (1e-1, 1e-2, 1e-3, 1e-4):
        b = oracle.HMatrix.compress_sparse(s, r, c, v, eps).rank_stats()["bytes"]
        assert b >= prev
        prev = b


def test_weak_needs_larger_rank(oracle):                                                # :272-281
    eps = 1e-4
    r, c, v, coords = P.poisson2d_block(32)
    ss = oracle.Structure(coords, 32, 2.0, False)
    sw = oracle.Structure(coords, 32, 2.0, True)
    ist = oracle.HMatrix.compress_sparse(ss, r, c, v, eps).invert(eps)
    iwk = oracle.HMatrix.compress_sparse(sw, r, c, v, eps).invert(eps)
    assert iwk.rank_stats()["largest_rank"] >= ist.rank_stats()["largest_rank"]


def test_recompress(oracle):                                                            # :283-294
    r, c, v, coords = P.poisson2d_block(32)
    s = oracle.Structure(coords, 32)
    H = oracle.HMatrix.compress_sparse(s, r, c, v, 1e-10)
    inv = H.invert(1e-6)
    before = inv.rank_stats()["largest_rank"]
    A = np.zeros((1024, 1024))
    np.add.at(A, (r, c), v)
    exact = np.linalg.inv(A)
    inv.recompress(1e-3)
    assert inv.rank_stats()["largest_rank"] <= before
    assert np.linalg.norm(inv.to_dense() - exact) <= 1e-2 * np.linalg.norm(exact)


def test_leaf_memory_cap(oracle):                                                       # :305-309
    s, (r, c, v) = fixture(oracle, 32, 32)
    with pytest.raises(oracle.OracleError) as ei:
        oracle.HMatrix.compress_sparse(s, r, c, v, 1e-4, cap=64)
    assert ei.value.code == 3
