// =============================================================================
// acr_oracle.cpp — CPU ORACLE (TEST INFRASTRUCTURE ONLY; NOT THE PRODUCT)
//
// A from-scratch C++17 restatement of the reference ACR hierarchical-matrix
// path (arXiv 1701.00182, mounted at /root/reference/proj), used as the parity
// checker for the sm_100a implementation and as the CPU baseline timed by
// bench.py.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it.  The product (libacrgpu.so) never links it.
//
// Parity status: the reference cannot be compiled here (Eigen 3.4, doctest and
// CLI11 are absent; proj/core/CMakeLists.txt:1), and it ships no golden
// vectors.  This restatement is pinned by re-running the reference's own
// tolerance/property tests against it (tests/test_oracle_*.py, citing
// proj/tests/*.cpp line by line).  Dense linear algebra mirrors Eigen's
// algorithm classes (unpivoted Householder QR, two-sided Jacobi SVD, partial
// pivot LU + Hager/Higham 1-norm rcond) written from textbook descriptions.
//
// Followed reference code (file:line, relative to /root/reference/proj):
//   cluster tree / admissibility ....... core/src/cluster.cpp:9-126
//   truncate_impl / dense_to_lowrank ... core/src/hmatrix.cpp:56-99
//   build_from_sparse / compress ....... core/src/hmatrix.cpp:108-168,664-676
//   build_from_dense ................... core/src/hmatrix.cpp:170-197
//   node_apply[_trans] ................. core/src/hmatrix.cpp:203-238
//   add_node (hadd/hsub) ............... core/src/hmatrix.cpp:242-263,712-724
//   deposit / flush .................... core/src/hmatrix.cpp:352-392
//   mult_to_lowrank / mult_add ......... core/src/hmatrix.cpp:397-479
//   invert_node ........................ core/src/hmatrix.cpp:483-534
//   rank stats / footprint ............. core/src/hmatrix.cpp:538-554,758-767
//   recompress ......................... core/src/hmatrix.cpp:623-662
//   happly ............................. core/src/hmatrix.cpp:695-710
//   red/black positions ................ core/src/acr.cpp:46-58
//   reduce_level / apex / factor ....... core/src/acr.cpp:70-160
//   solve .............................. core/src/acr.cpp:162-229
//   bytes / stats / level info ......... core/src/acr.cpp:231-300
//   lift_hmatrix / acr_factor .......... core/src/acr.cpp:316-384
//   eliminate_around / forward / back .. core/include/acr/acr.hpp:78-132
//   arithmetic slack (eps*0.5) ......... core/include/acr/acr.hpp:178-181
//   DenseKernel (exact oracle mode) .... core/include/acr/acr.hpp:26-38
//
// Plane parallelism: `threads` > 1 runs the independent planes of a level
// concurrently (the reference's only parallel axis, core/src/parallel.cpp);
// per-plane arithmetic is unchanged, so results are bitwise identical for every
// thread count (reference contract, proj/tests/test_parallel.cpp:75-89).
// =============================================================================
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <numeric>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- errors
enum ErrCode { OK = 0, E_DIMENSION = 1, E_SINGULAR = 2, E_LEAFMEM = 3, E_USAGE = 4, E_INTERNAL = 9 };

struct OracleError : std::runtime_error {
    int code, level, plane;
    OracleError(int c, const std::string& m, int lv = -1, int pl = -1)
        : std::runtime_error(m), code(c), level(lv), plane(pl) {}
};

// ---------------------------------------------------------------- flop ledger
// Nominal, implementation-independent counts; shared formulas
// with the GPU accounting in paper_1701_00182_b200/csrc/flops.h.
enum FlopClass { F_GEMM = 0, F_GEQRF, F_ORGQR, F_SVD, F_LU, F_APPLY, F_NCLASS };
static std::atomic<long long> g_flops[F_NCLASS];
static std::atomic<long long> g_trunc_calls{0};
static inline void addf(FlopClass c, double f) { g_flops[c].fetch_add((long long)f, std::memory_order_relaxed); }

// optional truncation trace (m, n, K, ku, kv, r) for kernel-design statistics
static std::mutex g_trace_mu;
static bool g_trace_on = false;
static std::vector<std::array<int, 6>> g_trace;

// ---------------------------------------------------------------- dense matrix
struct Mat {
    int r = 0, c = 0;
    std::vector<double> a;  // column-major
    Mat() = default;
    Mat(int r_, int c_) : r(r_), c(c_), a((size_t)r_ * c_, 0.0) {}
    double& operator()(int i, int j) { return a[(size_t)j * r + i]; }
    double operator()(int i, int j) const { return a[(size_t)j * r + i]; }
    double* col(int j) { return a.data() + (size_t)j * r; }
    const double* col(int j) const { return a.data() + (size_t)j * r; }
    size_t size() const { return a.size(); }
};

static Mat identity(int m, int n) {
    Mat I(m, n);
    for (int i = 0; i < std::min(m, n); ++i) I(i, i) = 1.0;
    return I;
}

// C(ci.., cj..) += alpha * op(A) * op(B); views by pointer + leading dimension.
// Loop orders are fixed per transpose case, so every column of C is produced
// by the same instruction sequence regardless of how many columns there are.
static void gemm(bool ta, bool tb, int m, int n, int k, double alpha, const double* A, int lda,
                 const double* B, int ldb, double* C, int ldc) {
    if (m <= 0 || n <= 0 || k <= 0) return;
    addf(F_GEMM, 2.0 * m * n * k);
    if (!ta && !tb) {
        for (int j = 0; j < n; ++j) {
            double* cj = C + (size_t)j * ldc;
            for (int p = 0; p < k; ++p) {
                const double b = alpha * B[(size_t)j * ldb + p];
                if (b == 0.0) continue;
                const double* ap = A + (size_t)p * lda;
                for (int i = 0; i < m; ++i) cj[i] += ap[i] * b;
            }
        }
    } else if (ta && !tb) {
        for (int j = 0; j < n; ++j) {
            const double* bj = B + (size_t)j * ldb;
            for (int i = 0; i < m; ++i) {
                const double* ai = A + (size_t)i * lda;
                double s = 0;
                for (int p = 0; p < k; ++p) s += ai[p] * bj[p];
                C[(size_t)j * ldc + i] += alpha * s;
            }
        }
    } else if (!ta && tb) {
        for (int j = 0; j < n; ++j) {
            double* cj = C + (size_t)j * ldc;
            for (int p = 0; p < k; ++p) {
                const double b = alpha * B[(size_t)p * ldb + j];
                if (b == 0.0) continue;
                const double* ap = A + (size_t)p * lda;
                for (int i = 0; i < m; ++i) cj[i] += ap[i] * b;
            }
        }
    } else {
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < m; ++i) {
                double s = 0;
                for (int p = 0; p < k; ++p) s += A[(size_t)i * lda + p] * B[(size_t)p * ldb + j];
                C[(size_t)j * ldc + i] += alpha * s;
            }
    }
}

static Mat matmul(const Mat& A, const Mat& B, bool ta = false, bool tb = false) {
    const int m = ta ? A.c : A.r, k = ta ? A.r : A.c, n = tb ? B.r : B.c;
    Mat C(m, n);
    gemm(ta, tb, m, n, k, 1.0, A.a.data(), A.r, B.a.data(), B.r, C.a.data(), C.r);
    return C;
}

// ---------------------------------------------------------------- Householder QR
// Unpivoted Householder QR of A (m x K): R = top ku rows (upper trapezoidal,
// ku x K), Q = explicit thin factor (m x ku), ku = min(m, K).
// Eigen::HouseholderQR semantics (hmatrix.cpp:62-63,80-81): reflector
// H = I - tau v v^T with v(0) = 1, beta = -sign(c0) * ||x||; tau = 0 when the
// sub-diagonal tail is exactly zero.
static void householder_qr(const Mat& A, Mat& R, Mat* Q) {
    const int m = A.r, K = A.c, ku = std::min(m, K);
    Mat W = A;
    std::vector<double> tau(ku, 0.0);
    const double tiny = std::numeric_limits<double>::min();
    for (int j = 0; j < ku; ++j) {
        double* wj = W.col(j);
        const double c0 = wj[j];
        double tail = 0;
        for (int i = j + 1; i < m; ++i) tail += wj[i] * wj[i];
        double beta;
        if (tail <= tiny) {
            tau[j] = 0.0;
            beta = c0;
            for (int i = j + 1; i < m; ++i) wj[i] = 0.0;
        } else {
            beta = std::sqrt(c0 * c0 + tail);
            if (c0 >= 0) beta = -beta;
            const double inv = 1.0 / (c0 - beta);
            for (int i = j + 1; i < m; ++i) wj[i] *= inv;
            tau[j] = (beta - c0) / beta;
        }
        wj[j] = beta;
        if (tau[j] == 0.0) continue;
        for (int c = j + 1; c < K; ++c) {
            double* wc = W.col(c);
            double s = wc[j];
            for (int i = j + 1; i < m; ++i) s += wj[i] * wc[i];
            s *= tau[j];
            wc[j] -= s;
            for (int i = j + 1; i < m; ++i) wc[i] -= s * wj[i];
        }
    }
    if (m >= K) addf(F_GEQRF, 2.0 * m * K * K - 2.0 / 3.0 * K * K * K);
    else addf(F_GEQRF, 2.0 * K * m * m - 2.0 / 3.0 * m * m * m);
    R = Mat(ku, K);
    for (int c = 0; c < K; ++c)
        for (int i = 0; i <= std::min(c, ku - 1); ++i) R(i, c) = W(i, c);
    if (!Q) return;
    Mat& q = *Q;
    q = identity(m, ku);
    for (int j = ku - 1; j >= 0; --j) {
        if (tau[j] == 0.0) continue;
        const double* v = W.col(j);
        for (int c = j; c < ku; ++c) {
            double* qc = q.col(c);
            double s = qc[j];
            for (int i = j + 1; i < m; ++i) s += v[i] * qc[i];
            s *= tau[j];
            qc[j] -= s;
            for (int i = j + 1; i < m; ++i) qc[i] -= s * v[i];
        }
    }
    addf(F_ORGQR, 2.0 * m * ku * ku - 2.0 / 3.0 * ku * ku * ku);
}

// ---------------------------------------------------------------- Jacobi SVD
// Two-sided cyclic Jacobi SVD of a square matrix (Eigen::JacobiSVD's algorithm
// class, hmatrix.cpp:67,89,632,641): sweep pairs (p > q), symmetrise the 2x2
// pivot block with a left rotation, diagonalise it with a symmetric Jacobi
// rotation, stop when every off-diagonal entry is below 2*eps*max|diag|.
// Non-square inputs are first reduced to square by Householder QR (Eigen's QR
// preconditioner).  Singular values are returned in descending order.
struct SVDResult {
    std::vector<double> s;
    Mat U, V;  // thin: U (rows x p), V (cols x p), p = min(rows, cols)
};

static void svd_square(const Mat& M, SVDResult& out, bool want_vectors) {
    const int n = M.r;
    Mat W = M;
    double scale = 0;
    for (double v : W.a) scale = std::max(scale, std::fabs(v));
    if (!(scale > 0) || !std::isfinite(scale)) scale = 1.0;
    for (double& v : W.a) v /= scale;
    Mat U = want_vectors ? identity(n, n) : Mat();
    Mat V = want_vectors ? identity(n, n) : Mat();
    const double tiny = std::numeric_limits<double>::min();
    const double prec = 2.0 * std::numeric_limits<double>::epsilon();
    double maxdiag = 0;
    for (int i = 0; i < n; ++i) maxdiag = std::max(maxdiag, std::fabs(W(i, i)));
    bool done = false;
    int sweeps = 0;
    while (!done && sweeps < 100) {
        done = true;
        ++sweeps;
        for (int p = 1; p < n; ++p)
            for (int q = 0; q < p; ++q) {
                const double thr = std::max(tiny, prec * maxdiag);
                if (!(std::fabs(W(p, q)) > thr || std::fabs(W(q, p)) > thr)) continue;
                done = false;
                // 2x2 block [[a b][c d]] on rows/cols (q, p)
                const double a = W(q, q), b = W(q, p), c = W(p, q), d = W(p, p);
                // left rotation G1 = [[c1 s1][-s1 c1]] making G1^T B symmetric
                double c1 = 1, s1 = 0;
                const double diff = b - c;
                if (std::fabs(diff) >= tiny) {
                    const double rho = (a + d) / diff;
                    s1 = 1.0 / std::sqrt(1.0 + rho * rho);
                    c1 = rho * s1;
                }
                const double x = c1 * a - s1 * c, y = c1 * b - s1 * d, z = s1 * b + c1 * d;
                // symmetric Jacobi J = [[cj sj][-sj cj]] with J^T S J diagonal
                double cj = 1, sj = 0;
                if (y != 0.0) {
                    const double tau = (z - x) / (2.0 * y);
                    const double t = (tau >= 0 ? 1.0 : -1.0) / (std::fabs(tau) + std::sqrt(1.0 + tau * tau));
                    cj = 1.0 / std::sqrt(1.0 + t * t);
                    sj = t * cj;
                }
                // L = G1 * J
                const double l11 = c1 * cj - s1 * sj, l12 = c1 * sj + s1 * cj;
                const double l21 = -s1 * cj - c1 * sj, l22 = -s1 * sj + c1 * cj;
                // W <- L^T W (rows q, p)
                for (int k = 0; k < n; ++k) {
                    const double wq = W(q, k), wp = W(p, k);
                    W(q, k) = l11 * wq + l21 * wp;
                    W(p, k) = l12 * wq + l22 * wp;
                }
                // W <- W J (cols q, p)
                for (int k = 0; k < n; ++k) {
                    const double wq = W(k, q), wp = W(k, p);
                    W(k, q) = cj * wq - sj * wp;
                    W(k, p) = sj * wq + cj * wp;
                }
                if (want_vectors) {
                    for (int k = 0; k < n; ++k) {
                        const double uq = U(k, q), up = U(k, p);
                        U(k, q) = l11 * uq + l21 * up;
                        U(k, p) = l12 * uq + l22 * up;
                        const double vq = V(k, q), vp = V(k, p);
                        V(k, q) = cj * vq - sj * vp;
                        V(k, p) = sj * vq + cj * vp;
                    }
                }
                maxdiag = std::max(maxdiag, std::max(std::fabs(W(p, p)), std::fabs(W(q, q))));
            }
    }
    std::vector<int> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    std::vector<double> sv(n);
    for (int i = 0; i < n; ++i) sv[i] = std::fabs(W(i, i));
    std::stable_sort(idx.begin(), idx.end(), [&](int i, int j) { return sv[i] > sv[j]; });
    out.s.resize(n);
    for (int i = 0; i < n; ++i) out.s[i] = sv[idx[i]] * scale;
    if (want_vectors) {
        out.U = Mat(n, n);
        out.V = Mat(n, n);
        for (int t = 0; t < n; ++t) {
            const int i = idx[t];
            const double sg = W(i, i) < 0 ? -1.0 : 1.0;
            for (int k = 0; k < n; ++k) {
                out.U(k, t) = sg * U(k, i);
                out.V(k, t) = V(k, i);
            }
        }
    }
    addf(F_SVD, 21.0 * n * n * n);
}

static void svd(const Mat& M, SVDResult& out, bool want_vectors) {
    if (M.r == M.c) return svd_square(M, out, want_vectors);
    if (M.r > M.c) {
        Mat R, Q;
        householder_qr(M, R, want_vectors ? &Q : nullptr);  // R: c x c
        SVDResult inner;
        svd_square(R, inner, want_vectors);
        out.s = inner.s;
        if (want_vectors) {
            out.U = matmul(Q, inner.U);
            out.V = inner.V;
        }
        return;
    }
    Mat T(M.c, M.r);
    for (int i = 0; i < M.r; ++i)
        for (int j = 0; j < M.c; ++j) T(j, i) = M(i, j);
    SVDResult inner;
    svd(T, inner, want_vectors);
    out.s = inner.s;
    if (want_vectors) {
        out.U = inner.V;
        out.V = inner.U;
    }
}

// ---------------------------------------------------------------- LU inverse
// Partial-pivot LU, Hager/Higham 1-norm condition estimate and explicit
// inverse (Eigen::PartialPivLU + rcond + inverse, hmatrix.cpp:485-494,
// acr.cpp:23-29).  Returns rcond; `inv` receives A^{-1}.
static double lu_inverse(const Mat& A, Mat& inv) {
    const int n = A.r;
    Mat LU = A;
    std::vector<int> piv(n);
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = std::fabs(LU(k, k));
        for (int i = k + 1; i < n; ++i)
            if (std::fabs(LU(i, k)) > best) {
                best = std::fabs(LU(i, k));
                p = i;
            }
        piv[k] = p;
        if (p != k)
            for (int c = 0; c < n; ++c) std::swap(LU(k, c), LU(p, c));
        const double d = LU(k, k);
        if (d != 0.0) {
            for (int i = k + 1; i < n; ++i) LU(i, k) /= d;
            for (int c = k + 1; c < n; ++c) {
                const double f = LU(k, c);
                if (f == 0.0) continue;
                for (int i = k + 1; i < n; ++i) LU(i, c) -= LU(i, k) * f;
            }
        }
    }
    auto solve = [&](std::vector<double>& x) {  // A x = b in place
        for (int k = 0; k < n; ++k) std::swap(x[k], x[piv[k]]);
        for (int k = 0; k < n; ++k)
            for (int i = k + 1; i < n; ++i) x[i] -= LU(i, k) * x[k];
        for (int k = n - 1; k >= 0; --k) {
            x[k] /= LU(k, k);
            for (int i = 0; i < k; ++i) x[i] -= LU(i, k) * x[k];
        }
    };
    auto solve_t = [&](std::vector<double>& x) {  // A^T x = b in place
        for (int k = 0; k < n; ++k) {
            for (int i = 0; i < k; ++i) x[k] -= LU(i, k) * x[i];
            x[k] /= LU(k, k);
        }
        for (int k = n - 1; k >= 0; --k)
            for (int i = k + 1; i < n; ++i) x[k] -= LU(i, k) * x[i];
        for (int k = n - 1; k >= 0; --k) std::swap(x[k], x[piv[k]]);
    };
    double anorm = 0;
    for (int c = 0; c < n; ++c) {
        double s = 0;
        for (int i = 0; i < n; ++i) s += std::fabs(A(i, c));
        anorm = std::max(anorm, s);
    }
    bool zero_pivot = false;
    for (int k = 0; k < n; ++k)
        if (LU(k, k) == 0.0) zero_pivot = true;
    double rcond = 0.0;
    if (anorm > 0 && !zero_pivot) {
        // Hager's estimator of ||A^{-1}||_1
        std::vector<double> x(n, 1.0 / n), y, z;
        double est = 0;
        for (int it = 0; it < 5; ++it) {
            y = x;
            solve(y);
            double ny = 0;
            for (double v : y) ny += std::fabs(v);
            if (it > 0 && ny <= est) break;
            est = ny;
            z.assign(n, 0.0);
            for (int i = 0; i < n; ++i) z[i] = y[i] >= 0 ? 1.0 : -1.0;
            solve_t(z);
            int jmax = 0;
            for (int i = 1; i < n; ++i)
                if (std::fabs(z[i]) > std::fabs(z[jmax])) jmax = i;
            double ztx = 0;
            for (int i = 0; i < n; ++i) ztx += z[i] * x[i];
            if (it > 0 && std::fabs(z[jmax]) <= ztx) break;
            x.assign(n, 0.0);
            x[jmax] = 1.0;
        }
        // Higham's alternative lower bound guards against Hager's failure cases
        std::vector<double> alt(n);
        for (int i = 0; i < n; ++i) alt[i] = (i % 2 ? -1.0 : 1.0) * (1.0 + double(i) / std::max(1, n - 1));
        solve(alt);
        double na = 0;
        for (double v : alt) na += std::fabs(v);
        est = std::max(est, 2.0 * na / (3.0 * n));
        rcond = (est > 0 && std::isfinite(est)) ? 1.0 / (anorm * est) : 0.0;
    }
    inv = Mat(n, n);
    if (!zero_pivot) {
        std::vector<double> e(n);
        for (int c = 0; c < n; ++c) {
            std::fill(e.begin(), e.end(), 0.0);
            e[c] = 1.0;
            solve(e);
            std::copy(e.begin(), e.end(), inv.col(c));
        }
    }
    addf(F_LU, 2.0 * n * n * n);  // 2/3 n^3 (getrf) + 4/3 n^3 (getri)
    return rcond;
}

// ---------------------------------------------------------------- cluster tree
struct Box {
    double x0 = 0, x1 = 0, y0 = 0, y1 = 0;
    double diam() const { return std::sqrt((x1 - x0) * (x1 - x0) + (y1 - y0) * (y1 - y0)); }
    double dist(const Box& o) const {
        const double dx = std::max({0.0, o.x0 - x1, x0 - o.x1});
        const double dy = std::max({0.0, o.y0 - y1, y0 - o.y1});
        return std::sqrt(dx * dx + dy * dy);
    }
};

struct Cluster {
    int begin = 0, end = 0;
    Box box;
    std::unique_ptr<Cluster> lo, hi;
    bool leaf() const { return !lo; }
};

// Median bisection along the longer box side with a stable sort
// (cluster.cpp:39-80): deterministic, contiguous tree-order ranges.
struct ClusterTree {
    std::unique_ptr<Cluster> root;
    std::vector<int> perm, iperm;  // tree pos -> original, original -> tree pos
    int leaf_size = 0;

    ClusterTree(const std::vector<double>& xy, int leaf) : leaf_size(leaf) {
        const int N = (int)(xy.size() / 2);
        if (N == 0) throw OracleError(E_USAGE, "ClusterTree: empty point set");
        if (leaf < 1) throw OracleError(E_USAGE, "ClusterTree: leaf_size must be >= 1");
        perm.resize(N);
        std::iota(perm.begin(), perm.end(), 0);
        std::function<std::unique_ptr<Cluster>(int, int)> make = [&](int b, int e) {
            auto c = std::make_unique<Cluster>();
            c->begin = b;
            c->end = e;
            Box bx;
            bx.x0 = bx.x1 = xy[2 * perm[b]];
            bx.y0 = bx.y1 = xy[2 * perm[b] + 1];
            for (int i = b + 1; i < e; ++i) {
                const double x = xy[2 * perm[i]], y = xy[2 * perm[i] + 1];
                bx.x0 = std::min(bx.x0, x);
                bx.x1 = std::max(bx.x1, x);
                bx.y0 = std::min(bx.y0, y);
                bx.y1 = std::max(bx.y1, y);
            }
            c->box = bx;
            if (e - b > leaf_size) {
                const int axis = (bx.x1 - bx.x0) >= (bx.y1 - bx.y0) ? 0 : 1;
                std::stable_sort(perm.begin() + b, perm.begin() + e,
                                 [&](int p, int q) { return xy[2 * p + axis] < xy[2 * q + axis]; });
                const int mid = b + (e - b) / 2;
                c->lo = make(b, mid);
                c->hi = make(mid, e);
            }
            return c;
        };
        root = make(0, N);
        iperm.resize(N);
        for (int i = 0; i < N; ++i) iperm[perm[i]] = i;
    }
    int size() const { return (int)perm.size(); }
};

enum Kind { DENSE = 0, RK = 1, BRANCH = 2 };

struct BNode {  // block cluster tree node
    const Cluster* row = nullptr;
    const Cluster* col = nullptr;
    Kind kind = DENSE;
    std::array<std::unique_ptr<BNode>, 4> ch;
};

// Standard (min diam <= eta*dist) or weak (disjoint ranges) admissibility;
// quadtree subdivision while both clusters split (cluster.cpp:94-126).
struct BlockTree {
    std::shared_ptr<ClusterTree> tree;
    double eta;
    int weak;
    std::unique_ptr<BNode> root;
    BlockTree(std::shared_ptr<ClusterTree> t, double eta_, int weak_) : tree(std::move(t)), eta(eta_), weak(weak_) {
        if (!(eta > 0)) throw OracleError(E_USAGE, "BlockClusterTree: eta must be positive");
        root = build(tree->root.get(), tree->root.get());
    }
    bool admissible(const Cluster* t, const Cluster* s) const {
        if (weak) return t->end <= s->begin || s->end <= t->begin;
        return std::min(t->box.diam(), s->box.diam()) <= eta * t->box.dist(s->box);
    }
    std::unique_ptr<BNode> build(const Cluster* t, const Cluster* s) const {
        auto n = std::make_unique<BNode>();
        n->row = t;
        n->col = s;
        if (admissible(t, s)) {
            n->kind = RK;
        } else if (!t->leaf() && !s->leaf()) {
            n->kind = BRANCH;
            const Cluster* tc[2] = {t->lo.get(), t->hi.get()};
            const Cluster* sc[2] = {s->lo.get(), s->hi.get()};
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 2; ++j) n->ch[i * 2 + j] = build(tc[i], sc[j]);
        } else {
            n->kind = DENSE;
        }
        return n;
    }
};

// ---------------------------------------------------------------- H-matrix
struct HNode {
    int rb = 0, re = 0, cb = 0, ce = 0;
    Kind kind = DENSE;
    Mat D;     // dense leaf
    Mat U, V;  // Rk leaf: U (rows x k), V (cols x k), block = U V^T
    std::array<std::unique_ptr<HNode>, 4> ch;
    int rows() const { return re - rb; }
    int cols() const { return ce - cb; }
    int rank() const { return U.c; }
};

using HPtr = std::unique_ptr<HNode>;

static HPtr clone(const HNode& n) {
    auto c = std::make_unique<HNode>();
    c->rb = n.rb; c->re = n.re; c->cb = n.cb; c->ce = n.ce;
    c->kind = n.kind;
    c->D = n.D;
    c->U = n.U;
    c->V = n.V;
    if (n.kind == BRANCH)
        for (int i = 0; i < 4; ++i) c->ch[i] = clone(*n.ch[i]);
    return c;
}

static HPtr zero_like(const HNode& n) {
    auto c = std::make_unique<HNode>();
    c->rb = n.rb; c->re = n.re; c->cb = n.cb; c->ce = n.ce;
    c->kind = n.kind;
    if (n.kind == DENSE) c->D = Mat(n.rows(), n.cols());
    if (n.kind == RK) {
        c->U = Mat(n.rows(), 0);
        c->V = Mat(n.cols(), 0);
    }
    if (n.kind == BRANCH)
        for (int i = 0; i < 4; ++i) c->ch[i] = zero_like(*n.ch[i]);
    return c;
}

static bool same_structure(const HNode& a, const HNode& b) {
    if (a.rb != b.rb || a.re != b.re || a.cb != b.cb || a.ce != b.ce || a.kind != b.kind) return false;
    if (a.kind == BRANCH)
        for (int i = 0; i < 4; ++i)
            if (!same_structure(*a.ch[i], *b.ch[i])) return false;
    return true;
}

struct HMatrix {
    std::shared_ptr<ClusterTree> tree;
    HPtr root;
    double eps = 0;
    HMatrix() = default;
    HMatrix(std::shared_ptr<ClusterTree> t, HPtr r, double e) : tree(std::move(t)), root(std::move(r)), eps(e) {}
    HMatrix(const HMatrix& o) : tree(o.tree), root(o.root ? clone(*o.root) : nullptr), eps(o.eps) {}
    HMatrix& operator=(const HMatrix& o) {
        if (this != &o) {
            tree = o.tree;
            root = o.root ? clone(*o.root) : nullptr;
            eps = o.eps;
        }
        return *this;
    }
    HMatrix(HMatrix&&) = default;
    HMatrix& operator=(HMatrix&&) = default;
    int dim() const { return root ? root->rows() : 0; }
};

// ---- rank truncation (hmatrix.cpp:56-84)
// U (m x K), V (n x K) -> U (m x r), V (n x r): QR both, SVD of the core
// Ru Rv^T, keep sigma_i > max(eps*sigma_1, abs_cutoff), absorb sigma into U.
static void truncate(Mat& U, Mat& V, double eps, double abs_cutoff = 0.0) {
    const int m = U.r, n = V.r, K = U.c;
    if (K == 0) return;
    g_trunc_calls.fetch_add(1, std::memory_order_relaxed);
    const int ku = std::min(m, K), kv = std::min(n, K);
    Mat Ru, Rv, Qu, Qv;
    householder_qr(U, Ru, &Qu);
    householder_qr(V, Rv, &Qv);
    Mat core = matmul(Ru, Rv, false, true);  // ku x kv
    SVDResult sv;
    svd(core, sv, true);
    int r = 0;
    if (!sv.s.empty() && sv.s[0] > 0.0) {
        const double cut = std::max(eps * sv.s[0], abs_cutoff);
        while (r < (int)sv.s.size() && sv.s[r] > cut) ++r;
    }
    if (g_trace_on) {
        std::lock_guard<std::mutex> lk(g_trace_mu);
        g_trace.push_back({m, n, K, ku, kv, r});
    }
    Mat Us(ku, r), Vs(kv, r);
    for (int t = 0; t < r; ++t)
        for (int i = 0; i < ku; ++i) Us(i, t) = sv.U(i, t) * sv.s[t];
    for (int t = 0; t < r; ++t)
        for (int i = 0; i < kv; ++i) Vs(i, t) = sv.V(i, t);
    U = matmul(Qu, Us);
    V = matmul(Qv, Vs);
}

// ---- dense block -> outer product (hmatrix.cpp:87-99)
static void dense_to_lowrank(const Mat& M, double eps, Mat& U, Mat& V) {
    SVDResult sv;
    svd(M, sv, true);
    int r = 0;
    if (!sv.s.empty() && sv.s[0] > 0.0) {
        const double cut = eps * sv.s[0];
        while (r < (int)sv.s.size() && sv.s[r] > cut) ++r;
    }
    U = Mat(M.r, r);
    V = Mat(M.c, r);
    for (int t = 0; t < r; ++t) {
        for (int i = 0; i < M.r; ++i) U(i, t) = sv.U(i, t) * sv.s[t];
        for (int i = 0; i < M.c; ++i) V(i, t) = sv.V(i, t);
    }
}

// ---- construction (hmatrix.cpp:108-197)
struct Entry {
    int r, c;
    double v;
};

static HPtr build_sparse(const BNode& bn, std::vector<Entry> ent, double eps, long cap) {
    auto h = std::make_unique<HNode>();
    h->rb = bn.row->begin; h->re = bn.row->end;
    h->cb = bn.col->begin; h->ce = bn.col->end;
    const int m = h->rows(), nn = h->cols();
    if (bn.kind == DENSE) {
        h->kind = DENSE;
        if (8L * m * nn > cap)
            throw OracleError(E_LEAFMEM, "dense leaf of " + std::to_string(m) + "x" + std::to_string(nn) +
                                             " exceeds memory cap");
        h->D = Mat(m, nn);
        for (const auto& e : ent) h->D(e.r - h->rb, e.c - h->cb) += e.v;
    } else if (bn.kind == RK) {
        h->kind = RK;
        std::vector<int> cols;
        for (const auto& e : ent) cols.push_back(e.c);
        std::sort(cols.begin(), cols.end());
        cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
        const int c = (int)cols.size();
        if (8L * (m + nn) * c > cap)
            throw OracleError(E_LEAFMEM, "low-rank leaf factor of width " + std::to_string(c) +
                                             " exceeds memory cap");
        h->U = Mat(m, c);
        h->V = Mat(nn, c);
        for (const auto& e : ent) {
            const int j = (int)(std::lower_bound(cols.begin(), cols.end(), e.c) - cols.begin());
            h->U(e.r - h->rb, j) += e.v;
        }
        for (int j = 0; j < c; ++j) h->V(cols[j] - h->cb, j) = 1.0;
        truncate(h->U, h->V, eps);
    } else {
        h->kind = BRANCH;
        std::array<std::vector<Entry>, 4> part;
        const int rmid = bn.ch[0]->row->end, cmid = bn.ch[0]->col->end;
        for (const auto& e : ent) part[(e.r < rmid ? 0 : 2) + (e.c < cmid ? 0 : 1)].push_back(e);
        ent.clear();
        ent.shrink_to_fit();
        for (int i = 0; i < 4; ++i) h->ch[i] = build_sparse(*bn.ch[i], std::move(part[i]), eps, cap);
    }
    return h;
}

static HPtr build_dense(const BNode& bn, const Mat& P, double eps, long cap) {
    auto h = std::make_unique<HNode>();
    h->rb = bn.row->begin; h->re = bn.row->end;
    h->cb = bn.col->begin; h->ce = bn.col->end;
    const int m = h->rows(), nn = h->cols();
    if (bn.kind != BRANCH && 8L * m * nn > cap)
        throw OracleError(E_LEAFMEM, "leaf exceeds memory cap");
    if (bn.kind == BRANCH) {
        h->kind = BRANCH;
        for (int i = 0; i < 4; ++i) h->ch[i] = build_dense(*bn.ch[i], P, eps, cap);
        return h;
    }
    Mat blk(m, nn);
    for (int j = 0; j < nn; ++j)
        for (int i = 0; i < m; ++i) blk(i, j) = P(h->rb + i, h->cb + j);
    if (bn.kind == DENSE) {
        h->kind = DENSE;
        h->D = std::move(blk);
    } else {
        h->kind = RK;
        dense_to_lowrank(blk, eps, h->U, h->V);
    }
    return h;
}

// ---- leafwise apply (hmatrix.cpp:203-238); X/Y are (rows x k) column-major
// panels with leading dimension ld; row offsets xoff/yoff.
static void apply_node(const HNode& n, const double* X, int ldx, int xoff, double* Y, int ldy, int yoff,
                       int k, bool trans) {
    if (n.kind == BRANCH) {
        for (int i = 0; i < 4; ++i) apply_node(*n.ch[i], X, ldx, xoff, Y, ldy, yoff, k, trans);
        return;
    }
    const int in_b = trans ? n.rb : n.cb, out_b = trans ? n.cb : n.rb;
    const double* x = X + (in_b - xoff);
    double* y = Y + (out_b - yoff);
    if (n.kind == DENSE) {
        if (!trans) gemm(false, false, n.rows(), k, n.cols(), 1.0, n.D.a.data(), n.rows(), x, ldx, y, ldy);
        else gemm(true, false, n.cols(), k, n.rows(), 1.0, n.D.a.data(), n.rows(), x, ldx, y, ldy);
        return;
    }
    const int r = n.rank();
    if (r == 0) return;
    const Mat& In = trans ? n.U : n.V;    // contracted against X
    const Mat& Out = trans ? n.V : n.U;   // expands into Y
    Mat T(r, k);
    gemm(true, false, r, k, In.r, 1.0, In.a.data(), In.r, x, ldx, T.a.data(), r);
    gemm(false, false, Out.r, k, r, 1.0, Out.a.data(), Out.r, T.a.data(), r, y, ldy);
}

// ---- H-addition (hmatrix.cpp:242-263)
static void add_node(HNode& c, const HNode& a, double alpha, double eps) {
    if (c.kind == DENSE) {
        for (size_t i = 0; i < c.D.size(); ++i) c.D.a[i] += alpha * a.D.a[i];
    } else if (c.kind == RK) {
        if (a.rank() == 0) return;
        Mat U(c.rows(), c.rank() + a.rank()), V(c.cols(), c.rank() + a.rank());
        std::copy(c.U.a.begin(), c.U.a.end(), U.a.begin());
        std::copy(c.V.a.begin(), c.V.a.end(), V.a.begin());
        for (size_t i = 0; i < a.U.size(); ++i) U.a[c.U.size() + i] = alpha * a.U.a[i];
        std::copy(a.V.a.begin(), a.V.a.end(), V.a.begin() + c.V.size());
        truncate(U, V, eps);
        c.U = std::move(U);
        c.V = std::move(V);
    } else {
        for (int i = 0; i < 4; ++i) add_node(*c.ch[i], *a.ch[i], alpha, eps);
    }
}

// ---- multiplication (hmatrix.cpp:352-479)
// Low-rank contributions are queued per target Rk leaf and folded in with one
// truncation per leaf at the end of each mult_add call.
struct Pending {
    HNode* target;
    std::vector<std::pair<Mat, Mat>> parts;
};
struct Accum {
    std::vector<Pending> list;  // in first-deposit order
    void push(HNode* t, Mat U, Mat V) {
        for (auto& p : list)
            if (p.target == t) {
                p.parts.emplace_back(std::move(U), std::move(V));
                return;
            }
        list.push_back(Pending{t, {}});
        list.back().parts.emplace_back(std::move(U), std::move(V));
    }
};

static Mat rows_of(const Mat& M, int r0, int nr) {
    Mat S(nr, M.c);
    for (int j = 0; j < M.c; ++j) std::copy(M.col(j) + r0, M.col(j) + r0 + nr, S.col(j));
    return S;
}

static void deposit(HNode& c, const Mat& U, const Mat& V, Accum& acc) {
    if (U.c == 0) return;
    if (c.kind == DENSE) {
        gemm(false, true, c.rows(), c.cols(), U.c, 1.0, U.a.data(), U.r, V.a.data(), V.r, c.D.a.data(), c.D.r);
    } else if (c.kind == RK) {
        acc.push(&c, U, V);
    } else {
        for (int i = 0; i < 4; ++i) {
            HNode& s = *c.ch[i];
            deposit(s, rows_of(U, s.rb - c.rb, s.rows()), rows_of(V, s.cb - c.cb, s.cols()), acc);
        }
    }
}

static void flush(Accum& acc, double eps) {
    for (auto& p : acc.list) {
        HNode& t = *p.target;
        int extra = 0;
        for (auto& uv : p.parts) extra += uv.first.c;
        const int k0 = t.rank();
        Mat U(t.rows(), k0 + extra), V(t.cols(), k0 + extra);
        std::copy(t.U.a.begin(), t.U.a.end(), U.a.begin());
        std::copy(t.V.a.begin(), t.V.a.end(), V.a.begin());
        size_t ou = t.U.size(), ov = t.V.size();
        for (auto& uv : p.parts) {
            std::copy(uv.first.a.begin(), uv.first.a.end(), U.a.begin() + ou);
            std::copy(uv.second.a.begin(), uv.second.a.end(), V.a.begin() + ov);
            ou += uv.first.size();
            ov += uv.second.size();
        }
        truncate(U, V, eps);
        t.U = std::move(U);
        t.V = std::move(V);
    }
    acc.list.clear();
}

static void product_lowrank(const HNode& A, const HNode& B, double eps, Mat& U, Mat& V) {
    if (A.kind == RK) {  // (U_A V_A^T) B = U_A (B^T V_A)^T
        U = A.U;
        V = Mat(B.cols(), A.rank());
        if (A.rank() > 0) apply_node(B, A.V.a.data(), A.V.r, B.rb, V.a.data(), V.r, B.cb, A.rank(), true);
        return;
    }
    if (B.kind == RK) {  // A (U_B V_B^T) = (A U_B) V_B^T
        V = B.V;
        U = Mat(A.rows(), B.rank());
        if (B.rank() > 0) apply_node(A, B.U.a.data(), B.U.r, A.cb, U.a.data(), U.r, A.rb, B.rank(), false);
        return;
    }
    if (A.kind == DENSE && B.kind == DENSE) {
        dense_to_lowrank(matmul(A.D, B.D), eps, U, V);
        return;
    }
    if (A.kind == BRANCH && B.kind == BRANCH) {
        std::array<Mat, 8> pu, pv;
        std::array<const HNode*, 8> ar{}, bc{};
        int total = 0, t = 0;
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j)
                for (int k = 0; k < 2; ++k) {
                    ar[t] = A.ch[i * 2 + k].get();
                    bc[t] = B.ch[k * 2 + j].get();
                    product_lowrank(*ar[t], *bc[t], eps, pu[t], pv[t]);
                    total += pu[t].c;
                    ++t;
                }
        U = Mat(A.rows(), total);
        V = Mat(B.cols(), total);
        int off = 0;
        for (t = 0; t < 8; ++t) {
            for (int c = 0; c < pu[t].c; ++c) {
                std::copy(pu[t].col(c), pu[t].col(c) + pu[t].r, U.col(off + c) + (ar[t]->rb - A.rb));
                std::copy(pv[t].col(c), pv[t].col(c) + pv[t].r, V.col(off + c) + (bc[t]->cb - B.cb));
            }
            off += pu[t].c;
        }
        truncate(U, V, eps);
        return;
    }
    // mixed dense/branch (unbalanced trees)
    if (A.kind == DENSE) {  // B branch: (B^T A^T)^T
        Mat Xt(A.cols(), A.rows());
        for (int i = 0; i < A.rows(); ++i)
            for (int j = 0; j < A.cols(); ++j) Xt(j, i) = A.D(i, j);
        Mat Y(B.cols(), A.rows());
        apply_node(B, Xt.a.data(), Xt.r, B.rb, Y.a.data(), Y.r, B.cb, A.rows(), true);
        Mat Yt(A.rows(), B.cols());
        for (int i = 0; i < Y.r; ++i)
            for (int j = 0; j < Y.c; ++j) Yt(j, i) = Y(i, j);
        dense_to_lowrank(Yt, eps, U, V);
        return;
    }
    Mat Y(A.rows(), B.cols());
    apply_node(A, B.D.a.data(), B.D.r, A.cb, Y.a.data(), Y.r, A.rb, B.cols(), false);
    dense_to_lowrank(Y, eps, U, V);
}

static void mult_add_rec(HNode& C, const HNode& A, const HNode& B, double alpha, double eps, Accum& acc) {
    if (A.kind == BRANCH && B.kind == BRANCH && C.kind == BRANCH) {
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j)
                for (int k = 0; k < 2; ++k)
                    mult_add_rec(*C.ch[i * 2 + j], *A.ch[i * 2 + k], *B.ch[k * 2 + j], alpha, eps, acc);
        return;
    }
    Mat U, V;
    product_lowrank(A, B, eps, U, V);
    for (double& v : U.a) v *= alpha;
    deposit(C, U, V, acc);
}

static void mult_add(HNode& C, const HNode& A, const HNode& B, double alpha, double eps) {
    Accum acc;
    mult_add_rec(C, A, B, alpha, eps, acc);
    flush(acc, eps);
}

// ---- inversion (hmatrix.cpp:483-534): recursive 2x2 Schur complement
static HPtr invert_node(const HNode& n, double eps) {
    if (n.kind == DENSE) {
        auto out = std::make_unique<HNode>();
        out->rb = n.rb; out->re = n.re; out->cb = n.cb; out->ce = n.ce;
        out->kind = DENSE;
        const double rc = lu_inverse(n.D, out->D);
        if (!(rc > 1e-14))
            throw OracleError(E_SINGULAR, "singular dense pivot on cluster rows [" + std::to_string(n.rb) + ", " +
                                              std::to_string(n.re) + "), rcond=" + std::to_string(rc));
        return out;
    }
    if (n.kind != BRANCH) throw OracleError(E_INTERNAL, "invert_node: admissible diagonal block");
    const HNode &A11 = *n.ch[0], &A12 = *n.ch[1], &A21 = *n.ch[2], &A22 = *n.ch[3];
    HPtr X11 = invert_node(A11, eps);
    HPtr T12 = zero_like(A12);
    mult_add(*T12, *X11, A12, 1.0, eps);
    HPtr T21 = zero_like(A21);
    mult_add(*T21, A21, *X11, 1.0, eps);
    HPtr S = clone(A22);
    mult_add(*S, A21, *T12, -1.0, eps);
    HPtr X22 = invert_node(*S, eps);
    S.reset();
    HPtr C12 = zero_like(A12);
    mult_add(*C12, *T12, *X22, -1.0, eps);
    HPtr C21 = zero_like(A21);
    mult_add(*C21, *X22, *T21, -1.0, eps);
    HPtr C11 = std::move(X11);
    mult_add(*C11, *T12, *C21, -1.0, eps);
    auto out = std::make_unique<HNode>();
    out->rb = n.rb; out->re = n.re; out->cb = n.cb; out->ce = n.ce;
    out->kind = BRANCH;
    out->ch[0] = std::move(C11);
    out->ch[1] = std::move(C12);
    out->ch[2] = std::move(C21);
    out->ch[3] = std::move(X22);
    return out;
}

// ---- accounting (hmatrix.cpp:538-554)
struct RankStats {
    double average_rank = 0;
    int largest_rank = 0;
    int dense_leaf_count = 0;
    int lowrank_leaf_count = 0;
    long bytes = 0;
};

static void stats_walk(const HNode& n, RankStats& s, long& rsum) {
    if (n.kind == DENSE) {
        ++s.dense_leaf_count;
        s.bytes += 8L * n.rows() * n.cols();
    } else if (n.kind == RK) {
        ++s.lowrank_leaf_count;
        s.largest_rank = std::max(s.largest_rank, n.rank());
        rsum += n.rank();
        s.bytes += 8L * (n.rows() + n.cols()) * n.rank();
    } else {
        for (int i = 0; i < 4; ++i) stats_walk(*n.ch[i], s, rsum);
    }
}

static RankStats rank_stats(const HNode& root) {
    RankStats s;
    long rsum = 0;
    stats_walk(root, s, rsum);
    if (s.lowrank_leaf_count > 0) s.average_rank = double(rsum) / s.lowrank_leaf_count;
    return s;
}

static void merge_stats(RankStats& into, const RankStats& s) {  // acr.cpp:10-18
    const long c0 = into.lowrank_leaf_count, c1 = s.lowrank_leaf_count;
    if (c0 + c1 > 0) into.average_rank = (into.average_rank * c0 + s.average_rank * c1) / double(c0 + c1);
    into.largest_rank = std::max(into.largest_rank, s.largest_rank);
    into.dense_leaf_count += s.dense_leaf_count;
    into.lowrank_leaf_count += s.lowrank_leaf_count;
    into.bytes += s.bytes;
}

static void to_dense_walk(const HNode& n, Mat& P) {
    if (n.kind == BRANCH) {
        for (int i = 0; i < 4; ++i) to_dense_walk(*n.ch[i], P);
        return;
    }
    for (int j = 0; j < n.cols(); ++j)
        for (int i = 0; i < n.rows(); ++i) {
            double v = 0;
            if (n.kind == DENSE) v = n.D(i, j);
            else
                for (int t = 0; t < n.rank(); ++t) v += n.U(i, t) * n.V(j, t);
            P(n.rb + i, n.cb + j) = v;
        }
}

// ---- stored-inverse recompression (hmatrix.cpp:623-662)
static double scale_walk(const HNode& n) {
    if (n.kind == BRANCH) {
        double s = 0;
        for (int i = 0; i < 4; ++i) s = std::max(s, scale_walk(*n.ch[i]));
        return s;
    }
    if (n.kind == DENSE) {
        if (n.D.size() == 0) return 0;
        SVDResult sv;
        svd(n.D, sv, false);
        return sv.s[0];
    }
    if (n.rank() == 0) return 0;
    Mat Ru, Rv;
    householder_qr(n.U, Ru, nullptr);
    householder_qr(n.V, Rv, nullptr);
    SVDResult sv;
    svd(matmul(Ru, Rv, false, true), sv, false);
    return sv.s[0];
}

static void recompress_walk(HNode& n, double abs_cut) {
    if (n.kind == BRANCH) {
        for (int i = 0; i < 4; ++i) recompress_walk(*n.ch[i], abs_cut);
    } else if (n.kind == RK && n.rank() > 0) {
        truncate(n.U, n.V, 0.0, abs_cut);
    }
}

static void recompress(HMatrix& H, double eps) {
    if (!H.root) return;
    const double row_safety = 0.05;
    const double scale = scale_walk(*H.root);
    if (scale > 0) recompress_walk(*H.root, row_safety * eps * scale);
}

// ---- public-ish H operations
static HMatrix h_compress_sparse(const BlockTree& bt, const std::vector<Entry>& ent_orig, double eps, long cap) {
    const auto& ip = bt.tree->iperm;
    std::vector<Entry> ent;
    ent.reserve(ent_orig.size());
    for (const auto& e : ent_orig) ent.push_back(Entry{ip[e.r], ip[e.c], e.v});
    return HMatrix(bt.tree, build_sparse(*bt.root, std::move(ent), eps, cap), eps);
}

static Mat h_apply(const HMatrix& H, const Mat& X) {  // original ordering (hmatrix.cpp:695-706)
    if (!H.root) throw OracleError(E_DIMENSION, "happly: H-matrix not initialized");
    if (X.r != H.dim()) throw OracleError(E_DIMENSION, "happly: row count mismatch");
    const auto& perm = H.tree->perm;
    Mat Xp(X.r, X.c), Yp(X.r, X.c), Y(X.r, X.c);
    for (int j = 0; j < X.c; ++j)
        for (int i = 0; i < X.r; ++i) Xp(i, j) = X(perm[i], j);
    apply_node(*H.root, Xp.a.data(), Xp.r, 0, Yp.a.data(), Yp.r, 0, X.c, false);
    for (int j = 0; j < X.c; ++j)
        for (int i = 0; i < X.r; ++i) Y(perm[i], j) = Yp(i, j);
    return Y;
}

static HMatrix h_multiply(const HMatrix& A, const HMatrix& B, double eps) {
    if (A.tree != B.tree) throw OracleError(E_DIMENSION, "hmultiply: operands must share one cluster tree");
    HMatrix C(A.tree, zero_like(*A.root), A.eps);
    mult_add(*C.root, *A.root, *B.root, 1.0, eps);
    return C;
}

static HMatrix h_invert(const HMatrix& H, double eps) {
    return HMatrix(H.tree, invert_node(*H.root, eps), eps);
}

// ---------------------------------------------------------------- ACR driver
// Block = H-matrix (HMatrix mode) or dense matrix (Dense mode, exact oracle).
struct Block {
    bool h = true;
    HMatrix H;
    Mat D;  // dense mode, original ordering
};

struct Arith {
    bool hmode = true;
    double eps = 1e-3;        // arithmetic tolerance (config eps * 0.5)
    double store_eps = 0.0;   // stored-inverse tolerance (config eps)

    Block invert(const Block& a, int level, int plane) const {
        Block out;
        out.h = hmode;
        try {
            if (hmode) out.H = h_invert(a.H, eps);
            else {
                const double rc = lu_inverse(a.D, out.D);
                if (!(rc > 1e-14))
                    throw OracleError(E_SINGULAR, "diagonal block is numerically singular (rcond " +
                                                      std::to_string(rc) + ")");
            }
        } catch (const OracleError& e) {
            if (e.code == E_SINGULAR) throw OracleError(E_SINGULAR, e.what(), level, plane);
            throw;
        }
        return out;
    }
    Block multiply(const Block& a, const Block& b) const {
        Block out;
        out.h = hmode;
        if (hmode) out.H = h_multiply(a.H, b.H, eps);
        else out.D = matmul(a.D, b.D);
        return out;
    }
    void multiply_add(Block& c, const Block& a, const Block& b, double alpha) const {
        if (hmode) mult_add(*c.H.root, *a.H.root, *b.H.root, alpha, eps);
        else gemm(false, false, c.D.r, c.D.c, a.D.c, alpha, a.D.a.data(), a.D.r, b.D.a.data(), b.D.r, c.D.a.data(), c.D.r);
    }
    Block zeros_like(const Block& a) const {
        Block out;
        out.h = hmode;
        if (hmode) out.H = HMatrix(a.H.tree, orc::zero_like(*a.H.root), a.H.eps);
        else out.D = Mat(a.D.r, a.D.c);
        return out;
    }
    Mat apply(const Block& a, const Mat& x) const {
        if (hmode) return h_apply(a.H, x);
        Mat y(a.D.r, x.c);
        gemm(false, false, a.D.r, x.c, a.D.c, 1.0, a.D.a.data(), a.D.r, x.a.data(), x.r, y.a.data(), y.r);
        return y;
    }
    long bytes(const Block& a) const {
        if (hmode) return rank_stats(*a.H.root).bytes;
        return 8L * a.D.r * a.D.c;
    }
    void collect(const Block& a, RankStats& s) const {
        if (hmode) merge_stats(s, rank_stats(*a.H.root));
    }
    void recompress_stored(Block& a) const {
        if (hmode && store_eps > eps) recompress(a.H, store_eps);
    }
};

using OB = std::optional<Block>;

static std::vector<int> eliminated_positions(int m) {  // acr.cpp:46-51
    std::vector<int> v;
    for (int j = 0; j < m; j += 2) v.push_back(j);
    if (m % 2 == 1 && !v.empty()) v.pop_back();
    return v;
}
static std::vector<int> retained_positions(int m) {  // acr.cpp:53-58
    std::vector<int> v;
    for (int j = 1; j < m; j += 2) v.push_back(j);
    if (m % 2 == 1) v.push_back(m - 1);
    return v;
}

struct Level {
    int plane_count = 0;
    std::vector<int> elim, ret;
    std::vector<OB> E, F, Dinv;
};

struct Apex {
    std::vector<Block> Dinv;
    std::vector<OB> E, F;
};

struct Factorization {
    Arith ar;
    std::vector<Level> levels;
    Apex apex;
    int plane_dim = 0, plane_count = 0;
    double flops[F_NCLASS] = {0};
    long long trunc_calls = 0;
};

// run f(i) for i in [0, count) on up to `threads` workers; rethrow the error
// of the lowest failing index (the one a sequential sweep would report).
static void parallel_for(int count, int threads, const std::function<void(int)>& f) {
    if (threads <= 1 || count <= 1) {
        for (int i = 0; i < count; ++i) f(i);
        return;
    }
    std::vector<std::exception_ptr> errs(count);
    std::atomic<int> next{0};
    auto work = [&]() {
        for (;;) {
            const int i = next.fetch_add(1);
            if (i >= count) return;
            try {
                f(i);
            } catch (...) {
                errs[i] = std::current_exception();
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::min(threads, count); ++t) pool.emplace_back(work);
    for (auto& t : pool) t.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

struct RetainedUpdate {  // acr.hpp:71-76
    Block D;
    OB E, F;
};

// Eq. (6) of the paper, acr.hpp:78-107
static RetainedUpdate eliminate_around(const Arith& ar, const Block& Dj, const Block* Ej, const Block* Fj,
                                       const Block* Dlo, const Block* Elo, const Block* Flo,
                                       const Block* Dhi, const Block* Ehi, const Block* Fhi) {
    RetainedUpdate out;
    out.D = Dj;
    if (Dlo) {
        Block T = ar.multiply(*Ej, *Dlo);
        if (Flo) ar.multiply_add(out.D, T, *Flo, -1.0);
        if (Elo) {
            Block En = ar.zeros_like(Dj);
            ar.multiply_add(En, T, *Elo, -1.0);
            out.E = std::move(En);
        }
    }
    if (Dhi) {
        Block T = ar.multiply(*Fj, *Dhi);
        if (Ehi) ar.multiply_add(out.D, T, *Ehi, -1.0);
        if (Fhi) {
            Block Fn = ar.zeros_like(Dj);
            ar.multiply_add(Fn, T, *Fhi, -1.0);
            out.F = std::move(Fn);
        }
    }
    return out;
}

static const Block* at(const std::vector<OB>& v, int j) {
    if (j < 0 || j >= (int)v.size() || !v[j]) return nullptr;
    return &*v[j];
}

static Level reduce_level(const Arith& ar, int lvl, std::vector<OB>& D, std::vector<OB>& E, std::vector<OB>& F,
                          int threads) {
    const int m = (int)D.size();
    Level L;
    L.plane_count = m;
    L.elim = eliminated_positions(m);
    L.ret = retained_positions(m);
    L.E = std::move(E);
    L.F = std::move(F);
    L.Dinv.resize(m);
    std::vector<char> is_elim(m, 0);
    for (int e : L.elim) is_elim[e] = 1;
    parallel_for((int)L.elim.size(), threads, [&](int t) {
        const int e = L.elim[t];
        L.Dinv[e] = ar.invert(*D[e], lvl, e);
    });
    const int mn = (int)L.ret.size();
    std::vector<OB> Dn(mn), En(mn), Fn(mn);
    parallel_for(mn, threads, [&](int t) {
        const int j = L.ret[t];
        const bool lo = j > 0 && is_elim[j - 1];
        const bool hi = j + 1 < m && is_elim[j + 1];
        RetainedUpdate u = eliminate_around(ar, *D[j], at(L.E, j), at(L.F, j), lo ? &*L.Dinv[j - 1] : nullptr,
                                            at(L.E, j - 1), at(L.F, j - 1), hi ? &*L.Dinv[j + 1] : nullptr,
                                            at(L.E, j + 1), at(L.F, j + 1));
        Dn[t] = std::move(u.D);
        if (u.E) En[t] = std::move(u.E);
        else if (t > 0 && L.ret[t - 1] == j - 1) En[t] = *L.E[j];
        if (u.F) Fn[t] = std::move(u.F);
        else if (t + 1 < mn && L.ret[t + 1] == j + 1) Fn[t] = *L.F[j];
    });
    D = std::move(Dn);
    E = std::move(En);
    F = std::move(Fn);
    parallel_for((int)L.elim.size(), threads, [&](int t) { ar.recompress_stored(*L.Dinv[L.elim[t]]); });
    return L;
}

static Apex factor_apex(const Arith& ar, int lvl, std::vector<OB>& D, std::vector<OB>& E, std::vector<OB>& F) {
    const int s = (int)D.size();
    Apex ap;
    ap.E = std::move(E);
    ap.F = std::move(F);
    for (int i = 0; i < s; ++i) {  // block Thomas (acr.cpp:123-144)
        Block Di = std::move(*D[i]);
        if (i > 0) {
            Block T = ar.multiply(*ap.E[i], ap.Dinv[i - 1]);
            ar.multiply_add(Di, T, *ap.F[i - 1], -1.0);
        }
        ap.Dinv.push_back(ar.invert(Di, lvl, i));
    }
    for (auto& d : ap.Dinv) ar.recompress_stored(d);
    return ap;
}

// forward_rhs / back_substitute (acr.hpp:111-132)
static Mat forward_rhs(const Arith& ar, const Mat& fj, const Block* Ej, const Block* Dlo, const Mat* flo,
                       const Block* Fj, const Block* Dhi, const Mat* fhi) {
    Mat out = fj;
    if (Dlo && flo) {
        Mat t = ar.apply(*Ej, ar.apply(*Dlo, *flo));
        for (size_t i = 0; i < out.size(); ++i) out.a[i] -= t.a[i];
    }
    if (Dhi && fhi) {
        Mat t = ar.apply(*Fj, ar.apply(*Dhi, *fhi));
        for (size_t i = 0; i < out.size(); ++i) out.a[i] -= t.a[i];
    }
    return out;
}

static Mat back_substitute(const Arith& ar, const Block& Dinv, const Mat& fe, const Block* Ee, const Mat* ulo,
                           const Block* Fe, const Mat* uhi) {
    Mat r = fe;
    if (Ee && ulo) {
        Mat t = ar.apply(*Ee, *ulo);
        for (size_t i = 0; i < r.size(); ++i) r.a[i] -= t.a[i];
    }
    if (Fe && uhi) {
        Mat t = ar.apply(*Fe, *uhi);
        for (size_t i = 0; i < r.size(); ++i) r.a[i] -= t.a[i];
    }
    return ar.apply(Dinv, r);
}

// f: per plane a (dim x nrhs) panel.  Columns are processed independently with
// a fixed loop order, so multi-RHS solves equal single-RHS solves bitwise.
static std::vector<Mat> solve(const Factorization& fa, const std::vector<Mat>& f, int threads) {
    const Arith& ar = fa.ar;
    if ((int)f.size() != fa.plane_count)
        throw OracleError(E_DIMENSION, "solve: right-hand side has " + std::to_string(f.size()) +
                                           " planes, factorization has " + std::to_string(fa.plane_count));
    std::vector<std::vector<Mat>> fs;
    fs.push_back(f);
    for (const auto& L : fa.levels) {
        const auto& cur = fs.back();
        const int m = L.plane_count;
        std::vector<Mat> next(L.ret.size());
        parallel_for((int)L.ret.size(), threads, [&](int t) {
            const int j = L.ret[t];
            const bool lo = j > 0 && L.Dinv[j - 1].has_value();
            const bool hi = j + 1 < m && L.Dinv[j + 1].has_value();
            next[t] = forward_rhs(ar, cur[j], at(L.E, j), lo ? &*L.Dinv[j - 1] : nullptr, lo ? &cur[j - 1] : nullptr,
                                  at(L.F, j), hi ? &*L.Dinv[j + 1] : nullptr, hi ? &cur[j + 1] : nullptr);
        });
        fs.push_back(std::move(next));
    }
    // apex (acr.cpp:162-178)
    const auto& g0 = fs.back();
    const int s = (int)fa.apex.Dinv.size();
    std::vector<Mat> g(s), u(s);
    for (int i = 0; i < s; ++i) {
        g[i] = g0[i];
        if (i > 0) {
            Mat t = ar.apply(*fa.apex.E[i], ar.apply(fa.apex.Dinv[i - 1], g[i - 1]));
            for (size_t q = 0; q < g[i].size(); ++q) g[i].a[q] -= t.a[q];
        }
    }
    for (int i = s - 1; i >= 0; --i) {
        Mat r = g[i];
        if (i + 1 < s) {
            Mat t = ar.apply(*fa.apex.F[i], u[i + 1]);
            for (size_t q = 0; q < r.size(); ++q) r.a[q] -= t.a[q];
        }
        u[i] = ar.apply(fa.apex.Dinv[i], r);
    }
    for (int li = (int)fa.levels.size() - 1; li >= 0; --li) {
        const auto& L = fa.levels[li];
        const auto& fl = fs[li];
        const int m = L.plane_count;
        std::vector<Mat> ul(m);
        for (size_t t = 0; t < L.ret.size(); ++t) ul[L.ret[t]] = std::move(u[t]);
        parallel_for((int)L.elim.size(), threads, [&](int t) {
            const int e = L.elim[t];
            ul[e] = back_substitute(ar, *L.Dinv[e], fl[e], at(L.E, e), e > 0 ? &ul[e - 1] : nullptr, at(L.F, e),
                                    e + 1 < m ? &ul[e + 1] : nullptr);
        });
        u = std::move(ul);
    }
    return u;
}

}  // namespace orc

// =============================================================================
// extern "C" surface (ctypes; tests + bench only)
// =============================================================================
using namespace orc;

extern "C" {

struct orc_config {
    int mode;             // 0 = H-matrix, 1 = dense
    double eps;
    double eta;
    int leaf_size;
    int weak;             // 0 = standard admissibility, 1 = weak
    int stop_planes;
    long leaf_memory_cap;
    int threads;
};

struct orc_error {
    int code;
    int level;
    int plane;
    char msg[256];
};

static void set_err(orc_error* err, int code, const char* msg, int level = -1, int plane = -1) {
    if (!err) return;
    err->code = code;
    err->level = level;
    err->plane = plane;
    std::snprintf(err->msg, sizeof(err->msg), "%s", msg);
}

#define ORC_TRY(err, ...)                                                 \
    try {                                                                  \
        __VA_ARGS__                                                        \
    } catch (const OracleError& e) {                                       \
        set_err(err, e.code, e.what(), e.level, e.plane);                  \
    } catch (const std::exception& e) {                                    \
        set_err(err, E_INTERNAL, e.what());                                \
    }

void orc_flops_reset() {
    for (auto& f : g_flops) f.store(0);
    g_trunc_calls.store(0);
}
void orc_flops_read(double* out) {
    for (int i = 0; i < F_NCLASS; ++i) out[i] = (double)g_flops[i].load();
    out[F_NCLASS] = (double)g_trunc_calls.load();
}
void orc_trace_enable(int on) {
    std::lock_guard<std::mutex> lk(g_trace_mu);
    g_trace_on = on != 0;
    g_trace.clear();
}
long orc_trace_read(int* out, long cap) {
    std::lock_guard<std::mutex> lk(g_trace_mu);
    const long n = (long)g_trace.size();
    if (out)
        for (long i = 0; i < std::min(n, cap); ++i)
            for (int k = 0; k < 6; ++k) out[i * 6 + k] = g_trace[i][k];
    return n;
}

// ---- structure --------------------------------------------------------------
struct orc_bct {
    std::shared_ptr<ClusterTree> tree;
    std::unique_ptr<BlockTree> bt;
};

void* orc_bct_create(int dim, const double* xy, int leaf, double eta, int weak, orc_error* err) {
    set_err(err, OK, "");
    ORC_TRY(err, {
        auto* b = new orc_bct;
        b->tree = std::make_shared<ClusterTree>(std::vector<double>(xy, xy + 2L * dim), leaf);
        b->bt = std::make_unique<BlockTree>(b->tree, eta, weak);
        return b;
    })
    return nullptr;
}
void orc_bct_free(void* p) { delete (orc_bct*)p; }

void orc_bct_perm(void* p, int* perm) {
    auto* b = (orc_bct*)p;
    std::copy(b->tree->perm.begin(), b->tree->perm.end(), perm);
}

// cluster tree summary: leaf count, depth
void orc_bct_cluster_info(void* p, int* leaves, int* depth) {
    auto* b = (orc_bct*)p;
    std::function<void(const Cluster*, int)> walk = [&](const Cluster* c, int d) {
        if (c->leaf()) {
            ++*leaves;
            *depth = std::max(*depth, d);
            return;
        }
        walk(c->lo.get(), d + 1);
        walk(c->hi.get(), d + 1);
    };
    *leaves = 0;
    *depth = 0;
    walk(b->tree->root.get(), 0);
}

// leaves in depth-first (child 0..3) order: rb, re, cb, ce, kind; returns count
long orc_bct_leaves(void* p, int* out, long cap) {
    auto* b = (orc_bct*)p;
    long n = 0;
    std::function<void(const BNode&)> walk = [&](const BNode& bn) {
        if (bn.kind == BRANCH) {
            for (int i = 0; i < 4; ++i) walk(*bn.ch[i]);
            return;
        }
        if (out && n < cap) {
            int* o = out + 5 * n;
            o[0] = bn.row->begin; o[1] = bn.row->end; o[2] = bn.col->begin; o[3] = bn.col->end; o[4] = bn.kind;
        }
        ++n;
    };
    walk(*b->bt->root);
    return n;
}

// ---- H-matrix handles (test surface, mirrors hmatrix.hpp:62-108) ------------
void* orc_h_compress_sparse(void* pb, long nnz, const int* rows, const int* cols, const double* vals, double eps,
                            long cap, orc_error* err) {
    set_err(err, OK, "");
    ORC_TRY(err, {
        auto* b = (orc_bct*)pb;
        std::vector<Entry> ent(nnz);
        const int dim = b->tree->size();
        for (long i = 0; i < nnz; ++i) {
            if (rows[i] < 0 || rows[i] >= dim || cols[i] < 0 || cols[i] >= dim)
                throw OracleError(E_DIMENSION, "PlaneBlock: entry index out of range");
            ent[i] = Entry{rows[i], cols[i], vals[i]};
        }
        return new HMatrix(h_compress_sparse(*b->bt, ent, eps, cap));
    })
    return nullptr;
}

void* orc_h_compress_dense(void* pb, const double* A, double eps, orc_error* err) {
    set_err(err, OK, "");
    ORC_TRY(err, {
        auto* b = (orc_bct*)pb;
        const int n = b->tree->size();
        const auto& perm = b->tree->perm;
        Mat P(n, n);
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) P(i, j) = A[(size_t)perm[j] * n + perm[i]];
        return new HMatrix(b->tree, build_dense(*b->bt->root, P, eps, 2L << 30), eps);
    })
    return nullptr;
}

void orc_h_free(void* h) { delete (HMatrix*)h; }
void* orc_h_clone(void* h) { return new HMatrix(*(HMatrix*)h); }

void orc_h_to_dense(void* ph, double* out) {  // original ordering, column-major
    auto* H = (HMatrix*)ph;
    const int n = H->dim();
    Mat P(n, n);
    to_dense_walk(*H->root, P);
    const auto& perm = H->tree->perm;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) out[(size_t)perm[j] * n + perm[i]] = P(i, j);
}

int orc_h_apply(void* ph, int nrhs, const double* X, double* Y, orc_error* err) {
    set_err(err, OK, "");
    ORC_TRY(err, {
        auto* H = (HMatrix*)ph;
        const int n = H->dim();
        Mat x(n, nrhs);
        std::copy(X, X + (size_t)n * nrhs, x.a.begin());
        Mat y = h_apply(*H, x);
        std::copy(y.a.begin(), y.a.end(), Y);
        return 0;
    })
    return err ? err->code : -1;
}

int orc_h_apply_checked(void* ph, int rows, int nrhs, const double* X, double* Y, orc_error* err) {
    set_err(err, OK, "");
    auto* H = (HMatrix*)ph;
    if (rows != H->dim()) {
        set_err(err, E_DIMENSION, "happly: row count mismatch");
        return E_DIMENSION;
    }
    return orc_h_apply(ph, nrhs, X, Y, err);
}

void* orc_h_multiply(void* a, void* b, double eps, orc_error* err) {
    set_err(err, OK, "");
    ORC_TRY(err, { return new HMatrix(h_multiply(*(HMatrix*)a, *(HMatrix*)b, eps)); })
    return nullptr;
}

int orc_h_multiply_add(void* c, void* a, void* b, double alpha, double eps, orc_error* err) {
    set_err(err, OK, "");
    ORC_TRY(err, {
        mult_add(*((HMatrix*)c)->root, *((HMatrix*)a)->root, *((HMatrix*)b)->root, alpha, eps);
        return 0;
    })
    return err ? err->code : -1;
}

void* orc_h_add(void* a, void* b, double alpha, double eps, orc_error* err) {
    set_err(err, OK, "");
    ORC_TRY(err, {
        auto* A = (HMatrix*)a;
        auto* B = (HMatrix*)b;
        if (A->tree != B->tree || !same_structure(*A->root, *B->root))
            throw OracleError(E_DIMENSION, "H-matrix operands must share one block structure");
        auto* C = new HMatrix(*A);
        add_node(*C->root, *B->root, alpha, eps);
        return C;
    })
    return nullptr;
}

void* orc_h_invert(void* a, double eps, orc_error* err) {
    set_err(err, OK, "");
    ORC_TRY(err, { return new HMatrix(h_invert(*(HMatrix*)a, eps)); })
    return nullptr;
}

void orc_h_recompress(void* a, double eps) { recompress(*(HMatrix*)a, eps); }

void orc_h_rank_stats(void* a, double* avg, int* largest, int* ndense, int* nrk, long* bytes) {
    RankStats s = rank_stats(*((HMatrix*)a)->root);
    *avg = s.average_rank;
    *largest = s.largest_rank;
    *ndense = s.dense_leaf_count;
    *nrk = s.lowrank_leaf_count;
    *bytes = s.bytes;
}

// leaf ranks in depth-first order (-1 for dense leaves)
long orc_h_leaf_ranks(void* a, int* out, long cap) {
    long n = 0;
    std::function<void(const HNode&)> walk = [&](const HNode& h) {
        if (h.kind == BRANCH) {
            for (int i = 0; i < 4; ++i) walk(*h.ch[i]);
            return;
        }
        if (out && n < cap) out[n] = h.kind == RK ? h.rank() : -1;
        ++n;
    };
    walk(*((HMatrix*)a)->root);
    return n;
}

// truncate_lowrank (hmatrix.hpp:106-108) on explicit factors; returns rank r,
// Uout (m x r) and Vout (n x r) must hold m*K and n*K doubles.
int orc_truncate(int m, int n, int K, const double* U, const double* V, double eps, double abs_cut, double* Uout,
                 double* Vout) {
    Mat u(m, K), v(n, K);
    std::copy(U, U + (size_t)m * K, u.a.begin());
    std::copy(V, V + (size_t)n * K, v.a.begin());
    truncate(u, v, eps, abs_cut);
    std::copy(u.a.begin(), u.a.end(), Uout);
    std::copy(v.a.begin(), v.a.end(), Vout);
    return u.c;
}

// singular values of a (r x c) column-major matrix, descending
void orc_svd_values(int r, int c, const double* A, double* s) {
    Mat M(r, c);
    std::copy(A, A + (size_t)r * c, M.a.begin());
    SVDResult sv;
    svd(M, sv, false);
    std::copy(sv.s.begin(), sv.s.end(), s);
}

double orc_lu_inverse(int n, const double* A, double* inv) {
    Mat M(n, n), I;
    std::copy(A, A + (size_t)n * n, M.a.begin());
    const double rc = lu_inverse(M, I);
    std::copy(I.a.begin(), I.a.end(), inv);
    return rc;
}

// ---- ACR factor / solve -------------------------------------------------------
// System layout (shared with the product's C-ABI, include/acrgpu.h):
//   blocks 0..n-1 = D(j), n..2n-2 = E(j) for j = 1..n-1 (couples j -> j-1),
//   2n-1..3n-3 = F(j) for j = 0..n-2 (couples j -> j+1); block b's COO entries
//   are [blk_off[b], blk_off[b+1]) of rows/cols/vals (plane-local indices).
struct orc_fact {
    Factorization fa;
};

void* orc_factor(int n, int dim, const double* xy, const long* blk_off, const int* rows, const int* cols,
                 const double* vals, const orc_config* cfg, orc_error* err) {
    set_err(err, OK, "");
    ORC_TRY(err, {
        if (n < 1 || dim < 1) throw OracleError(E_DIMENSION, "acr_factor: empty system");
        if (cfg->stop_planes < 1) throw OracleError(E_USAGE, "acr_factor: stop_planes must be >= 1");
        const int nb = 3 * n - 2;
        std::vector<std::vector<Entry>> blocks(nb);
        for (int b = 0; b < nb; ++b) {
            for (long i = blk_off[b]; i < blk_off[b + 1]; ++i) {
                if (rows[i] < 0 || rows[i] >= dim || cols[i] < 0 || cols[i] >= dim)
                    throw OracleError(E_DIMENSION, "PlaneBlock: entry index out of range");
                blocks[b].push_back(Entry{rows[i], cols[i], vals[i]});
            }
        }
        auto* out = new orc_fact;
        Factorization& fa = out->fa;
        fa.plane_dim = dim;
        fa.plane_count = n;
        fa.ar.hmode = cfg->mode == 0;
        fa.ar.eps = fa.ar.hmode ? cfg->eps * 0.5 : 0.0;  // acr.hpp:178-181
        fa.ar.store_eps = fa.ar.hmode ? cfg->eps : 0.0;
        const int th = std::max(1, cfg->threads);
        std::vector<OB> D(n), E(n), F(n);
        std::vector<int> bid(nb);
        std::iota(bid.begin(), bid.end(), 0);
        std::unique_ptr<orc_bct> st;
        if (fa.ar.hmode) {  // lift_hmatrix (acr.cpp:316-333)
            st = std::make_unique<orc_bct>();
            st->tree = std::make_shared<ClusterTree>(std::vector<double>(xy, xy + 2L * dim), cfg->leaf_size);
            st->bt = std::make_unique<BlockTree>(st->tree, cfg->eta, cfg->weak);
        }
        parallel_for(nb, th, [&](int b) {
            Block blk;
            blk.h = fa.ar.hmode;
            if (fa.ar.hmode) blk.H = h_compress_sparse(*st->bt, blocks[b], cfg->eps, cfg->leaf_memory_cap);
            else {
                blk.D = Mat(dim, dim);
                for (const auto& e : blocks[b]) blk.D(e.r, e.c) += e.v;
            }
            if (b < n) D[b] = std::move(blk);
            else if (b < 2 * n - 1) E[b - n + 1] = std::move(blk);
            else F[b - (2 * n - 1)] = std::move(blk);
        });
        int lvl = 0;
        while ((int)D.size() > cfg->stop_planes) fa.levels.push_back(reduce_level(fa.ar, lvl++, D, E, F, th));
        fa.apex = factor_apex(fa.ar, lvl, D, E, F);
        return out;
    })
    return nullptr;
}

void orc_factor_free(void* f) { delete (orc_fact*)f; }

// f, u: [nrhs][n][dim] (plane-major per right-hand side)
int orc_solve(void* pf, int nrhs, const double* f, double* u, int threads, orc_error* err) {
    set_err(err, OK, "");
    ORC_TRY(err, {
        const Factorization& fa = ((orc_fact*)pf)->fa;
        const int n = fa.plane_count, d = fa.plane_dim;
        std::vector<Mat> planes(n, Mat(d, nrhs));
        for (int r = 0; r < nrhs; ++r)
            for (int j = 0; j < n; ++j)
                std::copy(f + ((size_t)r * n + j) * d, f + ((size_t)r * n + j + 1) * d, planes[j].col(r));
        std::vector<Mat> x = solve(fa, planes, threads);
        for (int r = 0; r < nrhs; ++r)
            for (int j = 0; j < n; ++j) std::copy(x[j].col(r), x[j].col(r) + d, u + ((size_t)r * n + j) * d);
        return 0;
    })
    return err ? err->code : -1;
}

// factor_bytes (acr.cpp:231-248), inverse rank stats (acr.cpp:250-258)
void orc_factor_stats(void* pf, double* avg, int* largest, int* ndense, int* nrk, long* inv_bytes, long* factor_bytes) {
    const Factorization& fa = ((orc_fact*)pf)->fa;
    const Arith& ar = fa.ar;
    RankStats s;
    long total = 0;
    for (const auto& L : fa.levels) {
        for (const auto& b : L.E)
            if (b) total += ar.bytes(*b);
        for (const auto& b : L.F)
            if (b) total += ar.bytes(*b);
        for (const auto& b : L.Dinv)
            if (b) {
                total += ar.bytes(*b);
                ar.collect(*b, s);
            }
    }
    for (const auto& b : fa.apex.E)
        if (b) total += ar.bytes(*b);
    for (const auto& b : fa.apex.F)
        if (b) total += ar.bytes(*b);
    for (const auto& b : fa.apex.Dinv) {
        total += ar.bytes(b);
        ar.collect(b, s);
    }
    *avg = s.average_rank;
    *largest = s.largest_rank;
    *ndense = s.dense_leaf_count;
    *nrk = s.lowrank_leaf_count;
    *inv_bytes = s.bytes;
    *factor_bytes = total;
}

// level_info (acr.cpp:260-300); arrays of length >= levels+1; returns count
int orc_level_info(void* pf, int cap, int* level, int* plane_count, int* eliminated, long* bytes, int* largest,
                   double* avg) {
    const Factorization& fa = ((orc_fact*)pf)->fa;
    const Arith& ar = fa.ar;
    int k = 0;
    for (size_t i = 0; i < fa.levels.size() && k < cap; ++i, ++k) {
        const auto& L = fa.levels[i];
        RankStats s;
        long b = 0;
        for (const auto& x : L.Dinv)
            if (x) {
                b += ar.bytes(*x);
                ar.collect(*x, s);
            }
        for (const auto& x : L.E)
            if (x) b += ar.bytes(*x);
        for (const auto& x : L.F)
            if (x) b += ar.bytes(*x);
        level[k] = (int)i;
        plane_count[k] = L.plane_count;
        eliminated[k] = (int)L.elim.size();
        bytes[k] = b;
        largest[k] = s.largest_rank;
        avg[k] = s.average_rank;
    }
    if (k < cap) {
        RankStats s;
        long b = 0;
        for (const auto& x : fa.apex.Dinv) {
            b += ar.bytes(x);
            ar.collect(x, s);
        }
        for (const auto& x : fa.apex.E)
            if (x) b += ar.bytes(*x);
        for (const auto& x : fa.apex.F)
            if (x) b += ar.bytes(*x);
        level[k] = (int)fa.levels.size();
        plane_count[k] = (int)fa.apex.Dinv.size();
        eliminated[k] = plane_count[k];
        bytes[k] = b;
        largest[k] = s.largest_rank;
        avg[k] = s.average_rank;
        ++k;
    }
    return k;
}

// Leaf ranks of a stored inverse: level li (== levels for the apex), plane j.
long orc_factor_dinv_ranks(void* pf, int li, int j, int* out, long cap) {
    const Factorization& fa = ((orc_fact*)pf)->fa;
    const Block* b = nullptr;
    if (li < (int)fa.levels.size()) b = at(fa.levels[li].Dinv, j);
    else if (j < (int)fa.apex.Dinv.size()) b = &fa.apex.Dinv[j];
    if (!b || !b->h) return -1;
    long n = 0;
    std::function<void(const HNode&)> walk = [&](const HNode& h) {
        if (h.kind == BRANCH) {
            for (int i = 0; i < 4; ++i) walk(*h.ch[i]);
            return;
        }
        if (out && n < cap) out[n] = h.kind == RK ? h.rank() : -1;
        ++n;
    };
    walk(*b->H.root);
    return n;
}

}  // extern "C"
