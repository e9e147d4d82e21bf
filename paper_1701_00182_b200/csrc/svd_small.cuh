// Register-resident one-sided Jacobi SVD for blocks of at most 32 x 32 (one
// warp per block) and 64 x 64 (four warps per block).
//
// Layout: one-sided Jacobi on the augmented matrix [A; I], A = M or M^T with
// rows >= cols.  Each thread owns ONE ROW in registers -- a row of A or a row of
// the right-rotation accumulator V -- so a column rotation is applied by every
// thread to two of its own registers with no data movement; only the three
// inner products per column pair need communication (warp reduce-scatter, plus
// one shared-memory combine across the two A-row warps of the 64 variant).
// Pairs follow the round-robin tournament; instead of indexing registers
// dynamically, the columns are moved through the fixed circle permutation
// after every round, so all register indices are compile-time constants and a
// full sweep (NC-1 rounds) returns every column to its original slot.
// Rotation parameters use two reciprocal square roots (no divisions):
//   d = beta - alpha, g = 2 gamma, w = 1/sqrt(d^2 + g^2), q = (1 + |d| w)/2,
//   c = sqrt(q), s = sign(d) g w / (2 sqrt(q))      (|theta| <= pi/4).
//
// Same algorithm class as the reference's JacobiSVD (hmatrix.cpp:67,89): the
// singular triplets agree to rounding; rank decisions use the reference rule
// sigma_i > max(eps * sigma_1, abs_cut) (hmatrix.cpp:70-74).
#pragma once

namespace acrgpu {

constexpr double JEPS = 2.2204460492503131e-16;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// lanes l and l^16 end with the warp sum of v[l & 15]
__device__ __forceinline__ double reduce_scatter16(double (&v)[16], int lane) {
#pragma unroll
    for (int h = 8; h >= 1; h >>= 1) {
        const bool up = (lane & h) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = up ? v[i] : v[i + h];
            const double keep = up ? v[i + h] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
        }
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

template <int NC>
__device__ __forceinline__ void circle_permute(double (&a)[NC]) {
    constexpr int NP = NC / 2;
    const double b0 = a[1];
    const double tl = a[2 * (NP - 1)];
#pragma unroll
    for (int k = NP - 1; k >= 2; --k) a[2 * k] = a[2 * (k - 1)];
    a[2] = b0;
#pragma unroll
    for (int k = 0; k <= NP - 2; ++k) a[2 * k + 1] = a[2 * k + 3];
    a[2 * NP - 1] = tl;
}

// Rotate iff the pair is not yet orthogonal to working precision and neither
// column is numerically zero (norm below ~eps * ||A||_F: such columns carry only
// rounding noise, whose relative orthogonality can never converge).
__device__ __forceinline__ bool jacobi_params(double al, double be, double ga, double tol2, double zthr, double& c,
                                              double& s) {
    c = 1.0;
    s = 0.0;
    if (!(ga * ga > tol2 * al * be) || !(al > zthr) || !(be > zthr)) return false;
    const double d = be - al, g = 2.0 * ga;
    const double h = fma(d, d, g * g);
    if (!(h > 0.0) || !isfinite(h)) return false;
    const double w = rsqrt(h);
    const double q = fma(0.5 * fabs(d), w, 0.5);
    const double rq = rsqrt(q);
    c = q * rq;
    s = 0.5 * copysign(1.0, d) * g * w * rq;
    return s != 0.0;
}

__device__ __forceinline__ void rot2(double& x, double& y, double c, double s) {
    const double nx = fma(c, x, -s * y);
    const double ny = fma(s, x, c * y);
    x = nx;
    y = ny;
}

// ---------------------------------------------------------------- 32 x 32, one warp
// a: this lane's row of A (row index = lane); v: this lane's row of V.
__device__ int warp_jacobi32(double (&a)[32], double (&v)[32], int rows, bool want_v) {
    const int lane = threadIdx.x & 31;
    const double tol = (double)(rows > 1 ? rows : 1) * JEPS;
    const double tol2 = tol * tol;
    double fro = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) fro = fma(a[j], a[j], fro);
#pragma unroll
    for (int o = 16; o; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
    const double zthr = fro * (16.0 * JEPS * JEPS);
    for (int sweep = 0; sweep < 40; ++sweep) {
        bool any = false;
        for (int round = 0; round < 31; ++round) {
            double r[16];
            double al, be, ga;
#pragma unroll
            for (int k = 0; k < 16; ++k) r[k] = a[2 * k] * a[2 * k];
            al = reduce_scatter16(r, lane);
#pragma unroll
            for (int k = 0; k < 16; ++k) r[k] = a[2 * k + 1] * a[2 * k + 1];
            be = reduce_scatter16(r, lane);
#pragma unroll
            for (int k = 0; k < 16; ++k) r[k] = a[2 * k] * a[2 * k + 1];
            ga = reduce_scatter16(r, lane);
            double c, s;
            const bool rot = jacobi_params(al, be, ga, tol2, zthr, c, s);  // lane l: pair l & 15
            if (__any_sync(0xffffffffu, rot)) {
                any = true;
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const double ck = __shfl_sync(0xffffffffu, c, k);
                    const double sk = __shfl_sync(0xffffffffu, s, k);
                    rot2(a[2 * k], a[2 * k + 1], ck, sk);
                    if (want_v) rot2(v[2 * k], v[2 * k + 1], ck, sk);
                }
            }
            circle_permute<32>(a);
            if (want_v) circle_permute<32>(v);
        }
        if (!any) return sweep + 1;
    }
    return 40;
}

// ---------------------------------------------------------------- 32 x 32, one warp, column per lane
// Lane j owns column j of A (a[i], i = row) and column j of V.  In round r lane j
// is paired with partner(j, r) (round-robin tournament); the pair exchanges its
// columns with register shuffles, both lanes compute the same rotation from
// bitwise-identical inner products, and each lane updates its own column.  No
// reductions, no register permutation.
__device__ __forceinline__ int rr_partner32(int x, int r) {
    // circle method over 32 players, player 0 fixed, 31 rounds
    if (x == 0) return 1 + r;
    const int y = x - 1;
    int yp = (2 * r - y) % 31;
    if (yp < 0) yp += 31;
    return yp == y ? 0 : 1 + yp;
}

__device__ int warp_jacobi32c(double (&a)[32], double (&v)[32], bool want_v, double zthr_floor) {
    const int lane = threadIdx.x & 31;
    const double tol = 32.0 * JEPS;
    const double tol2 = tol * tol;
    double own = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) own = fma(a[i], a[i], own);
    double fro = own;
#pragma unroll
    for (int o = 16; o; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
    const double zthr = fmax(fro * (16.0 * JEPS * JEPS), zthr_floor);
    for (int sweep = 0; sweep < 40; ++sweep) {
        bool any = false;
        for (int round = 0; round < 31; ++round) {
            const int p = rr_partner32(lane, round);
            const bool low = lane < p;
            double pa[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) pa[i] = __shfl_sync(0xffffffffu, a[i], p);
            // inner products in the pair's canonical orientation (low column first)
            double s0 = 0, s1 = 0, s2 = 0, t0 = 0, t1 = 0, t2 = 0;
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                const double xl = low ? a[i] : pa[i], xh = low ? pa[i] : a[i];
                const double yl = low ? a[i + 1] : pa[i + 1], yh = low ? pa[i + 1] : a[i + 1];
                s0 = fma(xl, xl, s0);
                s1 = fma(xh, xh, s1);
                s2 = fma(xl, xh, s2);
                t0 = fma(yl, yl, t0);
                t1 = fma(yh, yh, t1);
                t2 = fma(yl, yh, t2);
            }
            const double al = s0 + t0, be = s1 + t1, ga = s2 + t2;
            double c, s;
            const bool rot = jacobi_params(al, be, ga, tol2, zthr, c, s);
            if (__any_sync(0xffffffffu, rot)) {
                any = true;
                // low:  a' = c a - s pa      high: a' = s pa + c a
                const double sl = low ? -s : s;
#pragma unroll
                for (int i = 0; i < 32; ++i) a[i] = fma(sl, pa[i], c * a[i]);
                if (want_v) {
#pragma unroll
                    for (int i0 = 0; i0 < 32; i0 += 8) {
                        double pv[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) pv[i] = __shfl_sync(0xffffffffu, v[i0 + i], p);
#pragma unroll
                        for (int i = 0; i < 8; ++i) v[i0 + i] = fma(sl, pv[i], c * v[i0 + i]);
                    }
                }
            }
        }
        if (!any) return sweep + 1;
    }
    return 40;
}

// sigma of column (lane) -> sig; rank position of column (lane) -> pos; rank r (warp-uniform)
__device__ void warp_sigma_rank32(const double (&a)[32], int cols, double eps, double abs_cut, double& sig, int& pos,
                                  int& r) {
    const int lane = threadIdx.x & 31;
    double t[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) t[k] = a[k] * a[k];
    const double s0 = reduce_scatter16(t, lane);
#pragma unroll
    for (int k = 0; k < 16; ++k) t[k] = a[16 + k] * a[16 + k];
    const double s1 = reduce_scatter16(t, lane);
    sig = lane < cols ? sqrt(lane < 16 ? s0 : s1) : -1.0;
    pos = 0;
    double smax = sig;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const double w = __shfl_sync(0xffffffffu, sig, i);
        pos += (w > sig) || (w == sig && i < lane);
        smax = fmax(smax, w);
    }
    int cnt = 0;
    if (smax > 0.0) {
        const double cut = fmax(eps * smax, abs_cut);
        cnt = __popc(__ballot_sync(0xffffffffu, lane < cols && sig > cut));
    }
    r = cnt;
}

// ---------------------------------------------------------------- 64 x 64, four warps
// warps 0,1: rows 0-31 / 32-63 of A; warps 2,3: rows 0-31 / 32-63 of V.
struct Smem64 {
    double red[2][2][3][32];  // [buffer][A-warp][alpha,beta,gamma][pair]
    double fro[2];
};

__device__ int cta_jacobi64(double (&a)[64], int rows, bool want_v, Smem64& sm) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool awarp = warp < 2;
    const double tol = (double)(rows > 1 ? rows : 1) * JEPS;
    const double tol2 = tol * tol;
    if (awarp) {
        double f = 0;
#pragma unroll
        for (int j = 0; j < 64; ++j) f = fma(a[j], a[j], f);
#pragma unroll
        for (int o = 16; o; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
        if (lane == 0) sm.fro[warp] = f;
    }
    __syncthreads();
    const double zthr = (sm.fro[0] + sm.fro[1]) * (16.0 * JEPS * JEPS);
    int buf = 0;
    for (int sweep = 0; sweep < 40; ++sweep) {
        int any = 0;
        for (int round = 0; round < 63; ++round) {
            if (awarp) {
                double r[16];
#pragma unroll
                for (int half = 0; half < 2; ++half) {
#pragma unroll
                    for (int k = 0; k < 16; ++k) r[k] = a[2 * (16 * half + k)] * a[2 * (16 * half + k)];
                    const double al = reduce_scatter16(r, lane);
#pragma unroll
                    for (int k = 0; k < 16; ++k) r[k] = a[2 * (16 * half + k) + 1] * a[2 * (16 * half + k) + 1];
                    const double be = reduce_scatter16(r, lane);
#pragma unroll
                    for (int k = 0; k < 16; ++k) r[k] = a[2 * (16 * half + k)] * a[2 * (16 * half + k) + 1];
                    const double ga = reduce_scatter16(r, lane);
                    if ((lane >> 4) == half) {
                        sm.red[buf][warp][0][lane] = al;
                        sm.red[buf][warp][1][lane] = be;
                        sm.red[buf][warp][2][lane] = ga;
                    }
                }
            }
            __syncthreads();
            if (!awarp && !want_v) {
                buf ^= 1;
                continue;
            }
            const double al = sm.red[buf][0][0][lane] + sm.red[buf][1][0][lane];
            const double be = sm.red[buf][0][1][lane] + sm.red[buf][1][1][lane];
            const double ga = sm.red[buf][0][2][lane] + sm.red[buf][1][2][lane];
            double c, s;
            const bool rot = jacobi_params(al, be, ga, tol2, zthr, c, s);  // lane l: pair l
            if (__any_sync(0xffffffffu, rot)) {
                any = 1;
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    const double ck = __shfl_sync(0xffffffffu, c, k);
                    const double sk = __shfl_sync(0xffffffffu, s, k);
                    rot2(a[2 * k], a[2 * k + 1], ck, sk);
                }
            }
            circle_permute<64>(a);
            buf ^= 1;
        }
        if (!__syncthreads_or(any)) return sweep + 1;
    }
    return 40;
}

// column norms of A (64 columns) and rank positions; results for column j on
// every thread via smem arrays sig[64], pos[64]; returns r.
struct SigSmem64 {
    double part[2][64];
    double sig[64];
    int pos[64];
    int r;
};

__device__ int cta_sigma_rank64(const double (&a)[64], int cols, double eps, double abs_cut, SigSmem64& sm) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < 2) {
        double t[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int k = 0; k < 16; ++k) t[k] = a[16 * q + k] * a[16 * q + k];
            const double s = reduce_scatter16(t, lane);
            if (lane < 16) sm.part[warp][16 * q + lane] = s;
        }
    }
    __syncthreads();
    if (threadIdx.x < 64) {
        const int j = threadIdx.x;
        sm.sig[j] = j < cols ? sqrt(sm.part[0][j] + sm.part[1][j]) : -1.0;
    }
    __syncthreads();
    if (threadIdx.x < 64) {
        const int j = threadIdx.x;
        const double v = sm.sig[j];
        int p = 0;
        for (int i = 0; i < 64; ++i) {
            const double w = sm.sig[i];
            p += (w > v) || (w == v && i < j);
        }
        sm.pos[j] = p;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double smax = 0;
        for (int j = 0; j < cols; ++j) smax = fmax(smax, sm.sig[j]);
        int r = 0;
        if (smax > 0.0) {
            const double cut = fmax(eps * smax, abs_cut);
            for (int j = 0; j < cols; ++j) r += sm.sig[j] > cut;
        }
        sm.r = r;
    }
    __syncthreads();
    return sm.r;
}

// One product part in "row-producer" form: A[i, j] += alpha * sum_t P(i, t) Q(j, t)
// over i in [pd, pd+pr), j in [qd, qd+qr).  P(i,t) = P[i*ps + t*pt], Q(j,t) = Q[j*qs + t*qt].
// upper: P and Q are upper-trapezoidal R factors (entries with t < row are zero).
struct RowPart {
    const double* P;
    const double* Q;
    long ps, pt, qs, qt;
    int pd, pr, qd, qr;
    int k;
    int upper;
    double alpha;
};

// Accumulate a part into register rows: thread with row index `row` (< NC, or -1
// if it owns no A row).  Q is staged in shared memory Qs[NC][TC+1] by `nthr`
// cooperating threads (sync: per-warp __syncwarp when nthr == 32, else CTA).
template <int NC, int TC>
__device__ void rows_accumulate(double (&a)[NC], int row, const RowPart& p, double (*Qs)[TC + 1], int tid, int nthr) {
    const bool own = row >= p.pd && row < p.pd + p.pr;
    const int ir = row - p.pd;
    for (int t0 = 0; t0 < p.k; t0 += TC) {
        const int tn = min(TC, p.k - t0);
        if (nthr == 32) __syncwarp(); else __syncthreads();
        for (int e = tid; e < NC * TC; e += nthr) {
            const int j = e % NC, t = e / NC;
            double q = 0.0;
            const int jr = j - p.qd;
            if (t < tn && jr >= 0 && jr < p.qr && !(p.upper && t0 + t < jr)) q = p.Q[jr * p.qs + (long)(t0 + t) * p.qt];
            Qs[j][t] = q;
        }
        if (nthr == 32) __syncwarp(); else __syncthreads();
        if (own) {
            for (int t = 0; t < tn; ++t) {
                double pv = (p.upper && t0 + t < ir) ? 0.0 : p.P[ir * p.ps + (long)(t0 + t) * p.pt];
                pv *= p.alpha;
#pragma unroll
                for (int j = 0; j < NC; ++j) a[j] = fma(pv, Qs[j][t], a[j]);
            }
        }
    }
    if (nthr == 32) __syncwarp(); else __syncthreads();
}

}  // namespace acrgpu
