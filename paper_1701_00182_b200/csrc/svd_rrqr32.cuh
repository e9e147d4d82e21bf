// Rank-revealing truncated SVD of blocks up to 32 x 32, one warp per block.
//
//   1. Householder QR with column pivoting (column per lane, fully unrolled) on
//      M (m x n); it stops as soon as every remaining column norm is below
//      delta, a threshold 1e-3 below the truncation cutoff: M P = Q [R; ~0] with
//      R of rp <= min(m, n) rows, and the dropped remainder has norm
//      <= sqrt(32) * delta = 1e-3 * cutoff, so every singular value above the
//      cutoff is reproduced to 1e-3 of the cutoff and rank decisions match the
//      reference (hmatrix.cpp:70-74) except for values within that band.
//   2. One-sided Jacobi on A' = R^T (n x rp): columns of A' are rows of R, one
//      column per lane; each round a lane exchanges its column with its
//      round-robin partner by register shuffles, both lanes form the same
//      rotation from bitwise-identical inner products.  The QR
//      preconditioning (Drmac-Veselic) and the reduced column count rp make
//      this converge in a few short sweeps.
//   3. U' = Q [J_r Sigma_r; 0] (reflectors applied per lane), V' = P W_r Sigma_r^{-1},
//      with J_r Sigma_r = R W_r Sigma_r^{-1} (R = J W^T), so J is never accumulated.
//
// Mathematically the same truncated SVD the reference computes with QR(U),
// QR(V) and JacobiSVD of the core (hmatrix.cpp:56-84).
#pragma once

namespace acrgpu {

struct Warp32Smem {
    double H[32][33];  // H[k][i]: essential part of reflector k (i > k)
    double T[32][33];  // staging: formation chunks, then the R^T transpose
    double tau[32];
    int perm[32];
};

__device__ __forceinline__ int rr_partner(int x, int r, int P) {
    // circle method over P (even) players, player 0 fixed, P-1 rounds
    if (x == 0) return 1 + r;
    const int y = x - 1;
    int yp = (2 * r - y) % (P - 1);
    if (yp < 0) yp += P - 1;
    return yp == y ? 0 : 1 + yp;
}

// Phase 1+2.  In: lane j holds column j of M in a[0..m).  Out: returns rp;
// lane c < rp holds column c of W = R^T J in a[0..n); sm.H / sm.tau / sm.perm describe
// Q and P, sm.T holds R^T.  (v / want_v: unused, kept for call-site compatibility.)
__device__ int warp_rrqr_jacobi32(double (&a)[32], double (&v)[32], int m, int n, double delta_rel,
                                  double abs_delta, bool want_v, Warp32Smem& sm, unsigned long long* wt = nullptr) {
    const int lane = threadIdx.x & 31;
    const unsigned FULL = 0xffffffffu;
    int perm_j = lane;
    // column norms and pivot threshold
    double c2 = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) c2 = fma(a[i], a[i], c2);
    double cmax = lane < n ? c2 : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) cmax = fmax(cmax, __shfl_xor_sync(FULL, cmax, o));
    const double d1 = delta_rel * sqrt(cmax);
    const double delta2 = fmax(d1 * d1, abs_delta * abs_delta);
    const int kmax = m < n ? m : n;
    int rp = 0;
    // ---- QR with column pivoting, stopped at the numerical rank.
    // The step loop is rolled (one copy of the code for every k): a fully unrolled
    // 32-step loop is ~40k SASS instructions, and a warp running it alone (the top
    // cyclic-reduction levels, a handful of tasks per launch) stalls on instruction
    // fetch.  Per-k register indexing becomes masks over the unrolled i loops; every
    // FMA sequence is the one of the unrolled form (leading terms are exact zeros or
    // ones), so the results are bitwise unchanged.
#pragma unroll 1
    for (int k = 0; k < kmax; ++k) {
        double nr = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const double ai = i >= k ? a[i] : 0.0;
            nr = fma(ai, ai, nr);
        }
        double best = (lane >= k && lane < n) ? nr : -1.0;
        int bidx = lane;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const double ob = __shfl_xor_sync(FULL, best, o);
            const int oi = __shfl_xor_sync(FULL, bidx, o);
            if (ob > best || (ob == best && oi < bidx)) {
                best = ob;
                bidx = oi;
            }
        }
        if (!(best > delta2)) break;
        if (bidx != k) {
            const int src = lane == k ? bidx : (lane == bidx ? k : lane);
#pragma unroll
            for (int i = 0; i < 32; ++i) a[i] = __shfl_sync(FULL, a[i], src);
            perm_j = __shfl_sync(FULL, perm_j, src);
        }
        // lane k publishes its column; every lane derives the reflector from it
        if (lane == k) {
#pragma unroll
            for (int i = 0; i < 32; ++i) sm.H[k][i] = a[i];
        }
        __syncwarp();
        const double* hk = sm.H[k];
        double tail = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const double h = i > k ? hk[i] : 0.0;
            tail = fma(h, h, tail);
        }
        const double c0 = hk[k];
        double tau = 0.0, inv = 0.0, beta = c0;
        if (tail > 2.2250738585072014e-308) {
            beta = sqrt(c0 * c0 + tail);
            if (c0 >= 0) beta = -beta;
            inv = 1.0 / (c0 - beta);
            tau = (beta - c0) / beta;
        }
        // v = [0 (i < k); 1; hk[i] * inv (i > k)], formed once (v[] is free during the QR)
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = i > k ? (tau != 0.0 ? hk[i] * inv : 0.0) : (i == k ? 1.0 : 0.0);
        if (lane > k && tau != 0.0) {
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < 32; ++i) s = fma(v[i], a[i], s);
            s *= tau;
#pragma unroll
            for (int i = 0; i < 32; ++i) a[i] = fma(-s, v[i], a[i]);
        }
        __syncwarp();  // all lanes read the raw column before lane k stores the reflector
        if (lane == k) {
            // the stored reflector (Q for the write phase): [0; 1; v] in full length
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                sm.H[k][i] = v[i];
                if (i == k) a[i] = beta;
            }
            sm.tau[k] = tau;
        }
        rp = k + 1;
    }
    sm.perm[lane] = perm_j;
    // ---- A' = R^T: lane c < rp takes row c of R
#pragma unroll
    for (int i = 0; i < 32; ++i) sm.T[lane][i] = (i < rp && i <= lane) ? a[i] : 0.0;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) a[j] = lane < rp ? sm.T[j][lane] : 0.0;
    __syncwarp();
    if (wt) {
        w32_mark(1, *wt);
        if (lane == 0) atomicAdd(&g_w32_cyc[7], (unsigned long long)rp);
    }
    if (rp < 2) return rp;
    // ---- one-sided Jacobi on the rp columns of A'
    const int P = rp + (rp & 1);
    const double tol = (double)(n > 1 ? n : 1) * JEPS;
    const double tol2 = tol * tol;
    double own = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) own = fma(a[i], a[i], own);
    double fro = own;
#pragma unroll
    for (int o = 16; o; o >>= 1) fro += __shfl_xor_sync(FULL, fro, o);
    const double zthr = fro * (16.0 * JEPS * JEPS);
    for (int sweep = 0; sweep < 40; ++sweep) {
        bool any = false;
        // circle-method partner (rr_partner) stepped incrementally: no integer modulo per round
        const int y = lane - 1;
        int yp = y <= 0 ? 0 : (P - 1) - y;
        for (int round = 0; round < P - 1; ++round) {
            const int p = lane >= P ? lane : (lane == 0 ? 1 + round : (yp == y ? 0 : 1 + yp));
            yp += 2;
            if (yp >= P - 1) yp -= P - 1;
            const bool low = lane < p;
            double pa[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) pa[i] = __shfl_sync(FULL, a[i], p);
            // own / partner / cross inner products; both lanes of a pair run the same FMA
            // sequence on the same values, so (alpha, beta, gamma) are bitwise identical
            double so0 = 0, so1 = 0, sp0 = 0, sp1 = 0, sx0 = 0, sx1 = 0;
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                so0 = fma(a[i], a[i], so0);
                so1 = fma(a[i + 1], a[i + 1], so1);
                sp0 = fma(pa[i], pa[i], sp0);
                sp1 = fma(pa[i + 1], pa[i + 1], sp1);
                sx0 = fma(a[i], pa[i], sx0);
                sx1 = fma(a[i + 1], pa[i + 1], sx1);
            }
            const double so = so0 + so1, sp = sp0 + sp1, sx = sx0 + sx1;
            double c, s;
            bool rot = false;
            if (p != lane) rot = jacobi_params(low ? so : sp, low ? sp : so, sx, tol2, zthr, c, s);
            if (!rot) {
                c = 1.0;
                s = 0.0;
            }
            if (__any_sync(FULL, rot)) {
                any = true;
                const double sl = low ? -s : s;
#pragma unroll
                for (int i = 0; i < 32; ++i) a[i] = fma(sl, pa[i], c * a[i]);
            }
        }
        if (wt && lane == 0) atomicAdd(&g_w32_cyc[6], 1ull);
        if (!any) break;
    }
    if (wt) w32_mark(2, *wt);
    return rp;
}

// sigma (lane c < rp), descending position and rank r (warp-uniform).
__device__ __forceinline__ void warp_sigma_pos32(const double (&a)[32], int rp, double eps, double abs_cut, double& sig,
                                                 int& pos, int& r, double& smax) {
    const int lane = threadIdx.x & 31;
    double s = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) s = fma(a[i], a[i], s);
    sig = lane < rp ? sqrt(s) : -1.0;
    pos = 0;
    smax = fmax(sig, 0.0);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const double w = __shfl_sync(0xffffffffu, sig, i);
        pos += (w > sig) || (w == sig && i < lane);
        smax = fmax(smax, w);
    }
    r = 0;
    if (smax > 0.0) {
        const double cut = fmax(eps * smax, abs_cut);
        r = __popc(__ballot_sync(0xffffffffu, lane < rp && sig > cut));
    }
}

// Phase 3: write U' (m x r) = Q [J Sigma; 0] and V' (n x r) = P W Sigma^{-1}.
// J Sigma is recovered as R W Sigma^{-1} (R = J W^T), with R^T still staged in sm.T,
// so the Jacobi sweeps never accumulate J.
__device__ void warp_write32(double (&a)[32], int m, int n, int rp, double sig, int pos, int r, Warp32Smem& sm,
                             double* Uo, double* Vo) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    if (lane < rp && pos < r) {
        const double inv = 1.0 / sig;
        double* w = Vo + (size_t)pos * n;
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < n) w[sm.perm[j]] = a[j] * inv;
        // x = R W_c / sigma in place over a[]: R is upper triangular (R[i][j] = T[j][i] = 0
        // for j < i), so x[i] only needs a[j >= i], which are not yet overwritten
        double (&x)[32] = a;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            double acc = 0.0;
            if (i < rp) {
#pragma unroll
                for (int j = i; j < 32; ++j) acc = fma(sm.T[j][i], a[j], acc);  // R[i][j] = T[j][i]
            }
            x[i] = acc * inv;
        }
#pragma unroll 1
        for (int k = rp - 1; k >= 0; --k) {
            const double tk = sm.tau[k];
            if (tk != 0.0) {
                const double* hk = sm.H[k];  // [0 (i < k); 1; v]
                double s = 0.0;
#pragma unroll
                for (int i = 0; i < 32; ++i) s = fma(hk[i], x[i], s);
                s *= tk;
#pragma unroll
                for (int i = 0; i < 32; ++i) x[i] = fma(-s, hk[i], x[i]);
            }
        }
        double* u = Uo + (size_t)pos * m;
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (i < m) u[i] = x[i];
    }
    __syncwarp();
}

// Dense * dense formation on the FP64 tensor cores: M = Ad (m x k, ld m) * Bd (k x n, ld k),
// m, n, k <= 32, returned column per lane (a[i] = M[i][lane]).  Ad is staged as T[t][i] and Bd
// as H[t][j] (coalesced predicated loads, all in flight), the 4 x 4 tiles of M are accumulated
// in DMMA fragments (mma.sync.m8n8k4.f64, 16 per k-step of 4), and the fragments are turned
// into columns through sm.T.  Returns the zero-operand flags like warp_accumulate32.
__device__ int warp_dd32_mma(double (&a)[32], const double* Ad, const double* Bd, int m, int k, int n, Warp32Smem& sm) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
    bool nzP = false, nzQ = false;
    __syncwarp();
#pragma unroll
    for (int t8 = 0; t8 < 32; t8 += 8) {
        double xv[8], yv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int t = t8 + u;
            xv[u] = (t < k && lane < m) ? Ad[lane + (long)t * m] : 0.0;  // Ad[i = lane][t]
            yv[u] = (t < k && lane < n) ? Bd[t + (long)lane * k] : 0.0;  // Bd[t][j = lane]
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            nzP |= xv[u] != 0.0;
            nzQ |= yv[u] != 0.0;
            sm.T[t8 + u][lane] = xv[u];
            sm.H[t8 + u][lane] = yv[u];
        }
    }
    __syncwarp();
    double c[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) c[i][j][0] = c[i][j][1] = 0.0;
    for (int k0 = 0; k0 < k; k0 += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            af[i] = sm.T[k0 + t4][8 * i + g];  // A[g][t4] of row tile i
            bf[i] = sm.H[k0 + t4][8 * i + g];  // B[t4][g] of column tile i
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma8x8x4(c[i][j][0], c[i][j][1], af[i], bf[j]);
    }
    __syncwarp();
    // C[g][2 t4 + q] of tile (i, j) = M[8 i + g][8 j + 2 t4 + q] -> sm.T[col][row]
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            sm.T[8 * j + 2 * t4][8 * i + g] = c[i][j][0];
            sm.T[8 * j + 2 * t4 + 1][8 * i + g] = c[i][j][1];
        }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] = (i < m && lane < n) ? sm.T[lane][i] : 0.0;
    __syncwarp();
    return (nzP ? 1 : 0) | (nzQ ? 2 : 0);
}

// Truncation-task formation on the FP64 tensor cores: M += alpha P Q^T for one part, staged
// like warp_accumulate32 (T[t][i] = alpha P(i, t), H[t][j] = Q(j, t), zero outside the part's
// rows / columns) and accumulated into the 4 x 4 tiles of DMMA fragments c (kept across the
// parts of a task); warp_frags_to_cols turns them into columns once at the end.
__device__ int warp_accumulate32_mma(double (&c)[4][4][2], const RowPart& p, Warp32Smem& sm) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
    constexpr int TC = 32;
    const int jr = lane - p.qd;
    const bool own = jr >= 0 && jr < p.qr;
    const int ir = lane - p.pd;
    const bool prow = ir >= 0 && ir < p.pr;
    bool nzP = false, nzQ = false;
    for (int t0 = 0; t0 < p.k; t0 += TC) {
        const int tn = min(TC, p.k - t0);
        __syncwarp();
#pragma unroll
        for (int t8 = 0; t8 < TC; t8 += 8) {
            if (t8 < tn) {
                double xv[8], yv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int t = t8 + u;
                    xv[u] = (t < tn && prow) ? p.alpha * p.P[ir * p.ps + (long)(t0 + t) * p.pt] : 0.0;
                    yv[u] = (t < tn && own) ? p.Q[jr * p.qs + (long)(t0 + t) * p.qt] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    nzP |= xv[u] != 0.0;
                    nzQ |= yv[u] != 0.0;
                    sm.T[t8 + u][lane] = xv[u];
                    sm.H[t8 + u][lane] = yv[u];
                }
            }
        }
        __syncwarp();
        for (int k0 = 0; k0 < tn; k0 += 4) {
            const bool kok = k0 + t4 < tn;
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                af[i] = kok ? sm.T[k0 + t4][8 * i + g] : 0.0;
                bf[i] = kok ? sm.H[k0 + t4][8 * i + g] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma8x8x4(c[i][j][0], c[i][j][1], af[i], bf[j]);
        }
    }
    __syncwarp();
    return (nzP ? 1 : 0) | (nzQ ? 2 : 0);
}

__device__ void warp_frags_to_cols(const double (&c)[4][4][2], double (&a)[32], Warp32Smem& sm) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            sm.T[8 * j + 2 * t4][8 * i + g] = c[i][j][0];
            sm.T[8 * j + 2 * t4 + 1][8 * i + g] = c[i][j][1];
        }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] = sm.T[lane][i];
    __syncwarp();
}

}  // namespace acrgpu
