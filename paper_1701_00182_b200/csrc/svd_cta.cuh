// CTA-wide rank-revealing truncated SVD (blocks up to 64 x 64 in shared memory,
// larger cores of the QR route in global workspace).  Same three stages as the
// warp engine (svd_rrqr32.cuh):
//   1. Householder QR with column pivoting, stopped when every remaining column
//      norm is below delta (1e-3 below the truncation cutoff);
//   2. one-sided Jacobi on A' = R^T (rp columns), warp per column pair,
//      round-robin order, rotation parameters from two reciprocal square roots;
//   3. U' = Q [J Sigma; 0], V' = P W Sigma^{-1}.
// Reference semantics: truncate_impl / dense_to_lowrank, hmatrix.cpp:56-99.
#pragma once
// (included inside namespace acrgpu by kernels.cu, after arena_alloc)

// CTA-engine phase timing (clock64 deltas of thread 0, summed over tasks): diagnostics only.
// [0] tasks [1] rrqr [2] jacobi [3] write [4] sum rp [5] sum cols [6] jacobi sweeps
__device__ unsigned long long g_cta_cyc[8];

struct CtaSvdWork {
    double* A;      // rows x cols (ld = lda): input, then R + reflectors
    int lda;
    double* W;      // cols x rp (ld = ldw): A' = R^T, then W = A' J
    int ldw;
    double* J;      // rp x rp (ld = ldj)
    int ldj;
    double* tau;    // >= min(rows, cols)
    double* nrm;    // >= cols
    double* sig;    // >= cols
    int* perm;      // >= cols
    int* order;     // >= cols
};

// Returns rp.  delta2: squared pivot threshold.  NT threads, NW warps.
// One barrier per pivot step (two when the pivot moves): the update pass that
// applies reflector k also leaves, per column, the norm over rows > k (pivot
// choice) and over rows > k+1 (the next reflector's tail), and each warp's
// best candidate; every thread then picks the pivot and derives the reflector
// scalars itself.  Reflector k is applied unscaled (v = [1; x / (c0 - beta)])
// and stored scaled one step later, when column k is no longer read.
template <int NT>
__device__ int cta_rrqr(const CtaSvdWork& w, int rows, int cols, double delta2) {
    constexpr int NW = NT / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ double sh_wbest[2][NW];  // per-warp pivot candidates, double-buffered by step parity
    __shared__ int sh_wpiv[2][NW];
    double* A = w.A;
    const int lda = w.lda;
    double* tail = w.sig;  // norm over rows > k of each remaining column
    for (int j = threadIdx.x; j < cols; j += NT) w.perm[j] = j;
    const int kmax = rows < cols ? rows : cols;
    {
        double best = -1.0;
        int bi = cols;
        for (int j = warp; j < cols; j += NW) {
            const double* cj = A + (size_t)j * lda;
            double s = 0, tl = 0;
#pragma unroll 4
            for (int i = lane; i < rows; i += 32) {
                s = fma(cj[i], cj[i], s);
                if (i > 0) tl = fma(cj[i], cj[i], tl);
            }
            s = warp_sum(s);
            tl = warp_sum(tl);
            if (lane == 0) {
                w.nrm[j] = s;
                tail[j] = tl;
            }
            if (s > best) {
                best = s;
                bi = j;
            }
        }
        if (lane == 0) {
            sh_wbest[0][warp] = best;
            sh_wpiv[0][warp] = bi;
        }
    }
    __syncthreads();
    int rp = 0;
    double p_inv = 0.0, p_beta = 0.0, p_tau = 0.0;
    for (int k = 0; k < kmax; ++k) {
        double best = -1.0;
        int piv = cols;
        for (int q = 0; q < NW; ++q) {
            const double b = sh_wbest[k & 1][q];
            const int i = sh_wpiv[k & 1][q];
            if (b > best || (b == best && i < piv)) {
                best = b;
                piv = i;
            }
        }
        if (!(best > delta2)) break;
        if (piv != k) {
            double* ck = A + (size_t)k * lda;
            double* cp = A + (size_t)piv * lda;
            for (int i = threadIdx.x; i < rows; i += NT) {
                const double t = ck[i];
                ck[i] = cp[i];
                cp[i] = t;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                const int t = w.perm[k];
                w.perm[k] = w.perm[piv];
                w.perm[piv] = t;
                double tn = w.nrm[k];
                w.nrm[k] = w.nrm[piv];
                w.nrm[piv] = tn;
                tn = tail[k];
                tail[k] = tail[piv];
                tail[piv] = tn;
            }
            __syncthreads();
        }
        double* ck = A + (size_t)k * lda;
        const double c0 = ck[k], t = tail[k];
        double beta, tk, inv;
        if (t > 2.2250738585072014e-308) {
            beta = sqrt(c0 * c0 + t);
            if (c0 >= 0) beta = -beta;
            inv = 1.0 / (c0 - beta);
            tk = (beta - c0) / beta;
        } else {
            inv = 0.0;
            tk = 0.0;
            beta = c0;
        }
        if (threadIdx.x == 0) w.tau[k] = tk;
        if (k > 0) {  // store reflector k-1 (column k-1 is not read in this step)
            double* cq = A + (size_t)(k - 1) * lda;
            for (int i = k + threadIdx.x; i < rows; i += NT) cq[i] = p_tau != 0.0 ? cq[i] * p_inv : 0.0;
            if (threadIdx.x == 0) cq[k - 1] = p_beta;
        }
        // apply reflector k to the remaining columns; refresh norms; warp-local pivot candidates
        double wb = -1.0;
        int wi = cols;
        // RQ columns per warp iteration (j, j + NW, ...): their reductions are independent, so
        // the shuffle trees interleave; per-column arithmetic and pivot order are unchanged
#ifndef ACRGPU_RRQR_Q
#define ACRGPU_RRQR_Q 4
#endif
        constexpr int RQ = ACRGPU_RRQR_Q;
        for (int j = k + 1 + warp; j < cols; j += RQ * NW) {
            double* cq[RQ];
            bool has[RQ];
#pragma unroll
            for (int q = 0; q < RQ; ++q) {
                has[q] = j + q * NW < cols;
                cq[q] = A + (size_t)(has[q] ? j + q * NW : j) * lda;
            }
            double sq[RQ];
#pragma unroll
            for (int q = 0; q < RQ; ++q) sq[q] = 0.0;
            if (tk != 0.0) {
#pragma unroll 2
                for (int i = k + 1 + lane; i < rows; i += 32) {
                    const double v = ck[i];
#pragma unroll
                    for (int q = 0; q < RQ; ++q)
                        if (has[q]) sq[q] = fma(v, cq[q][i], sq[q]);
                }
#pragma unroll
                for (int o = 16; o; o >>= 1)
#pragma unroll
                    for (int q = 0; q < RQ; ++q) sq[q] += __shfl_xor_sync(0xffffffffu, sq[q], o);
#pragma unroll
                for (int q = 0; q < RQ; ++q) sq[q] = has[q] ? fma(sq[q], inv, cq[q][k]) * tk : 0.0;
            }
            double nn[RQ], tl[RQ];
#pragma unroll
            for (int q = 0; q < RQ; ++q) nn[q] = tl[q] = 0.0;
#pragma unroll 2
            for (int i = k + 1 + lane; i < rows; i += 32) {
                const double ci = ck[i];
#pragma unroll
                for (int q = 0; q < RQ; ++q)
                    if (has[q]) {
                        const double v = fma(-(sq[q] * inv), ci, cq[q][i]);
                        cq[q][i] = v;
                        nn[q] = fma(v, v, nn[q]);
                        if (i > k + 1) tl[q] = fma(v, v, tl[q]);
                    }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1)
#pragma unroll
                for (int q = 0; q < RQ; ++q) {
                    nn[q] += __shfl_xor_sync(0xffffffffu, nn[q], o);
                    tl[q] += __shfl_xor_sync(0xffffffffu, tl[q], o);
                }
            if (lane == 0) {
#pragma unroll
                for (int q = 0; q < RQ; ++q)
                    if (has[q]) {
                        cq[q][k] -= sq[q];
                        w.nrm[j + q * NW] = nn[q];
                        tail[j + q * NW] = tl[q];
                    }
            }
#pragma unroll
            for (int q = 0; q < RQ; ++q)
                if (has[q] && nn[q] > wb) {
                    wb = nn[q];
                    wi = j + q * NW;
                }
        }
        p_inv = inv;
        p_beta = beta;
        p_tau = tk;
        if (lane == 0) {
            sh_wbest[(k + 1) & 1][warp] = wb;
            sh_wpiv[(k + 1) & 1][warp] = wi;
        }
        __syncthreads();
        rp = k + 1;
    }
    if (rp > 0) {
        double* cq = A + (size_t)(rp - 1) * lda;
        for (int i = rp + threadIdx.x; i < rows; i += NT) cq[i] = p_tau != 0.0 ? cq[i] * p_inv : 0.0;
        if (threadIdx.x == 0) cq[rp - 1] = p_beta;
    }
    __syncthreads();
    return rp;
}

// One-sided Jacobi on W (rows x cols), warp per pair, J (cols x cols) accumulated
// when non-null.  sig[] receives column norms.
template <int NT>
__device__ void cta_jacobi(double* W, int ldw, int rows, int cols, double* J, int ldj, double* sig) {
    constexpr int NW = NT / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (J)
        for (int e = threadIdx.x; e < cols * cols; e += NT) {
            const int i = e % cols, j = e / cols;
            J[i + (size_t)j * ldj] = (i == j) ? 1.0 : 0.0;
        }
    __shared__ double sh_fro[NW];
    {
        double f = 0;
        for (int j = warp; j < cols; j += NW)
            #pragma unroll 4
            for (int i = lane; i < rows; i += 32) f = fma(W[i + (size_t)j * ldw], W[i + (size_t)j * ldw], f);
        f = warp_sum(f);
        if (lane == 0) sh_fro[warp] = f;
    }
    __syncthreads();
    double fro = 0;
    for (int i = 0; i < NW; ++i) fro += sh_fro[i];
    const double zthr = fro * (16.0 * JEPS * JEPS);
    const double tol = (double)(rows > 1 ? rows : 1) * JEPS;
    const double tol2 = tol * tol;
    if (cols > 1) {
        const int P = cols + (cols & 1);
        for (int sweep = 0; sweep < 40; ++sweep) {
            int rotated = 0;
            for (int r = 0; r < P - 1; ++r) {
                for (int pi = warp; pi < P / 2; pi += NW) {
                    int p, q;
                    if (pi == 0) {
                        p = 0;
                        q = 1 + r;
                    } else {
                        int a = r + pi, b = r - pi;
                        a %= (P - 1);
                        b %= (P - 1);
                        if (b < 0) b += P - 1;
                        p = 1 + a;
                        q = 1 + b;
                    }
                    if (p > q) { const int t = p; p = q; q = t; }
                    if (q >= cols) continue;
                    double* ap = W + (size_t)p * ldw;
                    double* aq = W + (size_t)q * ldw;
                    double al = 0, be = 0, ga = 0;
                    #pragma unroll 4
                    for (int e = lane; e < rows; e += 32) {
                        const double x = ap[e], y = aq[e];
                        al = fma(x, x, al);
                        be = fma(y, y, be);
                        ga = fma(x, y, ga);
                    }
                    al = warp_sum(al);
                    be = warp_sum(be);
                    ga = warp_sum(ga);
                    double c, s;
                    if (!jacobi_params(al, be, ga, tol2, zthr, c, s)) continue;
                    #pragma unroll 4
                    for (int e = lane; e < rows; e += 32) rot2(ap[e], aq[e], c, s);
                    if (J) {
                        double* vp = J + (size_t)p * ldj;
                        double* vq = J + (size_t)q * ldj;
                        for (int e = lane; e < cols; e += 32) rot2(vp[e], vq[e], c, s);
                    }
                    rotated = 1;
                }
                __syncthreads();
            }
            if (threadIdx.x == 0) atomicAdd(&g_cta_cyc[6], 1ull);
            if (!__syncthreads_or(rotated)) break;
        }
    }
    for (int j = warp; j < cols; j += NW) {
        double s = 0;
        #pragma unroll 4
        for (int e = lane; e < rows; e += 32) s = fma(W[e + (size_t)j * ldw], W[e + (size_t)j * ldw], s);
        s = warp_sum(s);
        if (lane == 0) sig[j] = sqrt(s);
    }
    __syncthreads();
}

// Full engine on w.A (rows x cols).  Returns the truncated rank r (CTA-uniform);
// order[t] = Jacobi column of the t-th largest sigma; *smax_out = sigma_1.
// rp_cap: columns the caller's W/J buffers can hold; a larger numerical rank moves
// W and J to `spill` (device arena) -- CTA-uniform decision.
template <int NT>
__device__ int cta_trunc_svd(CtaSvdWork& w, int rows, int cols, double eps, double abs_cut, bool values_only,
                             int* rp_out, double* smax_out, int rp_cap, const Arena* spill, double* w_alt = nullptr,
                             size_t w_alt_cap = 0) {
    __shared__ int sh_r;
    __shared__ double sh_smax;
    __shared__ double* sh_spill;
    // pivot threshold from the largest column norm (a lower bound of sigma_1)
    double cm = 0;
    {
        __shared__ double redm[NT / 32];
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int j = warp; j < cols; j += NT / 32) {
            double s = 0;
            #pragma unroll 4
            for (int i = lane; i < rows; i += 32) s = fma(w.A[i + (size_t)j * w.lda], w.A[i + (size_t)j * w.lda], s);
            cm = fmax(cm, warp_sum(s));
        }
        if (lane == 0) redm[warp] = cm;
        __syncthreads();
        cm = 0;
        for (int i = 0; i < NT / 32; ++i) cm = fmax(cm, redm[i]);
        __syncthreads();
    }
    const double drel = values_only ? 1e-10 : 1.8e-4 * eps;
    const double dabs = values_only ? 0.0 : 1.8e-4 * abs_cut;
    const double d1 = drel * sqrt(cm);
    const double delta2 = fmax(d1 * d1, dabs * dabs);
    unsigned long long ct0 = clock64();
    const int rp = cta_rrqr<NT>(w, rows, cols, delta2);
    *rp_out = rp;
    if (threadIdx.x == 0) {
        const unsigned long long t = clock64();
        atomicAdd(&g_cta_cyc[0], 1ull);
        atomicAdd(&g_cta_cyc[1], t - ct0);
        atomicAdd(&g_cta_cyc[4], (unsigned long long)rp);
        atomicAdd(&g_cta_cyc[5], (unsigned long long)cols);
        ct0 = t;
    }
    if (rp == 0) {
        *smax_out = 0.0;
        return 0;
    }
    if (rp > rp_cap) {
        if (threadIdx.x == 0)
            sh_spill = spill ? arena_alloc(*spill, (unsigned long long)cols * rp + (unsigned long long)rp * rp + 16) : nullptr;
        __syncthreads();
        if (sh_spill == nullptr) {  // no room: report rank 0 (arena overflow flag raised)
            *smax_out = 0.0;
            return 0;
        }
        w.W = sh_spill;
        w.ldw = cols;
        w.J = sh_spill + (size_t)cols * rp;
        w.ldj = rp;
    }
    // a faster home for W offered by the caller (shared memory while the core is in global)
    if (w_alt != nullptr && rp <= rp_cap && (size_t)cols * rp <= w_alt_cap) {
        w.W = w_alt;
        w.ldw = cols;
    }
    // A' = R^T (cols x rp)
    for (int e = threadIdx.x; e < cols * rp; e += NT) {
        const int j = e % cols, c = e / cols;
        w.W[j + (size_t)c * w.ldw] = j >= c ? w.A[c + (size_t)j * w.lda] : 0.0;
    }
    __syncthreads();
    cta_jacobi<NT>(w.W, w.ldw, cols, rp, nullptr, w.ldj, w.sig);  // J recovered as R W Sigma^{-2} at write time
    for (int j = threadIdx.x; j < rp; j += NT) {
        const double v = w.sig[j];
        int pos = 0;
        for (int i = 0; i < rp; ++i) {
            const double u = w.sig[i];
            pos += (u > v) || (u == v && i < j);
        }
        w.order[pos] = j;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double s0 = w.sig[w.order[0]];
        int r = 0;
        if (s0 > 0.0) {
            const double cut = fmax((values_only ? 0.0 : eps) * s0, abs_cut);
            while (r < rp && w.sig[w.order[r]] > cut) ++r;
        }
        sh_r = r;
        sh_smax = s0;
        atomicAdd(&g_cta_cyc[2], clock64() - ct0);
    }
    __syncthreads();
    *smax_out = sh_smax;
    return sh_r;
}

// U' (rows x r, ld ldu) = Q [J Sigma; 0];  V' (cols x r, ld ldv) = P W Sigma^{-1}.
template <int NT>
__device__ void cta_trunc_write(const CtaSvdWork& w, int rows, int cols, int rp, int r, double* Uo, int ldu, double* Vo,
                                int ldv) {
    constexpr int NW = NT / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned long long wt0 = clock64();
    // J_r Sigma_r = R W_r Sigma_r^{-1}  (R = J W^T: the rp x cols upper rows of the pivoted QR)
    for (int e = threadIdx.x; e < rows * r; e += NT) {
        const int i = e % rows, t = e / rows;
        const int c = w.order[t];
        double acc = 0.0;
        if (i < rp)
            for (int j = i; j < cols; ++j) acc = fma(w.A[i + (size_t)j * w.lda], w.W[j + (size_t)c * w.ldw], acc);
        Uo[i + (size_t)t * ldu] = acc / w.sig[c];
    }
    for (int e = threadIdx.x; e < cols * r; e += NT) {
        const int j = e % cols, t = e / cols;
        const int c = w.order[t];
        Vo[w.perm[j] + (size_t)t * ldv] = w.W[j + (size_t)c * w.ldw] / w.sig[c];
    }
    __syncthreads();
    // apply the reflectors of the pivoted QR in reverse order, warp per column
    for (int t = warp; t < r; t += NW) {
        double* x = Uo + (size_t)t * ldu;
        for (int k = rp - 1; k >= 0; --k) {
            const double tk = w.tau[k];
            if (tk == 0.0) continue;
            const double* v = w.A + (size_t)k * w.lda;
            double s = 0;
            #pragma unroll 4
            for (int i = k + 1 + lane; i < rows; i += 32) s = fma(v[i], x[i], s);
            s = (warp_sum(s) + x[k]) * tk;
            __syncwarp();
            if (lane == 0) x[k] -= s;
            #pragma unroll 4
            for (int i = k + 1 + lane; i < rows; i += 32) x[i] = fma(-s, v[i], x[i]);
            __syncwarp();
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(&g_cta_cyc[3], clock64() - wt0);
}


