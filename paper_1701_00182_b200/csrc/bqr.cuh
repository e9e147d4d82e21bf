// Blocked Householder QR (compact WY) for the tall factors of the QR-route
// truncation, Uc (m x K) and Vc (n x K) in arena workspace.  (Included inside
// namespace acrgpu by kernels.cu.)
//
// Panels of nb = 16 columns are factored in shared memory with the unblocked
// reflector loop (Eigen HouseholderQR conventions, hmatrix.cpp:62-63), the
// triangular factor T of Q_p = I - V T V^T is formed (LAPACK dlarft, forward /
// columnwise), and the trailing columns are updated as two FP64 tensor-core
// products, W = V^T A and A -= V (T^T W) (mma.sync m8n8k4 f64, DMMA), with V
// and W staged in shared memory and A streamed from L2 with register
// prefetch.  The same panels applied in reverse give Q [X; 0] for the outputs
// (bqr_apply).
//
// DMMA m8n8k4 fragment layout (checked by tools/dmma_layout.cu): lane = 4 g + t;
// A (8x4): A[g][t];  B (4x8): B[t][g];  C/D (8x8): C[g][2t], C[g][2t+1].
#pragma once

constexpr int BQR_NB = 16;
constexpr int BQR_LDW = 20;  // W (16 x ncol) leading dimension: == 4 mod 16 -> conflict-free fragments
constexpr int BQR_SCRATCH = 2 * 32 * 16 + 32;  // panel_qr_reg reduction scratch (<= 32 warps, double-buffered)

// smem leading dimension of an h-row panel: == 4 (mod 16) doubles, so the DMMA
// fragment loads (8 rows x 4 columns or 4 rows x 8 columns) hit 16 distinct banks.
__host__ __device__ __forceinline__ int bqr_ldp(int h) { return h + ((20 - (h & 15)) & 15); }

// Minimum shared-memory doubles bqr / bqr_apply need for `rows` rows and `cols` columns.
__host__ __device__ inline size_t bqr_smem_doubles(int rows, int cols) {
    return BQR_SCRATCH + (size_t)bqr_ldp(rows) * BQR_NB + 2 * BQR_NB * BQR_NB + (size_t)BQR_LDW * (((cols + 7) / 8) * 8) + 64;
}


// Unblocked Householder on a smem panel P (h x nb, ld ldp); tau[nb].  One barrier per
// column: every thread derives (beta, tau, 1/(c0-beta)) from the column's tail norm,
// which the warp that updated that column in the previous step left in sh_tail; the
// reflector is applied unscaled (v = [1; x * inv]) and column j is scaled one step later.
template <int NT>
__device__ void panel_qr(double* P, int h, int ldp, int nb, double* tau) {
    constexpr int NW = NT / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ double sh_tail[BQR_NB];
    const int kmax = h < nb ? h : nb;
    if (warp == 0) {
        double s = 0;
        for (int i = 1 + lane; i < h; i += 32) s = fma(P[i], P[i], s);
        s = warp_sum(s);
        if (lane == 0) sh_tail[0] = s;
    }
    __syncthreads();
    double p_inv = 0, p_beta = 0, p_tau = 0;
    for (int j = 0; j < kmax; ++j) {
        const double* pj = P + (size_t)j * ldp;
        const double tail = sh_tail[j], c0 = pj[j];
        double beta, tj, inv;
        if (tail <= 2.2250738585072014e-308) {
            tj = 0.0;
            beta = c0;
            inv = 0.0;
        } else {
            beta = sqrt(c0 * c0 + tail);
            if (c0 >= 0) beta = -beta;
            inv = 1.0 / (c0 - beta);
            tj = (beta - c0) / beta;
        }
        if (threadIdx.x == 0) tau[j] = tj;
        if (j > 0) {  // finish column j-1 (no longer read)
            double* pp = P + (size_t)(j - 1) * ldp;
            for (int i = j + threadIdx.x; i < h; i += NT) pp[i] = p_tau != 0.0 ? pp[i] * p_inv : 0.0;
            if (threadIdx.x == 0) pp[j - 1] = p_beta;
        }
        for (int c = j + 1 + warp; c < nb; c += NW) {
            double* pc = P + (size_t)c * ldp;
            const bool next = c == j + 1;
            double tl = 0;
            if (tj != 0.0) {
                double s = 0;
                for (int i = j + 1 + lane; i < h; i += 32) s = fma(pj[i], pc[i], s);
                s = (fma(warp_sum(s), inv, pc[j])) * tj;
                if (lane == 0) pc[j] -= s;
                const double si = s * inv;
                for (int i = j + 1 + lane; i < h; i += 32) {
                    const double x = fma(-si, pj[i], pc[i]);
                    pc[i] = x;
                    if (i > j + 1) tl = fma(x, x, tl);
                }
            } else if (next) {
                for (int i = j + 2 + lane; i < h; i += 32) tl = fma(pc[i], pc[i], tl);
            }
            if (next) {
                tl = warp_sum(tl);
                if (lane == 0) sh_tail[j + 1] = tl;
            }
        }
        p_inv = inv;
        p_beta = beta;
        p_tau = tj;
        __syncthreads();
    }
    if (kmax > 0) {
        double* pp = P + (size_t)(kmax - 1) * ldp;
        for (int i = kmax + threadIdx.x; i < h; i += NT) pp[i] = p_tau != 0.0 ? pp[i] * p_inv : 0.0;
        if (threadIdx.x == 0) pp[kmax - 1] = p_beta;
    }
    __syncthreads();
}

// Register-resident panel factorization: thread i owns panel rows i, i + NT, ...
// (RPT rows, all 16 columns in registers).  Per column one CTA-wide reduction of
// 16 sums (tail norm + the 15 dot products with the remaining columns, warp
// reduce-scatter then a 16-thread combine), after which every thread derives the
// reflector scalars itself and updates its rows.  The panel is read from and
// written back to W (global, rows j0.., columns j0..j0+nb), and the explicit
// reflector block V (h x 16, zero columns past nb) is left in smem P (ld ldp).
// scratch: >= 2 * NW * 16 + 32 doubles of shared memory.
template <int NT, int RPT>
__device__ void panel_qr_reg(double* Wp, int ld, int h, int nb, double* tau, double* P, int ldp, double* scratch) {
    constexpr int NW = NT / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* red = scratch;            // 2 x NW x 16 warp partials (double-buffered by column parity)
    double* rowj = red + 2 * NW * 16;  // 2 x 16: row j of the panel (double-buffered)
    double x[RPT][BQR_NB];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int i = threadIdx.x + r * NT;
#pragma unroll
        for (int c = 0; c < BQR_NB; ++c) x[r][c] = (i < h && c < nb) ? Wp[i + (size_t)c * ld] : 0.0;
    }
    const int kmax = h < nb ? h : nb;
#pragma unroll
    for (int j = 0; j < BQR_NB; ++j) {
        if (j < kmax) {
        double v[BQR_NB];
#pragma unroll
        for (int c = 0; c < BQR_NB; ++c) v[c] = 0.0;
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const int i = threadIdx.x + r * NT;
            if (i > j && i < h) {
                const double xj = x[r][j];
                v[j] = fma(xj, xj, v[j]);
#pragma unroll
                for (int c = j + 1; c < BQR_NB; ++c) v[c] = fma(xj, x[r][c], v[c]);
            }
            if (i == j) {
#pragma unroll
                for (int c = j; c < BQR_NB; ++c) rowj[(j & 1) * 16 + c] = x[r][c];
            }
        }
        const double part = reduce_scatter16(v, lane);
        double* rb = red + (j & 1) * NW * 16;
        if (lane < 16) rb[warp * 16 + lane] = part;
        __syncthreads();
        // every warp forms the 16 column totals itself (lane l < 16 sums slot l over the warps,
        // in warp order) and shares them by shuffles: one barrier per column instead of two
        double tot = 0;
        if (lane < 16)
            for (int w = 0; w < NW; ++w) tot += rb[w * 16 + lane];
        double fin[BQR_NB];
#pragma unroll
        for (int c = 0; c < BQR_NB; ++c) fin[c] = __shfl_sync(0xffffffffu, tot, c);
        const double* rj = rowj + (j & 1) * 16;
        const double tail = fin[j], c0 = rj[j];
        double beta, tj, inv;
        if (tail <= 2.2250738585072014e-308) {
            tj = 0.0;
            beta = c0;
            inv = 0.0;
        } else {
            beta = sqrt(c0 * c0 + tail);
            if (c0 >= 0) beta = -beta;
            inv = 1.0 / (c0 - beta);
            tj = (beta - c0) / beta;
        }
        if (threadIdx.x == 0) tau[j] = tj;
        double sc[BQR_NB];
#pragma unroll
        for (int c = j + 1; c < BQR_NB; ++c) sc[c] = fma(fin[c], inv, rj[c]) * tj;  // (v_j . a_c) tau_j
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const int i = threadIdx.x + r * NT;
            if (i > j) {
                const double vj = x[r][j] * inv;
#pragma unroll
                for (int c = j + 1; c < BQR_NB; ++c) x[r][c] = fma(-sc[c], vj, x[r][c]);
                x[r][j] = tj != 0.0 ? vj : 0.0;
            } else if (i == j) {
#pragma unroll
                for (int c = j + 1; c < BQR_NB; ++c) x[r][c] -= sc[c];
                x[r][j] = beta;
            }
        }
        }
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int i = threadIdx.x + r * NT;
        if (i < h) {
#pragma unroll
            for (int c = 0; c < BQR_NB; ++c) {
                if (c < nb) Wp[i + (size_t)c * ld] = x[r][c];
                P[i + (size_t)c * ldp] = c < nb ? (i > c ? x[r][c] : (i == c ? 1.0 : 0.0)) : 0.0;
            }
        }
    }
    __syncthreads();
}

// Turn the factored panel P (h x nb, ld ldp: R above the diagonal, reflectors below)
// into the explicit reflector block V (h x BQR_NB, in place; columns >= nb zeroed).
template <int NT>
__device__ void panel_explicit_v(double* P, int h, int ldp, int nb) {
    __syncthreads();
    for (int e = threadIdx.x; e < h * BQR_NB; e += NT) {
        const int i = e % h, l = e / h;
        double& x = P[i + (size_t)l * ldp];
        if (l >= nb) x = 0.0;
        else if (i < l) x = 0.0;
        else if (i == l) x = 1.0;
    }
    __syncthreads();
}

// T (16 x 16, ld BQR_NB, upper; zero past nb) of Q = H_0 ... H_{nb-1} = I - V T V^T from the
// explicit V (h x 16, ld ldp).  G = V^T V by DMMA (three 8x8 tiles, one warp each), then the
// dlarft recurrence T[i][q] = -tau_q sum_{i<=l<q} T[i][l] G[l][q]: row i depends only on
// row i, so lane i of warp 0 runs it from registers with no synchronisation.
template <int NT>
__device__ void panel_T(const double* V, int h, int ldp, int nb, const double* tau, double* T, double* G) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    if (warp < 3) {
        const int mt = warp == 2 ? 1 : 0, nt = warp == 0 ? 0 : 1;  // tiles (0,0), (0,1), (1,1)
        double a0 = 0, a1 = 0, b0 = 0, b1 = 0;
        int k0 = 0;
        for (; k0 + 8 <= h; k0 += 8) {
            const int ra = k0 + t, rb = k0 + 4 + t;
            dmma8x8x4(a0, a1, V[ra + (size_t)(g + 8 * mt) * ldp], V[ra + (size_t)(g + 8 * nt) * ldp]);
            dmma8x8x4(b0, b1, V[rb + (size_t)(g + 8 * mt) * ldp], V[rb + (size_t)(g + 8 * nt) * ldp]);
        }
        for (; k0 < h; k0 += 4) {
            const int ra = k0 + t;
            const bool ok = ra < h;
            dmma8x8x4(a0, a1, ok ? V[ra + (size_t)(g + 8 * mt) * ldp] : 0.0, ok ? V[ra + (size_t)(g + 8 * nt) * ldp] : 0.0);
        }
        const int l = 8 * mt + g, q = 8 * nt + 2 * t;
        G[l + q * BQR_NB] = a0 + b0;
        G[l + (q + 1) * BQR_NB] = a1 + b1;
    }
    __syncthreads();
    if (warp == 0 && lane < BQR_NB) {
        const int i = lane;
        double tr[BQR_NB];
#pragma unroll
        for (int q = 0; q < BQR_NB; ++q) {
            double s = 0;
#pragma unroll
            for (int l = 0; l < q; ++l)
                if (l >= i) s = fma(tr[l], G[l + q * BQR_NB], s);
            const double tq = q < nb ? tau[q] : 0.0;
            tr[q] = i < q ? -tq * s : (i == q ? tq : 0.0);
        }
#pragma unroll
        for (int q = 0; q < BQR_NB; ++q) T[i + q * BQR_NB] = tr[q];
    }
    __syncthreads();
}

// A (h x nc, global, ld lda) <- (I - V op(T) V^T) A with V (h x 16, smem, ld ldv, explicit,
// zero columns past nb) and T (16 x 16, smem).  trans: op(T) = T^T (apply Q^T).
// Ws: smem scratch of ws_cap >= BQR_LDW * ceil8(nc) doubles; Tpad: 16 x 17 smem scratch.
// All NT threads participate.
template <int NT>
__device__ void wy_update(double* A, int lda, int h, int nc, const double* V, int ldv, const double* T, bool trans,
                          double* Ws, int ws_cap, double* Tpad) {
    constexpr int NW = NT / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int nct = (nc + 7) >> 3;
    const int slice = BQR_LDW * nct * 8;
    // split the h-reduction of step 1 over idle warps (partials in separate W slices)
    int nsp = NW / nct;
    nsp = nsp < 1 ? 1 : (nsp > 4 ? 4 : nsp);
    while (nsp > 1 && nsp * slice > ws_cap) --nsp;
    const int kchunk = (((h + nsp - 1) / nsp) + 31) & ~31;
    // 1. W = V^T A  (16 x nc): unit = (8-column tile, row chunk); two 8-row halves
    for (int u = warp; u < nct * nsp; u += NW) {
        const int ct = u % nct, sp = u / nct;
        const int c = ct * 8 + g;
        const bool cok = c < nc;
        const double* a = A + (size_t)(cok ? c : 0) * lda;
        double p0 = 0, p1 = 0, q0 = 0, q1 = 0, r0 = 0, r1 = 0, s0 = 0, s1 = 0;
        const int kb = sp * kchunk, ke = min(h, kb + kchunk);
        for (int k0 = kb; k0 < ke; k0 += 32) {
            double bv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int row = k0 + 4 * q + t;
                bv[q] = (row < ke && cok) ? a[row] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int row = k0 + 4 * q + t;
                const bool ok = row < ke;
                const double v0 = ok ? V[row + (size_t)g * ldv] : 0.0;
                const double v1 = ok ? V[row + (size_t)(g + 8) * ldv] : 0.0;
                if (q & 1) {
                    dmma8x8x4(r0, r1, v0, bv[q]);
                    dmma8x8x4(s0, s1, v1, bv[q]);
                } else {
                    dmma8x8x4(p0, p1, v0, bv[q]);
                    dmma8x8x4(q0, q1, v1, bv[q]);
                }
            }
        }
        // C fragment: row g (reflector index), columns 2t, 2t+1 of the tile
        double* w = Ws + (size_t)sp * slice + (size_t)(ct * 8 + 2 * t) * BQR_LDW;
        w[g] = p0 + r0;
        w[g + 8] = q0 + s0;
        w[BQR_LDW + g] = p1 + r1;
        w[BQR_LDW + g + 8] = q1 + s1;
    }
    __syncthreads();
    // 2. W <- -op(T) (sum of slices): thread per (column, output row), in place by
    // column-disjoint chunks; T staged with ld 17 (conflict-free for both transposes)
    for (int e = threadIdx.x; e < BQR_NB * BQR_NB; e += NT) Tpad[(e % BQR_NB) + (e / BQR_NB) * (BQR_NB + 1)] = T[e];
    // fold the row-slice partial sums into slice 0 first (same summation order as summing
    // them inside the product below; keeps the unrolled product free of a runtime loop,
    // which the compiler had expanded to ~40k instructions)
    if (nsp > 1) {
        for (int e = threadIdx.x; e < nct * 8 * BQR_NB; e += NT) {
            const int k = e % BQR_NB, c = e / BQR_NB;
            double wk = Ws[k + (size_t)c * BQR_LDW];
#pragma unroll 1
            for (int sp = 1; sp < nsp; ++sp) wk += Ws[(size_t)sp * slice + k + (size_t)c * BQR_LDW];
            Ws[k + (size_t)c * BQR_LDW] = wk;
        }
    }
    __syncthreads();
    {
        const int tot = nct * 8 * BQR_NB;
        for (int base = 0; base < tot; base += 4 * NT) {
            double y[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = base + threadIdx.x + q * NT;
                y[q] = 0.0;
                if (e < tot) {
                    const int i = e % BQR_NB, c = e / BQR_NB;
                    double s = 0;
#pragma unroll
                    for (int k = 0; k < BQR_NB; ++k) {
                        const double wk = Ws[k + (size_t)c * BQR_LDW];
                        s = fma(trans ? Tpad[k + i * (BQR_NB + 1)] : Tpad[i + k * (BQR_NB + 1)], wk, s);
                    }
                    y[q] = -s;
                }
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = base + threadIdx.x + q * NT;
                if (e < tot) Ws[(e % BQR_NB) + (size_t)(e / BQR_NB) * BQR_LDW] = y[q];
            }
        }
    }
    __syncthreads();
    // 3. A += V W: units of (8-column tile, 64-row chunk); W fragments stay in registers,
    // the chunk's 8 C fragments are loaded before the 32 DMMAs
    const int nrc = (h + 63) >> 6;
    for (int u = warp; u < nct * nrc; u += NW) {
        const int ct = u % nct, rc = u / nct;
        double wb[4];
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) wb[ks] = Ws[(ks * 4 + t) + (size_t)(ct * 8 + g) * BQR_LDW];
        const int c0 = ct * 8 + 2 * t;
        const bool ok0 = c0 < nc, ok1 = c0 + 1 < nc;
        double* a0 = A + (size_t)(ok0 ? c0 : 0) * lda;
        double* a1 = A + (size_t)(ok1 ? c0 + 1 : 0) * lda;
        const int rb = rc * 64;
        double d[8][2];
#pragma unroll
        for (int rt = 0; rt < 8; ++rt) {
            const int row = rb + rt * 8 + g;
            const bool rok = row < h;
            d[rt][0] = (rok && ok0) ? a0[row] : 0.0;
            d[rt][1] = (rok && ok1) ? a1[row] : 0.0;
        }
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
#pragma unroll
            for (int rt = 0; rt < 8; ++rt) {
                const int row = rb + rt * 8 + g;
                dmma8x8x4(d[rt][0], d[rt][1], row < h ? V[row + (size_t)(ks * 4 + t) * ldv] : 0.0, wb[ks]);
            }
#pragma unroll
        for (int rt = 0; rt < 8; ++rt) {
            const int row = rb + rt * 8 + g;
            if (row < h) {
                if (ok0) a0[row] = d[rt][0];
                if (ok1) a1[row] = d[rt][1];
            }
        }
    }
    __syncthreads();
}

// Blocked QR of W (rows x cols, ld) in place; tau[cols]; Tall: per-panel T factors
// (ceil(cols/nb) x BQR_NB x BQR_NB); smem of smem_doubles >= bqr_smem_doubles(rows, cols).
template <int NT>
__device__ void bqr(double* W, int ld, int rows, int cols, double* tau, double* Tall, double* smem, size_t smem_doubles) {
    const int kmax = rows < cols ? rows : cols;
    double* G = smem;
    double* Ts = G + BQR_NB * BQR_NB;
    double* scratch = Ts + BQR_NB * BQR_NB;
    double* P = scratch + BQR_SCRATCH;
    double* Ws = P + (size_t)bqr_ldp(rows) * BQR_NB;
    const int ws_cap = (int)(smem_doubles - (size_t)(Ws - smem));
    for (int j0 = 0; j0 < kmax; j0 += BQR_NB) {
        const int h = rows - j0;
        const int ldp = bqr_ldp(h);
        const int nb = kmax - j0 < BQR_NB ? kmax - j0 : BQR_NB;
        unsigned long long ph_t0 = clock64();
        if (h <= NT) {
            panel_qr_reg<NT, 1>(W + j0 + (size_t)j0 * ld, ld, h, nb, tau + j0, P, ldp, scratch);

        } else {
            for (int e = threadIdx.x; e < h * nb; e += NT) {
                const int i = e % h, c = e / h;
                P[i + (size_t)c * ldp] = W[(j0 + i) + (size_t)(j0 + c) * ld];
            }
            __syncthreads();
            panel_qr<NT>(P, h, ldp, nb, tau + j0);
            for (int e = threadIdx.x; e < h * nb; e += NT) {
                const int i = e % h, c = e / h;
                W[(j0 + i) + (size_t)(j0 + c) * ld] = P[i + (size_t)c * ldp];
            }
            panel_explicit_v<NT>(P, h, ldp, nb);
        }
        PHASE_MARK(10);
        panel_T<NT>(P, h, ldp, nb, tau + j0, Ts, G);
        PHASE_MARK(11);
        double* Tp = Tall + (size_t)(j0 / BQR_NB) * BQR_NB * BQR_NB;
        for (int e = threadIdx.x; e < BQR_NB * BQR_NB; e += NT) Tp[e] = Ts[e];
        const int nc = cols - j0 - nb;
        if (nc > 0) wy_update<NT>(W + j0 + (size_t)(j0 + nb) * ld, ld, h, nc, P, ldp, Ts, true, Ws, ws_cap, scratch);
        __syncthreads();
        PHASE_MARK(12);
    }
}

// Y (rows x ncol, ld ldy) <- Q Y with Q from bqr (panels applied in reverse order);
// smem of smem_doubles >= bqr_smem_doubles(rows, ncol).
template <int NT>
__device__ void bqr_apply(const double* W, int ldw, int rows, int k, const double* Tall, double* Y, int ldy, int ncol,
                          double* smem, size_t smem_doubles) {
    const int np = (k + BQR_NB - 1) / BQR_NB;
    double* Ts = smem + BQR_NB * BQR_NB;
    double* scratch = Ts + BQR_NB * BQR_NB;
    double* P = scratch + BQR_SCRATCH;
    double* Ws = P + (size_t)bqr_ldp(rows) * BQR_NB;
    const int ws_cap = (int)(smem_doubles - (size_t)(Ws - smem));
    for (int p = np - 1; p >= 0; --p) {
        const int j0 = p * BQR_NB;
        const int nb = k - j0 < BQR_NB ? k - j0 : BQR_NB;
        const int h = rows - j0;
        const int ldp = bqr_ldp(h);
        const double* Tp = Tall + (size_t)p * BQR_NB * BQR_NB;
        __syncthreads();
        for (int e = threadIdx.x; e < BQR_NB * BQR_NB; e += NT) Ts[e] = Tp[e];
        for (int e = threadIdx.x; e < h * nb; e += NT) {
            const int i = e % h, c = e / h;
            P[i + (size_t)c * ldp] = W[(j0 + i) + (size_t)(j0 + c) * ldw];
        }
        panel_explicit_v<NT>(P, h, ldp, nb);
        wy_update<NT>(Y + j0, ldy, h, ncol, P, ldp, Ts, false, Ws, ws_cap, scratch);
    }
    __syncthreads();
}
