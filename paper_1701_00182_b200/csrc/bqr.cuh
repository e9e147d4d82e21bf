// Blocked Householder QR (compact WY) for the tall factors of the QR-route
// truncation, Uc (m x K) and Vc (n x K) in arena workspace.  (Included inside
// namespace acrgpu by kernels.cu.)
//
// Panels of nb columns are factored in shared memory with the unblocked
// reflector loop (Eigen HouseholderQR conventions, hmatrix.cpp:62-63), the
// triangular factor T of Q_p = I - V T V^T is formed (LAPACK dlarft, forward /
// columnwise), and the trailing columns are updated in ONE pass each,
// A <- A - V (T^T (V^T A)), warp per column with the column streamed from
// global memory.  The same panels applied in reverse give Q [X; 0] for the
// outputs (bqr_apply).  Versus the column-at-a-time loop this reads the
// trailing matrix K/nb times instead of K times.
#pragma once

constexpr int BQR_NB = 16;

// Unblocked Householder on a smem panel P (h x nb, ld h); tau[nb]; returns nothing.
template <int NT>
__device__ void panel_qr(double* P, int h, int nb, double* tau, double* red) {
    constexpr int NW = NT / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ double sh_beta, sh_tau, sh_inv;
    const int kmax = h < nb ? h : nb;
    for (int j = 0; j < kmax; ++j) {
        double* pj = P + (size_t)j * h;
        double part = 0;
        for (int i = j + 1 + threadIdx.x; i < h; i += NT) part = fma(pj[i], pj[i], part);
        part = warp_sum(part);
        __syncthreads();
        if (lane == 0) red[warp] = part;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tail = 0;
            for (int w = 0; w < NW; ++w) tail += red[w];
            const double c0 = pj[j];
            if (tail <= 2.2250738585072014e-308) {
                sh_tau = 0.0;
                sh_beta = c0;
                sh_inv = 0.0;
            } else {
                double beta = sqrt(c0 * c0 + tail);
                if (c0 >= 0) beta = -beta;
                sh_inv = 1.0 / (c0 - beta);
                sh_tau = (beta - c0) / beta;
                sh_beta = beta;
            }
            tau[j] = sh_tau;
        }
        __syncthreads();
        const double tj = sh_tau, inv = sh_inv;
        for (int i = j + 1 + threadIdx.x; i < h; i += NT) pj[i] = tj != 0.0 ? pj[i] * inv : 0.0;
        __syncthreads();
        if (threadIdx.x == 0) pj[j] = sh_beta;
        if (tj != 0.0)
            for (int c = j + 1 + warp; c < nb; c += NW) {
                double* pc = P + (size_t)c * h;
                double s = 0;
                for (int i = j + 1 + lane; i < h; i += 32) s = fma(pj[i], pc[i], s);
                s = (warp_sum(s) + pc[j]) * tj;
                if (lane == 0) pc[j] -= s;
                for (int i = j + 1 + lane; i < h; i += 32) pc[i] = fma(-s, pj[i], pc[i]);
            }
        __syncthreads();
    }
}

// T (nb x nb, ld BQR_NB, upper) of Q = H_0 ... H_{nb-1} = I - V T V^T; V = unit lower
// trapezoidal reflectors stored in P (h x nb).  G = V^T V computed warp per entry.
template <int NT>
__device__ void panel_T(const double* P, int h, int nb, const double* tau, double* T, double* G) {
    constexpr int NW = NT / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = warp; e < nb * nb; e += NW) {
        const int l = e % nb, q = e / nb;  // G[l][q] = v_l . v_q for l < q
        if (l >= q) continue;
        const double* vl = P + (size_t)l * h;
        const double* vq = P + (size_t)q * h;
        // v_l(i) = 0 for i < l, 1 at i = l;  v_q(i) = 0 for i < q, 1 at i = q  (l < q)
        double s = 0;
        for (int i = q + 1 + lane; i < h; i += 32) s = fma(vl[i], vq[i], s);
        s = warp_sum(s);
        if (lane == 0) G[l + q * BQR_NB] = s + vl[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 0; q < nb; ++q) {
            const double tq = tau[q];
            for (int i = 0; i < q; ++i) {
                double s = 0;
                for (int l = i; l < q; ++l) s = fma(T[i + l * BQR_NB], G[l + q * BQR_NB], s);
                T[i + q * BQR_NB] = -tq * s;
            }
            T[q + q * BQR_NB] = tq;
            for (int i = q + 1; i < BQR_NB; ++i) T[i + q * BQR_NB] = 0.0;
        }
    }
    __syncthreads();
}

// y (length h, global) <- (I - V op(T) V^T) y for one column; warp-cooperative.
// trans: op(T) = T^T (apply Q^T), else T (apply Q).  V: explicit unit-lower reflector
// block in shared memory (zeros above the diagonal, ones on it, zero columns past nb).
__device__ __forceinline__ void wy_column(double* y, int h, const double* V, int ldv, int nb, const double* T, bool trans) {
    const int lane = threadIdx.x & 31;
    double w[BQR_NB];
#pragma unroll
    for (int l = 0; l < BQR_NB; ++l) w[l] = 0.0;
#pragma unroll 2
    for (int i = lane; i < h; i += 32) {
        const double yi = y[i];
#pragma unroll
        for (int l = 0; l < BQR_NB; ++l) w[l] = fma(V[i + (size_t)l * ldv], yi, w[l]);
    }
    const double wl = reduce_scatter16(w, lane);  // lane l (and l^16) holds (V^T y)_{l&15}
    double t = 0.0;
    const int me = lane & 15;
#pragma unroll
    for (int k = 0; k < BQR_NB; ++k) {
        const double wk = __shfl_sync(0xffffffffu, wl, k);
        const double Tv = trans ? T[k + me * BQR_NB] : T[me + k * BQR_NB];  // op(T)[me][k]
        if (k < nb && me < nb) t = fma(Tv, wk, t);
    }
    double tt[BQR_NB];
#pragma unroll
    for (int l = 0; l < BQR_NB; ++l) tt[l] = __shfl_sync(0xffffffffu, t, l);
#pragma unroll 2
    for (int i = lane; i < h; i += 32) {
        double yi = y[i];
#pragma unroll
        for (int l = 0; l < BQR_NB; ++l) yi = fma(-V[i + (size_t)l * ldv], tt[l], yi);
        y[i] = yi;
    }
}

// Turn the factored panel P (h x nb: R above the diagonal, reflectors below) into the
// explicit reflector block V (h x BQR_NB, in place; columns >= nb zeroed).
template <int NT>
__device__ void panel_explicit_v(double* P, int h, int nb) {
    __syncthreads();
    for (int e = threadIdx.x; e < h * BQR_NB; e += NT) {
        const int i = e % h, l = e / h;
        if (l >= nb) P[e] = 0.0;
        else if (i < l) P[e] = 0.0;
        else if (i == l) P[e] = 1.0;
    }
    __syncthreads();
}

// Blocked QR of W (rows x cols, ld) in place; tau[cols]; Tall: per-panel T factors
// (ceil(cols/nb) x BQR_NB x BQR_NB); smem: >= rows * BQR_NB + 2 * BQR_NB^2 doubles.
template <int NT>
__device__ void bqr(double* W, int ld, int rows, int cols, double* tau, double* Tall, double* smem, size_t smem_doubles,
                    double* red) {
    constexpr int NW = NT / 32;
    const int warp = threadIdx.x >> 5;
    const int kmax = rows < cols ? rows : cols;
    double* G = smem;
    double* Ts = G + BQR_NB * BQR_NB;
    double* P = Ts + BQR_NB * BQR_NB;
    for (int j0 = 0; j0 < kmax; j0 += BQR_NB) {
        const int h = rows - j0;
        const int nb = kmax - j0 < BQR_NB ? kmax - j0 : BQR_NB;  // caller guarantees rows * BQR_NB <= pcap
        // load panel rows j0.., columns j0..j0+nb
        for (int e = threadIdx.x; e < h * nb; e += NT) {
            const int i = e % h, c = e / h;
            P[e] = W[(j0 + i) + (size_t)(j0 + c) * ld];
        }
        __syncthreads();
        panel_qr<NT>(P, h, nb, tau + j0, red);
        for (int e = threadIdx.x; e < BQR_NB * BQR_NB; e += NT) {
            G[e] = 0.0;
            Ts[e] = 0.0;
        }
        __syncthreads();
        panel_T<NT>(P, h, nb, tau + j0, Ts, G);
        double* Tp = Tall + (size_t)(j0 / BQR_NB) * BQR_NB * BQR_NB;
        for (int e = threadIdx.x; e < BQR_NB * BQR_NB; e += NT) Tp[e] = Ts[e];
        for (int e = threadIdx.x; e < h * nb; e += NT) {
            const int i = e % h, c = e / h;
            W[(j0 + i) + (size_t)(j0 + c) * ld] = P[e];
        }
        panel_explicit_v<NT>(P, h, nb);
        // trailing update: A <- (I - V T^T V^T) A  (Q_p^T applied), warp per column
        for (int c = j0 + nb + warp; c < cols; c += NW)
            wy_column(W + j0 + (size_t)c * ld, h, P, h, nb, Ts, true);
        __syncthreads();
    }
}

// Y (rows x ncol, ld ldy) <- Q Y with Q from bqr (panels applied in reverse order);
// each panel's reflector block is staged in shared memory (smem >= rows * BQR_NB + BQR_NB^2).
template <int NT>
__device__ void bqr_apply(const double* W, int ldw, int rows, int k, const double* Tall, double* Y, int ldy, int ncol,
                          double* smem) {
    constexpr int NW = NT / 32;
    const int warp = threadIdx.x >> 5;
    const int np = (k + BQR_NB - 1) / BQR_NB;
    double* Ts = smem;
    double* P = smem + BQR_NB * BQR_NB;
    for (int p = np - 1; p >= 0; --p) {
        const int j0 = p * BQR_NB;
        const int nb = k - j0 < BQR_NB ? k - j0 : BQR_NB;
        const int h = rows - j0;
        const double* Tp = Tall + (size_t)p * BQR_NB * BQR_NB;
        __syncthreads();
        for (int e = threadIdx.x; e < BQR_NB * BQR_NB; e += NT) Ts[e] = Tp[e];
        for (int e = threadIdx.x; e < h * nb; e += NT) {
            const int i = e % h, c = e / h;
            P[e] = W[(j0 + i) + (size_t)(j0 + c) * ldw];
        }
        panel_explicit_v<NT>(P, h, nb);
        for (int c = warp; c < ncol; c += NW) wy_column(Y + j0 + (size_t)c * ldy, h, P, h, nb, Ts, false);
    }
    __syncthreads();
}
