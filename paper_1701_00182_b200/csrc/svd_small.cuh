// Shared warp-level helpers of the FP64 truncation engines (svd_rrqr32.cuh,
// svd_cta.cuh, bqr.cuh): warp reductions, the Jacobi rotation parameters and the
// "row-producer" description of one product part.
// Rotation parameters use two reciprocal square roots (no divisions):
//   d = beta - alpha, g = 2 gamma, w = 1/sqrt(d^2 + g^2), q = (1 + |d| w)/2,
//   c = sqrt(q), s = sign(d) g w / (2 sqrt(q))      (|theta| <= pi/4).
// Same algorithm class as the reference's JacobiSVD (hmatrix.cpp:67,89): rank
// decisions use the reference rule sigma_i > max(eps * sigma_1, abs_cut)
// (hmatrix.cpp:70-74).
#pragma once

namespace acrgpu {

constexpr double JEPS = 2.2204460492503131e-16;

// FP64 tensor-core step D += A B, mma.sync.aligned.m8n8k4 (DMMA; tcgen05 has no f64 kind).
// Fragment layout (checked by tools/dmma_layout.cu): lane = 4 g + t;  A (8x4): A[g][t];
// B (4x8): B[t][g];  C/D (8x8): lane holds C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

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

}  // namespace acrgpu
