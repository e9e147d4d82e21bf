// Vector kernels of the GPU Krylov drivers (engine.cu: acrgpu_pcg / acrgpu_refine):
// the block-tridiagonal operator as one CSR SpMV, deterministic dot products and the
// PCG / refinement vector updates.  Reference: core/src/krylov.cpp:38-133 (pcg,
// iterative_refinement), core/src/block.cpp:89-107 (apply).
//
// All of it is HBM-bound streaming (7-point operators: ~7 nonzeros per row); a dot
// product is a fixed-shape two-stage tree (KRY_G partial sums of a grid-stride loop,
// then one CTA), so every reduction is bitwise reproducible run to run.
#include <cuda_runtime.h>

#include "kernels.hpp"

namespace acrgpu {

constexpr int KRY_NT = 256;

__global__ void __launch_bounds__(KRY_NT) k_csr_spmv(const long* __restrict__ ptr, const int* __restrict__ col,
                                                     const double* __restrict__ val, const double* __restrict__ x,
                                                     const double* __restrict__ b, double* __restrict__ y, long nrows) {
    for (long i = blockIdx.x * (long)KRY_NT + threadIdx.x; i < nrows; i += (long)gridDim.x * KRY_NT) {
        double s = 0.0;
        for (long e = ptr[i]; e < ptr[i + 1]; ++e) s = fma(val[e], x[col[e]], s);
        y[i] = b ? b[i] - s : s;
    }
}

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    v = threadIdx.x < KRY_NT / 32 ? red[threadIdx.x] : 0.0;
    if (w == 0) {
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    return v;  // valid in thread 0
}

__global__ void __launch_bounds__(KRY_NT) k_dot_part(const double* __restrict__ x, const double* __restrict__ y, long n,
                                                     double* __restrict__ part) {
    __shared__ double red[KRY_NT / 32];
    double s = 0.0;
    for (long i = blockIdx.x * (long)KRY_NT + threadIdx.x; i < n; i += (long)gridDim.x * KRY_NT) s = fma(x[i], y[i], s);
    s = block_sum(s, red);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(KRY_NT) k_dot_fin(const double* __restrict__ part, int np, double* __restrict__ out) {
    __shared__ double red[KRY_NT / 32];
    double s = 0.0;
    for (int i = threadIdx.x; i < np; i += KRY_NT) s += part[i];
    s = block_sum(s, red);
    if (threadIdx.x == 0) *out = s;
}

// x += alpha p;  r -= alpha Ap
__global__ void __launch_bounds__(KRY_NT) k_cg_update(double* __restrict__ x, double* __restrict__ r,
                                                      const double* __restrict__ p, const double* __restrict__ ap,
                                                      double alpha, long n) {
    for (long i = blockIdx.x * (long)KRY_NT + threadIdx.x; i < n; i += (long)gridDim.x * KRY_NT) {
        x[i] = fma(alpha, p[i], x[i]);
        r[i] = fma(-alpha, ap[i], r[i]);
    }
}

// p = z + beta p
__global__ void __launch_bounds__(KRY_NT) k_xpby(double* __restrict__ p, const double* __restrict__ z, double beta, long n) {
    for (long i = blockIdx.x * (long)KRY_NT + threadIdx.x; i < n; i += (long)gridDim.x * KRY_NT) p[i] = fma(beta, p[i], z[i]);
}

// x += z
__global__ void __launch_bounds__(KRY_NT) k_vadd(double* __restrict__ x, const double* __restrict__ z, long n) {
    for (long i = blockIdx.x * (long)KRY_NT + threadIdx.x; i < n; i += (long)gridDim.x * KRY_NT) x[i] += z[i];
}

static int grid_for(long n) {
    const long g = (n + KRY_NT - 1) / KRY_NT;
    return (int)(g < 148L * 8 ? (g > 0 ? g : 1) : 148L * 8);
}

void launch_csr_spmv(cudaStream_t st, const long* ptr, const int* col, const double* val, const double* x,
                     const double* b, double* y, long nrows) {
    ProfScope _ps(st, "k_csr_spmv", grid_for(nrows));
    k_csr_spmv<<<grid_for(nrows), KRY_NT, 0, st>>>(ptr, col, val, x, b, y, nrows);
}

void launch_dot(cudaStream_t st, const double* x, const double* y, long n, double* part, double* out) {
    {
        ProfScope _ps(st, "k_dot_part", KRY_G);
        k_dot_part<<<KRY_G, KRY_NT, 0, st>>>(x, y, n, part);
    }
    ProfScope _ps(st, "k_dot_fin", 1);
    k_dot_fin<<<1, KRY_NT, 0, st>>>(part, KRY_G, out);
}

void launch_cg_update(cudaStream_t st, double* x, double* r, const double* p, const double* ap, double alpha, long n) {
    ProfScope _ps(st, "k_cg_update", grid_for(n));
    k_cg_update<<<grid_for(n), KRY_NT, 0, st>>>(x, r, p, ap, alpha, n);
}

void launch_xpby(cudaStream_t st, double* p, const double* z, double beta, long n) {
    ProfScope _ps(st, "k_xpby", grid_for(n));
    k_xpby<<<grid_for(n), KRY_NT, 0, st>>>(p, z, beta, n);
}

void launch_vadd(cudaStream_t st, double* x, const double* z, long n) {
    ProfScope _ps(st, "k_vadd", grid_for(n));
    k_vadd<<<grid_for(n), KRY_NT, 0, st>>>(x, z, n);
}

}  // namespace acrgpu
