// Microbenchmark of the blocked Householder QR (bqr.cuh) used by the QR-route
// truncation: one CTA (512 threads) per m x K matrix, phase cycle breakdown,
// and a correctness check ||R^T R - A^T A|| / ||A^T A||.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 tools/bqr_bench.cu -o tools/bqr_bench
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <random>
#include "../paper_1701_00182_b200/csrc/svd_small.cuh"
namespace acrgpu {
__device__ unsigned long long g_phase_cyc[16];
#define PHASE_MARK(i)                                                          \
    do {                                                                       \
        if (threadIdx.x == 0) {                                                \
            const unsigned long long t_ = clock64();                           \
            atomicAdd(&g_phase_cyc[i], t_ - ph_t0);                            \
            ph_t0 = t_;                                                        \
        }                                                                      \
    } while (0)
#include "../paper_1701_00182_b200/csrc/bqr.cuh"
}  // namespace acrgpu
using namespace acrgpu;

constexpr int NT = 512;
constexpr size_t SMEM_D = 27328;

__global__ void __launch_bounds__(NT, 1) kbqr(double* A, int m, int K, double* tau, double* Tall) {
    extern __shared__ double smem[];
    double* a = A + (size_t)blockIdx.x * m * K;
    const int npan = (K + BQR_NB - 1) / BQR_NB;
    bqr<NT>(a, m, m, K, tau + (size_t)blockIdx.x * K, Tall + (size_t)blockIdx.x * npan * 256, smem, SMEM_D);
}

int main(int argc, char** argv) {
    const int m = argc > 1 ? atoi(argv[1]) : 276;
    const int K = argc > 2 ? atoi(argv[2]) : 69;
    const int nmat = argc > 3 ? atoi(argv[3]) : 148 * 4;
    const int reps = 5;
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd;
    std::vector<double> h((size_t)m * K * nmat);
    for (auto& x : h) x = nd(rng);
    // decaying column scales like an H-arithmetic concatenation
    for (int t = 0; t < nmat; ++t)
        for (int j = 0; j < K; ++j)
            for (int i = 0; i < m; ++i) h[(size_t)t * m * K + i + (size_t)j * m] *= pow(10.0, -8.0 * ((j * 7) % K) / K);
    double *dA, *dA0, *dtau, *dT;
    const int npan = (K + 15) / 16;
    cudaMalloc(&dA, h.size() * 8);
    cudaMalloc(&dA0, h.size() * 8);
    cudaMalloc(&dtau, (size_t)nmat * K * 8);
    cudaMalloc(&dT, (size_t)nmat * npan * 256 * 8);
    cudaMemcpy(dA0, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(kbqr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(SMEM_D * 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaMemcpy(dA, dA0, h.size() * 8, cudaMemcpyDeviceToDevice);
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_phase_cyc, z, sizeof(z));
        cudaEventRecord(e0);
        kbqr<<<nmat, NT, SMEM_D * 8>>>(dA, m, K, dtau, dT);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    unsigned long long ph[16];
    cudaMemcpyFromSymbol(ph, g_phase_cyc, sizeof(ph));
    std::vector<double> R((size_t)m * K);
    cudaMemcpy(R.data(), dA, R.size() * 8, cudaMemcpyDeviceToHost);
    // check matrix 0: R^T R vs A^T A
    double num = 0, den = 0;
    for (int p = 0; p < K; ++p)
        for (int q = 0; q < K; ++q) {
            double g = 0, rr = 0;
            for (int i = 0; i < m; ++i) g += h[i + (size_t)p * m] * h[i + (size_t)q * m];
            for (int i = 0; i <= std::min(std::min(p, q), m - 1); ++i) rr += R[i + (size_t)p * m] * R[i + (size_t)q * m];
            num += (g - rr) * (g - rr);
            den += g * g;
        }
    const double fl = (m >= K ? 2.0 * m * K * K - 2.0 / 3 * K * K * K : 2.0 * K * m * m - 2.0 / 3 * m * m * m) * nmat;
    const double cta_cyc = (double)(ph[10] + ph[11] + ph[12]) / nmat;
    printf("{\"m\": %d, \"K\": %d, \"nmat\": %d, \"ms\": %.4f, \"tflops\": %.3f, \"relerr\": %.3e, \"cyc_per_cta\": %.0f, "
           "\"panel\": %.0f, \"T\": %.0f, \"update\": %.0f, \"err\": \"%s\"}\n",
           m, K, nmat, best, fl / best / 1e9, sqrt(num / den), cta_cyc, (double)ph[10] / nmat, (double)ph[11] / nmat,
           (double)ph[12] / nmat, cudaGetErrorString(err));
    return 0;
}
