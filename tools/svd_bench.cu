// Microbenchmark of the register-resident Jacobi SVD engines (svd_small.cuh):
// sweeps, latency and accuracy on synthetic blocks with decaying spectra.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <random>
#include "../paper_1701_00182_b200/csrc/svd_small.cuh"
#include "../paper_1701_00182_b200/csrc/svd_rrqr32.cuh"
using namespace acrgpu;

__device__ int g_sweeps[64];

__global__ void bench32(const double* M, int nmat, double* sig_out, int* sweeps_out, long long* cycles) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * 4 + warp;
    if (t >= nmat) return;
    double a[32], v[32];
    for (int j = 0; j < 32; ++j) { a[j] = M[(size_t)t * 1024 + lane + j * 32]; v[j] = (j == lane) ? 1.0 : 0.0; }
    long long c0 = clock64();
    const int sw = warp_jacobi32(a, v, 32, true);
    if (lane == 0) sweeps_out[t] = sw;
    long long c1 = clock64();
    double sig; int pos, r;
    warp_sigma_rank32(a, 32, 5e-7, 0.0, sig, pos, r);
    sig_out[(size_t)t * 32 + pos] = sig;
    if (lane == 0) cycles[t] = c1 - c0;
}

__global__ void bench32c(const double* M, int nmat, double* sig_out, int* sweeps_out, long long* cycles, double floor_rel) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * 4 + warp;
    if (t >= nmat) return;
    double a[32], v[32];
    double fro = 0;
    for (int i = 0; i < 32; ++i) { a[i] = M[(size_t)t * 1024 + i + lane * 32]; v[i] = (i == lane) ? 1.0 : 0.0; fro += a[i]*a[i]; }
    for (int o = 16; o; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
    long long c0 = clock64();
    const int sw = warp_jacobi32c(a, v, true, fro * floor_rel * floor_rel);
    long long c1 = clock64();
    double s = 0; for (int i = 0; i < 32; ++i) s += a[i]*a[i];
    double sig = sqrt(s);
    int pos = 0;
    for (int i = 0; i < 32; ++i) { double w = __shfl_sync(0xffffffffu, sig, i); pos += (w > sig) || (w == sig && i < lane); }
    sig_out[(size_t)t * 32 + pos] = sig;
    if (lane == 0) { cycles[t] = c1 - c0; sweeps_out[t] = sw; }
}

// QR-preconditioned variant: A = QR (Householder, column per lane, fully unrolled),
// then one-sided Jacobi on R^T (rows of R become columns).
__global__ void bench32q(const double* M, int nmat, double* sig_out, int* sweeps_out, long long* cycles, double floor_rel) {
    __shared__ double T[4][32][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * 4 + warp;
    if (t >= nmat) return;
    double a[32], v[32];
    double fro = 0;
    for (int i = 0; i < 32; ++i) { a[i] = M[(size_t)t * 1024 + i + lane * 32]; v[i] = (i == lane) ? 1.0 : 0.0; fro += a[i]*a[i]; }
    for (int o = 16; o; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
    long long c0 = clock64();
#pragma unroll
    for (int j = 0; j < 31; ++j) {
        double beta = 0, tau = 0, inv = 0;
        if (lane == j) {
            double tail = 0;
#pragma unroll
            for (int i = j + 1; i < 32; ++i) tail = fma(a[i], a[i], tail);
            const double c0v = a[j];
            if (tail > 2.2250738585072014e-308) {
                beta = sqrt(c0v * c0v + tail);
                if (c0v >= 0) beta = -beta;
                inv = 1.0 / (c0v - beta);
                tau = (beta - c0v) / beta;
            } else { beta = c0v; tau = 0; inv = 0; }
#pragma unroll
            for (int i = j + 1; i < 32; ++i) a[i] *= inv;
            a[j] = beta;
        }
        tau = __shfl_sync(0xffffffffu, tau, j);
        double vv[32];
#pragma unroll
        for (int i = j + 1; i < 32; ++i) vv[i] = __shfl_sync(0xffffffffu, a[i], j);
        if (lane > j && tau != 0.0) {
            double sdot = a[j];
#pragma unroll
            for (int i = j + 1; i < 32; ++i) sdot = fma(vv[i], a[i], sdot);
            sdot *= tau;
            a[j] -= sdot;
#pragma unroll
            for (int i = j + 1; i < 32; ++i) a[i] = fma(-sdot, vv[i], a[i]);
        }
    }
    // transpose R (upper) through smem: lane k gets row k of R
#pragma unroll
    for (int i = 0; i < 32; ++i) T[warp][i][lane] = (i <= lane) ? a[i] : 0.0;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) a[j] = T[warp][lane][j];
    __syncwarp();
    const int sw = warp_jacobi32c(a, v, true, fro * floor_rel * floor_rel);
    long long c1 = clock64();
    double s = 0; for (int i = 0; i < 32; ++i) s += a[i]*a[i];
    double sig = sqrt(s);
    int pos = 0;
    for (int i = 0; i < 32; ++i) { double w = __shfl_sync(0xffffffffu, sig, i); pos += (w > sig) || (w == sig && i < lane); }
    sig_out[(size_t)t * 32 + pos] = sig;
    if (lane == 0) { cycles[t] = c1 - c0; sweeps_out[t] = sw; }
}

__global__ void bench32r(const double* M, int nmat, double* sig_out, int* sweeps_out, long long* cycles, double eps) {
    __shared__ Warp32Smem sm[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * 2 + warp;
    if (t >= nmat) return;
    double a[32], v[32];
    for (int i = 0; i < 32; ++i) a[i] = M[(size_t)t * 1024 + i + lane * 32];
    long long c0 = clock64();
    const int rp = warp_rrqr_jacobi32(a, v, 32, 32, 1e-3 * eps / 5.66, 0.0, true, sm[warp]);
    double sig, smax; int pos, r;
    warp_sigma_pos32(a, rp, eps, 0.0, sig, pos, r, smax);
    long long c1 = clock64();
    for (int k = lane; k < 32; k += 32) sig_out[(size_t)t * 32 + k] = 0.0;
    __syncwarp();
    if (lane < rp) sig_out[(size_t)t * 32 + pos] = sig;
    if (lane == 0) { cycles[t] = c1 - c0; sweeps_out[t] = rp; }
}

int main(int argc, char** argv) {
    const int nmat = 4096;
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd;
    std::vector<double> M((size_t)nmat * 1024);
    for (int t = 0; t < nmat; ++t) {
        // M = sum_k s_k x_k y_k^T with s_k = 10^(-k * decay)
        const int kind = t % 3;
        const double decay = kind == 0 ? 0.0 : (kind == 1 ? 0.5 : 0.25);
        const int K = 48;
        for (int k = 0; k < K; ++k) {
            double x[32], y[32];
            for (int i = 0; i < 32; ++i) { x[i] = nd(rng); y[i] = nd(rng); }
            const double s = pow(10.0, -decay * k);
            for (int j = 0; j < 32; ++j)
                for (int i = 0; i < 32; ++i) M[(size_t)t * 1024 + i + j * 32] += s * x[i] * y[j];
        }
    }
    double *dM, *dS; int* dw; long long* dc;
    cudaMalloc(&dM, M.size() * 8); cudaMalloc(&dS, (size_t)nmat * 32 * 8); cudaMalloc(&dw, 4 * nmat); cudaMalloc(&dc, 8 * nmat);
    cudaMemcpy(dM, M.data(), M.size() * 8, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        bench32<<<(nmat + 3) / 4, 128>>>(dM, nmat, dS, dw, dc);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("warp32: %d SVDs in %.3f ms (%.2f us/SVD amortized) err=%s\n", nmat, ms, 1000 * ms / nmat, cudaGetErrorString(cudaGetLastError()));
    }
    std::vector<long long> cyc(nmat);
    std::vector<int> sw(nmat);
    cudaMemcpy(cyc.data(), dc, 8 * nmat, cudaMemcpyDeviceToHost);
    cudaMemcpy(sw.data(), dw, 4 * nmat, cudaMemcpyDeviceToHost);
    double avg[3] = {0, 0, 0}, asw[3] = {0, 0, 0};
    for (int t = 0; t < nmat; ++t) { avg[t % 3] += cyc[t] / (nmat / 3.0); asw[t % 3] += sw[t] / (nmat / 3.0); }
    printf("cycles per SVD (latency): full-rank %.0f, decay0.5 %.0f, decay0.25 %.0f\n", avg[0], avg[1], avg[2]);
    printf("sweeps: full-rank %.2f, decay0.5 %.2f, decay0.25 %.2f\n", asw[0], asw[1], asw[2]);
    std::vector<double> sref((size_t)nmat * 32), sc((size_t)nmat * 32);
    cudaMemcpy(sref.data(), dS, sref.size() * 8, cudaMemcpyDeviceToHost);
    for (int variant = 0; variant < 4; ++variant) {
        const double fl = variant % 2 ? 1e-11 : 0.0;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (variant < 2) bench32c<<<(nmat + 3) / 4, 128>>>(dM, nmat, dS, dw, dc, fl);
            else bench32q<<<(nmat + 3) / 4, 128>>>(dM, nmat, dS, dw, dc, fl);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("%s floor %.0e: %d SVDs in %.3f ms err=%s\n", variant < 2 ? "col32" : "qr+col32", fl, nmat, ms, cudaGetErrorString(cudaGetLastError()));
        }
        cudaMemcpy(cyc.data(), dc, 8 * nmat, cudaMemcpyDeviceToHost);
        cudaMemcpy(sw.data(), dw, 4 * nmat, cudaMemcpyDeviceToHost);
        cudaMemcpy(sc.data(), dS, sc.size() * 8, cudaMemcpyDeviceToHost);
        double avg2[3] = {0, 0, 0}, asw2[3] = {0, 0, 0}, maxrel = 0;
        for (int t = 0; t < nmat; ++t) {
            avg2[t % 3] += cyc[t] / (nmat / 3.0); asw2[t % 3] += sw[t] / (nmat / 3.0);
            for (int k = 0; k < 32; ++k) { double a = sref[t*32+k], b = sc[t*32+k]; if (a > 1e-9 * sref[t*32]) maxrel = fmax(maxrel, fabs(a-b)/a); }
        }
        printf("  cycles: %.0f %.0f %.0f  sweeps: %.2f %.2f %.2f  max rel sigma diff (sigma>1e-9 s1) vs row engine: %.2e\n", avg2[0], avg2[1], avg2[2], asw2[0], asw2[1], asw2[2], maxrel);
    }
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        bench32r<<<(nmat + 1) / 2, 64>>>(dM, nmat, dS, dw, dc, 5e-7);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("rrqr32 eps 5e-7: %d SVDs in %.3f ms err=%s\n", nmat, ms, cudaGetErrorString(cudaGetLastError()));
    }
    cudaMemcpy(cyc.data(), dc, 8 * nmat, cudaMemcpyDeviceToHost);
    cudaMemcpy(sw.data(), dw, 4 * nmat, cudaMemcpyDeviceToHost);
    cudaMemcpy(sc.data(), dS, sc.size() * 8, cudaMemcpyDeviceToHost);
    {
        double avg2[3] = {0, 0, 0}, asw2[3] = {0, 0, 0}, maxrel = 0; int rankdiff = 0;
        for (int t = 0; t < nmat; ++t) {
            avg2[t % 3] += cyc[t] / (nmat / 3.0); asw2[t % 3] += sw[t] / (nmat / 3.0);
            int ra = 0, rb = 0;
            for (int k = 0; k < 32; ++k) { double a = sref[t*32+k], b = sc[t*32+k]; if (a > 1e-6 * sref[t*32]) maxrel = fmax(maxrel, fabs(a-b)/a);
                ra += a > 5e-7 * sref[t*32]; rb += b > 5e-7 * sc[t*32]; }
            rankdiff += ra != rb;
        }
        printf("  cycles: %.0f %.0f %.0f  rp: %.2f %.2f %.2f  max rel sigma diff (sigma>1e-6 s1): %.2e  rank mismatches: %d\n", avg2[0], avg2[1], avg2[2], asw2[0], asw2[1], asw2[2], maxrel, rankdiff);
    }
    return 0;
}
