// FP64 peak microbenchmark for B200 (sm_100a): DFMA (CUDA cores) and DMMA
// (mma.sync.m8n8k4.f64 tensor path). Result feeds the roofline denominator
// used by bench.py (MEASURED_PEAKS.json carries no FP64 figure).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[4][2];
    for (int i = 0; i < 4; ++i) { c[i][0] = 0; c[i][1] = 0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0;
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i < n; i += stride) b[i] = a[i];
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    // DFMA: blocks x threads x iters x 8 fma x 2 flop
    for (int rep = 0; rep < 2; ++rep) {
        int blocks = sms * 8, threads = 256, iters = 20000;
        dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * (double)iters * blocks * threads;
        if (rep) printf("{\"kind\":\"dfma\",\"tflops\":%.3f}\n", flops / ms / 1e9);
    }
    for (int rep = 0; rep < 2; ++rep) {
        int blocks = sms * 8, threads = 256, iters = 20000;
        dmma_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e0);
        dmma_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        // per warp per mma: 8*8*4*2 = 512 flop
        double flops = 512.0 * 4 * (double)iters * blocks * (threads / 32);
        if (rep) printf("{\"kind\":\"dmma_m8n8k4\",\"tflops\":%.3f}\n", flops / ms / 1e9);
    }
    size_t n = (size_t)1 << 27;  // 2 GiB of double2 per buffer
    double2 *a, *b;
    cudaMalloc(&a, n * 16);
    cudaMalloc(&b, n * 16);
    cudaMemset(a, 0, n * 16);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        copy_kernel<<<sms * 16, 256>>>(a, b, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) printf("{\"kind\":\"copy\",\"gbs\":%.1f}\n", 2.0 * n * 16 / ms / 1e6);
    }
    cudaError_t err = cudaGetLastError();
    printf("{\"err\":\"%s\"}\n", cudaGetErrorString(err));
    return 0;
}
