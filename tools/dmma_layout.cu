// Checks the mma.sync.m8n8k4 f64 fragment layout assumed by bqr.cuh:
//   A (8x4 row): lane holds A[lane>>2][lane&3];  B (4x8 col): B[lane&3][lane>>2];
//   C/D (8x8): lane holds C[lane>>2][2*(lane&3) + i], i = 0, 1.
#include <cstdio>
#include <cmath>
__global__ void k(const double* A, const double* B, double* C) {
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    double a = A[g * 4 + t], b = B[t * 8 + g], d0 = 0, d1 = 0;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
    C[g * 8 + 2 * t] = d0;
    C[g * 8 + 2 * t + 1] = d1;
}
int main() {
    double hA[32], hB[32], hC[64], *dA, *dB, *dC;
    for (int i = 0; i < 32; ++i) { hA[i] = 1 + i * 0.37; hB[i] = 2 - i * 0.11; }
    cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dC, 512);
    cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dA, dB, dC);
    cudaMemcpy(hC, dC, 512, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) {
            double s = 0;
            for (int q = 0; q < 4; ++q) s += hA[i * 4 + q] * hB[q * 8 + j];
            err = fmax(err, fabs(s - hC[i * 8 + j]));
        }
    printf("{\"dmma_layout_maxerr\": %g}\n", err);
    return err < 1e-12 ? 0 : 1;
}
