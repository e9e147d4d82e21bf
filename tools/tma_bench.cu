// Microbenchmark: cost of cp.async.bulk (global -> shared) as a function of the copy size and of
// who issues it.  One CTA per SM; per CTA `nprod` producer warps stream `total` bytes from a private
// global region into a 4-slot shared ring, `sz` bytes per copy, waiting on an mbarrier every `batch`
// copies.  mode 0: lane 0 of each producer warp issues; mode 1: every lane issues its own copy.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/tma_bench.cu -o /tmp/tma_bench && /tmp/tma_bench
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned s32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool mtry(unsigned long long* b, unsigned ph) {
    unsigned ok;
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(s32(b)), "r"(ph) : "memory");
    return ok;
}
__global__ void __launch_bounds__(256, 1) k(const char* src, size_t per_cta, int sz, int mode, int nprod, unsigned long long* cyc) {
    extern __shared__ __align__(128) char sm[];
    __shared__ unsigned long long bar[16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x < 16) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(bar + threadIdx.x)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (warp >= nprod) return;
    const char* g = src + (size_t)blockIdx.x * per_cta + (size_t)warp * (per_cta / nprod);
    const size_t mine = per_cta / nprod;
    char* dst = sm + (size_t)warp * (160 * 1024 / nprod);
    const int ring = (160 * 1024 / nprod);
    const int per_batch = (ring / 2) / sz;
    const int batch_bytes = per_batch * sz;     // half a ring per mbarrier phase
    if (per_batch == 0) return;
    unsigned ph[2] = {0, 0};
    const unsigned long long t0 = clock64();
    size_t nb = 0;
    for (size_t off = 0; off + batch_bytes <= mine; off += batch_bytes, ++nb) {
        const int hb = (int)(nb & 1);
        const int half = hb * batch_bytes;
        unsigned long long* mb = bar + 2 * warp + hb;
        // the half ring being refilled must have landed (batch nb - 2)
        if (nb >= 2) { while (!mtry(mb, ph[hb])) {} ph[hb] ^= 1; }
        if (mode == 0) {
            if (lane == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(mb)), "r"(batch_bytes) : "memory");
                for (int i = 0; i < per_batch; ++i)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s32(dst + half + i * sz)), "l"(g + off + (size_t)i * sz), "r"(sz), "r"(s32(mb)) : "memory");
            }
        } else {
            if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(mb)), "r"(batch_bytes) : "memory");
            __syncwarp();
            for (int i = lane; i < per_batch; i += 32)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s32(dst + half + i * sz)), "l"(g + off + (size_t)i * sz), "r"(sz), "r"(s32(mb)) : "memory");
        }
    }
    for (int hb = 0; hb < 2; ++hb)
        if (nb > (size_t)hb) while (!mtry(bar + 2 * warp + hb, ph[hb])) {}
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}
int main() {
    setvbuf(stdout, nullptr, _IOLBF, 0);
    const size_t per_cta = 64ull << 20;  // 64 MiB per CTA, 9.25 GiB total
    const int nsm = 148;
    char* src;
    cudaMalloc(&src, per_cta * nsm);
    cudaMemset(src, 1, per_cta * nsm);
    unsigned long long* cyc;
    cudaMalloc(&cyc, nsm * 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int sizes[] = {256, 512, 1024, 2048, 4096, 8192, 32768};
    for (int nprod : {1, 2, 4})
        for (int mode : {0, 1})
            for (int sz : sizes) {
                k<<<nsm, 256, 160 * 1024>>>(src, per_cta, sz, mode, nprod, cyc);
                cudaEventRecord(e0);
                k<<<nsm, 256, 160 * 1024>>>(src, per_cta, sz, mode, nprod, cyc);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                const double ops = (double)per_cta / sz;  // per SM
                printf("nprod %d mode %d size %6d: %7.3f ms  %7.1f GB/s  %.1f cycles/op/SM (at 1.965 GHz)  err=%d\n", nprod, mode, sz, ms,
                       per_cta * nsm / ms / 1e6, ms * 1e-3 * 1.965e9 / ops, (int)cudaGetLastError());
            }
    return 0;
}
