// sm_100a kernels of the batched H-matrix arithmetic (FP64).
//
// Every kernel is "task-parallel": blockIdx.x indexes a structural task of a
// compiled plan, blockIdx.y the plane of the batch.  Sizes that depend on
// ranks are read from device memory, outputs of data-dependent size are carved
// from a device bump arena, so whole levels of the cyclic reduction are
// enqueued without host synchronisation.
//
// Reference operations (file:line relative to /root/reference/proj/core/src):
//   k_truncate      truncate_impl / flush / Branch*Branch agglomeration  hmatrix.cpp:56-84,373-392,415-440
//   k_dd_product    Dense*Dense -> dense_to_lowrank                       hmatrix.cpp:87-99,411-413
//   k_apply         node_apply / node_apply_trans (Rk*H, H*Rk products)   hmatrix.cpp:203-238,399-410
//   k_deposit       deposit into dense targets                            hmatrix.cpp:354-371
//   k_lu_inverse    PartialPivLU + rcond guard + inverse                  hmatrix.cpp:483-496
//   k_sigma1_*      scale_walk (largest leaf spectral norm)               hmatrix.cpp:623-642
//   k_matvec        happly / node_apply in the solve                      hmatrix.cpp:695-706
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <algorithm>
#include <cstdlib>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "kernels.hpp"
#include "structure.hpp"
#include "svd_small.cuh"
namespace acrgpu {
// warp-engine phase timing (clock64 deltas of lane 0 per task): diagnostics only
__device__ unsigned long long g_w32_cyc[8];
__device__ unsigned long long g_w32_cnt;
__device__ __forceinline__ void w32_mark(int i, unsigned long long& t0) {
    if ((threadIdx.x & 31) == 0) {
        const unsigned long long t = clock64();
        atomicAdd(&g_w32_cyc[i], t - t0);
        t0 = t;
    }
}
}  // namespace acrgpu
#include "svd_rrqr32.cuh"

namespace acrgpu {

constexpr int NT = 256;

// ------------------------------------------------------------------ helpers

__device__ double* arena_alloc(const Arena& a, unsigned long long n) {
    n = (n + 15ull) & ~15ull;  // 128-byte granules
    const unsigned long long off = atomicAdd(a.ctr, n);
    if (off + n > a.cap) {
        atomicExch(a.overflow, 1);
        return nullptr;
    }
    return a.base + off;
}

// ------------------------------------------------------------------ TMA bulk copies and mbarriers (PTX)
// cp.async.bulk global -> shared (SASS UBLKCP) completing on an mbarrier by transaction bytes; used by
// the solve's slab kernel (k_mv_slab_tma) and by the dense-leaf staging of k_dd_product.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    unsigned spins = 0;
    while (!mbar_try(b, parity))
        if (++spins > (1u << 27)) __trap();  // a lost arrival must not hang the device
}
// global -> shared bulk copy (TMA, SASS UBLKCP), bytes a multiple of 16, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// QR-route phase timing (clock64 deltas of thread 0, summed over CTAs): diagnostics only
__device__ unsigned long long g_phase_cyc[16];
__device__ unsigned long long g_phase_cnt;
// k_mv_slab_tma diagnostics (warp 0 / producer warp 0, lane 0): CTAs, CTA cycles, consumer cycles
// waiting for a full stage, consumer cycles between wait and release, producer cycles waiting for
// an empty stage, stages, leaf entries, producer cycles
__device__ unsigned long long g_mv_cyc[16];
#define PHASE_MARK(i)                                                          \
    do {                                                                       \
        if (threadIdx.x == 0) {                                                \
            const unsigned long long t_ = clock64();                           \
            atomicAdd(&g_phase_cyc[i], t_ - ph_t0);                            \
            ph_t0 = t_;                                                        \
        }                                                                      \
    } while (0)

#include "svd_cta.cuh"
#include "bqr.cuh"

__device__ __forceinline__ void add_flops(FlopLedger* L, int cls, double f) {
    if (L && f > 0) atomicAdd(&L->f[cls], f);
}

// nominal counts (identical formulas to oracle/acr_oracle.cpp)
__device__ __forceinline__ double fl_gemm(double m, double n, double k) { return (m > 0 && n > 0 && k > 0) ? 2 * m * n * k : 0; }
__device__ __forceinline__ double fl_geqrf(double m, double K) {
    return m >= K ? 2 * m * K * K - 2.0 / 3.0 * K * K * K : 2 * K * m * m - 2.0 / 3.0 * m * m * m;
}
__device__ __forceinline__ double fl_orgqr(double m, double ku) { return 2 * m * ku * ku - 2.0 / 3.0 * ku * ku * ku; }
// returns flops of the oracle's svd() of an r x c matrix, split into (svd, qr-ish, gemm)
__device__ void fl_svd(double r, double c, double& fsvd, double& fqr, double& fgemm) {
    if (r == c) { fsvd += 21 * r * r * r; return; }
    const double p = r < c ? r : c, q = r < c ? c : r;
    fqr += fl_geqrf(q, p) + fl_orgqr(q, p);
    fsvd += 21 * p * p * p;
    fgemm += fl_gemm(q, p, p);
}

// ------------------------------------------------------------------ part resolution
struct PartRes {
    const double* U;
    const double* V;
    int ldu, ldv, rank;
};

__device__ __forceinline__ PartRes resolve_part(const Part& p, const Slot* slots, int b, int B, const HView& C) {
    PartRes r{nullptr, nullptr, 0, 0, 0};
    if (p.src == S_SLOT) {
        const Slot s = slots[(size_t)p.id * B + b];
        r.rank = s.rank;
        if (s.rank > 0) {
            r.U = s.U + p.u_src;
            r.V = s.V + p.v_src;
            r.ldu = s.ldu;
            r.ldv = s.ldv;
        }
    } else if (p.src == S_CLEAF) {
        r.rank = C.rank[p.id];
        if (r.rank > 0) {
            r.U = C.U[p.id] + p.u_src;
            r.V = C.V[p.id] + p.v_src;
            r.ldu = p.rows_u;
            r.ldv = p.rows_v;
        }
    }
    return r;
}

// ------------------------------------------------------------------ truncation kernel
// One CTA per (task, plane).  Dense route (m, n <= DENSE_MAX): form the m x n
// block M = sum alpha U V^T in shared memory and SVD it directly -- the same
// singular triplets the reference obtains from QR(U), QR(V), SVD(Ru Rv^T),
// without the two QRs.  QR route (larger blocks): concatenate into an arena
// workspace, Householder QR both factors, SVD the ku x kv core, rebuild
// U' = Qu Us Sigma, V' = Qv Vs by applying the reflectors.
// Carve an engine workspace for blocks up to p x p out of `base`.
__device__ __forceinline__ CtaSvdWork cta_smem_work(double* base, int p, int rpcap) {
    CtaSvdWork w;
    w.A = base;
    w.lda = p;
    w.W = base + (size_t)p * p;
    w.ldw = p;
    w.J = w.W + (size_t)p * rpcap;
    w.ldj = rpcap;
    w.tau = w.J + (size_t)rpcap * rpcap;
    w.nrm = w.tau + p;
    w.sig = w.nrm + p;
    w.perm = (int*)(w.sig + p);
    w.order = w.perm + p;
    return w;
}

struct TruncArgs {
    const TruncTask* tasks;
    const Part* parts;
    Slot* slots;
    int B;
    double eps;
    const double* abs_cut;  // per plane (nullptr: 0)
    double* sig_out;        // values-only mode: sigma_1 per (task, plane)
    int values_only;
    Arena out_arena;        // persistent (flush) or transient (products)
    Arena work;             // transient workspace
    FlopLedger* flops;
    int dense_min_k;        // blocks <= DMAX take the dense route only when K >= this (else the QR route)
};

// C (ru x rv, ld ldc; shared memory) += alpha * A (ru x k) * B^T (rv x k), A/B column-major
// in global memory.  NTH threads as a GY x GX grid (GX = 16), each owning a TM x TN register
// tile (rows ty + GY i, columns tx + 16 j); k is staged through `stage`.
template <int NTH, int TM, int TN, bool TRI = false>
__device__ void gemm_nt_tiled(double* C, int ldc, const double* A, int lda, const double* B, int ldb, int ru, int rv, int k,
                              double alpha, double* stage, int stage_doubles, int ra0 = 0, int rb0 = 0) {
    constexpr int GX = 16, GY = NTH / GX;
    constexpr int RA = GY * TM, RB = GX * TN;
    int KC = stage_doubles / (RA + RB);
    if (KC > 32) KC = 32;
    double* As = stage;            // RA x KC
    double* Bs = stage + RA * KC;  // RB x KC
    const int ty = threadIdx.x % GY, tx = threadIdx.x / GY;  // consecutive lanes -> consecutive rows (no bank conflicts on C)
    double acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;
    for (int t0 = 0; t0 < k; t0 += KC) {
        const int kc = min(KC, k - t0);
        __syncthreads();
        // groups of 8 loads are issued before their shared-memory stores (a load-store loop
        // pays one memory round trip per iteration: the compiler cannot reorder across the
        // generic smem store)
        for (int e0 = threadIdx.x; e0 < RA * kc; e0 += 8 * NTH) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * NTH, i = e % RA, t = e / RA;
                v[u] = (e < RA * kc && i < ru && (!TRI || ra0 + i <= t0 + t)) ? A[i + (size_t)(t0 + t) * lda] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * NTH;
                if (e < RA * kc) As[(e % RA) + (e / RA) * RA] = v[u];
            }
        }
        for (int e0 = threadIdx.x; e0 < RB * kc; e0 += 8 * NTH) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * NTH, i = e % RB, t = e / RB;
                v[u] = (e < RB * kc && i < rv && (!TRI || rb0 + i <= t0 + t)) ? B[i + (size_t)(t0 + t) * ldb] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * NTH;
                if (e < RB * kc) Bs[(e % RB) + (e / RB) * RB] = v[u];
            }
        }
        __syncthreads();
        for (int t = 0; t < kc; ++t) {
            double a[TM], bb[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = As[ty + GY * i + t * RA];
#pragma unroll
            for (int j = 0; j < TN; ++j) bb[j] = Bs[tx + GX * j + t * RB];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], bb[j], acc[i][j]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int r = ty + GY * i, c = tx + GX * j;
            if (r < ru && c < rv) C[r + (size_t)c * ldc] += alpha * acc[i][j];
        }
    __syncthreads();
}

// shared memory of the QR-route kernel beyond the DMAX / RPCAP layout, up to the 227 KB a CTA
// may opt into (room for cores a little above DMAX, see core_mid)
constexpr int BIG_SMEM_EXTRA = 1400;

// QR = false: dense route only (the <= 64 class never takes the QR route); without the
// blocked-QR code the kernel fits 128 registers per thread, so two CTAs share an SM.
template <int DMAX, int RPCAP, int NTH, bool QR = true>
__global__ void __launch_bounds__(NTH, QR ? 1 : 2) k_truncate(TruncArgs args, BatchViews bv) {
    extern __shared__ double smem[];
    __shared__ int sh_K;
    __shared__ double* sh_ws;
    const TruncTask task = args.tasks[blockIdx.x];
    const int b = blockIdx.y;
    const int B = args.B;
    const HView& C = bv.c[b];
    const int m = task.m, n = task.n;
    const double abs_cut = args.abs_cut ? args.abs_cut[b] : 0.0;
    if (abs_cut < 0) return;  // recompress with zero matrix scale: leave untouched

    // total concatenated rank K
    if (threadIdx.x == 0) {
        int K = 0;
        for (int pi = task.pbeg; pi < task.pend; ++pi) K += resolve_part(args.parts[pi], args.slots, b, B, C).rank;
        sh_K = K;
    }
    __syncthreads();
    const int K = sh_K;

    auto write_out = [&](int r, double* U, double* V) {
        if (threadIdx.x != 0 || args.values_only) return;
        if (task.out_kind == 0) {
            Slot& s = args.slots[(size_t)task.out_id * B + b];
            s.rank = r;
            s.U = U;
            s.V = V;
            s.ldu = m;
            s.ldv = n;
        } else {
            C.rank[task.out_id] = r;
            C.U[task.out_id] = U;
            C.V[task.out_id] = V;
        }
    };

    if (K == 0) {
        write_out(0, nullptr, nullptr);
        if (args.values_only && threadIdx.x == 0) args.sig_out[(size_t)blockIdx.x * B + b] = 0.0;
        return;
    }

    const int ku = m < K ? m : K, kv = n < K ? n : K;
    double fsvd = 0, fqr = 0, fgemm = 0;
    __shared__ double* sh_out;

    if (m <= DMAX && n <= DMAX && (!QR || K >= args.dense_min_k)) {
        // ---------------- dense route: M = sum alpha U V^T in shared memory, rank-revealing SVD
        CtaSvdWork w = cta_smem_work(smem, DMAX, RPCAP);
        double* M = w.A;
        w.lda = m;
        for (int e = threadIdx.x; e < m * n; e += NTH) M[e] = 0.0;
        __syncthreads();
        for (int pi = task.pbeg; pi < task.pend; ++pi) {
            const Part p = args.parts[pi];
            const PartRes pr = resolve_part(p, args.slots, b, B, C);
            if (pr.rank == 0) continue;
            gemm_nt_tiled<NTH, DMAX * 16 / NTH, DMAX / 16>(M + p.u_dst + (size_t)p.v_dst * m, m, pr.U, pr.ldu, pr.V, pr.ldv, p.rows_u,
                                     p.rows_v, pr.rank, p.alpha, w.W, DMAX * RPCAP + RPCAP * RPCAP);
        }
        int rp;
        double smax;
        const int r = cta_trunc_svd<NTH>(w, m, n, args.eps, abs_cut, args.values_only != 0, &rp, &smax, RPCAP, &args.work);
        if (args.values_only) {
            if (threadIdx.x == 0) args.sig_out[(size_t)blockIdx.x * B + b] = smax;
        } else {
            if (threadIdx.x == 0) sh_out = r > 0 ? arena_alloc(args.out_arena, (unsigned long long)(m + n) * r) : nullptr;
            __syncthreads();
            double* out = sh_out;
            if (out) cta_trunc_write<NTH>(w, m, n, rp, r, out, m, out + (size_t)m * r, n);
            write_out(out ? r : 0, out, out ? out + (size_t)m * r : nullptr);
        }
        if (threadIdx.x == 0) {
            fqr += fl_geqrf(m, K) + fl_geqrf(n, K);
            fgemm += fl_gemm(ku, kv, K);
            if (!args.values_only) {
                fqr += fl_orgqr(m, ku) + fl_orgqr(n, kv);
                fgemm += fl_gemm(m, r, ku) + fl_gemm(n, r, kv);
            }
            const double qr_nominal = fqr;
            fl_svd(ku, kv, fsvd, fqr, fgemm);
            add_flops(args.flops, F_SVD, fsvd);
            add_flops(args.flops, F_GEQRF, fqr);
            add_flops(args.flops, F_GEMM, fgemm);
            // the dense route forms M (2 m n K) instead of the two QRs
            add_flops(args.flops, F_SKIP, fmax(0.0, qr_nominal - fl_gemm(m, n, K)));
        }
        return;
    }

    // ---------------- QR route
    if constexpr (!QR) {
        __trap();  // size class routing error: a block above DMAX reached the dense-only kernel
    } else {
    // workspace: Uc (m x K) | Vc (n x K) | tau_u (K) | tau_v (K) | [core engine work if too big for smem]
    const int pmax = ku > kv ? ku : kv;
    const bool core_in_smem = pmax <= DMAX;
    const size_t smem_doubles = (size_t)DMAX * DMAX + (size_t)DMAX * RPCAP + (size_t)RPCAP * RPCAP + 5 * DMAX + BIG_SMEM_EXTRA;
    // blocked QR staging (panel, W, T) in shared memory, or in global workspace for panels too
    // tall for it (C5's 2048-row leaves)
    const size_t bneed = bqr_smem_doubles(m > n ? m : n, K);
    const bool blocked = bneed <= smem_doubles;
    const int npan = (K + BQR_NB - 1) / BQR_NB + 1;
    const unsigned long long base_need =
        (unsigned long long)(m + n) * K + 2ull * K + 32 + 2ull * npan * BQR_NB * BQR_NB;
    // a core a little above DMAX (K up to ~155) still fits shared memory on its own: W = R^T
    // takes what is left (cols x rp, rp small) or spills to the arena like any oversized W
    const bool core_mid = !core_in_smem && (size_t)ku * kv + (size_t)5 * pmax + 8 + 2304 <= smem_doubles;
    const unsigned long long core_need = (core_in_smem || core_mid) ? 0ull : 3ull * pmax * pmax + 6ull * pmax + 64;
    if (threadIdx.x == 0) sh_ws = arena_alloc(args.work, base_need + core_need + (blocked ? 0ull : bneed));
    __syncthreads();
    double* ws = sh_ws;
    if (ws == nullptr) return;  // arena exhausted: flag raised, target left unchanged
    unsigned long long ph_t0 = clock64();
    if (threadIdx.x == 0) {
        atomicAdd(&g_phase_cnt, 1ull);
        atomicAdd(&g_phase_cyc[6], (unsigned long long)K);
        atomicAdd(&g_phase_cyc[7], (unsigned long long)(m > n ? m : n));
        if (!core_in_smem && !core_mid) atomicAdd(&g_phase_cyc[8], 1ull);
        if (!blocked) atomicAdd(&g_phase_cyc[9], 1ull);
    }
    double* Uc = ws;
    double* Vc = Uc + (size_t)m * K;
    double* tau_u = Vc + (size_t)n * K;
    double* tau_v = tau_u + K;
    double* Tu = tau_v + K + 32;
    double* Tv = Tu + (size_t)npan * BQR_NB * BQR_NB;
    CtaSvdWork w = core_in_smem ? cta_smem_work(smem, DMAX, RPCAP)
                                : cta_smem_work(Tv + (size_t)npan * BQR_NB * BQR_NB, pmax, pmax);
    // Core too large for shared memory (K > 128; a quarter of C5's tasks): the core itself stays
    // in the global workspace (pivoted QR), but the per-column arrays the QR reads every step
    // and the Jacobi working matrix W = R^T (cols x rp, rp small) move to shared memory, which
    // is idle between the blocked QRs and the Q application.
    double* w_alt = nullptr;
    size_t w_alt_cap = 0;
    int rp_cap = core_in_smem ? RPCAP : pmax;
    if (core_mid) {
        double* small = smem + (smem_doubles - (size_t)5 * pmax - 8);
        w.A = smem;
        w.lda = ku;
        w.W = smem + (size_t)ku * kv;
        w.ldw = kv;
        w.J = nullptr;
        w.ldj = 0;
        w.tau = small;
        w.nrm = w.tau + pmax;
        w.sig = w.nrm + pmax;
        w.perm = (int*)(w.sig + pmax);
        w.order = w.perm + pmax;
        rp_cap = (int)((size_t)(small - w.W) / (size_t)kv);
    } else if (!core_in_smem && (size_t)5 * pmax + 64 <= smem_doubles / 4) {
        double* small = smem + (smem_doubles - (size_t)5 * pmax - 8);
        w.tau = small;
        w.nrm = w.tau + pmax;
        w.sig = w.nrm + pmax;
        w.perm = (int*)(w.sig + pmax);
        w.order = w.perm + pmax;
        w_alt = smem;
        w_alt_cap = (size_t)(small - smem);
    }
    for (size_t e = threadIdx.x; e < (size_t)(m + n) * K; e += NTH) ws[e] = 0.0;
    __syncthreads();
    {
        int off = 0;
        for (int pi = task.pbeg; pi < task.pend; ++pi) {
            const Part p = args.parts[pi];
            const PartRes pr = resolve_part(p, args.slots, b, B, C);
            if (pr.rank == 0) continue;
            for (int e = threadIdx.x; e < p.rows_u * pr.rank; e += NTH) {
                const int i = e % p.rows_u, t = e / p.rows_u;
                Uc[(p.u_dst + i) + (size_t)(off + t) * m] = p.alpha * pr.U[i + (size_t)t * pr.ldu];
            }
            for (int e = threadIdx.x; e < p.rows_v * pr.rank; e += NTH) {
                const int i = e % p.rows_v, t = e / p.rows_v;
                Vc[(p.v_dst + i) + (size_t)(off + t) * n] = pr.V[i + (size_t)t * pr.ldv];
            }
            off += pr.rank;
        }
    }
    __syncthreads();
    PHASE_MARK(0);
    double* qs = blocked ? smem : ws + base_need + core_need;
    const size_t qs_doubles = blocked ? smem_doubles : bneed;
    bqr<NTH>(Uc, m, m, K, tau_u, Tu, qs, qs_doubles);
    bqr<NTH>(Vc, n, n, K, tau_v, Tv, qs, qs_doubles);
    PHASE_MARK(1);
    // core = Ru Rv^T (ku x kv)
    double* core = w.A;
    w.lda = ku;
    if (core_in_smem) {
        for (int e = threadIdx.x; e < ku * kv; e += NTH) core[e] = 0.0;
        gemm_nt_tiled<NTH, DMAX * 16 / NTH, DMAX / 16, true>(core, ku, Uc, m, Vc, n, ku, kv, K, 1.0, w.W,
                                                               DMAX * RPCAP + RPCAP * RPCAP);
    } else {  // core above DMAX (shared memory or global workspace): 128 x 128 output tiles
        for (size_t e = threadIdx.x; e < (size_t)ku * kv; e += NTH) core[e] = 0.0;
        __syncthreads();
        double* stage = core_mid ? w.W : smem;
        const int stage_doubles = core_mid ? (int)(w.tau - w.W) : DMAX * RPCAP + RPCAP * RPCAP;
        for (int r0 = 0; r0 < ku; r0 += DMAX)
            for (int c0 = 0; c0 < kv; c0 += DMAX)
                gemm_nt_tiled<NTH, DMAX * 16 / NTH, DMAX / 16, true>(core + r0 + (size_t)c0 * ku, ku, Uc + r0, m,
                                                                       Vc + c0, n, min(DMAX, ku - r0),
                                                                       min(DMAX, kv - c0), K, 1.0, stage,
                                                                       stage_doubles, r0, c0);
    }
    PHASE_MARK(2);
    int rp;
    double smax;
    const int r = cta_trunc_svd<NTH>(w, ku, kv, args.eps, abs_cut, args.values_only != 0, &rp, &smax,
                                    rp_cap, &args.work, w_alt, w_alt_cap);
    PHASE_MARK(3);
    if (args.values_only) {
        if (threadIdx.x == 0) args.sig_out[(size_t)blockIdx.x * B + b] = smax;
    } else {
        if (threadIdx.x == 0) sh_out = r > 0 ? arena_alloc(args.out_arena, (unsigned long long)(m + n) * r) : nullptr;
        __syncthreads();
        double* out = sh_out;
        if (out) {
            double* Uo = out;
            double* Vo = out + (size_t)m * r;
            for (int e = threadIdx.x; e < m * r; e += NTH) Uo[e] = 0.0;
            for (int e = threadIdx.x; e < n * r; e += NTH) Vo[e] = 0.0;
            __syncthreads();
            cta_trunc_write<NTH>(w, ku, kv, rp, r, Uo, m, Vo, n);
            PHASE_MARK(4);
            bqr_apply<NTH>(Uc, m, m, ku, Tu, Uo, m, r, qs, qs_doubles);
            bqr_apply<NTH>(Vc, n, n, kv, Tv, Vo, n, r, qs, qs_doubles);
            PHASE_MARK(5);
        }
        write_out(out ? r : 0, out, out ? out + (size_t)m * r : nullptr);
    }
    if (threadIdx.x == 0) {
        fqr += fl_geqrf(m, K) + fl_geqrf(n, K);
        fgemm += fl_gemm(ku, kv, K);
        if (!args.values_only) {
            fqr += fl_orgqr(m, ku) + fl_orgqr(n, kv);
            fgemm += fl_gemm(m, r, ku) + fl_gemm(n, r, kv);
        }
        fl_svd(ku, kv, fsvd, fqr, fgemm);
        add_flops(args.flops, F_SVD, fsvd);
        add_flops(args.flops, F_GEQRF, fqr);
        add_flops(args.flops, F_GEMM, fgemm);
    }
    }  // QR
}

// ------------------------------------------------------------------ dense * dense product
struct DDArgs {
    const DDTask* tasks;
    Slot* slots;
    int B;
    double eps;
    Arena out_arena;
    FlopLedger* flops;
};

__global__ void __launch_bounds__(NT, 1) k_dd_product(DDArgs args, BatchViews bv) {
    extern __shared__ double smem[];
    __shared__ double* sh_out;
    const DDTask task = args.tasks[blockIdx.x];
    const int b = blockIdx.y;
    const int m = task.m, k = task.k, n = task.n;
    const double* Ad = bv.a[b].dense + task.da;
    const double* Bd = bv.b[b].dense + task.db;
    CtaSvdWork w = cta_smem_work(smem, DENSE_MAX, DENSE_MAX);
    double* M = w.A;
    w.lda = m;
    // operands staged in the (not yet used) W / J areas; a zero operand (off-diagonal leaves
    // of the diagonal level-0 couplings) is detected while staging and gives a rank-0 product
    double* As = w.W;
    double* Bs = w.J;
    auto zero_product = [&]() {
        if (threadIdx.x == 0) {
            Slot& s = args.slots[(size_t)task.prod * args.B + b];
            s.rank = 0;
            s.U = nullptr;
            s.V = nullptr;
            s.ldu = m;
            s.ldv = n;
            double fsvd = 0, fqr = 0, fgemm = fl_gemm(m, n, k);
            fl_svd(m, n, fsvd, fqr, fgemm);
            add_flops(args.flops, F_SVD, fsvd);
            add_flops(args.flops, F_GEQRF, fqr);
            add_flops(args.flops, F_GEMM, fgemm);
            add_flops(args.flops, F_SKIP, fsvd + fqr + fgemm);
        }
    };
    // Both leaves are contiguous in their dense pools: when sizes and addresses are 16-byte aligned
    // (always, for even leaf sizes) one thread brings them in as two TMA bulk copies on one mbarrier
    // -- both in flight at once, no register staging -- and the zero tests read shared memory.
    __shared__ unsigned long long dd_bar;
    const bool bulk = ((m * k) & 1) == 0 && ((k * n) & 1) == 0 &&
                      ((((unsigned long long)Ad | (unsigned long long)Bd) & 15ull) == 0) && ((smem_u32(As) | smem_u32(Bs)) & 15u) == 0;
    if (bulk) {
        if (threadIdx.x == 0) {
            mbar_init(&dd_bar, 1);
            fence_proxy_async();
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            mbar_arrive_tx(&dd_bar, (unsigned)(m * k + k * n) * 8u);
            bulk_g2s(As, Ad, (unsigned)(m * k) * 8u, &dd_bar);
            bulk_g2s(Bs, Bd, (unsigned)(k * n) * 8u, &dd_bar);
        }
        mbar_wait(&dd_bar, 0);
        int nz = 0;
        for (int e = threadIdx.x; e < m * k; e += NT) nz |= As[e] != 0.0;
        if (!__syncthreads_or(nz)) {
            zero_product();
            return;
        }
        nz = 0;
        for (int e = threadIdx.x; e < k * n; e += NT) nz |= Bs[e] != 0.0;
        if (!__syncthreads_or(nz)) {
            zero_product();
            return;
        }
    } else {
        int nz = 0;
        for (int e = threadIdx.x; e < m * k; e += NT) {
            const double v = Ad[e];
            nz |= v != 0.0;
            As[e] = v;
        }
        if (!__syncthreads_or(nz)) {
            zero_product();
            return;
        }
        nz = 0;
        for (int e = threadIdx.x; e < k * n; e += NT) {
            const double v = Bd[e];
            nz |= v != 0.0;
            Bs[e] = v;
        }
        if (!__syncthreads_or(nz)) {
            zero_product();
            return;
        }
    }
    // M = A B on the FP64 tensor cores: 8 x 8 output tiles over the warps, k-steps of 4
    // (mma.sync.m8n8k4.f64; fragment layout in bqr.cuh), operands from shared memory
    {
        const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
        const int tm = (m + 7) >> 3, tn = (n + 7) >> 3;
        for (int tile = threadIdx.x >> 5; tile < tm * tn; tile += NT / 32) {
            const int ti = tile % tm, tj = tile / tm;
            const int ra = 8 * ti + g, cb = 8 * tj + g;
            double d0 = 0.0, d1 = 0.0;
            for (int k0 = 0; k0 < k; k0 += 4) {
                const int kk = k0 + t;
                const double a = (ra < m && kk < k) ? As[ra + (size_t)kk * m] : 0.0;
                const double bb = (cb < n && kk < k) ? Bs[kk + (size_t)cb * k] : 0.0;
                dmma8x8x4(d0, d1, a, bb);
            }
            const int c0 = 8 * tj + 2 * t;
            if (ra < m) {
                if (c0 < n) M[ra + (size_t)c0 * m] = d0;
                if (c0 + 1 < n) M[ra + (size_t)(c0 + 1) * m] = d1;
            }
        }
    }
    __syncthreads();
    int rp;
    double smax;
    const int r = cta_trunc_svd<NT>(w, m, n, args.eps, 0.0, false, &rp, &smax, DENSE_MAX, nullptr);
    if (threadIdx.x == 0) sh_out = r > 0 ? arena_alloc(args.out_arena, (unsigned long long)(m + n) * r) : nullptr;
    __syncthreads();
    double* out = sh_out;
    if (out) cta_trunc_write<NT>(w, m, n, rp, r, out, m, out + (size_t)m * r, n);
    if (threadIdx.x == 0) {
        Slot& s = args.slots[(size_t)task.prod * args.B + b];
        s.rank = out ? r : 0;
        s.U = out;
        s.V = out ? out + (size_t)m * r : nullptr;
        s.ldu = m;
        s.ldv = n;
        double fsvd = 0, fqr = 0, fgemm = fl_gemm(m, n, k);
        fl_svd(m, n, fsvd, fqr, fgemm);
        add_flops(args.flops, F_SVD, fsvd);
        add_flops(args.flops, F_GEQRF, fqr);
        add_flops(args.flops, F_GEMM, fgemm);
    }
}

// ------------------------------------------------------------------ apply products
struct AllocArgs {
    const AllocTask* tasks;
    int ntasks;
    Slot* slots;
    int B;
    Arena arena;
};

__global__ void k_alloc_apply(AllocArgs args, BatchViews bv) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= args.ntasks * args.B) return;
    const int ti = idx / args.B, b = idx % args.B;
    const AllocTask t = args.tasks[ti];
    Slot s;
    s.pad = 0;
    if (t.kind == P_RK_LEFT) {
        const HView& A = bv.a[b];
        s.rank = A.rank[t.kx];
        s.U = s.rank ? A.U[t.kx] : nullptr;
        s.ldu = t.rows_alias;
        s.ldv = t.rows_out;
        s.V = s.rank ? arena_alloc(args.arena, (unsigned long long)t.rows_out * s.rank) : nullptr;
        if (s.rank && !s.V) s.rank = 0;
    } else {
        const HView& Bv = bv.b[b];
        s.rank = Bv.rank[t.kx];
        s.V = s.rank ? Bv.V[t.kx] : nullptr;
        s.ldv = t.rows_alias;
        s.ldu = t.rows_out;
        s.U = s.rank ? arena_alloc(args.arena, (unsigned long long)t.rows_out * s.rank) : nullptr;
        if (s.rank && !s.U) s.rank = 0;
    }
    args.slots[(size_t)t.prod * args.B + b] = s;
}

struct ApplyArgs {
    const ApplyTask* tasks;
    const ApplyLeaf* leaves;
    Slot* slots;
    int B;
    int nprod;        // T task t of the batch lives in slot (nprod + t)
    const int* x_ld;  // per task: leading dimension of X
    FlopLedger* flops;
};

struct ApplyTArgs {
    const ApplyTTask* tasks;
    Slot* slots;
    int B;
    int nprod;
    Arena arena;
    FlopLedger* flops;
};

// The apply products run on the FP64 tensor cores (mma.sync.m8n8k4.f64, DMMA; fragment layout
// in bqr.cuh), ONE WARP PER (task, plane) ITEM: a CTA holds eight items and strides over the
// grid, so the many rank-0 items of the level-0 couplings cost one slot read each instead of
// a CTA launch.  Operand fragments (8 rows x 4 columns) are read straight from L2/HBM with
// four k-steps of loads in flight; per output element the sum runs over the leaves in DFS
// order and over k-steps of 4 in order, whatever the batch.

// T = In^T X (rank x k) for one Rk leaf, once per (leaf, plane): 8 x 8 tiles of T per warp.
__device__ __forceinline__ void apply_t_item(const ApplyTArgs& args, const BatchViews& bv, const int ti, const int b,
                                             double& fl) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
    const ApplyTTask task = args.tasks[ti];
    Slot& out = args.slots[(size_t)(args.nprod + ti) * args.B + b];
    const Slot s = args.slots[(size_t)task.prod * args.B + b];
    const int k = s.rank;
    const bool trans = task.kind == P_RK_LEFT;
    const HView& H = trans ? bv.b[b] : bv.a[b];
    const int rr = k ? H.rank[task.id] : 0;
    if (rr == 0) {
        if (lane == 0) out.U = nullptr;
        return;
    }
    double* T = nullptr;
    if (lane == 0) {
        T = arena_alloc(args.arena, (unsigned long long)rr * k);
        out.U = T;
        out.rank = rr;
    }
    T = (double*)__shfl_sync(0xffffffffu, (unsigned long long)T, 0);
    if (!T) return;  // arena exhausted: flagged; the slabs skip this leaf
    const double* In = trans ? H.U[task.id] : H.V[task.id];
    const double* X = (trans ? bv.a[b].V[task.kx] : bv.b[b].U[task.kx]) + task.in_off;
    const int L = task.in_len, ldx = task.x_ld;
    const int nti = (rr + 7) >> 3, ntj = (k + 7) >> 3;
    for (int tile = 0; tile < nti * ntj; ++tile) {
        const int t0 = 8 * (tile % nti), c0 = 8 * (tile / nti);
        const bool aok = t0 + g < rr, bok = c0 + g < k;
        const double* ap = In + (size_t)(aok ? t0 + g : 0) * L;   // A[g][t] = In[j + (t0 + g) L]
        const double* bp = X + (size_t)(bok ? c0 + g : 0) * ldx;  // B[t][g] = X[j + (c0 + g) ldx]
        double d0 = 0.0, d1 = 0.0;
        for (int j0 = 0; j0 < L; j0 += 16) {
            double av[4], bw[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = j0 + 4 * q + t4;
                av[q] = (aok && j < L) ? ap[j] : 0.0;
                bw[q] = (bok && j < L) ? bp[j] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (j0 + 4 * q < L) dmma8x8x4(d0, d1, av[q], bw[q]);
        }
        const int tr = t0 + g, tc = c0 + 2 * t4;
        if (tr < rr) {
            if (tc < k) T[tr + (size_t)tc * rr] = d0;
            if (tc + 1 < k) T[tr + (size_t)(tc + 1) * rr] = d1;
        }
    }
    if (lane == 0) fl += 2.0 * rr * L * k;
}

__global__ void __launch_bounds__(NT) k_apply_t(const ApplyTArgs args, const __grid_constant__ BatchViews bv, const int ntasks) {
    const long total = (long)ntasks * args.B;
    double fl = 0;
    for (long w = (long)blockIdx.x * (NT / 32) + (threadIdx.x >> 5); w < total; w += (long)gridDim.x * (NT / 32))
        apply_t_item(args, bv, (int)(w / args.B), (int)(w % args.B), fl);
    if ((threadIdx.x & 31) == 0 && fl > 0) add_flops(args.flops, F_GEMM, fl);
}

// One output slab (<= 64 rows, all k columns) per warp: Y = sum over dense leaves of D (or D^T)
// X plus sum over Rk leaves of Out T, as 8 x 8 tiles of Y accumulated in DMMA fragments.
__device__ __forceinline__ void apply_item(const ApplyArgs& args, const BatchViews& bv, const int ti, const int b,
                                           double& fl) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
    const ApplyTask task = args.tasks[ti];
    const Slot s = args.slots[(size_t)task.prod * args.B + b];
    const int k = s.rank;
    if (k == 0) return;
    const bool trans = task.kind == P_RK_LEFT;
    const HView& H = trans ? bv.b[b] : bv.a[b];
    const double* X = trans ? bv.a[b].V[task.kx] : bv.b[b].U[task.kx];
    const int ldx = args.x_ld[ti];
    double* Y = trans ? s.V : s.U;
    const int ldy = trans ? s.ldv : s.ldu;
    const int r0 = task.r0, nr = task.r1 - task.r0;
    const int nti = (nr + 7) >> 3, ntj = (k + 7) >> 3;
    for (int tile = 0; tile < nti * ntj; ++tile) {
        const int rt = 8 * (tile % nti), c0 = 8 * (tile / nti);
        const int row = r0 + rt + g;  // this lane's A row (slab output space)
        const bool bok = c0 + g < k;
        double d0 = 0.0, d1 = 0.0;
        for (int li = task.lbeg; li < task.lend; ++li) {
            const ApplyLeaf L = args.leaves[li];
            const int out_len = trans ? L.n : L.m;
            const int o0 = max(r0 + rt, L.out_off), o1 = min(min(task.r1, r0 + rt + 8), L.out_off + out_len);
            if (o0 >= o1) continue;  // leaf misses this row tile
            const bool rok = row >= o0 && row < o1;
            const int lr = rok ? row - L.out_off : 0;
            const double* A;   // A[g][t] = A_(row, j) at A + j * ja (+ row offset folded in)
            long ja;
            const double* Bp;  // B[t][g] = contracted (j, column c0 + g) at Bp + j
            int len;
            if (L.kind == K_DENSE) {
                const double* D = H.dense + L.doff;
                len = trans ? L.m : L.n;
                if (!trans) { A = D + lr; ja = L.m; }
                else { A = D + (size_t)lr * L.m; ja = 1; }
                Bp = X + L.in_off + (size_t)(bok ? c0 + g : 0) * ldx;
            } else {
                const Slot ts = args.slots[(size_t)(args.nprod + L.tl) * args.B + b];
                const double* T = ts.U;
                if (!T) continue;
                len = ts.rank;
                A = (trans ? H.V[L.id] : H.U[L.id]) + lr;
                ja = out_len;
                Bp = T + (size_t)(bok ? c0 + g : 0) * len;
            }
            for (int j0 = 0; j0 < len; j0 += 16) {
                double av[4], bw[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int j = j0 + 4 * q + t4;
                    av[q] = (rok && j < len) ? A[(size_t)j * ja] : 0.0;
                    bw[q] = (bok && j < len) ? Bp[j] : 0.0;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (j0 + 4 * q < len) dmma8x8x4(d0, d1, av[q], bw[q]);
            }
            if (lane == 0 && c0 == 0) fl += 2.0 * (o1 - o0) * len * k;
        }
        const int yc = c0 + 2 * t4;
        if (rt + g < nr) {
            if (yc < k) Y[(row) + (size_t)yc * ldy] = d0;
            if (yc + 1 < k) Y[(row) + (size_t)(yc + 1) * ldy] = d1;
        }
    }
}

__global__ void __launch_bounds__(NT) k_apply(const ApplyArgs args, const __grid_constant__ BatchViews bv, const int ntasks) {
    const long total = (long)ntasks * args.B;
    double fl = 0;
    for (long w = (long)blockIdx.x * (NT / 32) + (threadIdx.x >> 5); w < total; w += (long)gridDim.x * (NT / 32))
        apply_item(args, bv, (int)(w / args.B), (int)(w % args.B), fl);
    if ((threadIdx.x & 31) == 0 && fl > 0) add_flops(args.flops, F_GEMM, fl);
}

// ------------------------------------------------------------------ dense-target deposits
struct DepArgs {
    const DepTask* tasks;
    const Part* parts;
    const Slot* slots;
    int B;
    FlopLedger* flops;
};

// Dense-target deposit on the FP64 tensor cores: warp per 8 x 8 tile of the target leaf (tile
// w, w + 8, ... of the leaf's tile grid), the tile held in DMMA accumulator fragments while every
// part is added in part order -- alpha U V^T as k-steps of 4 over the part's rank
// (mma.sync.m8n8k4.f64; alpha = +-1 is applied exactly to the U fragment), exact dense
// products A B likewise over their inner dimension.  U / V / A / B fragments come straight
// from L2 (8 rows x 4 columns per load).
__device__ __forceinline__ void deposit_item(const DepArgs& args, const BatchViews& bv, const int ti, const int b) {
    const DepTask task = args.tasks[ti];
    double* Cd = bv.c[b].dense + task.doff;
    const int m = task.m, n = task.n;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int tm = (m + 7) >> 3, tn = (n + 7) >> 3;
    double fl = 0;
    for (int tile = threadIdx.x >> 5; tile < tm * tn; tile += NT / 32) {
        const int ri = 8 * (tile % tm) + g;          // A-fragment row of this lane
        const int cj = 8 * (tile / tm) + g;          // B-fragment column of this lane
        const int c0 = 8 * (tile / tm) + 2 * t;      // accumulator columns c0, c0 + 1 (row ri)
        const bool rok = ri < m, cok = cj < n;
        double d0 = (rok && c0 < n) ? Cd[ri + (size_t)c0 * m] : 0.0;
        double d1 = (rok && c0 + 1 < n) ? Cd[ri + (size_t)(c0 + 1) * m] : 0.0;
        for (int pi = task.pbeg; pi < task.pend; ++pi) {
            const Part p = args.parts[pi];
            const double* A;
            const double* Bt;  // B fragment source: element (k, col) at Bt[k * bk + col * bc]
            long lda, bk, bc;
            int kk;
            double alpha = p.alpha;
            if (p.src == S_GEMM) {
                A = bv.a[b].dense + p.da;
                lda = m;
                Bt = bv.b[b].dense + p.db;
                bk = 1;
                bc = p.gk;
                kk = p.gk;
            } else {
                const Slot s = args.slots[(size_t)p.id * args.B + b];
                if (s.rank == 0) continue;
                A = s.U + p.u_src;
                lda = s.ldu;
                Bt = s.V + p.v_src;  // V^T: element (k, col) = V[col + k ldv]
                bk = s.ldv;
                bc = 1;
                kk = s.rank;
            }
            for (int k0 = 0; k0 < kk; k0 += 16) {  // four k-steps, fragment loads first
                double av[4], bw[4];
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    const int q = k0 + 4 * s + t;
                    av[s] = (rok && q < kk) ? alpha * A[ri + (size_t)q * lda] : 0.0;
                    bw[s] = (cok && q < kk) ? Bt[(size_t)q * bk + (size_t)cj * bc] : 0.0;
                }
#pragma unroll
                for (int s = 0; s < 4; ++s)
                    if (k0 + 4 * s < kk) dmma8x8x4(d0, d1, av[s], bw[s]);
            }
            if (tile == 0 && lane == 0) fl += 2.0 * m * n * kk;
        }
        if (rok && c0 < n) Cd[ri + (size_t)c0 * m] = d0;
        if (rok && c0 + 1 < n) Cd[ri + (size_t)(c0 + 1) * m] = d1;
    }
    if (threadIdx.x == 0) add_flops(args.flops, F_GEMM, fl);
}

// Grid-stride over (task, plane) items (see item_grid: capped for k_apply_t, whose many
// rank-0 items return at once; one CTA per item for the others).
__global__ void __launch_bounds__(NT) k_deposit(const DepArgs args, const __grid_constant__ BatchViews bv, const int ntasks) {
    const long total = (long)ntasks * args.B;
    for (long w = blockIdx.x; w < total; w += gridDim.x) {
        __syncthreads();  // shared staging of the previous item is no longer read
        deposit_item(args, bv, (int)(w / args.B), (int)(w % args.B));
    }
}

// ------------------------------------------------------------------ dense leaf inversion
struct LuArgs {
    const LuTask* tasks;
    DevError* err;
    unsigned long long call_id;
    FlopLedger* flops;
};

// CTA-wide (NT threads): Out = A^{-1} (n x n, n <= DENSE_MAX; A and Out in global or shared
// memory, ld n) by partial-pivot LU, and the reciprocal condition estimate (CTA-uniform
// return value).  smem: 2 n^2 + n doubles of workspace.  Ends with a barrier.
__device__ double lu_inverse_cta(const double* A, double* Out, const int n, double* smem) {
    __shared__ int piv[DENSE_MAX];
    __shared__ int sh_p;
    __shared__ double sh_rcond;
    __syncthreads();
    double* LU = smem;                 // n x n
    double* Ao = LU + n * n;           // original (for the 1-norm)
    double* vx = Ao + n * n;           // work vector (permutations of the condition estimate)
    for (int e = threadIdx.x; e < n * n; e += NT) {
        LU[e] = A[e];
        Ao[e] = A[e];
    }
    __syncthreads();
    bool zero_pivot = false;
    for (int k = 0; k < n; ++k) {
        if (threadIdx.x < 32) {
            double best = -1;
            int bi = k;
            for (int i = k + threadIdx.x; i < n; i += 32) {
                const double v = fabs(LU[i + k * n]);
                if (v > best) { best = v; bi = i; }
            }
            for (int o = 16; o; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            if (threadIdx.x == 0) { sh_p = bi; piv[k] = bi; }
        }
        __syncthreads();
        const int p = sh_p;
        if (p != k)
            for (int c = threadIdx.x; c < n; c += NT) {
                const double t = LU[k + c * n];
                LU[k + c * n] = LU[p + c * n];
                LU[p + c * n] = t;
            }
        __syncthreads();
        const double d = LU[k + k * n];
        if (d == 0.0) zero_pivot = true;
        if (d != 0.0) {
            for (int i = k + 1 + threadIdx.x; i < n; i += NT) LU[i + k * n] /= d;
            __syncthreads();
            const int rem = n - k - 1;
            for (int e = threadIdx.x; e < rem * rem; e += NT) {
                const int i = k + 1 + e % rem, c = k + 1 + e / rem;
                LU[i + c * n] -= LU[i + k * n] * LU[k + c * n];
            }
        }
        __syncthreads();
    }
    // Row permutation of the pivoting: (P b)[i] = b[perm[i]] (the swaps piv[0..n) in order).
    __shared__ int perm[DENSE_MAX];
    if (threadIdx.x == 0) {
        for (int i = 0; i < n; ++i) perm[i] = i;
        for (int k = 0; k < n; ++k) {
            const int t = perm[k];
            perm[k] = perm[piv[k]];
            perm[piv[k]] = t;
        }
    }
    zero_pivot = false;
    for (int k = 0; k < n; ++k) zero_pivot |= (LU[k + k * n] == 0.0);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned FULL = 0xffffffffu;
    // Warp-parallel triangular solves: lane owns rows lane and lane + 32 (y0, y1); each step
    // broadcasts the finished entry k from its owner lane.  Per element the updates run in
    // the same order as the sequential column-oriented substitution.
    auto own = [&](int k, double y0, double y1) { return __shfl_sync(FULL, k < 32 ? y0 : y1, k & 31); };
    auto lsolve = [&](double& y0, double& y1) {  // L y = y (unit lower)
        for (int k = 0; k < n - 1; ++k) {
            const double xk = own(k, y0, y1);
            if (lane > k && lane < n) y0 = fma(-LU[lane + k * n], xk, y0);
            if (lane + 32 > k && lane + 32 < n) y1 = fma(-LU[lane + 32 + k * n], xk, y1);
        }
    };
    auto usolve = [&](double& y0, double& y1) {  // U y = y
        for (int k = n - 1; k >= 0; --k) {
            if (lane == (k & 31)) {
                if (k < 32) y0 /= LU[k + k * n];
                else y1 /= LU[k + k * n];
            }
            const double xk = own(k, y0, y1);
            if (lane < k) y0 = fma(-LU[lane + k * n], xk, y0);
            if (lane + 32 < k) y1 = fma(-LU[lane + 32 + k * n], xk, y1);
        }
    };
    if (warp == 0) {
        // Hager / Higham 1-norm condition estimate (rcond of Eigen's PartialPivLU), warp 0
        double anorm = 0;
        for (int c = 0; c < n; ++c) {
            double s2 = 0;
            for (int i = lane; i < n; i += 32) s2 += fabs(Ao[i + c * n]);
            s2 = warp_sum(s2);
            anorm = fmax(anorm, s2);
        }
        const bool r0 = lane < n, r1 = lane + 32 < n;
        // The estimate is this kernel's critical path (up to 11 triangular sweeps of n dependent
        // steps on one warp, next to ~5 inverse columns per warp on the others): its sweeps
        // multiply by reciprocal pivots computed once instead of dividing at every step.  Only
        // the estimate (compared with 1e-14) sees the different rounding; the inverse divides.
        const double rd0 = (r0 && !zero_pivot) ? 1.0 / LU[lane + lane * n] : 0.0;
        const double rd1 = (r1 && !zero_pivot) ? 1.0 / LU[lane + 32 + (lane + 32) * n] : 0.0;
        auto usolve_r = [&](double& y0, double& y1) {  // U y = y, reciprocal pivots
            for (int k = n - 1; k >= 0; --k) {
                if (lane == (k & 31)) {
                    if (k < 32) y0 *= rd0;
                    else y1 *= rd1;
                }
                const double xk = own(k, y0, y1);
                if (lane < k) y0 = fma(-LU[lane + k * n], xk, y0);
                if (lane + 32 < k) y1 = fma(-LU[lane + 32 + k * n], xk, y1);
            }
        };
        auto solve = [&](double& y0, double& y1) {  // A x = b: x = U^-1 L^-1 P b
            __syncwarp();
            if (r0) vx[lane] = y0;
            if (r1) vx[lane + 32] = y1;
            __syncwarp();
            y0 = r0 ? vx[perm[lane]] : 0.0;
            y1 = r1 ? vx[perm[lane + 32]] : 0.0;
            lsolve(y0, y1);
            usolve_r(y0, y1);
        };
        auto solve_t = [&](double& y0, double& y1) {  // A^T x = b: x = P^T L^-T U^-T b
            for (int k = 0; k < n; ++k) {  // U^T w = b (forward, column-oriented)
                if (lane == (k & 31)) {
                    if (k < 32) y0 *= rd0;
                    else y1 *= rd1;
                }
                const double xk = own(k, y0, y1);
                if (lane > k && r0) y0 = fma(-LU[k + lane * n], xk, y0);
                if (lane + 32 > k && r1) y1 = fma(-LU[k + (lane + 32) * n], xk, y1);
            }
            for (int k = n - 1; k > 0; --k) {  // L^T v = w (unit upper)
                const double xk = own(k, y0, y1);
                if (lane < k) y0 = fma(-LU[k + lane * n], xk, y0);
                if (lane + 32 < k) y1 = fma(-LU[k + (lane + 32) * n], xk, y1);
            }
            __syncwarp();
            if (r0) vx[perm[lane]] = y0;
            if (r1) vx[perm[lane + 32]] = y1;
            __syncwarp();
            y0 = r0 ? vx[lane] : 0.0;
            y1 = r1 ? vx[lane + 32] : 0.0;
        };
        double rc = 0.0;
        if (anorm > 0 && !zero_pivot) {
            double est = 0;
            double x0 = r0 ? 1.0 / n : 0.0, x1 = r1 ? 1.0 / n : 0.0;  // current probe vector
            for (int it = 0; it < 5; ++it) {
                double z0 = x0, z1 = x1;
                solve(z0, z1);
                const double ny = warp_sum(fabs(z0) + fabs(z1));
                if (it > 0 && ny <= est) break;
                est = ny;
                z0 = r0 ? (z0 >= 0 ? 1.0 : -1.0) : 0.0;
                z1 = r1 ? (z1 >= 0 ? 1.0 : -1.0) : 0.0;
                solve_t(z0, z1);
                // first index of max |z|
                double zmax = fmax(r0 ? fabs(z0) : -1.0, r1 ? fabs(z1) : -1.0);
                int jmax = (r1 && fabs(z1) > (r0 ? fabs(z0) : -1.0)) ? lane + 32 : lane;
                for (int o = 16; o; o >>= 1) {
                    const double ob = __shfl_xor_sync(FULL, zmax, o);
                    const int oj = __shfl_xor_sync(FULL, jmax, o);
                    if (ob > zmax || (ob == zmax && oj < jmax)) {
                        zmax = ob;
                        jmax = oj;
                    }
                }
                const double ztx = warp_sum(z0 * x0 + z1 * x1);
                if (it > 0 && zmax <= ztx) break;
                x0 = (lane == jmax) ? 1.0 : 0.0;
                x1 = (lane + 32 == jmax) ? 1.0 : 0.0;
            }
            auto alt = [&](int i) { return ((i % 2) ? -1.0 : 1.0) * (1.0 + double(i) / (n > 1 ? n - 1 : 1)); };
            double z0 = r0 ? alt(lane) : 0.0, z1 = r1 ? alt(lane + 32) : 0.0;
            solve(z0, z1);
            const double na = warp_sum(fabs(z0) + fabs(z1));
            est = fmax(est, 2.0 * na / (3.0 * n));
            rc = (est > 0 && isfinite(est)) ? 1.0 / (anorm * est) : 0.0;
        }
        if (lane == 0) sh_rcond = rc;
    } else {
        // inverse, warps 1..NT/32-1: column c of A^{-1} = U^-1 L^-1 P e_c
        for (int c = warp - 1; c < n; c += NT / 32 - 1) {
            double* x = Out + (size_t)c * n;
            if (zero_pivot) {
                for (int i = lane; i < n; i += 32) x[i] = 0.0;
                continue;
            }
            double y0 = (lane < n && perm[lane] == c) ? 1.0 : 0.0;
            double y1 = (lane + 32 < n && perm[lane + 32] == c) ? 1.0 : 0.0;
            lsolve(y0, y1);
            usolve(y0, y1);
            if (lane < n) x[lane] = y0;
            if (lane + 32 < n) x[lane + 32] = y1;
        }
    }
    __syncthreads();
    return sh_rcond;
}

// rcond guard of the reference (hmatrix.cpp:485-494): the first failure by (call, plane) wins
__device__ __forceinline__ void lu_report(DevError* err, unsigned long long call_id, int b, double rcond, int rb, int re) {
    if (!(rcond > 1e-14) && threadIdx.x == 0) {
        const unsigned long long key = (call_id << 16) | (unsigned long long)b;
        const unsigned long long prev = atomicMin(&err->key, key);
        if (key < prev) {
            err->code = 2;
            err->rb = rb;
            err->re = re;
            err->rcond = rcond;
        }
    }
}

__global__ void __launch_bounds__(NT) k_lu_inverse(LuArgs args, BatchViews bv) {
    extern __shared__ double smem[];
    const LuTask task = args.tasks[blockIdx.x];
    const int b = blockIdx.y;
    const int n = task.m;
    const double rcond = lu_inverse_cta(bv.a[b].dense + task.doff, bv.c[b].dense + task.doff, n, smem);
    lu_report(args.err, args.call_id, b, rcond, task.rb, task.re);
    if (threadIdx.x == 0) add_flops(args.flops, F_LU, 2.0 * n * n * n);
}

// ------------------------------------------------------------------ scale_walk for dense leaves
struct Sig1Args {
    const long* doff;
    const int* dm;
    const int* dn;
    int nleaf;
    int B;
    double* sig_out;  // [leaf][b]
    FlopLedger* flops;
};

__global__ void __launch_bounds__(NT) k_sigma1_dense(Sig1Args args, BatchViews bv) {
    extern __shared__ double smem[];
    const int leaf = blockIdx.x, b = blockIdx.y;
    const int m = args.dm[leaf], n = args.dn[leaf];
    const double* D = bv.c[b].dense + args.doff[leaf];
    CtaSvdWork w = cta_smem_work(smem, DENSE_MAX, DENSE_MAX);
    w.lda = m;
    for (int e = threadIdx.x; e < m * n; e += NT) w.A[e] = D[e];
    __syncthreads();
    int rp;
    double smax;
    cta_trunc_svd<NT>(w, m, n, 0.0, 0.0, true, &rp, &smax, DENSE_MAX, nullptr);
    if (threadIdx.x == 0) {
        args.sig_out[(size_t)leaf * args.B + b] = smax;
        double fsvd = 0, fqr = 0, fgemm = 0;
        fl_svd(m, n, fsvd, fqr, fgemm);
        add_flops(args.flops, F_SVD, fsvd);
        add_flops(args.flops, F_GEQRF, fqr);
        add_flops(args.flops, F_GEMM, fgemm);
    }
}

// abs_cut[b] = 0.05 * eps * max(sig[.][b])  (recompress, hmatrix.cpp:655-662)
__global__ void k_scale_reduce(const double* sig_d, int nd, const double* sig_k, int nk, int B, double eps,
                               double* abs_cut) {
    const int b = blockIdx.x;
    double s = 0;
    for (int i = threadIdx.x; i < nd; i += blockDim.x) s = fmax(s, sig_d[(size_t)i * B + b]);
    for (int i = threadIdx.x; i < nk; i += blockDim.x) s = fmax(s, sig_k[(size_t)i * B + b]);
    s = warp_max(s);
    __shared__ double red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) m = fmax(m, red[i]);
        abs_cut[b] = m > 0 ? 0.05 * eps * m : -1.0;  // -1: scale 0, leave leaves untouched
    }
}

// ------------------------------------------------------------------ solve: batched H-matvec
// happly / node_apply in the solve (hmatrix.cpp:695-706; acr.cpp:180-229): y = base - H x
// for a batch of (H, x, base, y) items, x and y plane vectors in tree order with nrhs
// columns (ld dim).  HBM-bound: every stored entry of H is read exactly once.
//   phase 1 (k_mv_t):    T_k = V_k^T X[cols of leaf k] (rank x nrhs) once per (Rk leaf, item),
//                        into the transient arena; pointer table [item][leaf] at the arena base.
//   phase 2 (k_mv_slab): per <= 64-row output slab, y = base - sum_dense D X - sum_Rk U_k T_k.
// Per right-hand-side column the arithmetic is a fixed sequence (independent of nrhs and
// of the batch), so multi-RHS solves are bitwise equal to single-RHS ones.
struct MatvecArgs {
    const SlabTask* tasks;
    const ApplyLeaf* leaves;
    const MvLeaf* rk;     // Rk leaves of the root (phase 1)
    int nrk;
    int nbig;             // leading leaves of rk (sorted by decreasing n) with n >= MV1_BIG
    int nrhs;
    int dim;
    Arena arena;          // transient: [count x nrk T pointers | T blocks]
    FlopLedger* flops;
    int tma;              // 1: T blocks in the padded layout of the bulk-copy slab kernel (k_mv_slab_tma)
};
struct MatvecTma {        // extra arguments of k_mv_resolve / k_mv_slab_tma
    int nleaves;          // slab leaf records in total (tasks[ntasks - 1].lend)
    int* rec_cnt;         // resolved records per (item, slab)  [count x ntasks]
    void* rec;            // resolved records (TsMeta)          [count x nleaves], slab t of item b from b * nleaves + tasks[t].lbeg
    const MvCluster* cl;  // leaf clusters (packed-x blocks)
    int ncl;
    long xp_group;        // packed-x doubles per (item, RHS group)
    double* xp;           // packed x  [count][RHS group][xp_group]
};
constexpr int MV_RHS = 16;      // right-hand sides per pass (fixed register slots)

// Leading dimension of a rank-r T block in the padded layout: the smallest value >= r that is
// == 4 (mod 8).  Even (16-byte rows for cp.async.bulk) and conflict-free for the DMMA B
// fragment (lanes (g, t) read T[k + t][rhs g] = g * ld + t: 16 distinct 8-byte banks).
__host__ __device__ __forceinline__ int mv_ldt(int r) { return ((r + 3) & ~7) + 4; }

// Contraction order of a dense leaf whose column count n is a multiple of 32 (both slab kernels):
// position p = 4 s + t (k-step s, DMMA k index t) contracts column mv_col(p, n) = t (n / 4) + s, i.e.
// the four columns of a k-step come from the four quarters of the leaf.  The bulk-copy kernel
// brings such a leaf in as its four quarters (one 8 KB copy each for 64 x 64), padded by 4 doubles
// between quarters, and this order makes its A fragments conflict-free; the packed x block of the
// leaf's column cluster is stored in position order.  Other leaves: p.
__host__ __device__ __forceinline__ int mv_col(int p, int n) { return (p & 3) * (n >> 2) + (p >> 2); }
__host__ __device__ __forceinline__ int mv_pos(int c, int n) { return ((c % (n >> 2)) << 2) | (c / (n >> 2)); }

__device__ __forceinline__ double** mv_tptr(const MatvecArgs& a) { return (double**)a.arena.base; }

// Accumulation order of phase 2 (both slab kernels): every output element keeps FOUR partial
// sums; k-step s (four contracted entries) of the leaf at position i of the slab's leaf list
// goes to partial sum (s + 2 (i & 1)) mod 4, and the result is (p0 + p1) + (p2 + p3).  One DMMA
// chain per output tile would leave the FP64 tensor pipe idle two thirds of the time (its latency
// is far above its issue interval: profiles/r02_ncu_mv_slab_tma.txt); four chains per tile, and a
// different pair for consecutive short (rank <= 8) leaves, keep it fed.
template <int K>
__device__ __forceinline__ void mv_step(double (&acc)[4][4], double a, double b0, double b1) {
    dmma8x8x4(acc[K][0], acc[K][1], a, b0);
    dmma8x8x4(acc[K][2], acc[K][3], a, b1);
}
__device__ __forceinline__ void mv_acc_zero(double (&acc)[4][4]) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[k][i] = 0.0;
}
// element i (0: d00, 1: d01, 2: d10, 3: d11) of the combined accumulator
__device__ __forceinline__ double mv_acc_sum(const double (&acc)[4][4], int i) {
    return (acc[0][i] + acc[1][i]) + (acc[2][i] + acc[3][i]);
}

// Both phases run on the FP64 tensor cores (mma.sync.m8n8k4.f64, DMMA; fragment layout in
// bqr.cuh): the right-hand sides are always 16 zero-padded columns, so every output element
// is the same sequence of DMMA k-steps whatever nrhs is -- multi-RHS solves stay bitwise equal
// to single-RHS ones.
//
// Phase 1, one (item, Rk leaf) per WARP (eight per CTA, no barriers): T^T (16 x rank) =
// X^T (16 x n) V (n x rank), rank tiles of 8, k-steps of 4 rows.  V streams from HBM (each
// load = 8 rank columns x 4 consecutive rows, full 32-byte sectors), X from L2 (units are
// item-major, so the warps in flight share one item's X).
// The Rk leaf list is sorted by decreasing column count; its first nbig leaves (n >= 512) take a
// whole CTA each: the eight warps interleave the leaf's 32-row chunks and their partial T tiles
// are added in warp order (a lone warp streaming an 8192-row factor -- 256 dependent load rounds --
// was the critical path of every launch: ~0.3 ms of floor, 41 launches per solve).
__device__ __forceinline__ void mv_t_chunks(const double* vcol, bool vok, const double* xlo, const double* xhi, bool c_lo, bool c_hi,
                                            int n, int k_first, int k_step, int t4, double& d00, double& d01, double& d10,
                                            double& d11) {
    int k0 = k_first;
    for (; k0 + 32 <= n; k0 += k_step) {  // eight k-steps, loads first
        double va[8], xa[8], xb[8];
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const int j = k0 + 4 * s + t4;
            va[s] = vok ? vcol[j] : 0.0;
            xa[s] = c_lo ? xlo[j] : 0.0;
            xb[s] = c_hi ? xhi[j] : 0.0;
        }
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            dmma8x8x4(d00, d01, xa[s], va[s]);
            dmma8x8x4(d10, d11, xb[s], va[s]);
        }
    }
    // the (< 32-row) tail of the leaf belongs to the chunk sequence of whoever reaches it first
    if (k0 < n && k0 == (n & ~31)) {
        for (; k0 < n; k0 += 4) {
            const int j = k0 + t4;
            const bool jok = j < n;
            const double va = (vok && jok) ? vcol[j] : 0.0;
            dmma8x8x4(d00, d01, (c_lo && jok) ? xlo[j] : 0.0, va);
            dmma8x8x4(d10, d11, (c_hi && jok) ? xhi[j] : 0.0, va);
        }
    }
}

__global__ void __launch_bounds__(NT) k_mv_t(MatvecArgs args, const __grid_constant__ MatvecBatch mb) {
    __shared__ double part[NT / 32][MV_RHS][8];
    __shared__ double* sh_T;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
    const int ld = args.dim;
    const long nbig_ctas = (long)args.nbig * mb.count;
    if ((long)blockIdx.x < nbig_ctas) {
        // ---- one wide leaf per CTA
        const int b = (int)(blockIdx.x / args.nbig), li = (int)(blockIdx.x % args.nbig);
        const MvLeaf L = args.rk[li];
        const HView& H = mb.h[b];
        const int rr = H.rank[L.k];
        const int ldt = args.tma ? mv_ldt(rr) : rr;
        const int ncol = args.tma ? (args.nrhs + MV_RHS - 1) / MV_RHS * MV_RHS : args.nrhs;
        if (threadIdx.x == 0) {
            sh_T = rr > 0 ? arena_alloc(args.arena, (unsigned long long)ldt * ncol) : nullptr;
            mv_tptr(args)[(size_t)b * args.nrk + L.k] = sh_T;
        }
        __syncthreads();
        double* T = sh_T;
        if (T == nullptr) return;
        if (args.tma)
            for (int e = threadIdx.x; e < ldt * ncol; e += NT)
                if (e % ldt >= rr || e / ldt >= args.nrhs) T[e] = 0.0;
        const double* V = H.V[L.k];
        const int n = L.n;
        for (int c0 = 0; c0 < args.nrhs; c0 += MV_RHS) {
            const int nc = min(MV_RHS, args.nrhs - c0);
            const double* X = mb.x[b] + L.in_off + (size_t)c0 * ld;
            const bool c_lo = g < nc, c_hi = g + 8 < nc;
            for (int tc = 0; tc < rr; tc += 8) {
                const bool vok = tc + g < rr;
                double d00 = 0, d01 = 0, d10 = 0, d11 = 0;
                mv_t_chunks(V + (size_t)(vok ? tc + g : 0) * n, vok, X + (size_t)g * ld, X + (size_t)(g + 8) * ld, c_lo, c_hi, n,
                            32 * warp, 32 * (NT / 32), t4, d00, d01, d10, d11);
                // C[g][2 t4 + i]: RHS g (+8), rank tc + 2 t4 + i
                part[warp][g][2 * t4] = d00;
                part[warp][g][2 * t4 + 1] = d01;
                part[warp][g + 8][2 * t4] = d10;
                part[warp][g + 8][2 * t4 + 1] = d11;
                __syncthreads();
                if (threadIdx.x < MV_RHS * 8) {
                    const int c = threadIdx.x >> 3, tr = tc + (threadIdx.x & 7);
                    double sum = part[0][c][threadIdx.x & 7];
#pragma unroll
                    for (int w = 1; w < NT / 32; ++w) sum += part[w][c][threadIdx.x & 7];
                    if (tr < rr && c < nc) T[tr + (size_t)(c0 + c) * ldt] = sum;
                }
                __syncthreads();
            }
        }
        if (threadIdx.x == 0) add_flops(args.flops, F_APPLY, 2.0 * rr * n * args.nrhs);
        return;
    }
    // ---- every other leaf: one (item, leaf) per warp
    const int nsm = args.nrk - args.nbig;
    const long total = (long)nsm * mb.count;
    const long stride = (long)(gridDim.x - nbig_ctas) * (NT / 32);
    double fl = 0;
    for (long w = ((long)blockIdx.x - nbig_ctas) * (NT / 32) + warp; w < total; w += stride) {
        const int b = (int)(w / nsm), li = args.nbig + (int)(w % nsm);
        const MvLeaf L = args.rk[li];
        const HView& H = mb.h[b];
        const int rr = H.rank[L.k];
        double* T = nullptr;
        // T block: rank x nrhs (ld = rank), or -- for the bulk-copy slab kernel -- groups of 16
        // right-hand sides with ld = mv_ldt(rank), pad rows and pad columns zero
        const int ldt = args.tma ? mv_ldt(rr) : rr;
        const int ncol = args.tma ? (args.nrhs + MV_RHS - 1) / MV_RHS * MV_RHS : args.nrhs;
        if (lane == 0) {
            T = rr > 0 ? arena_alloc(args.arena, (unsigned long long)ldt * ncol) : nullptr;
            mv_tptr(args)[(size_t)b * args.nrk + L.k] = T;
        }
        T = (double*)__shfl_sync(0xffffffffu, (unsigned long long)T, 0);
        if (T == nullptr) continue;
        if (args.tma)
            for (int e = lane; e < ldt * ncol; e += 32)
                if (e % ldt >= rr || e / ldt >= args.nrhs) T[e] = 0.0;
        const double* V = H.V[L.k];
        const int n = L.n;
        for (int c0 = 0; c0 < args.nrhs; c0 += MV_RHS) {
            const int nc = min(MV_RHS, args.nrhs - c0);
            const double* X = mb.x[b] + L.in_off + (size_t)c0 * ld;
            const bool c_lo = g < nc, c_hi = g + 8 < nc;  // this lane's A rows (RHS g, g + 8)
            for (int tc = 0; tc < rr; tc += 8) {
                const bool vok = tc + g < rr;  // this lane's B column (rank tc + g)
                double d00 = 0, d01 = 0, d10 = 0, d11 = 0;  // C tiles: RHS 0-7 / 8-15 x rank tc..tc+7
                mv_t_chunks(V + (size_t)(vok ? tc + g : 0) * n, vok, X + (size_t)g * ld, X + (size_t)(g + 8) * ld, c_lo, c_hi, n,
                            0, 32, t4, d00, d01, d10, d11);
                // C[g][2 t4 + i]: RHS g (+8), rank tc + 2 t4 + i  ->  T[rank + rhs * ldt]
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int tr = tc + 2 * t4 + i;
                    if (tr < rr) {
                        if (c_lo) T[tr + (size_t)(c0 + g) * ldt] = i ? d01 : d00;
                        if (c_hi) T[tr + (size_t)(c0 + g + 8) * ldt] = i ? d11 : d10;
                    }
                }
            }
        }
        if (lane == 0) fl += 2.0 * rr * n * args.nrhs;
    }
    if (lane == 0 && fl > 0) add_flops(args.flops, F_APPLY, fl);
}

// Phase 2, one output slab (<= 64 rows) of one item per CTA: warp w owns rows 8w .. 8w+7 and
// all 16 right-hand sides (two 8 x 8 C tiles), so no cross-warp reduction.  The slab's leaf
// records are resolved once into shared memory; the contracted vectors (x chunk or T block)
// of a group of leaves are staged together (one barrier pair per group); each leaf is then
// contracted in DMMA k-steps of 4 with the operand rows streamed from HBM.
constexpr int MV_META = 96;       // leaf records resolved per pass
constexpr int MV_STAGE = 256;     // staged contracted entries per group
constexpr int MV_SLD = MV_STAGE + 4;  // Xs row stride (RHS-major): conflict-light B fragments
struct MvMeta {
    const double* A;    // operand column 0 at row 0 of the leaf (ld lda)
    const double* xin;  // contracted vector, column c at xin + c * ldx
    int len, lda, ldx, o0, o1, out_off;
    int perm;           // dense leaf with len % 32 == 0: contraction in mv_col order
};
__global__ void __launch_bounds__(NT) k_mv_slab(MatvecArgs args, const __grid_constant__ MatvecBatch mb) {
    __shared__ double Xs[MV_RHS * MV_SLD];
    __shared__ MvMeta meta[MV_META];
    const SlabTask task = args.tasks[blockIdx.x];
    const int b = blockIdx.y;
    const HView& H = mb.h[b];
    const double* X = mb.x[b];
    const double* base = mb.base[b];
    double* Y = mb.y[b];
    const int ld = args.dim;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
    const int row = task.r0 + 8 * warp + g;  // this lane's A row
    double* const* Tp = mv_tptr(args) + (size_t)b * args.nrk;
    double fl = 0;
    for (int c0 = 0; c0 < args.nrhs; c0 += MV_RHS) {
        const int nc = min(MV_RHS, args.nrhs - c0);
        double acc[4][4];  // [partial sum][rows 8w+g: RHS 2t4, 2t4+1 (tile 0), 8+2t4, 8+2t4+1 (tile 1)]
        mv_acc_zero(acc);
        for (int l0 = task.lbeg; l0 < task.lend; l0 += MV_META) {
            const int nl = min(MV_META, task.lend - l0);
            __syncthreads();
            if (threadIdx.x < nl) {
                const ApplyLeaf L = args.leaves[l0 + threadIdx.x];
                MvMeta m{nullptr, nullptr, 0, L.m, 0, max(task.r0, L.out_off), min(task.r1, L.out_off + L.m), L.out_off, 0};
                if (m.o0 < m.o1) {
                    if (L.kind == K_DENSE) {
                        m.A = H.dense + L.doff;
                        m.len = L.n;
                        m.perm = (L.n & 31) == 0 && L.n <= 64;
                        m.xin = X + L.in_off + (size_t)c0 * ld;
                        m.ldx = ld;
                    } else {
                        const int rr = H.rank[L.id];
                        const double* T = rr > 0 ? Tp[L.id] : nullptr;
                        if (T) {
                            m.A = H.U[L.id];
                            m.len = rr;
                            m.xin = T + (size_t)c0 * rr;
                            m.ldx = rr;
                        }
                    }
                }
                meta[threadIdx.x] = m;
            }
            __syncthreads();
            int q0 = 0;
            while (q0 < nl) {
                // group [q0, q1) of leaves whose contracted lengths (each rounded up to a k-step
                // of 4) fit MV_STAGE; a longer leaf is its own group, taken in chunks
                int q1 = q0, tot = 0;
                while (q1 < nl && (q1 == q0 || tot + ((meta[q1].len + 3) & ~3) <= MV_STAGE)) tot += (meta[q1++].len + 3) & ~3;
                for (int j0 = 0; j0 < max(tot, 1); j0 += MV_STAGE) {
                    const int jn = min(MV_STAGE, tot - j0);
                    __syncthreads();
                    for (int e = threadIdx.x; e < MV_STAGE * MV_RHS; e += NT) {
                        const int p = e % MV_STAGE, c = e / MV_STAGE;
                        double v = 0.0;
                        if (p < jn && c < nc) {
                            int q = q0, pos = j0 + p;
                            while (pos >= ((meta[q].len + 3) & ~3)) pos -= (meta[q++].len + 3) & ~3;
                            if (pos < meta[q].len) v = meta[q].xin[(meta[q].perm ? mv_col(pos, meta[q].len) : pos) + (size_t)c * meta[q].ldx];
                        }
                        Xs[c * MV_SLD + p] = v;
                    }
                    __syncthreads();
                    int off = 0;  // offset of leaf q's (padded) entries in the concatenation
                    for (int q = q0; q < q1; off += (meta[q].len + 3) & ~3, ++q) {
                        const MvMeta& m = meta[q];
                        const int lo = max(off, j0), hi = min(off + ((m.len + 3) & ~3), j0 + jn);
                        if (lo >= hi) continue;
                        if (8 * warp >= m.o1 - task.r0 || 8 * warp + 8 <= m.o0 - task.r0) continue;  // no rows here
                        const bool rok = row >= m.o0 && row < m.o1;
                        const double* A = m.A + (rok ? row - m.out_off : 0);
                        // B fragment of tile ct: B[k = t4][n = g] = x[j][RHS 8 ct + g]
                        const double* b0 = Xs + (size_t)g * MV_SLD + (off - j0);
                        const double* b1 = Xs + (size_t)(g + 8) * MV_SLD + (off - j0);
                        int j = lo - off;  // a multiple of 16 (leaf start, or a 256-entry chunk of a long leaf)
                        const int je = hi - off;
                        const bool par = ((l0 + q - task.lbeg) & 1) != 0;
                        auto run = [&](auto rot) {
                            constexpr int R = decltype(rot)::value;
                            for (; j + 16 <= je; j += 16) {
                                double a[4];
#pragma unroll
                                for (int s = 0; s < 4; ++s) {
                                    const int jj = j + 4 * s + t4;
                                    a[s] = (rok && jj < m.len) ? A[(size_t)(m.perm ? mv_col(jj, m.len) : jj) * m.lda] : 0.0;
                                }
                                mv_step<(0 + R) & 3>(acc, a[0], b0[j + t4], b1[j + t4]);
                                mv_step<(1 + R) & 3>(acc, a[1], b0[j + 4 + t4], b1[j + 4 + t4]);
                                mv_step<(2 + R) & 3>(acc, a[2], b0[j + 8 + t4], b1[j + 8 + t4]);
                                mv_step<(3 + R) & 3>(acc, a[3], b0[j + 12 + t4], b1[j + 12 + t4]);
                            }
                            if (j < je) {
                                double a[3];
#pragma unroll
                                for (int s = 0; s < 3; ++s) {
                                    const int jj = j + 4 * s + t4;
                                    a[s] = (rok && jj < m.len && j + 4 * s < je) ? A[(size_t)(m.perm ? mv_col(jj, m.len) : jj) * m.lda] : 0.0;
                                }
                                mv_step<(0 + R) & 3>(acc, a[0], b0[j + t4], b1[j + t4]);
                                if (j + 4 < je) mv_step<(1 + R) & 3>(acc, a[1], b0[j + 4 + t4], b1[j + 4 + t4]);
                                if (j + 8 < je) mv_step<(2 + R) & 3>(acc, a[2], b0[j + 8 + t4], b1[j + 8 + t4]);
                            }
                        };
                        if (par) run(std::integral_constant<int, 2>{});
                        else run(std::integral_constant<int, 0>{});
                    }
                }
                if (threadIdx.x == 0 && c0 == 0)
                    for (int q = q0; q < q1; ++q) fl += 2.0 * (meta[q].o1 - meta[q].o0) * meta[q].len * args.nrhs;
                q0 = q1;
            }
        }
        // C[g][2 t4 + i] of tile ct: row 8 warp + g, RHS 8 ct + 2 t4 + i
        const int r = 8 * warp + g;
        if (r < task.r1 - task.r0) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int ca = 2 * t4 + i, cb = 8 + 2 * t4 + i;
                if (ca < nc) {
                    const size_t o = (task.r0 + r) + (size_t)(c0 + ca) * ld;
                    const double s = mv_acc_sum(acc, i);
                    Y[o] = base ? base[o] - s : s;
                }
                if (cb < nc) {
                    const size_t o = (task.r0 + r) + (size_t)(c0 + cb) * ld;
                    const double s = mv_acc_sum(acc, 2 + i);
                    Y[o] = base ? base[o] - s : s;
                }
            }
        }
    }
    if (threadIdx.x == 0) add_flops(args.flops, F_APPLY, fl);
}

// ------------------------------------------------------------------ solve, phase 2 on the bulk-copy engine
// k_mv_slab_tma: the same slab contraction as k_mv_slab (same leaf order, same k-steps, same four
// partial sums per output element: bitwise the same result), fed by TMA bulk copies
// (cp.async.bulk global -> shared, SASS UBLKCP, completion on an mbarrier by transaction bytes)
// instead of per-lane loads.
//   * Persistent CTAs, two per SM (296), walk the (<= 64-row slab, item, RHS group) work items; the
//     stage ring of a CTA runs on across work items, so the next slab is fetched while the current
//     one is contracted.
//   * Warps 0-7 are consumers: warp w owns slab rows 8w .. 8w+7 and all 16 right-hand sides and reads
//     its DMMA fragments from shared memory (every layout below has a leading dimension == 4 mod 16
//     doubles: conflict-free 64-bit fragment loads).
//   * Warps 8-11 are producers.  They stream the slab's 64-byte leaf records, written in list order
//     by k_mv_resolve together with each leaf's place in the ring (stage entry, break flag), and issue
//     the copies: a 64 x 64 (or 32 x 32) dense leaf as its four column quarters (8 KB each), padded
//     by 4 doubles, contracted in mv_col order; the U columns of an Rk leaf as one 512-byte slab
//     segment per column in 68-double slots; the contracted vectors as ONE copy (the packed x block
//     of the leaf's column cluster, or the padded T block of the Rk leaf).  One warp issues a bulk
//     copy only every ~57-90 cycles (tools/tma_bench.cu, profiles/r02_tma_bench.txt), hence four.
//   * A stage holds up to 64 operand column slots and 1152 contracted-vector doubles (up to 16
//     leaves).  Pad columns of a leaf's last k-step hold stale finite operand data (the ring is
//     zeroed once) and multiply zeros of the contracted vector.
//   * Sources or sizes that are not 16-byte aligned (odd cluster sizes) and zero pads of partial RHS
//     groups are written by producer lanes with ordinary stores; a stage that received such stores is
//     fenced (fence.proxy.async) before its next bulk copies.
// Measured at C5 (16 RHS): 20.6 ms against 41.6 ms for the per-lane-load kernel; the limits now are
// the producers' per-copy issue cost for rank-sized U columns and the consumers' DMMA issue rate
// (device counters: acrgpu_profile_report's "#phase mv-slab-tma" line).
constexpr int TS_STAGES = 2;                 // per CTA; two CTAs per SM
constexpr int TS_SLOTS = 64;                 // operand column slots per stage
constexpr int TS_ALD = 68;                   // slot stride in doubles
constexpr int TS_XCAP = 1152;                // contracted-vector doubles per stage
constexpr int TS_XLD = 68;                   // x chunk stride between right-hand sides
constexpr int TS_MAXENT = 16;                // leaves per stage
constexpr int TS_PROD = 4;                   // producer warps (one warp issues a bulk copy every ~57-90 cycles: tools/tma_bench.cu)
constexpr int TS_NT = NT + 32 * TS_PROD;
constexpr int TS_STAGE_DOUBLES = TS_SLOTS * TS_ALD + TS_XCAP;
struct TsEnt {
    short slot, ksteps, xoff, ldx, o0, o1, par, gm;  // par: parity of the leaf's position in the slab's list; gm > 0: the four column quarters of a gm-row dense leaf
};
struct TsDesc {
    int nent, last;
    int dirty;  // acquire count of the last use in which a producer lane wrote stage data with ordinary stores
    int pad1;
    TsEnt ent[TS_MAXENT];
};
enum : unsigned char { TF_GROUPED = 1, TF_PERM = 2, TF_XBLOCK = 4, TF_BRK = 8, TF_WIDE = 16 };
struct TsMeta {        // one resolved, non-empty leaf of a slab with its place in the stage ring (k_mv_resolve -> producers)
    const double* A;   // operand column 0 at leaf row 0 (ld lda)
    const double* xin; // contracted vectors of the first RHS group: packed x block / raw x / padded T block
    int len, lda;      // contracted length (columns / rank), operand leading dimension
    int ldsrc;         // per-RHS copies (raw x, wide T block): source stride between right-hand sides
    int gstride;       // xin stride between RHS groups (doubles)
    TsEnt ent;         // the stage entry, precomputed (wide leaves: o0 / o1 / par only)
    short roff;        // o0's row inside the leaf
    short aslots;      // operand slots taken
    int xneed;         // contracted-vector doubles taken
    unsigned char flags;  // TF_GROUPED: four column quarters; TF_PERM: mv_col order; TF_XBLOCK: one copy brings the vectors;
                          // TF_BRK: commit the open stage first; TF_WIDE: more than TS_SLOTS columns, one stage per piece
    unsigned char pad[7];
};
static_assert(sizeof(TsMeta) == 64, "TsMeta is one 64-byte record");
constexpr size_t TS_SMEM = (size_t)TS_STAGES * TS_STAGE_DOUBLES * sizeof(double) + TS_STAGES * sizeof(TsDesc) +
                           TS_PROD * 32 * sizeof(TsMeta) + 2 * TS_STAGES * sizeof(unsigned long long);

// n doubles global -> shared by one lane: a bulk copy when everything is 16-byte aligned, else scalar
__device__ __forceinline__ bool ts_copy(double* dst, const double* src, int n, unsigned long long* bar, unsigned& tx) {
    if ((((unsigned long long)src | (unsigned long long)smem_u32(dst)) & 15ull) == 0 && (n & 1) == 0) {
        bulk_g2s(dst, src, (unsigned)n * 8u, bar);
        tx += (unsigned)n * 8u;
        return false;
    }
    for (int i = 0; i < n; ++i) dst[i] = src[i];
    return true;  // ordinary stores: the stage's next bulk copies need a proxy fence first
}

// Phase 1.5: one warp per (slab, item) resolves the slab's leaf list against the item's ranks and
// pointers and writes the non-empty leaves as compact 32-byte records, in list order.  The
// producers of k_mv_slab_tma then stream records (one coalesced load per 32 leaves, prefetched)
// instead of chasing record -> rank -> pointer chains, which is what bounded them.
__global__ void __launch_bounds__(NT) k_mv_resolve(MatvecArgs args, const MatvecTma tm, const __grid_constant__ MatvecBatch mb, const int ntasks) {
    const int lane = threadIdx.x & 31;
    const int ngroups = (args.nrhs + MV_RHS - 1) / MV_RHS;
    const long total = (long)ntasks * mb.count;
    const long npack = (long)tm.ncl * mb.count * ngroups;
    const long stride = (long)gridDim.x * (NT / 32);
    for (long w = (long)blockIdx.x * (NT / 32) + (threadIdx.x >> 5); w < total + npack; w += stride) {
        if (w >= total) {
            // pack task: the x entries of one leaf cluster, 16 right-hand sides, in contraction order
            const long u = w - total;
            const MvCluster C = tm.cl[u % tm.ncl];
            const int gi = (int)((u / tm.ncl) % ngroups), b = (int)(u / ((long)tm.ncl * ngroups));
            const double* x = mb.x[b] + C.in_off + (size_t)gi * MV_RHS * args.dim;
            double* dst = tm.xp + ((size_t)b * ngroups + gi) * tm.xp_group + C.xoff;
            const bool perm = (C.n & 31) == 0 && C.n <= 64;
            for (int e = lane; e < MV_RHS * C.ldx; e += 32) {
                const int c = e / C.ldx, pp = e - c * C.ldx;
                const int col = (perm && pp < C.n) ? mv_col(pp, C.n) : pp;
                dst[e] = (pp < C.n && gi * MV_RHS + c < args.nrhs) ? x[col + (size_t)c * args.dim] : 0.0;
            }
            continue;
        }
        const int t = (int)(w % ntasks), b = (int)(w / ntasks);
        const SlabTask task = args.tasks[t];
        const HView& H = mb.h[b];
        double* const* Tp = mv_tptr(args) + (size_t)b * args.nrk;
        TsMeta* out = (TsMeta*)tm.rec + (size_t)b * tm.nleaves + task.lbeg;
        int n = 0;
        // packing state of the stage ring (the producers follow the TF_BRK flags): slots and
        // contracted-vector doubles used and entries in the open stage
        int slots = 0, xs = 0, nent = 0;
        bool have_open = false, force = false;
        for (int l0 = task.lbeg; l0 < task.lend; l0 += 32) {
            TsMeta m{};
            bool ok = false;
            if (l0 + lane < task.lend) {
                const ApplyLeaf L = args.leaves[l0 + lane];
                const int o0 = max(task.r0, L.out_off), o1 = min(task.r1, L.out_off + L.m);
                if (o0 < o1) {
                    m.lda = L.m;
                    m.ent.o0 = (short)(o0 - task.r0);
                    m.ent.o1 = (short)(o1 - task.r0);
                    m.roff = (short)(o0 - L.out_off);
                    m.ent.par = (short)((l0 + lane - task.lbeg) & 1);
                    int dense = 0;
                    if (L.kind == K_DENSE) {
                        m.A = H.dense + L.doff;
                        m.len = L.n;
                        // packed x block of the column cluster (tl < 0: not one leaf cluster -> raw x, per-RHS copies)
                        dense = L.tl >= 0 ? 1 : 2;
                        m.xin = dense == 1 ? tm.xp + (size_t)b * ngroups * tm.xp_group + L.tl : mb.x[b] + L.in_off;
                        m.gstride = dense == 1 ? (int)tm.xp_group : MV_RHS * args.dim;
                        m.ldsrc = args.dim;
                        ok = L.n > 0;
                    } else {
                        const int rr = H.rank[L.id];
                        const double* T = rr > 0 ? Tp[L.id] : nullptr;
                        if (T) {
                            m.A = H.U[L.id];
                            m.len = rr;
                            m.xin = T;
                            m.gstride = MV_RHS * mv_ldt(rr);
                            m.ldsrc = mv_ldt(rr);
                            ok = true;
                        }
                    }
                    if (ok) {
                        const int n4 = (m.len + 3) & ~3;
                        const bool perm = dense && (m.len & 31) == 0 && m.len <= 64;
                        const bool wide = m.len > TS_SLOTS;
                        const bool xblock = dense == 1 || (!dense && !wide);
                        const int ldx = dense == 1 ? n4 + ((20 - (n4 & 15)) & 15) : (xblock ? mv_ldt(m.len) : TS_XLD);
                        const int gs = (m.len >> 2) * m.lda + 4;  // quarter stride
                        const bool grouped = perm && !wide && m.roff == 0 && o1 - o0 == m.lda && (m.lda & 1) == 0 &&
                                             (((unsigned long long)m.A) & 15ull) == 0;
                        m.aslots = (short)(grouped ? (4 * gs + TS_ALD - 1) / TS_ALD : n4);
                        m.xneed = MV_RHS * ldx;
                        m.ent.ksteps = (short)(n4 >> 2);
                        m.ent.ldx = (short)ldx;
                        m.ent.gm = (short)(grouped ? m.lda : 0);
                        m.flags = (grouped ? TF_GROUPED : 0) | (perm ? TF_PERM : 0) | (xblock ? TF_XBLOCK : 0) | (wide ? TF_WIDE : 0);
                    }
                }
            }
            const unsigned mask = __ballot_sync(0xffffffffu, ok);
            // the packing is sequential in list order: walk the batch's non-empty leaves
            for (unsigned rest = mask; rest; rest &= rest - 1) {
                const int i = __ffs(rest) - 1;
                const int as_i = __shfl_sync(0xffffffffu, (int)m.aslots, i), xn_i = __shfl_sync(0xffffffffu, m.xneed, i);
                const bool wide_i = (__shfl_sync(0xffffffffu, (int)m.flags, i) & TF_WIDE) != 0;
                bool brk;
                if (wide_i) {  // every piece takes a stage of its own; the next leaf starts a new one
                    brk = have_open;
                    slots = xs = nent = 0;
                    have_open = true;
                    force = true;
                    if (lane == i && brk) m.flags |= TF_BRK;
                } else {
                    brk = have_open && (force || slots + as_i > TS_SLOTS || xs + xn_i > TS_XCAP || nent == TS_MAXENT);
                    if (brk || !have_open) slots = xs = nent = 0;
                    if (lane == i) {
                        m.ent.slot = (short)slots;
                        m.ent.xoff = (short)xs;
                        if (brk) m.flags |= TF_BRK;
                    }
                    slots += as_i;
                    xs += xn_i;
                    ++nent;
                    have_open = true;
                    force = false;
                }
            }
            if (ok) out[n + __popc(mask & ((1u << lane) - 1u))] = m;
            n += __popc(mask);
        }
        if (lane == 0) tm.rec_cnt[(size_t)b * ntasks + t] = n;
    }
}

__global__ void __launch_bounds__(TS_NT, 2) k_mv_slab_tma(MatvecArgs args, const MatvecTma tm, const __grid_constant__ MatvecBatch mb, const int ntasks) {
    extern __shared__ __align__(128) unsigned char ts_raw[];
    double* stage0 = (double*)ts_raw;
    TsDesc* desc = (TsDesc*)(stage0 + (size_t)TS_STAGES * TS_STAGE_DOUBLES);
    TsMeta* meta_all = (TsMeta*)(desc + TS_STAGES);
    unsigned long long* full = (unsigned long long*)(meta_all + TS_PROD * 32);
    unsigned long long* empty = full + TS_STAGES;
    const int ld = args.dim;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // persistent CTAs: work item w = (RHS group, item, slab), slab fastest (neighbouring CTAs share
    // one item's x in L2); the stage ring runs on across work items, so the producers fetch the
    // next slab while the consumers finish the current one
    const int ngroups = (args.nrhs + MV_RHS - 1) / MV_RHS;
    const long total_work = (long)ntasks * mb.count * ngroups;
    // zeroed once: whatever a pad slot holds later is stale finite matrix data
    for (int e = threadIdx.x; e < TS_STAGES * TS_STAGE_DOUBLES; e += TS_NT) stage0[e] = 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < TS_STAGES; ++s) {
            mbar_init(full + s, TS_PROD);
            mbar_init(empty + s, NT / 32);
            desc[s].dirty = -2 * TS_STAGES;
        }
    }
    fence_proxy_async();
    __syncthreads();
    int stage = 0;
    unsigned phase = 0;
    if (warp >= NT / 32) {
        // ------------------------------------------------ producers: every producer warp runs the same
        // packing (same decisions from the same data); warp pw issues the copies of the columns
        // == pw (mod TS_PROD), warp 0 writes the descriptors and the zero pads
        const int pw = warp - NT / 32;
        TsMeta* meta = meta_all + pw * 32;
        double fl = 0;
        unsigned long long pc_wait = 0, pc_stages = 0, pc_ent = 0, pc_meta = 0, pc_copy = 0, pc_commit = 0, pc_items = 0;
        const unsigned long long pc_t0 = clock64();
        int use = 0;  // stages acquired so far (the same sequence in every producer warp)
        for (long w = blockIdx.x; w < total_work; w += gridDim.x) {
            const SlabTask task = args.tasks[w % ntasks];
            const int b = (int)((w / ntasks) % mb.count);
            const int c0 = (int)(w / ((long)ntasks * mb.count)) * MV_RHS;
            const int nc = min(MV_RHS, args.nrhs - c0);
            int nent = 0;  // entries of the open stage
            unsigned tx = 0;
            bool open = false;  // stage acquired (empty barrier passed)
            double* As = nullptr;
            double* Xs = nullptr;
            auto acquire = [&]() {
                const unsigned long long tw = clock64();
                mbar_wait(empty + stage, phase ^ 1u);
                pc_wait += clock64() - tw;
                ++pc_stages;
                // bulk copies over data this stage received by ordinary stores in its previous use
                // (unaligned copies, zero pads) are ordered behind them by a proxy fence; the common
                // path (aligned leaves, 16 right-hand sides) never needs one
                if (desc[stage].dirty >= use - TS_STAGES) fence_proxy_async();
                ++use;
                As = stage0 + (size_t)stage * TS_STAGE_DOUBLES;
                Xs = As + TS_SLOTS * TS_ALD;
                nent = 0, tx = 0;
                open = true;
            };
            auto commit = [&](int last) {
                const unsigned long long tc0 = clock64();
                if (lane == 0 && pw == 0) {
                    desc[stage].nent = nent;
                    desc[stage].last = last;
                }
                tx = (unsigned)__reduce_add_sync(0xffffffffu, tx);
                __syncwarp();
                if (lane == 0) mbar_arrive_tx(full + stage, tx);
                stage = stage + 1 == TS_STAGES ? 0 : stage + 1;
                phase ^= (stage == 0);
                open = false;
                pc_commit += clock64() - tc0;
            };
            const unsigned long long tm0 = clock64();
            ++pc_items;
            const int nrec = tm.rec_cnt[(size_t)b * ntasks + (int)(w % ntasks)];
            const TsMeta* recs = (const TsMeta*)tm.rec + (size_t)b * tm.nleaves + task.lbeg;
            TsMeta nxt{};
            if (lane < nrec) nxt = recs[lane];
            for (int l0 = 0; l0 < nrec; l0 += 32) {
                const int nl = min(32, nrec - l0);
                __syncwarp();
                meta[lane] = nxt;
                if (l0 + 32 + lane < nrec) nxt = recs[l0 + 32 + lane];  // in flight while this batch is issued
                __syncwarp();
                if (l0 == 0) pc_meta += clock64() - tm0;
                for (int q = 0; q < nl; ++q) {
                    const TsMeta m = meta[q];
                    const int nrow = m.ent.o1 - m.ent.o0;
                    if (lane == 0 && pw == 0 && c0 == 0) fl += 2.0 * nrow * m.len * args.nrhs;
                    const double* xin = m.xin + (size_t)(c0 / MV_RHS) * m.gstride;  // this RHS group's contracted vectors
                    if (!(m.flags & TF_WIDE)) {
                        // the stage entry and its place were computed by k_mv_resolve
                        if ((m.flags & TF_BRK) && open) commit(0);
                        if (!open) acquire();
                        if (lane == 0 && pw == 0) desc[stage].ent[nent] = m.ent;
                        const unsigned long long tk0 = clock64();
                        double* Ad = As + (size_t)m.ent.slot * TS_ALD;
                        if (m.flags & TF_GROUPED) {
                            const int G = pw + TS_PROD * lane, qn = (m.len >> 2) * m.lda;  // quarter G: qn contiguous doubles
                            if (G < 4) ts_copy(Ad + (size_t)G * (qn + 4), m.A + (size_t)G * qn, qn, full + stage, tx);  // aligned (k_mv_resolve)
                        } else if (pw == (int)(pc_ent % TS_PROD)) {
                            // the columns of a per-column leaf (the U columns of an Rk leaf: rank-many 512-byte
                            // copies) are all issued by ONE producer warp, one lane each, and consecutive
                            // leaves go to different warps: the four warps issue in parallel instead of
                            // walking every leaf in lockstep with one or two copies each
                            for (int c = lane; c < m.len; c += 32)
                                if (ts_copy(Ad + (size_t)((m.flags & TF_PERM) ? mv_pos(c, m.len) : c) * TS_ALD + m.ent.o0,
                                            m.A + (size_t)c * m.lda + m.roff, nrow, full + stage, tx))
                                    desc[stage].dirty = use - 1;
                        }
                        double* xd = Xs + m.ent.xoff;
                        if (m.flags & TF_XBLOCK) {
                            const bool xmine = (m.flags & TF_GROUPED) ? (lane == 0 && pw == nent % TS_PROD)
                                                                      : (lane == 31 && pw == (int)(pc_ent % TS_PROD));
                            if (xmine && ts_copy(xd, xin, m.xneed, full + stage, tx)) desc[stage].dirty = use - 1;
                        } else {
                            // raw x of a dense leaf whose columns are not one leaf cluster: per right-hand side
                            const int c = pw + TS_PROD * lane, pslots = 4 * m.ent.ksteps;
                            if (c < MV_RHS) {
                                double* d = xd + (size_t)c * TS_XLD;
                                if (c < nc) {
                                    for (int j = 0; j < m.len; ++j) d[j] = xin[((m.flags & TF_PERM) ? mv_col(j, m.len) : j) + (size_t)c * m.ldsrc];
                                    for (int j = m.len; j < pslots; ++j) d[j] = 0.0;
                                } else {
                                    for (int j = 0; j < pslots; ++j) d[j] = 0.0;
                                }
                                desc[stage].dirty = use - 1;
                            }
                        }
                        pc_copy += clock64() - tk0;
                        ++nent;
                        ++pc_ent;
                    } else {
                        // more than TS_SLOTS columns (an Rk leaf of rank > 64): one stage per piece of 64
                        for (int j0 = 0; j0 < m.len; j0 += TS_SLOTS) {
                            const int plen = min(TS_SLOTS, m.len - j0), pslots = (plen + 3) & ~3;
                            if (open) commit(0);
                            acquire();
                            if (lane == 0 && pw == 0) {
                                TsEnt e{0, (short)(pslots >> 2), 0, (short)TS_XLD, m.ent.o0, m.ent.o1, m.ent.par, 0};
                                desc[stage].ent[0] = e;
                            }
                            for (int c = pw + TS_PROD * lane; c < plen; c += 32 * TS_PROD)
                                if (ts_copy(As + (size_t)c * TS_ALD + m.ent.o0, m.A + (size_t)(j0 + c) * m.lda + m.roff, nrow,
                                            full + stage, tx))
                                    desc[stage].dirty = use - 1;
                            const int c = pw + TS_PROD * lane;
                            if (c < MV_RHS) {
                                double* d = Xs + (size_t)c * TS_XLD;
                                bool wrote = pslots > plen || c >= nc;
                                if (c < nc) {
                                    wrote |= ts_copy(d, xin + j0 + (size_t)c * m.ldsrc, plen, full + stage, tx);
                                    for (int j = plen; j < pslots; ++j) d[j] = 0.0;
                                } else {
                                    for (int j = 0; j < pslots; ++j) d[j] = 0.0;
                                }
                                if (wrote) desc[stage].dirty = use - 1;
                            }
                            nent = 1;
                            ++pc_ent;
                        }
                    }
                }
            }
            if (!open) acquire();
            commit(1);
        }
        if (lane == 0 && pw == 0) {
            add_flops(args.flops, F_APPLY, fl);
            atomicAdd(&g_mv_cyc[4], pc_wait);
            atomicAdd(&g_mv_cyc[5], pc_stages);
            atomicAdd(&g_mv_cyc[6], pc_ent);
            atomicAdd(&g_mv_cyc[7], clock64() - pc_t0);
            atomicAdd(&g_mv_cyc[8], pc_meta);
            atomicAdd(&g_mv_cyc[9], pc_copy);
            atomicAdd(&g_mv_cyc[10], pc_commit);
            atomicAdd(&g_mv_cyc[11], pc_items);
        }
    } else {
        // ------------------------------------------------ consumers
        const int g = lane >> 2, t4 = lane & 3;
        const int r = 8 * warp + g;  // this lane's slab row
        unsigned long long cc_wait = 0, cc_work = 0;
        const unsigned long long cc_t0 = clock64();
        for (long w = blockIdx.x; w < total_work; w += gridDim.x) {
            const SlabTask task = args.tasks[w % ntasks];
            const int b = (int)((w / ntasks) % mb.count);
            const int c0 = (int)(w / ((long)ntasks * mb.count)) * MV_RHS;
            const double* base = mb.base[b];
            double* Y = mb.y[b];
            const int nc = min(MV_RHS, args.nrhs - c0);
            double acc[4][4];  // [partial sum][rows 8w+g: RHS 2t4, 2t4+1 (tile 0), 8+2t4, 8+2t4+1 (tile 1)]
            mv_acc_zero(acc);
            // the base entries of this lane's four outputs, fetched ahead of the contraction
            double bs[4] = {0.0, 0.0, 0.0, 0.0};
            if (base && r < task.r1 - task.r0) {
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int ca = 2 * t4 + i, cb = 8 + 2 * t4 + i;
                    if (ca < nc) bs[i] = base[(task.r0 + r) + (size_t)(c0 + ca) * ld];
                    if (cb < nc) bs[2 + i] = base[(task.r0 + r) + (size_t)(c0 + cb) * ld];
                }
            }
            for (;;) {
                const unsigned long long tw0 = clock64();
                mbar_wait(full + stage, phase);
                const unsigned long long tw1 = clock64();
                cc_wait += tw1 - tw0;
                const double* As = stage0 + (size_t)stage * TS_STAGE_DOUBLES;
                const double* Xs = As + TS_SLOTS * TS_ALD;
                const TsDesc& D = desc[stage];
                const int nent = D.nent, last = D.last;
                for (int e = 0; e < nent; ++e) {
                    const TsEnt E = D.ent[e];
                    if (8 * warp >= E.o1 || 8 * warp + 8 <= E.o0) continue;  // no rows of this warp
                    const bool rok = r >= E.o0 && r < E.o1;
                    // per-column slots: position p at slot p (stride TS_ALD), rows at their slab position;
                    // quarters of a dense leaf: k-step s reads column s of quarter t4 (quarter stride gs)
                    const int gs = E.ksteps * E.gm + 4;
                    const double* A = E.gm ? As + (size_t)E.slot * TS_ALD + (size_t)t4 * gs + (r - E.o0)
                                           : As + (size_t)E.slot * TS_ALD + r + (size_t)t4 * TS_ALD;
                    const int st_u = E.gm ? E.gm : 4 * TS_ALD;  // stride of one k-step
                    const double* b0 = Xs + E.xoff + g * E.ldx + t4;
                    const double* b1 = b0 + 8 * E.ldx;
                    const int ks = E.ksteps;
                    auto run = [&](auto rot) {
                        constexpr int R = decltype(rot)::value;
                        int s = 0;
                        for (; s + 4 <= ks; s += 4) {
                            double a[4], x0[4], x1[4];
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                a[q] = rok ? A[(size_t)(s + q) * st_u] : 0.0;
                                x0[q] = b0[4 * (s + q)];
                                x1[q] = b1[4 * (s + q)];
                            }
                            mv_step<(0 + R) & 3>(acc, a[0], x0[0], x1[0]);
                            mv_step<(1 + R) & 3>(acc, a[1], x0[1], x1[1]);
                            mv_step<(2 + R) & 3>(acc, a[2], x0[2], x1[2]);
                            mv_step<(3 + R) & 3>(acc, a[3], x0[3], x1[3]);
                        }
                        if (s < ks) {
                            double a[3], x0[3], x1[3];
#pragma unroll
                            for (int q = 0; q < 3; ++q) {
                                const bool ok = s + q < ks;
                                a[q] = (rok && ok) ? A[(size_t)(s + q) * st_u] : 0.0;
                                x0[q] = ok ? b0[4 * (s + q)] : 0.0;
                                x1[q] = ok ? b1[4 * (s + q)] : 0.0;
                            }
                            mv_step<(0 + R) & 3>(acc, a[0], x0[0], x1[0]);
                            if (s + 1 < ks) mv_step<(1 + R) & 3>(acc, a[1], x0[1], x1[1]);
                            if (s + 2 < ks) mv_step<(2 + R) & 3>(acc, a[2], x0[2], x1[2]);
                        }
                    };
                    if (E.par) run(std::integral_constant<int, 2>{});
                    else run(std::integral_constant<int, 0>{});
                }
                __syncwarp();
                cc_work += clock64() - tw1;
                if (lane == 0) mbar_arrive(empty + stage);
                stage = stage + 1 == TS_STAGES ? 0 : stage + 1;
                phase ^= (stage == 0);
                if (last) break;
            }
            if (r < task.r1 - task.r0) {
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int ca = 2 * t4 + i, cb = 8 + 2 * t4 + i;
                    if (ca < nc) {
                        const size_t o = (task.r0 + r) + (size_t)(c0 + ca) * ld;
                        const double sv = mv_acc_sum(acc, i);
                        Y[o] = base ? bs[i] - sv : sv;
                    }
                    if (cb < nc) {
                        const size_t o = (task.r0 + r) + (size_t)(c0 + cb) * ld;
                        const double sv = mv_acc_sum(acc, 2 + i);
                        Y[o] = base ? bs[2 + i] - sv : sv;
                    }
                }
            }
        }
        if (threadIdx.x == 0) {
            atomicAdd(&g_mv_cyc[0], 1ull);
            atomicAdd(&g_mv_cyc[1], clock64() - cc_t0);
            atomicAdd(&g_mv_cyc[2], cc_wait);
            atomicAdd(&g_mv_cyc[3], cc_work);
        }
    }
}

// ------------------------------------------------------------------ solve, few right-hand sides
// With 1-4 right-hand sides the DMMA tiles above are mostly padding (16 RHS columns) and the
// per-leaf bookkeeping dominates: C2's leaves are 32 x 32 dense blocks and rank-5 factors.
// The same two phases on the FP64 FMA pipe, one coalesced 256-byte column segment per warp load:
//   phase 1 (k_mv_t1):    warp per (item, Rk leaf); lanes stride the leaf's columns j, eight
//                         rank columns of V per pass, a fixed shuffle tree per rank tile.
//   phase 2 (k_mv_slab1): CTA per (32-row half slab, item), lane = row; the leaves are
//                         flattened into a column table in shared memory and warp kc streams
//                         the columns s = kc (mod 8); the eight partial sums are combined in
//                         warp order.  x / T entries are warp-uniform loads from L1/L2.
// Per right-hand-side column the arithmetic is a fixed sequence, so solves with 1 to 4 columns
// are bitwise equal column by column; the 16-column DMMA path rounds differently (its own
// fixed sequence).
constexpr int MV1_KW = 8;

// lanes end with the warp sum of v[lane & 7]
__device__ __forceinline__ double reduce_scatter8(double (&v)[8], int lane) {
#pragma unroll
    for (int h = 4; h >= 1; h >>= 1) {
        const bool up = (lane & h) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = up ? v[i] : v[i + h];
            const double keep = up ? v[i + h] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
        }
    }
    double s = v[0];
    s += __shfl_xor_sync(0xffffffffu, s, 8);
    s += __shfl_xor_sync(0xffffffffu, s, 16);
    return s;
}

// one rank tile (8 columns of V from column tc) of T = V^T X over the chunks j0 = 32 (c0 + i dc):
// lanes end with the partial sum of rank column tc + (lane & 7), per right-hand side
template <int NR>
__device__ __forceinline__ void mv_t1_tile(const double* Vt, const double* X, int n, int ld, int nt, int nrhs, int c0, int dc,
                                           int lane, double (&out)[NR]) {
    double acc[NR][8];
#pragma unroll
    for (int c = 0; c < NR; ++c)
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[c][u] = 0.0;
#pragma unroll 2
    for (int j0 = 32 * c0; j0 < n; j0 += 32 * dc) {
        const int j = j0 + lane;
        const bool ok = j < n;
        double v[8], xv[NR];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = (ok && u < nt) ? Vt[(size_t)u * n + j] : 0.0;
#pragma unroll
        for (int c = 0; c < NR; ++c) xv[c] = (ok && c < nrhs) ? X[j + (size_t)c * ld] : 0.0;
#pragma unroll
        for (int c = 0; c < NR; ++c)
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[c][u] = fma(v[u], xv[c], acc[c][u]);
    }
#pragma unroll
    for (int c = 0; c < NR; ++c) out[c] = reduce_scatter8(acc[c], lane);
}

// The Rk leaf list is sorted by decreasing column count; the first nbig leaves
// take a whole CTA each (n >= 512): the eight warps interleave the leaf's 32-column chunks and their
// partial sums are added in warp order (a lone warp streaming a 2048-column factor was the
// critical path of the small-batch launches).  Every other leaf takes one warp.
// (threshold applied on the host: Engine::prepare_structure, n >= 512)
constexpr int MV1_RW = 32;  // rank columns per pass of the cooperative path
template <int NR>
__global__ void __launch_bounds__(NT, NR == 1 ? 4 : (NR == 2 ? 3 : 2)) k_mv_t1(MatvecArgs args, const __grid_constant__ MatvecBatch mb) {
    __shared__ double part[NT / 32][MV1_RW][NR];
    __shared__ double* sh_T;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ld = args.dim;
    const long nbig_ctas = (long)args.nbig * mb.count;
    double fl = 0;
    if ((long)blockIdx.x < nbig_ctas) {
        const int b = (int)(blockIdx.x / args.nbig), li = (int)(blockIdx.x % args.nbig);
        const MvLeaf L = args.rk[li];
        const HView& H = mb.h[b];
        const int rr = H.rank[L.k];
        if (threadIdx.x == 0) {
            sh_T = rr > 0 ? arena_alloc(args.arena, (unsigned long long)rr * args.nrhs) : nullptr;
            mv_tptr(args)[(size_t)b * args.nrk + L.k] = sh_T;
        }
        __syncthreads();
        double* T = sh_T;
        if (T == nullptr) return;
        const double* V = H.V[L.k];
        const double* X = mb.x[b] + L.in_off;
        for (int t0 = 0; t0 < rr; t0 += MV1_RW) {
            const int tw = min(MV1_RW, rr - t0);
            for (int tc = 0; tc < tw; tc += 8) {
                const int nt = min(8, tw - tc);
                double sv[NR];
                mv_t1_tile<NR>(V + (size_t)(t0 + tc) * L.n, X, L.n, ld, nt, args.nrhs, warp, NT / 32, lane, sv);
                if (lane < nt) {
#pragma unroll
                    for (int c = 0; c < NR; ++c) part[warp][tc + lane][c] = sv[c];
                }
            }
            __syncthreads();
            for (int e = threadIdx.x; e < tw * NR; e += NT) {
                const int t = e % tw, c = e / tw;
                if (c < args.nrhs) {
                    double sum = part[0][t][c];
#pragma unroll
                    for (int w = 1; w < NT / 32; ++w) sum += part[w][t][c];
                    T[t0 + t + (size_t)c * rr] = sum;
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) add_flops(args.flops, F_APPLY, 2.0 * rr * L.n * args.nrhs);
        return;
    }
    const long nsmall = (long)(args.nrk - args.nbig) * mb.count;
    const long stride = (long)(gridDim.x - nbig_ctas) * (NT / 32);
    for (long w = ((long)blockIdx.x - nbig_ctas) * (NT / 32) + warp; w < nsmall; w += stride) {
        const int nsm = args.nrk - args.nbig;
        const int b = (int)(w / nsm), li = args.nbig + (int)(w % nsm);
        const MvLeaf L = args.rk[li];
        const HView& H = mb.h[b];
        const int rr = H.rank[L.k];
        double* T = nullptr;
        if (lane == 0) {
            T = rr > 0 ? arena_alloc(args.arena, (unsigned long long)rr * args.nrhs) : nullptr;
            mv_tptr(args)[(size_t)b * args.nrk + L.k] = T;
        }
        T = (double*)__shfl_sync(0xffffffffu, (unsigned long long)T, 0);
        if (T == nullptr) continue;
        const double* V = H.V[L.k];
        const double* X = mb.x[b] + L.in_off;
        for (int tc = 0; tc < rr; tc += 8) {
            const int nt = min(8, rr - tc);
            double sv[NR];
            mv_t1_tile<NR>(V + (size_t)tc * L.n, X, L.n, ld, nt, args.nrhs, 0, 1, lane, sv);
#pragma unroll
            for (int c = 0; c < NR; ++c)
                if (lane < nt && c < args.nrhs) T[tc + lane + (size_t)c * rr] = sv[c];
        }
        if (lane == 0) fl += 2.0 * rr * L.n * args.nrhs;
    }
    if (lane == 0 && fl > 0) add_flops(args.flops, F_APPLY, fl);
}

// Phase 2.  The slab's leaves are resolved cooperatively (record, rank, U / T pointers: one
// round of parallel loads) and flattened into a column table in shared memory: entry s = one
// column of one leaf restricted to the slab's rows (pointer to its element at slab row 0,
// valid row range, pointer and stride of the x / T entry it multiplies).  Warp kc then
// streams the columns s = kc (mod 8) for row `lane`, sixteen loads in flight whatever the
// leaf boundaries.
constexpr int MV1_ML = 128;    // leaves per window
constexpr int MV1_KMAX = 1024; // columns per window
struct Mv1Leaf {
    const double* A;    // column 0, slab row 0
    const double* xin;
    int len, lda, ldx, o;  // o = o0 | o1 << 8 (rows relative to the slab)
};
template <int NR>
__global__ void __launch_bounds__(NT) k_mv_slab1(MatvecArgs args, const __grid_constant__ MatvecBatch mb) {
    static_assert(NT == 256 && MV1_KW == NT / 32, "8 warps = 8 column classes; one 32-row group per CTA");
    __shared__ Mv1Leaf meta[MV1_ML];
    __shared__ int pre[MV1_ML + 1];
    __shared__ const double* cA[MV1_KMAX];
    __shared__ const double* cX[MV1_KMAX];
    __shared__ int cLdx[MV1_KMAX];
    __shared__ int cO[MV1_KMAX];
    __shared__ double part[MV1_KW][32][NR];
    // CTA = one 32-row half of a slab (blockIdx.x = 2 slab + half): twice the CTAs per plane
    // for the small batches of the upper levels
    SlabTask task = args.tasks[blockIdx.x >> 1];
    task.r0 += 32 * (int)(blockIdx.x & 1);
    task.r1 = min(task.r1, task.r0 + 32);
    if (task.r0 >= task.r1) return;
    const int b = blockIdx.y;
    const HView& H = mb.h[b];
    const double* X = mb.x[b];
    const double* base = mb.base[b];
    double* Y = mb.y[b];
    const int ld = args.dim;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kc = warp;
    const int rrel = lane;  // this lane's row, relative to the half slab
    const int nrows = task.r1 - task.r0;
    double* const* Tp = mv_tptr(args) + (size_t)b * args.nrk;
    double acc[NR];
#pragma unroll
    for (int c = 0; c < NR; ++c) acc[c] = 0.0;
    double fl = 0;
    for (int l0 = task.lbeg; l0 < task.lend; l0 += MV1_ML) {
        const int nl = min(MV1_ML, task.lend - l0);
        __syncthreads();
        if (threadIdx.x < nl) {
            const ApplyLeaf L = args.leaves[l0 + threadIdx.x];
            Mv1Leaf m{nullptr, nullptr, 0, L.m, 0, 0};
            const int o0 = max(task.r0, L.out_off) - task.r0, o1 = min(task.r1, L.out_off + L.m) - task.r0;
            if (o0 < o1) {
                const double* A = nullptr;
                if (L.kind == K_DENSE) {
                    A = H.dense + L.doff;
                    m.len = L.n;
                    m.xin = X + L.in_off;
                    m.ldx = ld;
                } else {
                    const int rr = H.rank[L.id];
                    const double* T = rr > 0 ? Tp[L.id] : nullptr;
                    if (T) {
                        A = H.U[L.id];
                        m.len = rr;
                        m.xin = T;
                        m.ldx = rr;
                    }
                }
                // element (slab row 0, column 0): leaf row = slab row + r0 - out_off
                m.A = (const double*)((long long)A + 8ll * ((long long)task.r0 - L.out_off));
                m.o = o0 | (o1 << 8);
            }
            meta[threadIdx.x] = m;
        }
        __syncthreads();
        if (warp == 0) {  // exclusive prefix of the leaf lengths
            int v[MV1_ML / 32], run = 0;
#pragma unroll
            for (int i = 0; i < MV1_ML / 32; ++i) {
                const int q = lane * (MV1_ML / 32) + i;
                v[i] = q < nl ? meta[q].len : 0;
                run += v[i];
            }
            int incl = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            int excl = incl - run;
#pragma unroll
            for (int i = 0; i < MV1_ML / 32; ++i) {
                const int q = lane * (MV1_ML / 32) + i;
                if (q <= MV1_ML - 1) pre[q] = excl;
                excl += v[i];
            }
            if (lane == 31) pre[MV1_ML] = incl;
        }
        __syncthreads();
        const int K = pre[MV1_ML];
        for (int k0 = 0; k0 < K; k0 += MV1_KMAX) {
            const int kn = min(MV1_KMAX, K - k0);
            __syncthreads();
            for (int sidx = threadIdx.x; sidx < kn; sidx += NT) {
                const int k = k0 + sidx;
                int lo = 0, hi = MV1_ML - 1;  // last leaf q with pre[q] <= k
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (pre[mid] <= k) lo = mid; else hi = mid - 1;
                }
                const Mv1Leaf& m = meta[lo];
                const int j = k - pre[lo];
                cA[sidx] = m.A + (size_t)j * m.lda;
                cX[sidx] = m.xin + j;
                cLdx[sidx] = m.ldx;
                cO[sidx] = m.o;
                fl += 2.0 * ((m.o >> 8) - (m.o & 0xff)) * args.nrhs;
            }
            __syncthreads();
            {
                for (int s0 = kc; s0 < kn; s0 += MV1_KW * 16) {
                    double a[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        const int sx = s0 + MV1_KW * u;
                        bool ok = sx < kn;
                        const int sc = ok ? sx : 0;
                        const int o = cO[sc];
                        ok = ok && rrel >= (o & 0xff) && rrel < (o >> 8);
                        a[u] = ok ? cA[sc][rrel] : 0.0;
                    }
#pragma unroll
                    for (int c = 0; c < NR; ++c) {
                        if (c < args.nrhs) {
                            double xv[16];
#pragma unroll
                            for (int u = 0; u < 16; ++u) {
                                const int sx = s0 + MV1_KW * u;
                                xv[u] = sx < kn ? cX[sx][(size_t)c * cLdx[sx]] : 0.0;
                            }
#pragma unroll
                            for (int u = 0; u < 16; ++u) acc[c] = fma(a[u], xv[u], acc[c]);
                        }
                    }
                }
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NR; ++c) part[kc][rrel][c] = acc[c];
    __syncthreads();
    if (kc == 0 && rrel < nrows) {
#pragma unroll
        for (int c = 0; c < NR; ++c) {
            if (c < args.nrhs) {
                double sv = part[0][rrel][c];
#pragma unroll
                for (int w = 1; w < MV1_KW; ++w) sv += part[w][rrel][c];
                const size_t o = task.r0 + rrel + (size_t)c * ld;
                Y[o] = base ? base[o] - sv : sv;
            }
        }
    }
    fl = warp_sum(fl);
    if (lane == 0 && fl > 0) add_flops(args.flops, F_APPLY, fl);
}

// ------------------------------------------------------------------ misc kernels
// gather: out[j][r][i] = in[r][j][perm[i]] (to tree order);  scatter: inverse.
__global__ void k_permute_in(const double* in, double* out, const int* perm, int n, int dim, int nrhs) {
    const size_t total = (size_t)n * dim * nrhs;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const int i = e % dim;
        const size_t rest = e / dim;
        const int r = rest % nrhs;
        const int j = rest / nrhs;
        out[e] = in[((size_t)r * n + j) * dim + perm[i]];
    }
}

__global__ void k_permute_out(const double* in, double* out, const int* perm, int n, int dim, int nrhs) {
    const size_t total = (size_t)n * dim * nrhs;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const int i = e % dim;
        const size_t rest = e / dim;
        const int r = rest % nrhs;
        const int j = rest / nrhs;
        out[((size_t)r * n + j) * dim + perm[i]] = in[e];
    }
}

// zero a batch of views: dense slice (dsize doubles) and nk Rk leaves
__global__ void k_zero_views(BatchViews bv, long dsize, int nk) {
    const int b = blockIdx.y;
    const HView& v = bv.c[b];
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < dsize; e += (long)gridDim.x * blockDim.x)
        v.dense[e] = 0.0;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < nk; e += (long)gridDim.x * blockDim.x) {
        v.rank[e] = 0;
        v.U[e] = nullptr;
        v.V[e] = nullptr;
    }
}

// copy a batch of views a -> c (dense data + rank/pointer tables; U/V buffers shared)
__global__ void k_copy_views(BatchViews bv, long dsize, int nk) {
    const int b = blockIdx.y;
    const HView& s = bv.a[b];
    const HView& d = bv.c[b];
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < dsize; e += (long)gridDim.x * blockDim.x)
        d.dense[e] = s.dense[e];
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < nk; e += (long)gridDim.x * blockDim.x) {
        d.rank[e] = s.rank[e];
        d.U[e] = s.U[e];
        d.V[e] = s.V[e];
    }
}

// lift: scatter permuted COO entries into dense leaves (one block of entries per plane)
struct ScatterArgs {
    const int* rows;      // original indices
    const int* cols;
    const double* vals;
    const long* off;      // per batch element: entry range
    const int* iperm;
    const int* leaf_of;   // [rowleaf * nleafclusters + colleaf] -> dense id or -1-rk
    const int* cl_index;  // tree position -> leaf cluster index
    const int* cl_begin;  // leaf cluster -> first tree position
    int ncl;
    const long* d_off;    // dense id -> pool offset
    const int* d_rows;    // dense id -> rows
    const int* d_rb;
    const int* d_cb;
    int* rk_hits;         // count of entries landing in Rk leaves
};

__global__ void k_scatter(ScatterArgs a, BatchViews bv) {
    const int b = blockIdx.y;
    const long s = a.off[b], e = a.off[b + 1];
    double* dense = bv.c[b].dense;
    for (long i = s + blockIdx.x * (long)blockDim.x + threadIdx.x; i < e; i += (long)gridDim.x * blockDim.x) {
        const int r = a.iperm[a.rows[i]], c = a.iperm[a.cols[i]];
        const int lr = a.cl_index[r], lc = a.cl_index[c];
        const int leaf = a.leaf_of[(size_t)lr * a.ncl + lc];
        if (leaf >= 0) {
            const int m = a.d_rows[leaf];
            dense[a.d_off[leaf] + (r - a.d_rb[leaf]) + (size_t)(c - a.d_cb[leaf]) * m] += a.vals[i];
        } else {
            atomicAdd(a.rk_hits, 1);
        }
    }
}

__global__ void k_reset_counter(unsigned long long* ctr) { *ctr = 0; }
__global__ void k_set_counter(unsigned long long* ctr, unsigned long long v) { *ctr = v; }

// Factor compaction: copy every low-rank leaf (U then V) of a batch of stores into
// one exact-size buffer at host-computed offsets and repoint the leaf tables.
__global__ void k_compact(CompactArgs a) {
    const int leaf = blockIdx.x, s = blockIdx.y;
    const long off = a.off[(size_t)s * a.nleaf + leaf];
    if (off < 0) return;
    double** U = a.U[s];
    double** V = a.V[s];
    const int r = a.rank[s][leaf];
    const int m = a.km[leaf], n = a.kn[leaf];
    double* dst = a.base + off;
    const double* u = U[leaf];
    const double* v = V[leaf];
    for (long e = threadIdx.x; e < (long)m * r; e += blockDim.x) dst[e] = u[e];
    for (long e = threadIdx.x; e < (long)n * r; e += blockDim.x) dst[(long)m * r + e] = v[e];
    __syncthreads();
    if (threadIdx.x == 0 && a.repoint) {
        U[leaf] = dst;
        V[leaf] = dst + (long)m * r;
    }
}

__global__ void k_image_fix(ImageFix a) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= a.nk) return;
    const long off = (long)a.buf[a.offs + k];
    const int r = (int)a.buf[a.ranks + k];
    ((int*)(a.buf + a.irank))[k] = r;
    double** U = (double**)(a.buf + a.ptrs);
    double** V = U + a.nk;
    U[k] = off >= 0 ? a.buf + a.lr + off : nullptr;
    V[k] = off >= 0 ? a.buf + a.lr + off + (long)a.km[k] * r : nullptr;
}



// ------------------------------------------------------------------ register-resident small-block kernels
// Shared task plumbing: part ranks, output slot writes, nominal flops.
struct SmallTaskIO {
    __device__ static int total_rank(const TruncArgs& args, const TruncTask& task, int b, const HView& C) {
        int K = 0;
        for (int pi = task.pbeg; pi < task.pend; ++pi) K += resolve_part(args.parts[pi], args.slots, b, args.B, C).rank;
        return K;
    }
    __device__ static void write_out(const TruncArgs& args, const TruncTask& task, int b, const HView& C, int r,
                                     double* U, double* V) {
        if (args.values_only) return;
        if (task.out_kind == 0) {
            Slot& s = args.slots[(size_t)task.out_id * args.B + b];
            s.rank = r;
            s.U = U;
            s.V = V;
            s.ldu = task.m;
            s.ldv = task.n;
        } else {
            C.rank[task.out_id] = r;
            C.U[task.out_id] = U;
            C.V[task.out_id] = V;
        }
    }
    __device__ static void flops(const TruncArgs& args, int m, int n, int K, int r) {
        const int ku = m < K ? m : K, kv = n < K ? n : K;
        double fsvd = 0, fqr, fgemm;
        if (args.values_only) {
            fqr = fl_geqrf(m, K) + fl_geqrf(n, K);
            fgemm = fl_gemm(ku, kv, K);
        } else {
            fqr = fl_geqrf(m, K) + fl_orgqr(m, ku) + fl_geqrf(n, K) + fl_orgqr(n, kv);
            fgemm = fl_gemm(ku, kv, K) + fl_gemm(m, r, ku) + fl_gemm(n, r, kv);
        }
        const double qr_nominal = fqr;
        fl_svd(ku, kv, fsvd, fqr, fgemm);
        add_flops(args.flops, F_SVD, fsvd);
        add_flops(args.flops, F_GEQRF, fqr);
        add_flops(args.flops, F_GEMM, fgemm);
        // the warp engine forms M (2 m n K) instead of the two QRs
        add_flops(args.flops, F_SKIP, fmax(0.0, qr_nominal - fl_gemm(m, n, K)));
    }
    __device__ static RowPart row_part(const Part& p, const PartRes& pr, bool tall) {
        RowPart rp;
        rp.k = pr.rank;
        rp.upper = 0;
        rp.alpha = p.alpha;
        if (tall) {
            rp.P = pr.U; rp.ps = 1; rp.pt = pr.ldu; rp.pd = p.u_dst; rp.pr = p.rows_u;
            rp.Q = pr.V; rp.qs = 1; rp.qt = pr.ldv; rp.qd = p.v_dst; rp.qr = p.rows_v;
        } else {
            rp.P = pr.V; rp.ps = 1; rp.pt = pr.ldv; rp.pd = p.v_dst; rp.pr = p.rows_v;
            rp.Q = pr.U; rp.qs = 1; rp.qt = pr.ldu; rp.qd = p.u_dst; rp.qr = p.rows_u;
        }
        return rp;
    }
};

// ---- blocks <= 32 x 32: one warp per task
// mode 0: truncation task list (TruncArgs); mode 1: dense*dense products (DDArgs).
// Two warps per CTA, one task per warp (rank-revealing QR + Jacobi, svd_rrqr32.cuh).
template <int MODE>
__global__ void __launch_bounds__(64, 6) k_small32(TruncArgs targs, DDArgs dargs, int ntasks, BatchViews bv) {
    __shared__ Warp32Smem smem[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ti = blockIdx.x * 2 + warp;
    if (ti >= ntasks) return;
    Warp32Smem& sm = smem[warp];
    const int b = blockIdx.y;
    const HView& C = bv.c[b];
    int m, n, K;
    double eps, abs_cut = 0.0;
    bool values_only = false;
    TruncTask task{};
    DDTask dt{};
    if (MODE == 0) {
        task = targs.tasks[ti];
        m = task.m;
        n = task.n;
        eps = targs.eps;
        values_only = targs.values_only != 0;
        if (targs.abs_cut) {
            abs_cut = targs.abs_cut[b];
            if (abs_cut < 0) return;
        }
        K = 0;
        if (lane == 0) K = SmallTaskIO::total_rank(targs, task, b, C);
        K = __shfl_sync(0xffffffffu, K, 0);
        if (K == 0) {
            if (lane == 0) {
                SmallTaskIO::write_out(targs, task, b, C, 0, nullptr, nullptr);
                if (values_only) targs.sig_out[(size_t)ti * targs.B + b] = 0.0;
            }
            return;
        }
    } else {
        dt = dargs.tasks[ti];
        m = dt.m;
        n = dt.n;
        K = dt.k;
        eps = dargs.eps;
    }
    unsigned long long wt = clock64();
    if (lane == 0) atomicAdd(&g_w32_cnt, 1ull);
    double a[32], v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] = 0.0;
    if (MODE == 0) {
        double cf[4][4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) cf[i][j][0] = cf[i][j][1] = 0.0;
        for (int pi = task.pbeg; pi < task.pend; ++pi) {
            const Part p = targs.parts[pi];
            const PartRes pr = resolve_part(p, targs.slots, b, targs.B, C);
            if (pr.rank == 0) continue;
            warp_accumulate32_mma(cf, SmallTaskIO::row_part(p, pr, true), sm);
        }
        warp_frags_to_cols(cf, a, sm);
    } else {
        const double* Ad = bv.a[b].dense + dt.da;
        const double* Bd = bv.b[b].dense + dt.db;
        // A zero operand (the off-diagonal dense leaves of the diagonal level-0 couplings E/F)
        // gives a zero product, whose truncation is rank 0: skip the SVD.  The staging of the
        // product sees every entry of A (m x k) and B (k x n), so it doubles as the check.
        const int nz = warp_dd32_mma(a, Ad, Bd, m, dt.k, n, sm);
        if (!__any_sync(0xffffffffu, nz & 1) || !__any_sync(0xffffffffu, nz & 2)) {
            if (lane == 0) {
                Slot& s = dargs.slots[(size_t)dt.prod * dargs.B + b];
                s.rank = 0;
                s.U = nullptr;
                s.V = nullptr;
                s.ldu = m;
                s.ldv = n;
                double fsvd = 0, fqr = 0, fgemm = fl_gemm(m, n, dt.k);  // nominal work of the reference
                fl_svd(m, n, fsvd, fqr, fgemm);
                add_flops(dargs.flops, F_SVD, fsvd);
                add_flops(dargs.flops, F_GEQRF, fqr);
                add_flops(dargs.flops, F_GEMM, fgemm);
                add_flops(dargs.flops, F_SKIP, fsvd + fqr + fgemm);  // not executed
            }
            return;
        }
    }
    // pivot threshold 1e-3 below the cutoff (values-only: sigma_1 to ~1e-10)
    const double drel = values_only ? 1e-10 : 1.8e-4 * eps;
    const double dabs = values_only ? 0.0 : 1.8e-4 * abs_cut;
    w32_mark(0, wt);
    const int rp = warp_rrqr_jacobi32(a, v, m, n, drel, dabs, !values_only, sm, &wt);
    double sig, smax;
    int pos, r;
    warp_sigma_pos32(a, rp, values_only ? 0.0 : eps, abs_cut, sig, pos, r, smax);
    if (MODE == 0 && values_only) {
        if (lane == 0) {
            targs.sig_out[(size_t)ti * targs.B + b] = smax;
            SmallTaskIO::flops(targs, m, n, K, 0);
        }
        return;
    }
    double* out = nullptr;
    if (lane == 0 && r > 0) out = arena_alloc(MODE == 0 ? targs.out_arena : dargs.out_arena, (unsigned long long)(m + n) * r);
    out = (double*)__shfl_sync(0xffffffffu, (unsigned long long)out, 0);
    if (out == nullptr) r = 0;
    w32_mark(3, wt);
    if (r > 0) warp_write32(a, m, n, rp, sig, pos, r, sm, out, out + (size_t)m * r);
    w32_mark(4, wt);
    if (lane == 0) {
        if (MODE == 0) {
            SmallTaskIO::write_out(targs, task, b, C, r, out, out ? out + (size_t)m * r : nullptr);
            SmallTaskIO::flops(targs, m, n, K, r);
        } else {
            Slot& s = dargs.slots[(size_t)dt.prod * dargs.B + b];
            s.rank = r;
            s.U = out;
            s.V = out ? out + (size_t)m * r : nullptr;
            s.ldu = m;
            s.ldv = n;
            double fsvd = 0, fqr = 0, fgemm = fl_gemm(m, n, dt.k);
            fl_svd(m, n, fsvd, fqr, fgemm);
            add_flops(dargs.flops, F_SVD, fsvd);
            add_flops(dargs.flops, F_GEQRF, fqr);
            add_flops(dargs.flops, F_GEMM, fgemm);
        }
    }
}

// ------------------------------------------------------------------ fused leaf-level invert_node
// invert_node (hmatrix.cpp:483-534) of a branch whose four children are dense leaves <= 32:
// X11 = A11^-1;  T12 = X11 A12, T21 = A21 X11;  S = A22 - A21 T12;  X22 = S^-1;
// C12 = -T12 X22, C21 = -X22 T21;  X11 -= T12 C21 -- every product SVD-truncated at the
// arithmetic tolerance before it is added (the reference's dense * dense rule,
// hmatrix.cpp:411-413), as in the unfused plan.  One CTA per plane does the whole node in
// shared memory: the host-driven recursion spends 2 LU launches and 6 mult_adds (~25 dependent
// launches with their stream hand-overs, ~0.85 ms) on each of the dim/64 such nodes of every
// invert chain; here the six truncations (warp engine, T12 || T21 and C12 || C21 on two warps)
// and the two LU inversions run back to back.
struct Inv2Args {
    const Inv2Task* tasks;
    DevError* err;
    unsigned long long call_id;  // call_id: A11's inversion, call_id + 1: the Schur complement's
    double eps;
    FlopLedger* flops;
};

// warp: (Ad (m x k) Bd (k x n)) truncated at eps -> Uo (m x r, ld m), Vo (n x r, ld n); returns r
__device__ int warp_prod_trunc32(const double* Ad, const double* Bd, int m, int k, int n, double eps, Warp32Smem& sm,
                                 double* Uo, double* Vo, FlopLedger* flops) {
    const int lane = threadIdx.x & 31;
    double a[32], v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] = 0.0;
    const int nz = warp_dd32_mma(a, Ad, Bd, m, k, n, sm);
    double fsvd = 0, fqr = 0, fgemm = fl_gemm(m, n, k);  // nominal work of the reference
    fl_svd(m, n, fsvd, fqr, fgemm);
    if (lane == 0) {
        add_flops(flops, F_SVD, fsvd);
        add_flops(flops, F_GEQRF, fqr);
        add_flops(flops, F_GEMM, fgemm);
    }
    if (!__any_sync(0xffffffffu, nz & 1) || !__any_sync(0xffffffffu, nz & 2)) {
        if (lane == 0) add_flops(flops, F_SKIP, fsvd + fqr + fgemm);  // zero operand: rank 0, not executed
        return 0;
    }
    const int rp = warp_rrqr_jacobi32(a, v, m, n, 1.8e-4 * eps, 0.0, true, sm, nullptr);
    double sig, smax;
    int pos, r;
    warp_sigma_pos32(a, rp, eps, 0.0, sig, pos, r, smax);
    if (r > 0) warp_write32(a, m, n, rp, sig, pos, r, sm, Uo, Vo);
    return r;
}

// CTA: C (m x n, ld m) = C0 + alpha U V^T (C0 null: zero; C0 may alias C)
__device__ void cta_lowrank_set(double* C, int m, int n, const double* U, const double* V, int r, double alpha,
                                const double* C0, FlopLedger* flops) {
    for (int e = threadIdx.x; e < m * n; e += NT) {
        const int i = e % m, j = e / m;
        double acc = 0.0;
        for (int t = 0; t < r; ++t) acc = fma(U[i + t * m], V[j + t * n], acc);
        C[e] = fma(alpha, acc, C0 ? C0[e] : 0.0);
    }
    if (threadIdx.x == 0 && r > 0) add_flops(flops, F_GEMM, 2.0 * m * n * r);
}

constexpr int INV2_LU = 2 * 32 * 32 + 32;  // lu_inverse_cta workspace (doubles)
constexpr size_t INV2_SMEM = (INV2_LU + 3 * 1024 + 4 * 1024) * sizeof(double) + 2 * sizeof(Warp32Smem);
__global__ void __launch_bounds__(NT) k_invert2x2(Inv2Args args, BatchViews bv) {
    extern __shared__ double smem[];
    __shared__ int sh_r[2];
    const Inv2Task t = args.tasks[blockIdx.x];
    const int b = blockIdx.y;
    const double* A = bv.a[b].dense;
    double* X = bv.c[b].dense;
    const int m1 = t.m1, m2 = t.m2;
    double* luw = smem;
    double* T12 = luw + INV2_LU;
    double* T21 = T12 + 1024;
    double* S = T21 + 1024;
    double* UV = S + 1024;  // warp w: U at UV + 2048 w, V at UV + 2048 w + 1024
    Warp32Smem* wsm = (Warp32Smem*)(UV + 4096);
    const int warp = threadIdx.x >> 5;
    const double eps = args.eps;
    // X11 = A11^-1
    double rc = lu_inverse_cta(A + t.d11, X + t.d11, m1, luw);
    lu_report(args.err, args.call_id, b, rc, t.rb1, t.re1);
    // T12 = X11 A12 || T21 = A21 X11
    if (warp == 0) {
        const int r = warp_prod_trunc32(X + t.d11, A + t.d12, m1, m1, m2, eps, wsm[0], UV, UV + 1024, args.flops);
        if ((threadIdx.x & 31) == 0) sh_r[0] = r;
    } else if (warp == 1) {
        const int r = warp_prod_trunc32(A + t.d21, X + t.d11, m2, m1, m1, eps, wsm[1], UV + 2048, UV + 3072, args.flops);
        if ((threadIdx.x & 31) == 0) sh_r[1] = r;
    }
    __syncthreads();
    cta_lowrank_set(T12, m1, m2, UV, UV + 1024, sh_r[0], 1.0, nullptr, args.flops);
    cta_lowrank_set(T21, m2, m1, UV + 2048, UV + 3072, sh_r[1], 1.0, nullptr, args.flops);
    __syncthreads();
    // S = A22 - A21 T12
    if (warp == 0) {
        const int r = warp_prod_trunc32(A + t.d21, T12, m2, m1, m2, eps, wsm[0], UV, UV + 1024, args.flops);
        if ((threadIdx.x & 31) == 0) sh_r[0] = r;
    }
    __syncthreads();
    cta_lowrank_set(S, m2, m2, UV, UV + 1024, sh_r[0], -1.0, A + t.d22, args.flops);
    // X22 = S^-1 (lu_inverse_cta starts and ends with a barrier)
    rc = lu_inverse_cta(S, X + t.d22, m2, luw);
    lu_report(args.err, args.call_id + 1, b, rc, t.rb2, t.re2);
    // C12 = -T12 X22 || C21 = -X22 T21
    if (warp == 0) {
        const int r = warp_prod_trunc32(T12, X + t.d22, m1, m2, m2, eps, wsm[0], UV, UV + 1024, args.flops);
        if ((threadIdx.x & 31) == 0) sh_r[0] = r;
    } else if (warp == 1) {
        const int r = warp_prod_trunc32(X + t.d22, T21, m2, m2, m1, eps, wsm[1], UV + 2048, UV + 3072, args.flops);
        if ((threadIdx.x & 31) == 0) sh_r[1] = r;
    }
    __syncthreads();
    cta_lowrank_set(X + t.d12, m1, m2, UV, UV + 1024, sh_r[0], -1.0, nullptr, args.flops);
    cta_lowrank_set(X + t.d21, m2, m1, UV + 2048, UV + 3072, sh_r[1], -1.0, nullptr, args.flops);
    __syncthreads();
    // X11 -= T12 C21
    if (warp == 0) {
        const int r = warp_prod_trunc32(T12, X + t.d21, m1, m2, m1, eps, wsm[0], UV, UV + 1024, args.flops);
        if ((threadIdx.x & 31) == 0) sh_r[0] = r;
    }
    __syncthreads();
    cta_lowrank_set(X + t.d11, m1, m1, UV, UV + 1024, sh_r[0], -1.0, X + t.d11, args.flops);
    if (threadIdx.x == 0) add_flops(args.flops, F_LU, 2.0 * m1 * m1 * m1 + 2.0 * m2 * m2 * m2);
}

// sigma_1 of dense leaves (scale_walk, hmatrix.cpp:630-633), values only; <= 32: one warp per leaf.
__global__ void __launch_bounds__(64) k_sigma1_32(Sig1Args args, BatchViews bv) {
    __shared__ Warp32Smem smem[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int leaf = blockIdx.x * 2 + warp;
    if (leaf >= args.nleaf) return;
    const int b = blockIdx.y;
    const int m = args.dm[leaf], n = args.dn[leaf];
    const double* D = bv.c[b].dense + args.doff[leaf];
    double a[32], v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] = (lane < n && i < m) ? D[i + (size_t)lane * m] : 0.0;
    const int rp = warp_rrqr_jacobi32(a, v, m, n, 1e-10, 0.0, false, smem[warp]);
    double sig, smax;
    int pos, r;
    warp_sigma_pos32(a, rp, 0.0, 0.0, sig, pos, r, smax);
    if (lane == 0) {
        args.sig_out[(size_t)leaf * args.B + b] = smax;
        double fsvd = 0, fqr = 0, fgemm = 0;
        fl_svd(m, n, fsvd, fqr, fgemm);
        add_flops(args.flops, F_SVD, fsvd);
        add_flops(args.flops, F_GEQRF, fqr);
        add_flops(args.flops, F_GEMM, fgemm);
    }
}

// ------------------------------------------------------------------ launchers
static long g_launches = 0;
long launches_take() {
    const long v = g_launches;
    g_launches = 0;
    return v;
}

// Optional per-kernel device timing (ACRGPU_PROFILE=1): CUDA events around each
// launch on the launching stream, folded into per-kernel totals at prof_flush().
struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
    long ctas;
};
static std::vector<ProfRec> g_prof;
// recycled timing events (no create/destroy per launch), per device
static std::map<int, std::vector<cudaEvent_t>> g_ev_pool;
static cudaEvent_t ev_get() {
    int dev = 0;
    cudaGetDevice(&dev);
    auto& pool = g_ev_pool[dev];
    cudaEvent_t e;
    if (!pool.empty()) {
        e = pool.back();
        pool.pop_back();
    } else {
        cudaEventCreate(&e);
    }
    return e;
}
static void ev_put(cudaEvent_t e) {
    int dev = 0;
    cudaGetDevice(&dev);
    g_ev_pool[dev].push_back(e);
}
static std::vector<std::string> g_kernel_names;
static FlopLedger* g_report_ledger = nullptr;  // device ledgers [MAX_KERNELS] of the active context
int kernel_id(const char* name) {
    for (size_t i = 0; i < g_kernel_names.size(); ++i)
        if (g_kernel_names[i] == name) return (int)i;
    g_kernel_names.push_back(name);
    return (int)g_kernel_names.size() - 1;
}
static FlopLedger* ledger(FlopLedger* base, const char* name) {
    if (!base) return nullptr;
    const int id = kernel_id(name);
    return id < MAX_KERNELS ? base + id : base;
}
void set_report_ledger(FlopLedger* l) { g_report_ledger = l; }
static std::map<std::string, double> g_flop_acc;  // folded per-kernel nominal flops
static std::map<std::string, double> g_skip_acc;  // folded per-kernel nominal flops not executed
// Fold the device ledgers into the host accumulators (called before every ledger reset
// and by prof_report), so totals survive across factorizations.
void fold_ledger() {
    if (!g_report_ledger) return;
    std::vector<FlopLedger> led(MAX_KERNELS);
    cudaMemcpy(led.data(), g_report_ledger, MAX_KERNELS * sizeof(FlopLedger), cudaMemcpyDeviceToHost);
    for (size_t id = 0; id < g_kernel_names.size() && id < (size_t)MAX_KERNELS; ++id) {
        double fl = 0;
        for (int c = 0; c < F_NCLASS; ++c) fl += led[id].f[c];
        g_flop_acc[g_kernel_names[id]] += fl;
        g_skip_acc[g_kernel_names[id]] += led[id].f[F_SKIP];
    }
    cudaMemset(g_report_ledger, 0, MAX_KERNELS * sizeof(FlopLedger));
}
static std::map<std::string, std::tuple<double, long, long>> g_prof_acc;  // ms, launches, ctas
// -1: not yet read from ACRGPU_PROFILE; 0 off; 1 every kernel; 2 only the kernels in
// g_prof_sel (ACRGPU_PROFILE=name[,name...] or prof_select): events around the selected
// launches only, so a timed region can carry the dominant kernel's timing without
// paying two event records on every other launch.
static int g_prof_on = -1;
static std::vector<std::string> g_prof_sel;
void prof_select(const char* filter) {
    g_prof_sel.clear();
    if (!filter || !*filter || std::string(filter) == "0") {
        g_prof_on = 0;
        return;
    }
    const std::string f(filter);
    if (f == "1" || f == "*") {
        g_prof_on = 1;
        return;
    }
    size_t a = 0;
    while (a <= f.size()) {
        size_t b = f.find(',', a);
        if (b == std::string::npos) b = f.size();
        if (b > a) g_prof_sel.push_back(f.substr(a, b - a));
        a = b + 1;
    }
    g_prof_on = g_prof_sel.empty() ? 0 : 2;
}
static bool prof_on(const char* name) {
    if (g_prof_on < 0) prof_select(getenv("ACRGPU_PROFILE"));
    if (g_prof_on != 2) return g_prof_on == 1;
    for (const auto& s : g_prof_sel)
        if (s == name) return true;
    return false;
}
ProfScope::ProfScope(cudaStream_t s, const char* n, long c) : st(s), name(n), ctas(c) {
    ++g_launches;
    if (prof_on(n)) {
        a = ev_get();
        cudaEventRecord(a, st);
    }
}
ProfScope::~ProfScope() {
    static const bool dbg = getenv("ACRGPU_DEBUG_SYNC") != nullptr;
    if (dbg) {  // debugging aid: attribute launch / execution errors to the kernel
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            fprintf(stderr, "[acrgpu] %s (%ld CTAs): %s\n", name, ctas, cudaGetErrorString(e));
            abort();
        }
    }
    if (a) {
        cudaEvent_t b = ev_get();
        cudaEventRecord(b, st);
        g_prof.push_back({name, a, b, ctas});
    }
}
static std::vector<std::tuple<float, std::string, long>> g_top;  // slowest launches
void prof_flush() {
    if (g_prof.empty()) return;
    cudaDeviceSynchronize();
    for (auto& r : g_prof) {
        float ms = 0;
        cudaEventElapsedTime(&ms, r.a, r.b);
        g_top.emplace_back(ms, r.name, r.ctas);
        auto& acc = g_prof_acc[r.name];
        std::get<0>(acc) += ms;
        std::get<1>(acc) += 1;
        std::get<2>(acc) += r.ctas;
        ev_put(r.a);
        ev_put(r.b);
    }
    g_prof.clear();
    std::sort(g_top.begin(), g_top.end(), [](const auto& x, const auto& y) { return std::get<0>(x) > std::get<0>(y); });
    if (g_top.size() > 40) g_top.resize(40);
}
std::string prof_report(bool reset) {
    prof_flush();
    fold_ledger();
    std::string out;
    char buf[512];
    for (auto& [k, v] : g_prof_acc) {
        const double fl = g_flop_acc.count(k) ? g_flop_acc[k] : 0.0;
        const double sk = g_skip_acc.count(k) ? g_skip_acc[k] : 0.0;
        snprintf(buf, sizeof(buf), "%s %.3f %ld %ld %.6e %.6e\n", k.c_str(), std::get<0>(v), std::get<1>(v), std::get<2>(v), fl,
                 fl - sk);
        out += buf;
    }
    {
        unsigned long long ph[16], cnt = 0;
        cudaMemcpyFromSymbol(ph, g_phase_cyc, sizeof(ph));
        cudaMemcpyFromSymbol(&cnt, g_phase_cnt, sizeof(cnt));
        snprintf(buf, sizeof(buf), "#phase qr-route tasks %llu: concat %.3g qr %.3g core %.3g svd %.3g write %.3g applyq %.3g (Gcycles)"
                 " avgK %.1f avg_maxdim %.1f core_spill %llu unblocked %llu | bqr: panel %.3g T %.3g update %.3g\n",
                 cnt, ph[0] / 1e9, ph[1] / 1e9, ph[2] / 1e9, ph[3] / 1e9, ph[4] / 1e9, ph[5] / 1e9,
                 cnt ? (double)ph[6] / cnt : 0.0, cnt ? (double)ph[7] / cnt : 0.0, ph[8], ph[9], ph[10] / 1e9,
                 ph[11] / 1e9, ph[12] / 1e9);
        out += buf;
        unsigned long long cc[8];
        cudaMemcpyFromSymbol(cc, g_cta_cyc, sizeof(cc));
        const double cn = cc[0] ? (double)cc[0] : 1.0;
        snprintf(buf, sizeof(buf), "#phase cta-engine tasks %llu (cycles per task): rrqr %.0f jacobi %.0f write %.0f | "
                 "rp %.2f cols %.2f sweeps %.2f\n", cc[0], cc[1] / cn, cc[2] / cn, cc[3] / cn, cc[4] / cn, cc[5] / cn,
                 cc[6] / cn);
        out += buf;
        unsigned long long w[8], wc = 0;
        cudaMemcpyFromSymbol(w, g_w32_cyc, sizeof(w));
        cudaMemcpyFromSymbol(&wc, g_w32_cnt, sizeof(wc));
        const double d = wc ? (double)wc : 1.0;
        snprintf(buf, sizeof(buf), "#phase warp32 tasks %llu (cycles per task): load %.0f qr %.0f jacobi %.0f sigma %.0f "
                 "write %.0f | sweeps %.2f rp %.2f\n", wc, w[0] / d, w[1] / d, w[2] / d, w[3] / d, w[4] / d, w[6] / d, w[7] / d);
        out += buf;
        unsigned long long mv[16];
        cudaMemcpyFromSymbol(mv, g_mv_cyc, sizeof(mv));
        const double mc = mv[0] ? (double)mv[0] : 1.0;
        snprintf(buf, sizeof(buf), "#phase mv-slab-tma CTAs %llu (kcycles per CTA): total %.1f consumer wait %.1f work %.1f | "
                 "producer total %.1f wait-empty %.1f first-records %.1f copy-issue %.1f commit %.1f | stages %.1f entries %.1f "
                 "work items %.1f per CTA\n", mv[0], mv[1] / mc / 1e3, mv[2] / mc / 1e3, mv[3] / mc / 1e3, mv[7] / mc / 1e3,
                 mv[4] / mc / 1e3, mv[8] / mc / 1e3, mv[9] / mc / 1e3, mv[10] / mc / 1e3, mv[5] / mc, mv[6] / mc, mv[11] / mc);
        out += buf;
        if (reset) {
            const unsigned long long z8[8] = {};
            const unsigned long long z16[16] = {};
            cudaMemcpyToSymbol(g_mv_cyc, z16, sizeof(z16));
            cudaMemcpyToSymbol(g_w32_cyc, z8, sizeof(z8));
            cudaMemcpyToSymbol(g_w32_cnt, z8, sizeof(unsigned long long));
            const unsigned long long z[16] = {};
            cudaMemcpyToSymbol(g_phase_cyc, z, sizeof(z));
            cudaMemcpyToSymbol(g_phase_cnt, z, sizeof(unsigned long long));
            cudaMemcpyToSymbol(g_cta_cyc, z8, sizeof(z8));
        }
    }
    for (auto& [ms, name, ctas] : g_top) {
        snprintf(buf, sizeof(buf), "#top %s %.3f %ld\n", name.c_str(), ms, ctas);
        out += buf;
    }
    if (reset) {
        g_prof_acc.clear();
        g_flop_acc.clear();
        g_skip_acc.clear();
        g_top.clear();
    }
    return out;
}

static size_t trunc_smem() { return SMEM_TRUNC; }
constexpr int BIG_DMAX = 128, BIG_RPCAP = 56, BIG_NT = 512;
static size_t trunc_smem_big() {
    return ((size_t)BIG_DMAX * BIG_DMAX + (size_t)BIG_DMAX * BIG_RPCAP + (size_t)BIG_RPCAP * BIG_RPCAP + 5 * BIG_DMAX + 64 +
            BIG_SMEM_EXTRA) * sizeof(double);
}

void setup_kernels() {
    cudaFuncSetAttribute(k_truncate<64, 64, 256, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)trunc_smem());
    cudaFuncSetAttribute(k_truncate<BIG_DMAX, BIG_RPCAP, BIG_NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)trunc_smem_big());
    cudaFuncSetAttribute(k_dd_product, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)trunc_smem());
    cudaFuncSetAttribute(k_invert2x2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)INV2_SMEM);
    cudaFuncSetAttribute(k_lu_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)((2 * DENSE_MAX * DENSE_MAX + 2 * DENSE_MAX) * sizeof(double)));
    cudaFuncSetAttribute(k_sigma1_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)trunc_smem());
    cudaFuncSetAttribute(k_mv_slab_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TS_SMEM);
}

void launch_truncate(cudaStream_t st, int ntasks, const TruncTask* tasks, const Part* parts, Slot* slots, int B,
                     double eps, const double* abs_cut, double* sig_out, bool values_only, Arena out_arena,
                     Arena work, FlopLedger* flops, const BatchViews& bv, const char* name) {
    if (ntasks == 0 || B == 0) return;
    static const int dense_min_k = getenv("ACRGPU_DENSE_MIN_K") ? atoi(getenv("ACRGPU_DENSE_MIN_K")) : 0;
    TruncArgs a{tasks, parts, slots, B, eps, abs_cut, sig_out, values_only ? 1 : 0, out_arena, work,
                ledger(flops, name), dense_min_k};
    ProfScope _ps(st, name, (long)ntasks * B);
    k_truncate<BIG_DMAX, BIG_RPCAP, BIG_NT><<<dim3(ntasks, B), BIG_NT, trunc_smem_big(), st>>>(a, bv);
}

void launch_trunc_small(cudaStream_t st, int nc, int ntasks, const TruncTask* tasks, const Part* parts, Slot* slots,
                        int B, double eps, const double* abs_cut, double* sig_out, bool values_only, Arena out_arena,
                        Arena work, FlopLedger* flops, const BatchViews& bv) {
    if (ntasks == 0 || B == 0) return;
    const char* name = nc == 32 ? "k_trunc_small32" : "k_trunc_mid64";
    TruncArgs a{tasks, parts, slots, B, eps, abs_cut, sig_out, values_only ? 1 : 0, out_arena, work, ledger(flops, name)};
    DDArgs d{};
    ProfScope _ps(st, name, (long)ntasks * B);
    if (nc == 32) k_small32<0><<<dim3((ntasks + 1) / 2, B), 64, 0, st>>>(a, d, ntasks, bv);
    else k_truncate<64, 64, 256, false><<<dim3(ntasks, B), NT, trunc_smem(), st>>>(a, bv);
}

void launch_dd_small(cudaStream_t st, int nc, int ntasks, const DDTask* tasks, Slot* slots, int B, double eps,
                     Arena out_arena, FlopLedger* flops, const BatchViews& bv) {
    if (ntasks == 0 || B == 0) return;
    const char* name = nc == 32 ? "k_dd_small32" : "k_dd_mid64";
    DDArgs d{tasks, slots, B, eps, out_arena, ledger(flops, name)};
    TruncArgs a{};
    ProfScope _ps(st, name, (long)ntasks * B);
    if (nc == 32) k_small32<1><<<dim3((ntasks + 1) / 2, B), 64, 0, st>>>(a, d, ntasks, bv);
    else k_dd_product<<<dim3(ntasks, B), NT, trunc_smem(), st>>>(d, bv);
}

void launch_sigma1_small(cudaStream_t st, int nc, int nleaf, const long* doff, const int* dm, const int* dn, int B,
                         double* sig_out, FlopLedger* flops, const BatchViews& bv) {
    if (nleaf == 0 || B == 0) return;
    const char* name = nc == 32 ? "k_sigma1_32" : "k_sigma1_mid64";
    Sig1Args a{doff, dm, dn, nleaf, B, sig_out, ledger(flops, name)};
    ProfScope _ps(st, name, (long)nleaf * B);
    if (nc == 32) k_sigma1_32<<<dim3((nleaf + 1) / 2, B), 64, 0, st>>>(a, bv);
    else k_sigma1_dense<<<dim3(nleaf, B), NT, trunc_smem(), st>>>(a, bv);
}

// Grid of a grid-stride item kernel: `per_sm` resident CTAs on each of the 148 SMs, four
// rounds of them, never more CTAs than items (per_sm 0: one CTA per item).
static unsigned item_grid(long items, int per_sm) {
    const long cap = per_sm > 0 ? 148L * per_sm * 4 : items;
    return (unsigned)(items < cap ? (items > 0 ? items : 1) : cap);
}

// Grid of a warp-per-item kernel: one warp per item up to 8 resident CTAs of 8 warps on each of
// the 148 SMs (items beyond that are strided).
static unsigned warp_grid(long items) {
    const long ctas = (items + NT / 32 - 1) / (NT / 32);
    const long cap = 148L * 8;
    return (unsigned)(ctas < 1 ? 1 : (ctas < cap ? ctas : cap));
}

void launch_alloc_apply(cudaStream_t st, int ntasks, const AllocTask* tasks, Slot* slots, int B, Arena arena,
                        const BatchViews& bv) {
    if (ntasks == 0 || B == 0) return;
    AllocArgs a{tasks, ntasks, slots, B, arena};
    const int total = ntasks * B;
    ProfScope _ps(st, "k_alloc_apply", (long)((total + 127) / 128));
    k_alloc_apply<<<(total + 127) / 128, 128, 0, st>>>(a, bv);
}

void launch_apply_t(cudaStream_t st, int ntasks, const ApplyTTask* tasks, Slot* slots, int nprod, int B, Arena arena,
                    FlopLedger* flops, const BatchViews& bv) {
    if (ntasks == 0 || B == 0) return;
    ApplyTArgs a{tasks, slots, B, nprod, arena, ledger(flops, "k_apply_t")};
    ProfScope _ps(st, "k_apply_t", (long)ntasks * B);
    k_apply_t<<<warp_grid((long)ntasks * B), NT, 0, st>>>(a, bv, ntasks);
}

void launch_apply(cudaStream_t st, int ntasks, const ApplyTask* tasks, const ApplyLeaf* leaves, const int* x_ld,
                  Slot* slots, int nprod, int B, FlopLedger* flops, const BatchViews& bv) {
    if (ntasks == 0 || B == 0) return;
    ApplyArgs a{tasks, leaves, slots, B, nprod, x_ld, ledger(flops, "k_apply")};
    ProfScope _ps(st, "k_apply", (long)((ntasks)*(B)));
    k_apply<<<warp_grid((long)ntasks * B), NT, 0, st>>>(a, bv, ntasks);
}

void launch_deposit(cudaStream_t st, int ntasks, const DepTask* tasks, const Part* parts, const Slot* slots, int B,
                    FlopLedger* flops, const BatchViews& bv) {
    if (ntasks == 0 || B == 0) return;
    DepArgs a{tasks, parts, slots, B, ledger(flops, "k_deposit")};
    ProfScope _ps(st, "k_deposit", (long)((ntasks)*(B)));
    k_deposit<<<item_grid((long)ntasks * B, 0), NT, 0, st>>>(a, bv, ntasks);
}

void launch_lu(cudaStream_t st, int ntasks, const LuTask* tasks, DevError* err, unsigned long long call_id,
               FlopLedger* flops, const BatchViews& bv, int maxm) {
    if (ntasks == 0 || bv.count == 0) return;
    LuArgs a{tasks, err, call_id, ledger(flops, "k_lu_inverse")};
    const size_t sm = (2 * (size_t)maxm * maxm + 2 * maxm) * sizeof(double);
    ProfScope _ps(st, "k_lu_inverse", (long)((ntasks)*(bv.count)));
    k_lu_inverse<<<dim3(ntasks, bv.count), NT, sm, st>>>(a, bv);
}

void launch_invert2x2(cudaStream_t st, const Inv2Task* task, DevError* err, unsigned long long call_id, double eps,
                      FlopLedger* flops, const BatchViews& bv) {
    if (bv.count == 0) return;
    Inv2Args a{task, err, call_id, eps, ledger(flops, "k_invert2x2")};
    ProfScope _ps(st, "k_invert2x2", (long)bv.count);
    k_invert2x2<<<dim3(1, bv.count), NT, INV2_SMEM, st>>>(a, bv);
}

void launch_scale_reduce(cudaStream_t st, const double* sig_d, int nd, const double* sig_k, int nk, int B, double eps,
                         double* abs_cut) {
    if (B == 0) return;
    ProfScope _ps(st, "k_scale_reduce", (long)(B));
    k_scale_reduce<<<B, 256, 0, st>>>(sig_d, nd, sig_k, nk, B, eps, abs_cut);
}

void launch_matvec(cudaStream_t st, const MatvecPlan& mp, int nrhs, int dim, Arena arena, FlopLedger* flops, const MatvecBatch& mb) {
    const int ntasks = mp.ntasks, nrk = mp.nrk, nbig = mp.nbig;
    if (ntasks == 0 || mb.count == 0) return;
    // > 4 right-hand sides: phase 2 on the bulk-copy engine (ACRGPU_MV_LDG=1: the per-lane load kernel, A/B)
    const char* mv_env = getenv("ACRGPU_MV_LDG");  // read per call: the tests flip it between two solves
    const bool mv_ldg = mv_env && atoi(mv_env) != 0;
    // transient arena: [T pointers: count x nrk] [record counts: count x ntasks ints] [records: count x
    // nleaves x 64 bytes] [packed x: count x RHS groups x xp_group] then the bump-allocated T blocks
    const int ngroups = (nrhs + MV_RHS - 1) / MV_RHS;
    const unsigned long long tbl = ((unsigned long long)mb.count * nrk + 15ull) & ~15ull;
    const unsigned long long cnt_d = (((unsigned long long)mb.count * ntasks + 1) / 2 + 15ull) & ~15ull;
    const unsigned long long rec_d = ((unsigned long long)mb.count * mp.nleaves * (sizeof(TsMeta) / 8) + 15ull) & ~15ull;
    const unsigned long long xp_d = ((unsigned long long)mb.count * ngroups * mp.xp_group + 15ull) & ~15ull;
    const bool tma = nrhs > 4 && !mv_ldg && tbl + cnt_d + rec_d + xp_d < arena.cap / 2;
    MatvecArgs a{mp.tasks, mp.leaves, mp.rk, nrk, nbig, nrhs, dim, arena, ledger(flops, "k_mv_t"), tma ? 1 : 0};
    MatvecTma tm{mp.nleaves, nullptr, nullptr, mp.cl, mp.ncl, mp.xp_group, nullptr};
    if (tma) {
        tm.rec_cnt = (int*)(arena.base + tbl);
        tm.rec = (void*)(arena.base + tbl + cnt_d);
        tm.xp = arena.base + tbl + cnt_d + rec_d;
    }
    {
        ProfScope _ps(st, "k_set_counter", 1);
        k_set_counter<<<1, 1, 0, st>>>(arena.ctr, tma ? tbl + cnt_d + rec_d + xp_d : tbl);
    }
    // 1-4 right-hand sides: FMA-pipe kernels (lane = row / column, no padding);
    // more: 16-column DMMA tiles
    const int nr = nrhs <= 1 ? 1 : (nrhs <= 2 ? 2 : (nrhs <= 4 ? 4 : 0));
    if (nrk > 0) {
        ProfScope _ps(st, "k_mv_t", (long)nrk * mb.count);
        const unsigned grid = (unsigned)((long)nbig * mb.count) +
                              (nr ? warp_grid((long)(nrk - nbig) * mb.count) : item_grid(((long)(nrk - nbig) * mb.count + 7) / 8, 4));
        if (nr == 1) k_mv_t1<1><<<grid, NT, 0, st>>>(a, mb);
        else if (nr == 2) k_mv_t1<2><<<grid, NT, 0, st>>>(a, mb);
        else if (nr == 4) k_mv_t1<4><<<grid, NT, 0, st>>>(a, mb);
        else k_mv_t<<<grid, NT, 0, st>>>(a, mb);
    }
    if (a.tma) {
        const long warps = (long)ntasks * mb.count + (long)mp.ncl * mb.count * ngroups;
        ProfScope _ps(st, "k_mv_resolve", warps);
        k_mv_resolve<<<warp_grid(warps), NT, 0, st>>>(a, tm, mb, ntasks);
    }
    a.flops = ledger(flops, "k_mv_slab");
    ProfScope _ps(st, "k_mv_slab", (long)ntasks * mb.count);
    const dim3 grid(ntasks, mb.count), grid1(2 * ntasks, mb.count);
    if (nr == 1) k_mv_slab1<1><<<grid1, NT, 0, st>>>(a, mb);
    else if (nr == 2) k_mv_slab1<2><<<grid1, NT, 0, st>>>(a, mb);
    else if (nr == 4) k_mv_slab1<4><<<grid1, NT, 0, st>>>(a, mb);
    else if (a.tma) {
        const long work = (long)ntasks * mb.count * ngroups;
        k_mv_slab_tma<<<(unsigned)(work < 296 ? work : 296), TS_NT, TS_SMEM, st>>>(a, tm, mb, ntasks);
    }
    else k_mv_slab<<<grid, NT, 0, st>>>(a, mb);
}
void launch_permute_in(cudaStream_t st, const double* in, double* out, const int* perm, int n, int dim, int nrhs) {
    ProfScope _ps(st, "k_permute_in", (long)(1184));
    k_permute_in<<<1184, 256, 0, st>>>(in, out, perm, n, dim, nrhs);
}

void launch_permute_out(cudaStream_t st, const double* in, double* out, const int* perm, int n, int dim, int nrhs) {
    ProfScope _ps(st, "k_permute_out", (long)(1184));
    k_permute_out<<<1184, 256, 0, st>>>(in, out, perm, n, dim, nrhs);
}

void launch_zero_views(cudaStream_t st, const BatchViews& bv, long dsize, int nk) {
    if (bv.count == 0) return;
    const long work = dsize > nk ? dsize : nk;
    int gx = (int)((work + 255) / 256);
    if (gx > 64) gx = 64;
    if (gx < 1) gx = 1;
    ProfScope _ps(st, "k_zero_views", (long)((gx)*(bv.count)));
    k_zero_views<<<dim3(gx, bv.count), 256, 0, st>>>(bv, dsize, nk);
}

void launch_copy_views(cudaStream_t st, const BatchViews& bv, long dsize, int nk) {
    if (bv.count == 0) return;
    const long work = dsize > nk ? dsize : nk;
    int gx = (int)((work + 255) / 256);
    if (gx > 64) gx = 64;
    if (gx < 1) gx = 1;
    ProfScope _ps(st, "k_copy_views", (long)((gx)*(bv.count)));
    k_copy_views<<<dim3(gx, bv.count), 256, 0, st>>>(bv, dsize, nk);
}

void launch_scatter(cudaStream_t st, const ScatterLaunch& s, const BatchViews& bv) {
    if (bv.count == 0) return;
    ScatterArgs a{s.rows, s.cols, s.vals, s.off, s.iperm, s.leaf_of, s.cl_index, s.cl_begin, s.ncl,
                  s.d_off, s.d_rows, s.d_rb, s.d_cb, s.rk_hits};
    ProfScope _ps(st, "k_scatter", (long)((16)*(bv.count)));
    k_scatter<<<dim3(16, bv.count), 256, 0, st>>>(a, bv);
}

void launch_reset_counter(cudaStream_t st, unsigned long long* ctr) {
    ProfScope _ps(st, "k_reset_counter", (long)(1));
    k_reset_counter<<<1, 1, 0, st>>>(ctr);
}

void launch_image_fix(cudaStream_t st, const ImageFix& a) {
    if (a.nk == 0) return;
    ProfScope _ps(st, "k_image_fix", (long)((a.nk + 127) / 128));
    k_image_fix<<<(a.nk + 127) / 128, 128, 0, st>>>(a);
}

void launch_compact(cudaStream_t st, const CompactArgs& a, int nstores) {
    if (nstores == 0 || a.nleaf == 0) return;
    ProfScope _ps(st, "k_compact", (long)a.nleaf * nstores);
    k_compact<<<dim3(a.nleaf, nstores), 128, 0, st>>>(a);
}

}  // namespace acrgpu
