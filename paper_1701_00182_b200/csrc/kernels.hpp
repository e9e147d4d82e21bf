// Launch wrappers of the sm_100a kernels (kernels.cu); used by engine.cu.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "tasks.hpp"

namespace acrgpu {

constexpr int DENSE_MAX = 64;
constexpr int MAX_KERNELS = 32;             // per-kernel flop ledgers               // dense route / dense leaf limit
// dynamic smem of the 64-class kernels (k_truncate<64,..>, k_dd_product, k_sigma1_dense):
// one cta_smem_work(64, 64) = A, W, J (3 x 64 x 64) + tau/nrm/sig (3 x 64) doubles + perm/order
// (2 x 64) ints.  Sized exactly so that two CTAs fit on one SM.
constexpr size_t SMEM_TRUNC = (3 * 64 * 64 + 3 * 64) * 8 + 2 * 64 * 4 + 64;

struct ScatterLaunch {
    const int* rows;
    const int* cols;
    const double* vals;
    const long* off;
    const int* iperm;
    const int* leaf_of;
    const int* cl_index;
    const int* cl_begin;
    int ncl;
    const long* d_off;
    const int* d_rows;
    const int* d_rb;
    const int* d_cb;
    int* rk_hits;
};

struct CompactArgs {
    double* base;
    const long* off;      // [store][leaf] (-1: rank 0)
    double** const* U;    // per store: U pointer table
    double** const* V;
    int* const* rank;     // per store: rank table
    const int* km;
    const int* kn;
    int nleaf;
    int repoint;          // 1: the stores' U/V tables are redirected to the copies
};
void launch_compact(cudaStream_t st, const CompactArgs& a, int nstores);

// Wire image of one H-matrix (plane-partition exchange): after the bytes arrive,
// rebuild the int rank table and the U/V pointer tables inside the image.
struct ImageFix {
    double* buf;
    int nk;
    long offs, ranks, irank, ptrs, lr;  // section offsets (doubles)
    const int* km;
};
void launch_image_fix(cudaStream_t st, const ImageFix& a);

// Launch accounting (every launch) and, with ACRGPU_PROFILE=1, CUDA events around it on
// the launching stream (per-kernel device time in prof_report).
struct ProfScope {
    cudaStream_t st;
    const char* name;
    long ctas;
    cudaEvent_t a = nullptr;
    ProfScope(cudaStream_t s, const char* n, long c);
    ~ProfScope();
};

// Krylov vector kernels (krylov.cu)
constexpr int KRY_G = 296;  // partial sums per dot product (2 x 148 SMs)
void launch_csr_spmv(cudaStream_t st, const long* ptr, const int* col, const double* val, const double* x,
                     const double* b, double* y, long nrows);
void launch_dot(cudaStream_t st, const double* x, const double* y, long n, double* part, double* out);
void launch_cg_update(cudaStream_t st, double* x, double* r, const double* p, const double* ap, double alpha, long n);
void launch_xpby(cudaStream_t st, double* p, const double* z, double beta, long n);
void launch_vadd(cudaStream_t st, double* x, const double* z, long n);

void setup_kernels();
long launches_take();
std::string prof_report(bool reset);
void prof_select(const char* filter);
void set_report_ledger(FlopLedger* l);
void fold_ledger();
int kernel_id(const char* name);

void launch_truncate(cudaStream_t st, int ntasks, const TruncTask* tasks, const Part* parts, Slot* slots, int B,
                     double eps, const double* abs_cut, double* sig_out, bool values_only, Arena out_arena,
                     Arena work, FlopLedger* flops, const BatchViews& bv, const char* name = "k_truncate");
void launch_trunc_small(cudaStream_t st, int nc, int ntasks, const TruncTask* tasks, const Part* parts, Slot* slots,
                        int B, double eps, const double* abs_cut, double* sig_out, bool values_only, Arena out_arena,
                        Arena work, FlopLedger* flops, const BatchViews& bv);
void launch_dd_small(cudaStream_t st, int nc, int ntasks, const DDTask* tasks, Slot* slots, int B, double eps,
                     Arena out_arena, FlopLedger* flops, const BatchViews& bv);
void launch_sigma1_small(cudaStream_t st, int nc, int nleaf, const long* doff, const int* dm, const int* dn, int B,
                         double* sig_out, FlopLedger* flops, const BatchViews& bv);
void launch_dd(cudaStream_t st, int ntasks, const DDTask* tasks, Slot* slots, int B, double eps, Arena out_arena,
               FlopLedger* flops, const BatchViews& bv);
void launch_alloc_apply(cudaStream_t st, int ntasks, const AllocTask* tasks, Slot* slots, int B, Arena arena,
                        const BatchViews& bv);
void launch_apply_t(cudaStream_t st, int ntasks, const ApplyTTask* tasks, Slot* slots, int nprod, int B, Arena arena,
                    FlopLedger* flops, const BatchViews& bv);
void launch_apply(cudaStream_t st, int ntasks, const ApplyTask* tasks, const ApplyLeaf* leaves, const int* x_ld,
                  Slot* slots, int nprod, int B, FlopLedger* flops, const BatchViews& bv);
void launch_deposit(cudaStream_t st, int ntasks, const DepTask* tasks, const Part* parts, const Slot* slots, int B,
                    FlopLedger* flops, const BatchViews& bv);
void launch_lu(cudaStream_t st, int ntasks, const LuTask* tasks, DevError* err, unsigned long long call_id,
               FlopLedger* flops, const BatchViews& bv, int maxm);
void launch_invert2x2(cudaStream_t st, const Inv2Task* task, DevError* err, unsigned long long call_id, double eps,
                      FlopLedger* flops, const BatchViews& bv);
void launch_scale_reduce(cudaStream_t st, const double* sig_d, int nd, const double* sig_k, int nk, int B, double eps,
                         double* abs_cut);
// Batched solve matvec y = base - H x (two phases, see kernels.cu).  arena: transient
// workspace (reset by the call) for the per-leaf V^T x blocks.
void launch_matvec(cudaStream_t st, const MatvecPlan& mp, int nrhs, int dim, Arena arena, FlopLedger* flops, const MatvecBatch& mb);
void launch_permute_in(cudaStream_t st, const double* in, double* out, const int* perm, int n, int dim, int nrhs);
void launch_permute_out(cudaStream_t st, const double* in, double* out, const int* perm, int n, int dim, int nrhs);
void launch_zero_views(cudaStream_t st, const BatchViews& bv, long dsize, int nk);
void launch_copy_views(cudaStream_t st, const BatchViews& bv, long dsize, int nk);
void launch_scatter(cudaStream_t st, const ScatterLaunch& s, const BatchViews& bv);
void launch_reset_counter(cudaStream_t st, unsigned long long* ctr);

}  // namespace acrgpu
