/*
 * acrgpu.h — C-ABI of the B200-native ACR (Accelerated Cyclic Reduction)
 * hierarchical-matrix factor/solve path.  libacrgpu.so (sm_100a) implements it.
 *
 * Drop-in boundary: these entry points replace the H-matrix-mode bodies of the
 * reference's public API (all paths relative to /root/reference/proj):
 *
 *   acrgpu_factor        <- acr::acr_factor(const BlockTridiagonalSystem&, const AcrConfig&)
 *                           core/include/acr/acr.hpp:222, core/src/acr.cpp:366-384
 *                           (lift_hmatrix acr.cpp:316-333 + factor_impl acr.cpp:146-160)
 *   acrgpu_solve         <- acr::AcrFactorization::solve(const std::vector<Eigen::VectorXd>&) const
 *                           core/include/acr/acr.hpp:205, core/src/acr.cpp:350-352 (solve_impl 180-229);
 *                           nrhs > 1 = one pass for r right-hand sides
 *   acrgpu_stats         <- AcrFactorization::factor_bytes() / inverse_rank_stats()
 *                           acr.hpp:207-209, acr.cpp:231-258
 *   acrgpu_level_info    <- AcrFactorization::level_info()  acr.hpp:210, acr.cpp:260-300
 *   acrgpu_dinv_ranks    <- (test surface) leaf ranks of one stored inverse, rank_stats walk
 *                           core/src/hmatrix.cpp:538-554
 *   acrgpu_structure     <- ClusterTree / BlockClusterTree (core/src/cluster.cpp:39-126):
 *                           permutation + leaf table, for structure parity tests
 *   acrgpu_ctx_* / acrgpu_factor_destroy  <- object lifetimes (value types in the reference)
 *   acrgpu_factor_partitioned / acrgpu_comm_*
 *                        <- acr::execute_parallel_factor(system, plan, config)
 *                           core/include/acr/parallel.hpp:60-61, core/src/parallel.cpp:96-297;
 *                           plane ownership = plan_schedule(n, p) (parallel.cpp:383-405)
 *   acrgpu_messages      <- ParallelRun::ledger records (MessageLedger, parallel.hpp:24-48,
 *                           parallel.cpp:142-161,356-378)
 *
 * Errors map 1:1 onto the reference exception classes (core/include/acr/errors.hpp:10-60):
 *   ACRGPU_E_DIMENSION  DimensionError(plane)        ACRGPU_E_SINGULAR  SingularBlockError(level, plane)
 *   ACRGPU_E_LEAFMEM    LeafMemoryError               ACRGPU_E_USAGE     UsageError
 *   ACRGPU_E_DEVICE     CUDA / device-memory failure (no reference equivalent)
 *
 * System layout: 3n-2 sparse plane blocks in COO form (plane-local indices):
 *   block b in [0, n)        : D(b)
 *   block b in [n, 2n-1)     : E(j), j = b-n+1   (couples plane j to plane j-1; block.hpp:79-80)
 *   block b in [2n-1, 3n-2)  : F(j), j = b-2n+1  (couples plane j to plane j+1)
 *   block b owns entries [blk_off[b], blk_off[b+1]) of rows/cols/vals; duplicates are summed
 *   (PlaneBlock, core/src/block.cpp:7-29).  coords: 2*dim doubles (x0,y0,x1,y1,...) of the
 *   plane points, used for geometric clustering (one cluster tree shared by all blocks).
 * Vectors: f / u are [nrhs][n][dim] doubles, original (unpermuted) ordering.
 *
 * Ownership: caller owns every host buffer; the library owns device memory behind the
 * opaque handles until *_destroy.  A factor handle is immutable after acrgpu_factor;
 * solves on one handle are serialised on the context stream.  No callbacks.
 */
#ifndef ACRGPU_H
#define ACRGPU_H

#ifdef __cplusplus
extern "C" {
#endif

enum {
    ACRGPU_OK = 0,
    ACRGPU_E_DIMENSION = 1,
    ACRGPU_E_SINGULAR = 2,
    ACRGPU_E_LEAFMEM = 3,
    ACRGPU_E_USAGE = 4,
    ACRGPU_E_DEVICE = 5,
    ACRGPU_E_INDEFINITE = 6,   /* IndefiniteError (pcg: nonpositive curvature) */
    ACRGPU_E_DIVERGENCE = 7,   /* DivergenceError (iterative refinement) */
    ACRGPU_E_INTERNAL = 9
};

/* AcrConfig (core/include/acr/acr.hpp:15-23), H-matrix mode. */
typedef struct acrgpu_config {
    double eps;             /* truncation tolerance (arithmetic runs at eps*0.5, acr.hpp:178-181) */
    double eta;             /* admissibility parameter */
    int leaf_size;          /* cluster-tree leaf size (<= 64 on the GPU path) */
    int weak;               /* 0 = Admissibility::Standard, 1 = Admissibility::Weak */
    int stop_planes;        /* remaining plane count at which reduction stops (>= 1) */
    long leaf_memory_cap;   /* bytes per materialised leaf (hmatrix.hpp:60) */
    int flags;              /* ACRGPU_F_* below */
} acrgpu_config;

/* Deliberate, documented deviation switch: dense*dense leaf products that land
 * in dense target leaves are added exactly (GEMM) instead of SVD-truncated first
 * (reference quirk, hmatrix.cpp:411-413).  Off by default (reference semantics). */
#define ACRGPU_F_EXACT_DENSE_PRODUCTS 1

typedef struct acrgpu_error {
    int code;
    int level;       /* SingularBlockError level (-1 if n/a) */
    int plane;       /* SingularBlockError / DimensionError plane (-1 if n/a) */
    int row_begin;   /* failing dense pivot rows (tree order), -1 if n/a */
    int row_end;
    char msg[256];
} acrgpu_error;

typedef struct acrgpu_system {
    int n;                  /* plane count */
    int dim;                /* unknowns per plane */
    const double* coords;   /* 2*dim */
    const long* blk_off;    /* 3n-1 */
    const int* rows;
    const int* cols;
    const double* vals;
} acrgpu_system;

typedef struct acrgpu_rankstats {  /* RankStats (hmatrix.hpp:26-32) over stored inverses */
    double average_rank;
    int largest_rank;
    int dense_leaf_count;
    int lowrank_leaf_count;
    long inverse_bytes;
    long factor_bytes;             /* AcrFactorization::factor_bytes (acr.cpp:231-248) */
} acrgpu_rankstats;

typedef struct acrgpu_levelinfo {  /* LevelInfo (acr.hpp:185-192) */
    int level;
    int plane_count;
    int eliminated;
    long bytes;
    int largest_rank;
    double average_rank;
} acrgpu_levelinfo;

typedef struct acrgpu_timing {     /* device-event phase times of the last call (ms) */
    double lift_ms;
    double factor_ms;              /* includes lift */
    double solve_ms;
    double flops_nominal;          /* nominal FLOP count of the last factorization */
    double flops_svd, flops_qr, flops_gemm, flops_lu;
    long factor_launches;          /* kernels launched by the factorization */
    long solve_launches;           /* kernels launched by the last solve */
} acrgpu_timing;

typedef struct acrgpu_ctx acrgpu_ctx;
typedef struct acrgpu_fact acrgpu_fact;

/* Context on one CUDA device (device < 0: current device).  Destroying the
   context handle while factorizations built on it are alive is allowed: its
   device resources are released with the last of them.
   One context = one device = one worker of the reference's plane partition
   (parallel.cpp:96-297): a multi-GPU run creates one context per process / GPU and
   ties them together with a communicator handle (acrgpu_comm, below), rather than passing a device
   list to one context as SURVEY.md's sketch of the boundary did. */
int acrgpu_ctx_create(int device, acrgpu_ctx** out, acrgpu_error* err);
void acrgpu_ctx_destroy(acrgpu_ctx* ctx);

/* acr_factor in H-matrix mode.  System blocks are read from host memory (validated,
 * duplicate-merged and uploaded inside the call). */
int acrgpu_factor(acrgpu_ctx* ctx, const acrgpu_system* sys, const acrgpu_config* cfg,
                  acrgpu_fact** out, acrgpu_error* err);
/* Device-resident input: validate + upload once, then factor from HBM (no host input traffic). */
typedef struct acrgpu_dsystem acrgpu_dsystem;
int acrgpu_system_upload(acrgpu_ctx* ctx, const acrgpu_system* sys, acrgpu_dsystem** out, acrgpu_error* err);
void acrgpu_system_destroy(acrgpu_dsystem* sys);
int acrgpu_factor_resident(acrgpu_ctx* ctx, const acrgpu_dsystem* sys, const acrgpu_config* cfg,
                           acrgpu_fact** out, acrgpu_error* err);
void acrgpu_factor_destroy(acrgpu_fact* f);

/* AcrFactorization::solve for nrhs right-hand sides; f, u host pointers ([nrhs][n][dim]). */
int acrgpu_solve(acrgpu_fact* f, int nrhs, const double* f_host, double* u_host, acrgpu_error* err);
/* Same, with f and u already resident in device memory (device pointers). */
int acrgpu_solve_device(acrgpu_fact* f, int nrhs, const double* f_dev, double* u_dev, acrgpu_error* err);

int acrgpu_stats(acrgpu_fact* f, acrgpu_rankstats* out);
/* Fills up to cap entries (levels + apex); returns the count. */
int acrgpu_level_info(acrgpu_fact* f, acrgpu_levelinfo* out, int cap);
/* Leaf ranks (DFS order, -1 = dense leaf) of the stored inverse of plane j at level li
 * (li == number of levels: apex).  Returns the leaf count, -1 if absent. */
long acrgpu_dinv_ranks(acrgpu_fact* f, int li, int j, int* out, long cap);
int acrgpu_timing_get(acrgpu_fact* f, acrgpu_timing* out);

/* Structure only (no device work): permutation (tree pos -> original index, dim ints) and
 * leaf table (DFS order; rb, re, cb, ce, kind with kind 0 = dense, 1 = low-rank).
 * Returns the leaf count (leaves written up to cap), or -code on error. */
long acrgpu_structure(int dim, const double* coords, int leaf_size, double eta, int weak,
                      int* perm, int* leaves, long cap, acrgpu_error* err);

/* Per-kernel device time of the launches selected by acrgpu_profile_select / ACRGPU_PROFILE:
 * lines "kernel total_ms launches ctas nominal_flops executed_flops" (nominal = the reference
 * algorithm's count; executed = nominal minus the part the kernel skipped: zero-operand
 * products, the QRs the dense route replaces).  Returns the length written (NUL-terminated). */
long acrgpu_profile_report(char* buf, long cap, int reset);
/* Select which launches are timed (overrides ACRGPU_PROFILE): NULL / "" / "0" none, "1" / "*"
 * every kernel, else a comma-separated list of kernel names (e.g. "k_trunc_qr"). */
void acrgpu_profile_select(const char* filter);

/* ---- Plane partition over several GPUs (execute_parallel_factor, parallel.cpp:96-297).
 * Rank w owns the planes plan_schedule(n, p) assigns it (contiguous blocks at level 0;
 * retained planes keep their owner).  Per level every rank inverts its eliminated planes
 * and sends {Dinv_e, E_e, F_e} to the owner of each retained neighbour held by another
 * rank; the solve exchanges plane vectors the same way.  n and p must be powers of two,
 * stop_planes 1.  Results are bitwise identical for every p (test_parallel.cpp:75-89).
 *
 * Multi-process (one rank per GPU, NCCL point-to-point over NVLink): rank 0 calls
 * acrgpu_comm_unique_id, the id is broadcast out of band (e.g. torch.distributed), and
 * every rank calls acrgpu_comm_create on its device.  acrgpu_solve on such a handle fills
 * the planes this rank owns (other planes of u are set to 0).
 * In-process (acrgpu_comm_create_local): all p ranks run on the context's device in one
 * call; the handle holds every rank and acrgpu_solve returns the full solution.  Used to
 * check the partitioned data path on one GPU. */
#define ACRGPU_COMM_ID_BYTES 128
typedef struct acrgpu_comm acrgpu_comm;
int acrgpu_comm_unique_id(unsigned char* id /* ACRGPU_COMM_ID_BYTES */, acrgpu_error* err);
int acrgpu_comm_create(const unsigned char* id, int nranks, int rank, acrgpu_comm** out, acrgpu_error* err);
int acrgpu_comm_create_local(int nranks, acrgpu_comm** out, acrgpu_error* err);
/* Host-staged multi-process communicator (no NCCL): every wire image is copied to host memory
 * and moved by `fn`, called once per exchange phase with all of this rank's sends (to rank
 * dst[i], sbytes[i] bytes at sbuf[i]) and receives (from rank src[j] into rbuf[j], rbytes[j]
 * bytes).  Messages between one pair of ranks are posted in the same order on both sides, so
 * a point-to-point channel that keeps per-pair order (e.g. torch.distributed isend/irecv over
 * gloo) delivers them correctly.  Returns nonzero to abort the factorization (ACRGPU_E_DEVICE).
 * Used to run the partitioned data path across real processes without NVLink/NCCL. */
typedef int (*acrgpu_exchange_fn)(void* user, int nsend, const int* dst, const void* const* sbuf, const long* sbytes,
                                  int nrecv, const int* src, void* const* rbuf, const long* rbytes);
int acrgpu_comm_create_host(acrgpu_exchange_fn fn, void* user, int nranks, int rank, acrgpu_comm** out,
                            acrgpu_error* err);
void acrgpu_comm_destroy(acrgpu_comm* comm);
int acrgpu_factor_partitioned(acrgpu_ctx* ctx, acrgpu_comm* comm, const acrgpu_system* sys,
                              const acrgpu_config* cfg, acrgpu_fact** out, acrgpu_error* err);
/* Same, on a system already uploaded with acrgpu_system_upload. */
int acrgpu_factor_partitioned_resident(acrgpu_ctx* ctx, acrgpu_comm* comm, const acrgpu_dsystem* sys,
                                       const acrgpu_config* cfg, acrgpu_fact** out, acrgpu_error* err);
/* Cross-rank elimination payloads of a partitioned factorization (MessageRecord,
 * core/include/acr/parallel.hpp:24-30; recorded as in parallel.cpp:142-161): one record per
 * (eliminated plane, destination rank), bytes = memory_footprint of {Dinv, E, F} as sent
 * (before the stored-inverse trim) + 8*dim for the plane right-hand side.  Records of all
 * ranks held by this handle (every rank for an in-process communicator, this rank's own
 * sends for NCCL).  Returns the record count (written up to cap); 0 for acrgpu_factor. */
typedef struct acrgpu_message {
    int level;
    int from_plane;
    int to_plane;
    int solve_phase;               /* always 0 here; solve-phase {u} records follow from the plan */
    long bytes;
} acrgpu_message;
long acrgpu_messages(acrgpu_fact* f, acrgpu_message* out, long cap);

/* ---- Krylov drivers with the GPU factorization as preconditioner
 * (core/include/acr/krylov.hpp:8-35, core/src/krylov.cpp:38-133).  One right-hand side
 * f_dev and solution u_dev ([n][dim], device memory, original ordering) on an uploaded
 * system; the operator is applied as one CSR SpMV built from the system's COO blocks on
 * first use.  residual_history (host, may be NULL) receives the true relative residual
 * ||f - A u|| / ||f|| of every iteration (up to max_iterations entries).
 *   acrgpu_pcg     <- acr::pcg(system, precond, tol, max_iterations); precond may be NULL
 *                     (plain CG).  ACRGPU_E_INDEFINITE when p^T A p <= 0.
 *   acrgpu_refine  <- acr::iterative_refinement(system, precond, tol, max_iterations).
 *                     ACRGPU_E_DIVERGENCE after three consecutive residual increases.
 * Nonconvergence is reported in the trace (converged = 0), not as an error.  The
 * preconditioner must be a single-GPU factorization of a system of the same shape. */
typedef struct acrgpu_trace {
    int converged;
    int iterations;
    double apply_time;             /* mean seconds per preconditioner application (device events) */
    double total_time;             /* seconds */
} acrgpu_trace;
int acrgpu_pcg(acrgpu_ctx* ctx, const acrgpu_dsystem* sys, acrgpu_fact* precond, double tol, int max_iterations,
               const double* f_dev, double* u_dev, double* residual_history, acrgpu_trace* trace, acrgpu_error* err);
int acrgpu_refine(acrgpu_ctx* ctx, const acrgpu_dsystem* sys, acrgpu_fact* precond, double tol, int max_iterations,
                  const double* f_dev, double* u_dev, double* residual_history, acrgpu_trace* trace,
                  acrgpu_error* err);

/* Library build identification (sm arch, version). */
const char* acrgpu_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ACRGPU_H */
