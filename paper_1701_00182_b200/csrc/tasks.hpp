// Task descriptors shared by the host plan compiler (engine.cu) and the sm_100a
// kernels (kernels.cu).  All indices are RELATIVE to the operand view's node
// (dense ids / pool offsets / Rk ids minus the node's first ids), so one
// compiled plan serves every plane of a batch and every call on the same
// structural triple.
#pragma once

#include <cstdint>

namespace acrgpu {

constexpr int MAXB = 64;  // planes per batched launch

// Per-plane view of one H-matrix operand (node-relative base pointers).
struct HView {
    double* dense;  // dense pool slice of the node
    int* rank;      // rank[k_rel]
    double** U;     // U[k_rel]: rows x rank, column-major (ld = rows)
    double** V;     // V[k_rel]: cols x rank (ld = cols)
};

struct BatchViews {
    int count;
    HView c[MAXB], a[MAXB], b[MAXB];
};

// Product output (low-rank factors of A_sub * B_sub), one per (product, plane).
struct Slot {
    double* U;
    double* V;
    int rank;
    int ldu, ldv;
    int pad;
};

// Device bump allocator (stream-ordered; reset between operations).
struct Arena {
    double* base;
    unsigned long long cap;      // doubles
    unsigned long long* ctr;     // device counter (doubles used)
    int* overflow;               // device flag
};

// Leaf-level product kinds (reference mult_to_lowrank, hmatrix.cpp:397-454)
enum ProdKind : int {
    P_RK_LEFT = 0,   // A Rk:  U = A.U (alias), V = B^T A.V  (node_apply_trans)
    P_RK_RIGHT = 1,  // B Rk:  V = B.V (alias), U = A B.U    (node_apply)
    P_DD = 2,        // dense * dense -> SVD truncation
    P_BB = 3,        // branch * branch -> 8 sub-products, concat, truncate
};

// Allocation of an apply product's computed factor.
struct AllocTask {
    int prod;
    int kind;        // P_RK_LEFT / P_RK_RIGHT
    int kx;          // Rk leaf (relative) of A (RK_LEFT) or B (RK_RIGHT)
    int rows_out;    // rows of the computed factor
    int rows_alias;  // rows of the aliased factor (ld)
};

// One output slab of an apply product: Y[r0:r1, :k] = sum over leaves.
struct ApplyTask {
    int prod;
    int kind;        // P_RK_LEFT (transposed apply over B) / P_RK_RIGHT (apply over A)
    int kx;          // X source leaf
    int r0, r1;      // output rows of this slab
    int lbeg, lend;  // ApplyLeaf range
};

struct ApplyLeaf {
    int kind;        // K_DENSE / K_RK
    int id;          // relative Rk id (K_RK)
    long doff;       // relative dense pool offset (K_DENSE)
    int m, n;        // leaf rows / cols (untransposed)
    int in_off;      // X row of the leaf's first contracted index
    int out_off;     // Y row of the leaf's first output index (relative to slab output space)
    int tl;          // K_RK: index of the leaf's T task (T = In^T X, shared by all its slabs)
};

// T = In^T X for one Rk leaf of an apply product (In = U for the transposed apply, V
// otherwise), computed once and read by every output slab the leaf overlaps.  The
// result (rank x k, ld rank) lives in the transient arena; its pointer goes to slot
// (nprod + index) of the batch's slot table.
struct ApplyTTask {
    int prod;
    int kind;
    int kx;
    int id;          // relative Rk id
    int in_off;      // X row of the first contracted index
    int in_len;
    int x_ld;
};

struct DDTask {
    int prod;
    long da, db;     // relative dense offsets in A and B
    int m, k, n;
};

// Part of a concatenation [U_1 | U_2 | ...] / [V_1 | V_2 | ...].
enum PartSrc : int { S_SLOT = 0, S_CLEAF = 1, S_GEMM = 2 };
struct Part {
    int src;         // S_SLOT: product slot `id`; S_CLEAF: C's Rk leaf `id` (current value);
                     // S_GEMM: exact dense product A.D[da] * B.D[db] (deposit into dense only)
    int id;
    int u_src, v_src;    // first source row taken from U / V
    int u_dst, v_dst;    // first target row (placement inside the target block)
    int rows_u, rows_v;  // extent
    double alpha;
    long da, db;         // S_GEMM operands
    int gk;              // S_GEMM inner dimension
    int pad;
};

// Truncation of a concatenation (BB agglomeration -> slot, or flush -> C leaf).
struct TruncTask {
    int out_kind;    // 0 = product slot, 1 = C Rk leaf (persistent)
    int out_id;
    int m, n;
    int pbeg, pend;
};

// Dense-target deposit: C.D[doff] (m x n) += sum_parts alpha U V^T (in part order).
struct DepTask {
    long doff;
    int m, n;
    int pbeg, pend;
};

// Dense leaf inversion (LU + rcond guard), reference hmatrix.cpp:483-496.
struct LuTask {
    long doff;       // relative offset in A (input) and C (output) views
    int m;
    int rb, re;      // tree-order rows, for SingularBlockError messages
};

// invert_node of a branch whose four children are dense leaves <= 32 (k_invert2x2)
struct Inv2Task {
    long d11, d12, d21, d22;  // dense pool offsets of the children, relative to the node's view
    int m1, m2;               // rows of the first / second cluster
    int rb1, re1, rb2, re2;   // tree-order rows of the diagonal leaves (SingularBlockError)
};

// Error record (first error by (call, batch index) order wins).
struct DevError {
    unsigned long long key;  // (call_id << 16) | b ; ~0 = none
    int code;
    int rb, re;
    double rcond;
};

// Nominal FLOP ledger (SURVEY §8(d) formulas; same as oracle/acr_oracle.cpp).
// Nominal FLOPs of the reference algorithm by class (SURVEY §8(d) formulas), plus F_SKIP: the
// part of the nominal count a kernel did not execute (zero-operand products detected on the
// device; the two QRs the dense route replaces by forming M, net of that formation GEMM).
// executed = nominal - F_SKIP.
enum FlopClass : int { F_GEMM = 0, F_GEQRF, F_ORGQR, F_SVD, F_LU, F_APPLY, F_NCLASS, F_SKIP = F_NCLASS };
struct FlopLedger {
    double f[F_NCLASS + 1];
};

// Solve: batched H-matvec  y = base - H x  (or y = H x when base == nullptr).
struct SlabTask {      // output rows [r0, r1) of the tree-ordered plane vector
    int r0, r1;
    int lbeg, lend;    // ApplyLeaf range (non-transposed, in_off = leaf col, out_off = leaf row)
};
struct MvLeaf {         // Rk leaf k of the root: columns [in_off, in_off + n), rows m
    int k;
    int in_off;
    int n, m;
};
struct MvCluster {      // leaf cluster of the plane: packed-x block of its columns (k_mv_slab_tma)
    int in_off, n;      // first tree position, size
    int xoff, ldx;      // block offset (doubles, inside one item's RHS group) and its RHS stride
};
struct MatvecPlan {     // per-structure tables of the solve's batched H-matvec
    int ntasks;
    const SlabTask* tasks;
    const ApplyLeaf* leaves;  // slab leaves; dense leaves carry their column cluster's xoff in `tl`
    int nleaves;
    const MvLeaf* rk;
    int nrk, nbig;
    const MvCluster* cl;
    int ncl;
    long xp_group;      // packed-x doubles per (item, RHS group)
};
struct MatvecBatch {
    int count;
    HView h[MAXB];
    const double* x[MAXB];
    const double* base[MAXB];
    double* y[MAXB];
};

}  // namespace acrgpu
