// Launchers shared between the C-ABI layer and the kernel translation units.
#pragma once

#include "common.cuh"

namespace goat {

// ---------------------------------------------------------------- Sinkhorn
// Log-domain Sinkhorn on E_ij = coef * (gmax - G_ij) (sinkhorn.py:115-126),
// with the exact sweep semantics of sinkhorn_knopp (sinkhorn.py:60-85).
struct SkArgs {
    const void *G;      // n x n, element type = precision, leading dim ld
    int64_t ld;
    int n;              // columns (and rows unless m > 0)
    int m = 0;          // rows of a row-sharded block (0 = n)
    int single_pass = 0;  // row-sharded driver: run pass st->k only, then exit
    double *f[2];       // row potentials, ring of 2 (fp64)
    double *g[2];       // column potentials, ring of 2 (fp64)
    void *colpart;      // [nblk][ldp] per-CTA column partial sums (element type)
    int64_t ldp;
    double *devpart;    // [nblk] per-CTA max row deviation
    double *devcol;     // [merge blocks] max column deviation (pre-check)
    SkState *st;
    int nblk;           // CTAs of the pass kernel
    unsigned long long *dslot = nullptr;  // persistent driver: atomicMax dev slots [row k&1 | col]
    int slice_w = 0;    // cluster-split rows: columns per CTA rank
    int resident = 1;   // keep a CTA's single band in registers across sweeps
    int l2_last = 0;    // wide-row bulk copies carry an L2 evict_last hint (G fits in L2)
    int stages = 0;     // wide rows: shared-memory ring stages (0 = register path)
    unsigned long long *trace = nullptr;  // diagnostics: per-CTA phase timestamps of sweep trace_k
    int trace_k = -1;
    int stage_bytes = 0;
    int dbg = 0;        // timing experiments only (GOAT_SK_DBG): drop parts of the wide-row pass
};

struct SkPlan {
    int ch = 0;        // 16-byte chunks per thread
    int rows = 0;      // rows per band
    int nblk = 0;      // pass-kernel CTAs
    int merge_blocks = 0;
    bool persistent = false;  // one cooperative launch for the whole sweep loop
    int cl = 1;               // CTAs per row group (thread-block cluster) sharing each row
    int nt = 256;             // threads per CTA
    int ngrp = 0;             // row groups (= nblk / cl)
    int slice_w = 0;          // columns per CTA rank when cl > 1
    size_t colpart_bytes = 0;
    int stages = 0;           // wide rows: bulk-copy ring depth (0 = register prefetch)
    int stage_bytes = 0;
    size_t smem = 0;          // dynamic shared memory of the persistent kernel
    bool pipe = false;        // wide fp32 rows: decoupled bulk-copy pipeline (sk_pipe_kernel)
    bool tile = false;        // small n: shared-memory-resident tiles, one barrier per sweep (sk_tile_kernel)
    bool wide2 = false;       // 12288 < n <= 40960 fp32: 2-CTA clusters, registers hold y and the column sums (sk_wide_kernel)
    bool wide_tm = false;     // wide2 with rows parked in TMEM for a lagged finish (sk_wide_kernel<..., TM>)
    int tile_rows = 0;        // rows per row group of the tile kernel
};

// rows: rows of a row-sharded block (-1 = n); sharded: the plan serves single-pass
// launches of the row-sharded driver (no whole-LOT tile kernel).
template <class T> SkPlan sk_plan(int n, int num_sms, int rows = -1, bool sharded = false);
template <class T> void sk_launch_pass(const SkArgs &a, const SkPlan &p, cudaStream_t s);
template <class T> void sk_launch_merge(const SkArgs &a, const SkPlan &p, cudaStream_t s);
// All sweeps in one cooperative launch (bar: 2 unsigned of scratch).
template <class T> void sk_launch_persistent(const SkArgs &a, const SkPlan &p, unsigned *bar, cudaStream_t s);
// Q = exp(E + f + g) for the returned slot; optional fused partial sums:
// part[blk*4 + 0] = sum (Q-P)^2, [1] = <L,Q>.  P, L may be null.
// Row-sharded sweep (one rank's rows; the caller all-gathers `send` between):
//   sk_launch_shard_pass: pass st->k over the block (no-op once done), then
//     send[0..n) = fp64 column sums of the block, send[n] = its max row deviation;
//   sk_launch_shard_merge: fixed-order merge of recv[world][n+1], the stopping rule
//     and g_k (identical on every rank).
template <class T> void sk_launch_shard_pass(const SkArgs &a, const SkPlan &p, unsigned *bar, double *send,
                                             cudaStream_t s);
template <class T>
void sk_launch_shard_merge(const SkArgs &a, const double *recv, int world, unsigned char *bad, cudaStream_t s);
//   column repair round (only when the merge left the sweep pending):
//   sk_launch_shard_repair_pass: exact fp64 (max, sumexp) pairs of the flagged
//     columns over the block's rows -> pair[2n]; the caller all-gathers them;
//   sk_launch_shard_repair_merge: rank-order combine, finishes the sweep.
template <class T>
void sk_launch_shard_repair_pass(const SkArgs &a, const unsigned char *bad, double *pair, cudaStream_t s);
void sk_launch_shard_repair_merge(const SkArgs &a, const double *recv, int world, const unsigned char *bad,
                                  cudaStream_t s);
template <class T>
void sk_launch_emit(const SkArgs &a, T *Q, int64_t ldq, const T *P, int64_t ldp, const T *L,
                    int64_t ldl, double *part, int nblk, cudaStream_t s);

// ---------------------------------------------------------------- reductions
// Deterministic two-stage reductions (fixed grid, fixed order).
constexpr int kRedBlocks = 296;
template <class T>
void launch_minmax(const T *X, int64_t ld, int n, double *part, double *out2, cudaStream_t s, int rows = -1);
// D = P - Q: out[0]=<GQ,D>, [1]=<GP-GQ,D>, [2]=<GQ,Q>, [3]=|D|^2, [4]=<L,D>, [5]=<L,Q>
template <class T>
void launch_fw_dots(const T *GP, const T *GQ, const T *P, const T *Q, const T *L, int64_t ld, int n,
                    double *part, double *out6, cudaStream_t s, int rows = -1);
// out[0] = sum_ij A_ij * B_{p(i)p(j)}  (A, B fp64)
void launch_qap_perm(const double *A, int64_t lda, const double *B, int64_t ldb,
                     const int *perm, int n, double *part, double *out, cudaStream_t s);
// dst = scale * src (n x n, padding zeroed); *nonfinite <- 1 if some src entry is
// not finite (the reference's ValueError check, core.py:25, fused into the upload)
template <class T>
void launch_convert(const double *src, int64_t lds, T *dst, int64_t ldd, int n, double scale,
                    cudaStream_t s, int *nonfinite = nullptr);
template <class T>
void launch_convert_to_f64(const T *src, int64_t lds, double *dst, int64_t ldd, int n,
                           cudaStream_t s, int rows = -1);
template <class T> void launch_fill(T *dst, int64_t ld, int n, double value, cudaStream_t s, int rows = -1);
// Y = a*X + b*Y  (elementwise, matcher.py:197)
template <class T>
void launch_axpby(double a, const T *X, double b, T *Y, int64_t ld, int n, cudaStream_t s, int rows = -1);
// Q = permutation matrix of perm (core.py:64-70)
template <class T> void launch_perm_matrix(const int *perm, T *Q, int64_t ld, int n, cudaStream_t s);
// Y = X + L
template <class T>
void launch_add(const T *X, const T *L, T *Y, int64_t ld, int n, cudaStream_t s, int rows = -1);
// G_ij = (ra_i rb_j + ca_i cb_j) / n  (gradient at the barycenter, rank 2)
template <class T>
void launch_bary_grad(const T *A, int64_t lda, const T *B, int64_t ldb, T *G, int64_t ldg,
                      int n, double *vec4n, cudaStream_t s);
// 1 if X == X^T exactly, written to *flag (int)
template <class T>
void launch_is_symmetric(const T *X, int64_t ld, int n, int *flag, cudaStream_t s);
// Y = -log(X) (sinkhorn_knopp entry); *bad set to 1 if any X <= 0
template <class T>
void launch_neglog(const T *X, int64_t ldx, T *Y, int64_t ldy, int n, int *bad, cudaStream_t s);

// G_ij = (ra_i rb_j + ca_i cb_j) / n from the four degree vectors (vec4n = [ra|ca|rb|cb])
template <class T> void launch_bary_grad_vec(const double *vec4n, T *G, int64_t ldg, int n, cudaStream_t s);

// ---------------------------------------------------------------- sparse (CSR) adjacency (spmm.cu)
template <class T> struct DevCsr {
    const int64_t *rowptr = nullptr;  // [n+1]
    const int *col = nullptr;         // [nnz], strictly increasing within a row
    const T *val = nullptr;           // [nnz] or null: every stored entry is 1
    int64_t nnz = 0;
};
// out = alpha * (sum_t S_t D_t)^T, t < nterms (1 or 2).  S_t: `rows` CSR rows over
// column indices < (rows of D_t); D_t: row-major with `cols` columns, leading dim
// ld; out: cols x rows row-major, leading dim ldo (columns >= rows untouched).
template <class T>
void launch_spmm_t(int rows, int cols, int64_t ld, int64_t ldo, int nterms, const DevCsr<T> *S, const T *const *D,
                   double alpha, T *out, cudaStream_t s);
// flag[0] <- 0 unless rowptr spans [0, nnz], every row is strictly increasing with
// columns in [0, n), and the values are finite
template <class T> void launch_csr_check(const DevCsr<T> &a, int rows, int n, int *flag, cudaStream_t s);
size_t csr_transpose_scratch(int64_t nnz);
template <class T>
void launch_csr_transpose(const DevCsr<T> &a, int n, int64_t *rowptrT, int *colT, T *valT, void *scratch,
                          size_t scratch_bytes, cudaStream_t s);
template <class T> void launch_csr_equal(const DevCsr<T> &a, const DevCsr<T> &b, int n, int *flag, cudaStream_t s);
template <class T> void launch_csr_rowsum(const DevCsr<T> &a, int n, double *rs, cudaStream_t s);
// out[0] = sum_{(i,j) in A} A_ij B_{p(i) p(j)}  (fp64, fixed order; rowsum: n doubles of scratch)
template <class T>
void launch_csr_qap_perm(const DevCsr<T> &a, const DevCsr<T> &b, const int *perm, int n, double *rowsum, double *out,
                         cudaStream_t s);

// ---------------------------------------------------------------- GEMM
// C = alpha * op(A) op(B) + beta * C, op = transpose when trans != 0 (SIMT).
template <class T>
void gemm_simt(int m, int n, int k, double alpha, const T *A, int64_t lda, int transA,
               const T *B, int64_t ldb, int transB, double beta, T *C, int64_t ldc,
               cudaStream_t s);

// ---------------------------------------------------------------- LAP
// Certificate: strict row-argmax (sense-aware) forming a permutation.
template <class T>
void launch_lap_certificate(const T *M, int64_t ld, int n, int sense, int *cand, int *hits,
                            int *flag, cudaStream_t s);
// Exact shortest-augmenting-path LSAP with scipy's visiting order (lap.cu).
struct LapWork {
    double *u, *v, *spc;
    int *path, *row4col, *col4row, *rem;
    unsigned char *SR, *SC;
    int *status;
};
template <class T>
void launch_lap_sap(const T *M, int64_t ld, int n, int sense, const LapWork &w, cudaStream_t s, int warm = 0);
// eps-scaling auction + exact-repair preparation (lap.cu): fills w.u, w.v,
// w.row4col, w.col4row with a tight partial assignment and feasible duals for a
// warm-started launch_lap_sap.  counters: [0] assigned, [1] rounds, [2] capped, [3] freed rows.
struct AuctionWork {
    double *price, *row_bid_v;
    int *row_col, *col_row, *bid_row, *row_bid, *counters;
    unsigned long long *bid_val;
    unsigned *bar;
    double *part_w;  // [2 * kAucMaxCtas] per-CTA partial (best, second) of a shared row scan
    int *part_j;     // [kAucMaxCtas]
};
constexpr int kAucMaxCtas = 4096;
template <class T>
int launch_lap_auction(const T *M, int64_t ld, int n, int sense, double range, const LapWork &w,
                       const AuctionWork &aw, int num_sms, cudaStream_t s);

}  // namespace goat
