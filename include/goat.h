/*
 * goat.h -- C ABI of libgoat.so, the B200 (sm_100a) GOAT iteration.
 *
 * GOAT (arXiv 2111.05366) is Frank-Wolfe graph matching whose per-iteration
 * linear-assignment step is replaced by entropic Sinkhorn OT ("LOT").  The
 * reference (`otmatch`, pure Python/numpy) has no plugin registry; its one
 * strategy seam is the Frank-Wolfe core
 *     _fw_core(A, B, L, P0, opts) -> (assignment, history, iterations, converged)
 *     /root/reference/pkg/src/otmatch/matcher.py:177-212
 * which is what goat_fw_core() replaces.  The component entry points below
 * replace the functions _fw_core calls, so the reference's own component tests
 * can be restated against them.  Everything here takes plain pointers and
 * sizes; host matrices are float64 row-major with a leading dimension, exactly
 * the numpy arrays the reference passes (core.py:22).  The library never keeps
 * caller pointers after a call returns and never mutates inputs.
 *
 * Errors: every function returns GOAT_OK (0) or a GOAT_E* code; the message is
 * available from goat_last_error() (thread-local).  GOAT_EINVAL corresponds to
 * the reference's ValueError (core.py:23-26, matcher.py:52-66,105-106).
 * Sinkhorn non-convergence is NOT an error (sinkhorn.py:85).
 *
 * Threading: a handle is bound to one device and one stream and must not be
 * used from two threads at once; distinct handles may run concurrently.
 */
#ifndef GOAT_H
#define GOAT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GOAT_OK 0
#define GOAT_EINVAL 1  /* invalid argument (reference: ValueError) */
#define GOAT_ECUDA 2   /* CUDA runtime / launch failure */
#define GOAT_EOOM 3    /* device allocation failed */
#define GOAT_ENOTSUP 4 /* unsupported configuration */

#define GOAT_FP32 0    /* fp32 iterate, fp64 potentials and accumulators */
#define GOAT_FP64 1    /* fp64 throughout (reference arithmetic) */

#define GOAT_MINIMIZE 0
#define GOAT_MAXIMIZE 1

#define GOAT_STEP_EXACT_LAP 0 /* FAQ: matcher.py:191-192 */
#define GOAT_STEP_LOT 1       /* GOAT: matcher.py:193-194 */

/* GEMM engines for the gradient products (fp32 mode only; fp64 always SIMT). */
#define GOAT_GEMM_AUTO 0
#define GOAT_GEMM_SIMT 1     /* CUDA-core fp32 FMA */
#define GOAT_GEMM_TCGEN05 2  /* tcgen05/TMEM/TMA bf16-split, fp32 accumulate */

typedef struct goat_handle goat_handle;

typedef struct goat_config {
    int32_t device;     /* CUDA ordinal */
    int32_t precision;  /* GOAT_FP32 | GOAT_FP64 */
    int32_t gemm;       /* GOAT_GEMM_* */
    int32_t split_terms;/* bf16 terms per non-exact operand for GOAT_GEMM_TCGEN05 (2 or 3; 0 = default 3) */
} goat_config;

/* MatchOptions (matcher.py:32-50) + SinkhornParams (sinkhorn.py:21-32). */
typedef struct goat_options {
    int32_t max_iters;    /* matcher.py:45 (30) */
    int32_t max_sweeps;   /* sinkhorn.py:31 (1000) */
    int32_t sense;        /* GOAT_MAXIMIZE (matcher.py:50) */
    int32_t step_solver;  /* GOAT_STEP_LOT for GOAT */
    double fw_tol;        /* matcher.py:46 (1e-2) */
    double lam;           /* sinkhorn.py:30 (100) -- reg = 1/lam on the unit-range cost */
    double sk_tol;        /* sinkhorn.py:32 (1e-8) */
} goat_options;

/* _fw_core's return value plus the diagnostics the reference discards. */
typedef struct goat_fw_result {
    int64_t *assignment;     /* [n] out: permutation p[row] = col (lap.py:56-57) */
    double *hist_obj;        /* [max_iters+1] out: f(P_i), history[i][1] */
    double *hist_alpha;      /* [max_iters+1] out: alpha_i (entry 0 = NaN) */
    int32_t *lot_sweeps;     /* [max_iters] out or NULL */
    int32_t *lot_converged;  /* [max_iters] out or NULL */
    double *lot_dev;         /* [max_iters] out or NULL */
    int32_t iterations;      /* out */
    int32_t converged;       /* out */
    int32_t lap_certified;   /* out: 1 if the O(n^2) strict-argmax certificate fired */
    int32_t gpu_launches;    /* out: kernels launched by this call */
    double objective;        /* out: sum_ij A_ij B_{p(i)p(j)} on the inputs (core.py:120-124) */
    double time_ms[6];       /* out: gradient, lot, linesearch+update, lap, h2d+setup, total */
    int32_t *lot_fp64_from;  /* [max_iters] out or NULL: fp32 handles, sweeps done in fp32 before the LOT
                              * finished in fp64 arithmetic (-1: the whole LOT ran in the handle's precision) */
    double *lot_ms;          /* [max_iters] out or NULL: device time of each LOT step (CUDA events) */
} goat_fw_result;

int goat_create(goat_handle **out, const goat_config *cfg);
int goat_destroy(goat_handle *h);
const char *goat_last_error(void);
/* Reserve device workspace for order n up front (optional). */
int goat_reserve(goat_handle *h, int64_t n);

/* matcher.py:177-212 _fw_core on host float64 buffers.
 * L: seeded linear term (matcher.py:267) or NULL.  P0: initial iterate or NULL
 * for the barycenter J/n (core.py:89-93). */
int goat_fw_core(goat_handle *h, int64_t n,
                 const double *A, int64_t lda, const double *B, int64_t ldb,
                 const double *L, int64_t ldl, const double *P0, int64_t ldp,
                 const goat_options *opts, goat_fw_result *res);

/* Seeded _fw_core (matcher.py:245-269): the free blocks A22, B22 (nf x nf) and the
 * seed blocks A21, B21 (nf x m), A12, B12 (m x nf) of the seed-reordered,
 * shuffled inputs; the constant linear term L = A21 B21^T + A12^T B12
 * (matcher.py:267) is formed on the device.  objective = the free-block terms. */
int goat_fw_core_seeded(goat_handle *h, int64_t nf, int64_t m,
                        const double *A22, int64_t lda22, const double *B22, int64_t ldb22,
                        const double *A21, int64_t lda21, const double *A12, int64_t lda12,
                        const double *B21, int64_t ldb21, const double *B12, int64_t ldb12,
                        const double *P0, int64_t ldp, const goat_options *opts, goat_fw_result *res);

/* Same, inputs already resident on the handle's device (row-major, element
 * type = the handle's precision: float for GOAT_FP32, double for GOAT_FP64). */
int goat_fw_core_device(goat_handle *h, int64_t n,
                        const void *dA, int64_t lda, const void *dB, int64_t ldb,
                        const void *dL, int64_t ldl, const void *dP0, int64_t ldp,
                        const goat_options *opts, goat_fw_result *res);

/* Sparse adjacency (CSR).  Rows hold strictly increasing column indices; values
 * NULL means every stored entry is 1 (an unweighted graph).  Host calls take
 * float64 values; the _device variants take device pointers whose values have
 * the handle's element type.  The reference has no sparse input path (core.py:22
 * densifies everything); these entries replace _fw_core (matcher.py:177-212) and
 * gradient (matcher.py:100-107) for graphs held as CSR (BASELINE config 5). */
typedef struct goat_csr {
    const int64_t *rowptr;  /* [n+1], rowptr[0] = 0, rowptr[n] = nnz */
    const int32_t *colidx;  /* [nnz] */
    const void *values;     /* [nnz] or NULL */
    int64_t nnz;
} goat_csr;

int goat_fw_core_csr(goat_handle *h, int64_t n, const goat_csr *A, const goat_csr *B,
                     const double *L, int64_t ldl, const double *P0, int64_t ldp,
                     const goat_options *opts, goat_fw_result *res);
int goat_fw_core_csr_device(goat_handle *h, int64_t n, const goat_csr *dA, const goat_csr *dB,
                            const void *dL, int64_t ldl, const void *dP0, int64_t ldp,
                            const goat_options *opts, goat_fw_result *res);
/* gradient on CSR adjacency, dense host P -> dense host G (float64). */
int goat_gradient_csr(goat_handle *h, int64_t n, const goat_csr *A, const goat_csr *B,
                      const double *P, int64_t ldp, double *G, int64_t ldg);
/* timing hook: mean ms of `reps` CSR gradients on device CSR + dense device X (n x n). */
int goat_bench_gradient_csr(goat_handle *h, int64_t n, const goat_csr *dA, const goat_csr *dB,
                            const void *dX, int32_t reps, double *ms);

/* matcher.py:100-107  G = A P B^T + A^T P B  (host float64 in/out). */
int goat_gradient(goat_handle *h, int64_t n, const double *A, int64_t lda,
                  const double *B, int64_t ldb, const double *P, int64_t ldp,
                  double *G, int64_t ldg);

/* sinkhorn.py:103-130  lot(M, sense, params) -> Q, converged, sweeps, deviation. */
int goat_lot(goat_handle *h, int64_t n, const double *M, int64_t ldm, int32_t sense,
             double lam, int32_t max_sweeps, double tol, double *Q, int64_t ldq,
             int32_t *converged, int32_t *sweeps, double *deviation);

/* lot() on a device-resident M (element type = the handle's precision, leading
 * dimension round_up(n, 8), 16-byte aligned); Q is written on the device. */
int goat_lot_device(goat_handle *h, int64_t n, const void *dM, int64_t ldm, int32_t sense,
                    double lam, int32_t max_sweeps, double tol, void *dQ, int64_t ldq,
                    int32_t *converged, int32_t *sweeps, double *deviation);

/* sinkhorn.py:60-85  sinkhorn_knopp(K, params) on a strictly positive K. */
int goat_sinkhorn_knopp(goat_handle *h, int64_t n, const double *K, int64_t ldk,
                        int32_t max_sweeps, double tol, double *Q, int64_t ldq,
                        int32_t *converged, int32_t *sweeps, double *deviation);

/* matcher.py:110-122  (c2, c1) of the exact line search; L may be NULL. */
int goat_line_search_coeffs(goat_handle *h, int64_t n, const double *A, int64_t lda,
                            const double *B, int64_t ldb, const double *L, int64_t ldl,
                            const double *P, int64_t ldp, const double *Q, int64_t ldq,
                            double *c2, double *c1);

/* lap.py:48-58  solve_lap(M, sense): exact LAP on device (certificate fast
 * path, else the shortest-augmenting-path solver with scipy's visiting order). */
int goat_lap(goat_handle *h, int64_t n, const double *M, int64_t ldm, int32_t sense,
             int64_t *assignment, double *objective, int32_t *certified);

/* core.py:120-124  sum_ij A_ij B_{p(i) p(j)} (fp64, fixed reduction order). */
int goat_qap_objective_perm(goat_handle *h, int64_t n, const double *A, int64_t lda,
                            const double *B, int64_t ldb, const int64_t *perm,
                            double *objective);

/* Run subsequent work of this handle on `stream` (a cudaStream_t; NULL = the
 * handle's own stream).  Lets a caller bracket calls with its own CUDA events. */
int goat_set_stream(goat_handle *h, void *stream);

/* Measurement hook (bench.py roofline): `reps` back-to-back launches of the
 * fused Sinkhorn sweep kernel over the device matrix G (handle precision,
 * leading dim ld) at a mid-run sweep index; *ms_per_sweep = mean kernel time
 * from CUDA events on the handle's stream.  Algorithmic bytes per launch = n*n*elem. */
int goat_bench_sweep(goat_handle *h, int64_t n, const void *dG, int64_t ld, int32_t reps,
                     double *ms_per_sweep);

/* Measurement hook (bench.py GEMM TFLOP/s): the gradient A X B^T + A^T X B on
 * device matrices (handle precision, leading dim = n) `reps` times after one
 * untimed preparation; *ms = mean time per gradient (CUDA events), *products =
 * number of n^3 products it performed (2 symmetric, 4 directed), *terms = bf16
 * split terms issued per product on the tcgen05 path (0 on the SIMT path). */
int goat_bench_gradient(goat_handle *h, int64_t n, const void *dA, const void *dB, const void *dX,
                        int32_t reps, double *ms, int32_t *products, int32_t *terms);

/* lap.py:48-58 on a device matrix (handle precision, leading dim ldm); the
 * final projection of the row-sharded driver after it gathers G. */
int goat_lap_device(goat_handle *h, int64_t n, const void *dM, int64_t ldm, int32_t sense,
                    int64_t *assignment, double *objective, int32_t *certified);

/* ---- Row-sharded primitives (one process per GPU) ----------
 * The reference has no distributed path; these split _fw_core's per-iteration
 * work (matcher.py:177-212) by row blocks.  A rank owns rows [r0, r0+m) of the
 * n x n iterates P, Q, G; every block buffer is m x ld and full matrices are
 * n x ld with ld = round_up(n, 8) (device, handle precision).  The caller runs
 * the collectives between the calls (paper_2111_05366_b200/sharded.py: NCCL
 * through torch.distributed):
 *   gradient      all-gather Q -> goat_shard_gradient
 *   Sinkhorn      per sweep: goat_shard_lot_pass -> all-gather the (n+1)-vector
 *                 -> goat_shard_lot_merge (identical on every rank)
 *   line search   goat_shard_dots -> sum-allreduce of 6 doubles
 *   final LAP     all-gather G -> goat_lap_device.
 * dAT_rows = NULL declares A and B symmetric (G = 2 A Q B). */
int goat_shard_setup(goat_handle *h, int64_t n, int64_t m, const void *dA_rows, const void *dAT_rows,
                     const void *dB, int64_t ld);
/* G_r = (A_r Q) B^T + (A^T_r Q) B from the gathered Q (n x ld). */
/* Row-sharded setup on CSR adjacency (device pointers, values of the handle's
 * element type or NULL): this rank's m rows of A and of A^T (global column
 * indices; rowptr[0] = 0), and the whole B and B^T.  A^T rows and B^T are NULL
 * together for symmetric inputs.  The gradient then runs as SpMMs. */
int goat_shard_setup_csr(goat_handle *h, int64_t n, int64_t m, const goat_csr *dA_rows,
                         const goat_csr *dAT_rows, const goat_csr *dB, const goat_csr *dBT);
int goat_shard_gradient(goat_handle *h, const void *dQ_full, void *dOut_rows);
/* local (min, max) of a block (the LOT scale is global: min/max-allreduce). */
int goat_shard_minmax(goat_handle *h, const void *dX_rows, double *out2);
/* sinkhorn.py:103-130 set-up from the GLOBAL min/max of the cost. */
int goat_shard_lot_begin(goat_handle *h, int32_t sense, double lam, double gmin, double gmax,
                         int32_t max_sweeps, double tol);
/* one pass over the block: dSend[0..n) = fp64 column sums, dSend[n] = max row deviation.
 * No-op once the loop has stopped. */
int goat_shard_lot_pass(goat_handle *h, const void *dG_rows, double *dSend);
/* merge the gathered dRecv[world][n+1] in rank order: stopping rule + new column potentials.
 * A column sum that under/overflows leaves the sweep pending (passes and merges
 * are no-ops) until the repair round below has run. */
int goat_shard_lot_merge(goat_handle *h, const double *dRecv, int32_t world);
/* repair round: exact fp64 (max, sumexp) pairs of the flagged columns over the
 * block -> dPairs[2n]; all-gather; rank-order combine that finishes the sweep
 * (the multi-GPU form of the single-GPU exact column LSE). */
int goat_shard_lot_repair_pass(goat_handle *h, const void *dG_rows, double *dPairs);
int goat_shard_lot_repair_merge(goat_handle *h, const double *dRecvPairs, int32_t world);
/* loop state (synchronises): done, sweeps, converged, deviation, columns repaired so far,
 * repair round pending. */
int goat_shard_lot_status(goat_handle *h, int32_t *done, int32_t *sweeps, int32_t *converged,
                          double *deviation, int32_t *repaired, int32_t *pending);
/* fp32 handles: once the fp32 sweeps have stopped at the fp32 deviation floor (tol
 * below it), widen the block to fp64 and re-open the loop so passes/merges go on
 * in fp64 arithmetic from the same potentials (*started = 1); otherwise a no-op
 * (*started = 0).  Identical decision on every rank (the loop state is). */
int goat_shard_lot_refine(goat_handle *h, const void *dG_rows, int32_t *started);
/* Q_r = exp(E + f + g) of the returned iterate (1/n when the cost was constant). */
int goat_shard_lot_emit(goat_handle *h, const void *dG_rows, void *dQ_rows);
/* local line-search sums of goat_fw_core's dots: <GQ,D>, <GP-GQ,D>, <GQ,Q>, |D|^2, 0, 0 (D = P - Q). */
int goat_shard_dots(goat_handle *h, const void *GP, const void *GQ, const void *P, const void *Q,
                    double *out6);
/* Y = a X + b Y on a block (matcher.py:197); fill a block with a constant (core.py:89-93). */
int goat_shard_axpby(goat_handle *h, double a, const void *dX_rows, double b, void *dY_rows);
int goat_shard_fill(goat_handle *h, double value, void *dX_rows);

/* Library build/feature string, e.g. "goat sm_100a tcgen05". */
const char *goat_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GOAT_H */
