// Element-wise and reduction kernels of the GOAT iteration (HBM-bound).
//
// All reductions are two-stage with a fixed grid (kRedBlocks) and a fixed
// combine order, so results are bit-reproducible run to run -- the
// reference's determinism contract (test_matcher.py:160-170).
#include "kernels.cuh"

namespace goat {
namespace {

template <int NV>
__device__ void block_sum(double (&v)[NV], double *out /* NV, thread 0 only */) {
    __shared__ double s[NV][kThreads / 32];
#pragma unroll
    for (int q = 0; q < NV; ++q)
        for (int off = 16; off > 0; off >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], off);
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int q = 0; q < NV; ++q) s[q][threadIdx.x >> 5] = v[q];
    __syncthreads();
    if (threadIdx.x == 0)
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            double t = 0.0;
            for (int w = 0; w < kThreads / 32; ++w) t += s[q][w];
            out[q] = t;
        }
}

// Stage 2: one block sums `nb` partial vectors of width NV in fixed order.
template <int NV>
__global__ void finish_sum_kernel(const double *part, int nb, double *out) {
    double v[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = 0.0;
    // fixed per-thread order, then fixed tree: deterministic
    for (int b = threadIdx.x; b < nb; b += kThreads)
#pragma unroll
        for (int q = 0; q < NV; ++q) v[q] += part[b * NV + q];
    double r[NV];
    block_sum<NV>(v, r);
    if (threadIdx.x == 0)
#pragma unroll
        for (int q = 0; q < NV; ++q) out[q] = r[q];
}

template <class T>
__global__ void minmax_kernel(const T *X, int64_t ld, int n, int rows, double *part) {
    __shared__ double smin[kThreads / 32], smax[kThreads / 32];
    double lo = INFINITY, hi = -INFINITY;
    for (int i = blockIdx.x; i < rows; i += gridDim.x)
        for (int j = threadIdx.x; j < n; j += kThreads) {
            double x = (double)X[(int64_t)i * ld + j];
            lo = fmin(lo, x);
            hi = fmax(hi, x);
        }
    for (int off = 16; off > 0; off >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, off));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, off));
    }
    if ((threadIdx.x & 31) == 0) { smin[threadIdx.x >> 5] = lo; smax[threadIdx.x >> 5] = hi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 0; w < kThreads / 32; ++w) { lo = fmin(lo, smin[w]); hi = fmax(hi, smax[w]); }
        part[blockIdx.x * 2] = lo;
        part[blockIdx.x * 2 + 1] = hi;
    }
}

__global__ void minmax_finish_kernel(const double *part, int nb, double *out) {
    if (threadIdx.x) return;
    double lo = INFINITY, hi = -INFINITY;
    for (int b = 0; b < nb; ++b) { lo = fmin(lo, part[2 * b]); hi = fmax(hi, part[2 * b + 1]); }
    out[0] = lo;
    out[1] = hi;
}

// Line-search dots in difference form (D = P - Q formed per element, as the
// reference forms it at matcher.py:117, so small steps keep their sign):
//   [0] <GQ, D>   [1] <GP - GQ, D>   [2] <GQ, Q>   [3] |D|^2   [4] <L, D>   [5] <L, Q>
template <class T>
__global__ void fw_dots_kernel(const T *GP, const T *GQ, const T *P, const T *Q, const T *L, int64_t ld,
                               int n, int rows, double *part) {
    double v[6] = {0, 0, 0, 0, 0, 0};
    for (int i = blockIdx.x; i < rows; i += gridDim.x)
        for (int j = threadIdx.x; j < n; j += kThreads) {
            const int64_t o = (int64_t)i * ld + j;
            const double gq = GQ[o], gp = GP[o], q = Q[o];
            const double d = (double)P[o] - q;
            v[0] += gq * d;
            v[1] += (gp - gq) * d;
            v[2] += gq * q;
            v[3] += d * d;
            if (L) { const double l = L[o]; v[4] += l * d; v[5] += l * q; }
        }
    double r[6];
    block_sum<6>(v, r);
    if (threadIdx.x == 0)
        for (int q = 0; q < 6; ++q) part[blockIdx.x * 6 + q] = r[q];
}

__global__ void qap_perm_kernel(const double *A, int64_t lda, const double *B, int64_t ldb,
                                const int *perm, int n, double *part) {
    double v[1] = {0.0};
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const double *Bi = B + (int64_t)perm[i] * ldb;
        const double *Ai = A + (int64_t)i * lda;
        for (int j = threadIdx.x; j < n; j += kThreads) v[0] += Ai[j] * Bi[perm[j]];
    }
    double r[1];
    block_sum<1>(v, r);
    if (threadIdx.x == 0) part[blockIdx.x] = r[0];
}

template <class T>
__global__ void convert_kernel(const double *src, int64_t lds, T *dst, int64_t ldd, int n,
                               double scale, int *nonfinite) {
    bool bad = false;
    for (int i = blockIdx.x; i < n; i += gridDim.x)
        for (int j = threadIdx.x; j < ldd; j += kThreads) {
            const double x = (j < n) ? src[(int64_t)i * lds + j] : 0.0;
            bad |= !isfinite(x);
            dst[(int64_t)i * ldd + j] = (j < n) ? (T)(scale * x) : T(0);
        }
    if (nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) *nonfinite = 1;
}

template <class T>
__global__ void convert_to_f64_kernel(const T *src, int64_t lds, double *dst, int64_t ldd, int n, int rows) {
    for (int i = blockIdx.x; i < rows; i += gridDim.x)
        for (int j = threadIdx.x; j < n; j += kThreads) dst[(int64_t)i * ldd + j] = (double)src[(int64_t)i * lds + j];
}

template <class T>
__global__ void fill_kernel(T *dst, int64_t ld, int n, int rows, T value) {
    for (int i = blockIdx.x; i < rows; i += gridDim.x)
        for (int j = threadIdx.x; j < ld; j += kThreads) dst[(int64_t)i * ld + j] = (j < n) ? value : T(0);
}

template <class T>
__global__ void axpby_kernel(T a, const T *X, T b, T *Y, int64_t ld, int n, int rows) {
    for (int i = blockIdx.x; i < rows; i += gridDim.x)
        for (int j = threadIdx.x; j < n; j += kThreads) {
            const int64_t o = (int64_t)i * ld + j;
            Y[o] = a * X[o] + b * Y[o];
        }
}

template <class T>
__global__ void perm_matrix_kernel(const int *perm, T *Q, int64_t ld, int n) {
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const int pi = perm[i];
        for (int j = threadIdx.x; j < ld; j += kThreads) Q[(int64_t)i * ld + j] = (j == pi) ? T(1) : T(0);
    }
}

template <class T>
__global__ void add_kernel(const T *X, const T *L, T *Y, int64_t ld, int n, int rows) {
    for (int i = blockIdx.x; i < rows; i += gridDim.x)
        for (int j = threadIdx.x; j < n; j += kThreads) {
            const int64_t o = (int64_t)i * ld + j;
            Y[o] = X[o] + L[o];
        }
}

// Row sums (and column sums) of A and B in fp64: vec = [ra | ca | rb | cb].
template <class T>
__global__ void rowcol_sums_kernel(const T *A, int64_t lda, int n, double *rs, double *cs) {
    // one block per row for row sums; one thread per column for column sums
    __shared__ double s[kThreads / 32];
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        double v = 0.0;
        for (int j = threadIdx.x; j < n; j += kThreads) v += (double)A[(int64_t)i * lda + j];
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < kThreads / 32; ++w) t += s[w];
            rs[i] = t;
        }
        __syncthreads();
    }
    for (int j = blockIdx.x * kThreads + threadIdx.x; j < n; j += gridDim.x * kThreads) {
        double v = 0.0;
        for (int i = 0; i < n; ++i) v += (double)A[(int64_t)i * lda + j];
        cs[j] = v;
    }
}

template <class T>
__global__ void bary_grad_kernel(const double *ra, const double *ca, const double *rb,
                                 const double *cb, T *G, int64_t ldg, int n) {
    const double inv = 1.0 / (double)n;
    for (int i = blockIdx.x; i < n; i += gridDim.x)
        for (int j = threadIdx.x; j < ldg; j += kThreads)
            G[(int64_t)i * ldg + j] = (j < n) ? (T)((ra[i] * rb[j] + ca[i] * cb[j]) * inv) : T(0);
}

template <class T>
__global__ void symmetric_kernel(const T *X, int64_t ld, int n, int *flag) {
    for (int i = blockIdx.x; i < n; i += gridDim.x)
        for (int j = threadIdx.x; j < i; j += kThreads)
            if (X[(int64_t)i * ld + j] != X[(int64_t)j * ld + i]) *flag = 0;
}

template <class T>
__global__ void neglog_kernel(const T *X, int64_t ldx, T *Y, int64_t ldy, int n, int *bad) {
    for (int i = blockIdx.x; i < n; i += gridDim.x)
        for (int j = threadIdx.x; j < ldy; j += kThreads) {
            if (j >= n) { Y[(int64_t)i * ldy + j] = T(0); continue; }
            T x = X[(int64_t)i * ldx + j];
            if (!(x > T(0))) *bad = 1;
            Y[(int64_t)i * ldy + j] = -log(x);
        }
}

}  // namespace

template <class T>
void launch_minmax(const T *X, int64_t ld, int n, double *part, double *out2, cudaStream_t s, int rows) {
    minmax_kernel<T><<<kRedBlocks, kThreads, 0, s>>>(X, ld, n, rows < 0 ? n : rows, part); note_launch();
    minmax_finish_kernel<<<1, 32, 0, s>>>(part, kRedBlocks, out2); note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T>
void launch_fw_dots(const T *GP, const T *GQ, const T *P, const T *Q, const T *L, int64_t ld, int n,
                    double *part, double *out6, cudaStream_t s, int rows) {
    fw_dots_kernel<T><<<kRedBlocks, kThreads, 0, s>>>(GP, GQ, P, Q, L, ld, n, rows < 0 ? n : rows, part); note_launch();
    finish_sum_kernel<6><<<1, kThreads, 0, s>>>(part, kRedBlocks, out6); note_launch();
    GOAT_CHECK_LAUNCH();
}

void launch_qap_perm(const double *A, int64_t lda, const double *B, int64_t ldb, const int *perm,
                     int n, double *part, double *out, cudaStream_t s) {
    qap_perm_kernel<<<kRedBlocks, kThreads, 0, s>>>(A, lda, B, ldb, perm, n, part); note_launch();
    finish_sum_kernel<1><<<1, kThreads, 0, s>>>(part, kRedBlocks, out); note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T>
void launch_convert(const double *src, int64_t lds, T *dst, int64_t ldd, int n, double scale,
                    cudaStream_t s, int *nonfinite) {
    convert_kernel<T><<<std::min(n, 4096), kThreads, 0, s>>>(src, lds, dst, ldd, n, scale, nonfinite); note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T>
void launch_convert_to_f64(const T *src, int64_t lds, double *dst, int64_t ldd, int n, cudaStream_t s, int rows) {
    if (rows < 0) rows = n;
    convert_to_f64_kernel<T><<<std::max(1, std::min(rows, 4096)), kThreads, 0, s>>>(src, lds, dst, ldd, n, rows); note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T> void launch_fill(T *dst, int64_t ld, int n, double value, cudaStream_t s, int rows) {
    if (rows < 0) rows = n;
    fill_kernel<T><<<std::max(1, std::min(rows, 4096)), kThreads, 0, s>>>(dst, ld, n, rows, (T)value); note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T>
void launch_axpby(double a, const T *X, double b, T *Y, int64_t ld, int n, cudaStream_t s, int rows) {
    if (rows < 0) rows = n;
    axpby_kernel<T><<<std::max(1, std::min(rows, 4096)), kThreads, 0, s>>>((T)a, X, (T)b, Y, ld, n, rows); note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T> void launch_perm_matrix(const int *perm, T *Q, int64_t ld, int n, cudaStream_t s) {
    perm_matrix_kernel<T><<<std::min(n, 4096), kThreads, 0, s>>>(perm, Q, ld, n); note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T> void launch_add(const T *X, const T *L, T *Y, int64_t ld, int n, cudaStream_t s, int rows) {
    if (rows < 0) rows = n;
    add_kernel<T><<<std::max(1, std::min(rows, 4096)), kThreads, 0, s>>>(X, L, Y, ld, n, rows); note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T>
void launch_bary_grad(const T *A, int64_t lda, const T *B, int64_t ldb, T *G, int64_t ldg, int n,
                      double *vec4n, cudaStream_t s) {
    double *ra = vec4n, *ca = vec4n + n, *rb = vec4n + 2 * n, *cb = vec4n + 3 * n;
    const int nb = std::min(n, 1024);
    rowcol_sums_kernel<T><<<nb, kThreads, 0, s>>>(A, lda, n, ra, ca); note_launch();
    rowcol_sums_kernel<T><<<nb, kThreads, 0, s>>>(B, ldb, n, rb, cb); note_launch();
    bary_grad_kernel<T><<<std::min(n, 4096), kThreads, 0, s>>>(ra, ca, rb, cb, G, ldg, n); note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T> void launch_bary_grad_vec(const double *vec4n, T *G, int64_t ldg, int n, cudaStream_t s) {
    bary_grad_kernel<T><<<std::min(n, 4096), kThreads, 0, s>>>(vec4n, vec4n + n, vec4n + 2 * n, vec4n + 3 * n, G,
                                                                 ldg, n);
    note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T> void launch_is_symmetric(const T *X, int64_t ld, int n, int *flag, cudaStream_t s) {
    symmetric_kernel<T><<<std::min(n, 4096), kThreads, 0, s>>>(X, ld, n, flag); note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T>
void launch_neglog(const T *X, int64_t ldx, T *Y, int64_t ldy, int n, int *bad, cudaStream_t s) {
    neglog_kernel<T><<<std::min(n, 4096), kThreads, 0, s>>>(X, ldx, Y, ldy, n, bad); note_launch();
    GOAT_CHECK_LAUNCH();
}

#define GOAT_INST(T)                                                                                \
    template void launch_minmax<T>(const T *, int64_t, int, double *, double *, cudaStream_t, int);   \
    template void launch_fw_dots<T>(const T *, const T *, const T *, const T *, const T *, int64_t, int, \
                                    double *, double *, cudaStream_t, int);                          \
    template void launch_convert<T>(const double *, int64_t, T *, int64_t, int, double, cudaStream_t, int *); \
    template void launch_convert_to_f64<T>(const T *, int64_t, double *, int64_t, int, cudaStream_t, int); \
    template void launch_fill<T>(T *, int64_t, int, double, cudaStream_t, int);                      \
    template void launch_axpby<T>(double, const T *, double, T *, int64_t, int, cudaStream_t, int);  \
    template void launch_perm_matrix<T>(const int *, T *, int64_t, int, cudaStream_t);               \
    template void launch_add<T>(const T *, const T *, T *, int64_t, int, cudaStream_t, int);         \
    template void launch_bary_grad<T>(const T *, int64_t, const T *, int64_t, T *, int64_t, int,     \
                                      double *, cudaStream_t);                                       \
    template void launch_is_symmetric<T>(const T *, int64_t, int, int *, cudaStream_t);              \
    template void launch_bary_grad_vec<T>(const double *, T *, int64_t, int, cudaStream_t);          \
    template void launch_neglog<T>(const T *, int64_t, T *, int64_t, int, int *, cudaStream_t);
GOAT_INST(float)
GOAT_INST(double)
#undef GOAT_INST

}  // namespace goat
