// CUDA-core GEMM for the gradient products (matcher.py:107): used for the
// fp64 mode (the reference's arithmetic; fp64 tensor cores are not a B200
// lever for this shape) and as the fp32 fallback engine.  The fp32 hot path
// is the tcgen05 GEMM in gemm_tc.cu.
#include "kernels.cuh"

namespace goat {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <class T>
__global__ void __launch_bounds__(256) gemm_simt_kernel(int M, int N, int K, T alpha, const T *A,
                                                        int64_t lda, int tA, const T *B, int64_t ldb,
                                                        int tB, T beta, T *C, int64_t ldc) {
    __shared__ T As[BK][BM + 1];
    __shared__ T Bs[BK][BN + 1];
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
    for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            const int idx = tid + 256 * l;
            int m, k;
            if (!tA) { m = idx / BK; k = idx % BK; } else { m = idx % BM; k = idx / BM; }
            const int gm = m0 + m;
            int gk = k0 + k;
            T v = T(0);
            if (gm < M && gk < K) v = tA ? A[(int64_t)gk * lda + gm] : A[(int64_t)gm * lda + gk];
            As[k][m] = v;
            int n;
            if (!tB) { n = idx % BN; k = idx / BN; } else { n = idx / BK; k = idx % BK; }
            const int gn = n0 + n;
            gk = k0 + k;
            v = T(0);
            if (gn < N && gk < K) v = tB ? B[(int64_t)gn * ldb + gk] : B[(int64_t)gk * ldb + gn];
            Bs[k][n] = v;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            T a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[k][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gm = m0 + ty + 16 * i, gn = n0 + tx + 16 * j;
            if (gm < M && gn < N) {
                T *c = C + (int64_t)gm * ldc + gn;
                *c = (beta == T(0)) ? alpha * acc[i][j] : alpha * acc[i][j] + beta * *c;
            }
        }
}

}  // namespace

template <class T>
void gemm_simt(int m, int n, int k, double alpha, const T *A, int64_t lda, int transA, const T *B,
               int64_t ldb, int transB, double beta, T *C, int64_t ldc, cudaStream_t s) {
    dim3 grid(ceil_div(n, BN), ceil_div(m, BM));
    gemm_simt_kernel<T><<<grid, 256, 0, s>>>(m, n, k, (T)alpha, A, lda, transA, B, ldb, transB,
                                             (T)beta, C, ldc); note_launch();
    GOAT_CHECK_LAUNCH();
}

template void gemm_simt<float>(int, int, int, double, const float *, int64_t, int, const float *,
                               int64_t, int, double, float *, int64_t, cudaStream_t);
template void gemm_simt<double>(int, int, int, double, const double *, int64_t, int, const double *,
                                int64_t, int, double, double *, int64_t, cudaStream_t);

}  // namespace goat
