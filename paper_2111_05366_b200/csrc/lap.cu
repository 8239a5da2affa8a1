// Exact linear assignment on the device (final projection, matcher.py:211).
//
// Reference: lap.py:48-58 -> scipy.optimize.linear_sum_assignment (lap.py:55),
// a shortest-augmenting-path LSAP (Crouse 2016; restated in oracle/lsap.c).
//
// 1. Certificate (O(n^2), fully parallel): if every row's best column is
//    strictly better than the rest and those columns form a permutation, that
//    permutation attains sum_i max_j M_ij, an upper bound over all assignments,
//    so it is the unique optimum -- any exact solver, scipy included, returns it.
// 2. Otherwise one persistent CTA runs the same shortest-augmenting-path
//    search scipy runs, in the same visiting order ("remaining" list filled in
//    reverse and compacted by swap-removal; ties on the minimum resolved to the
//    last free column in scan order, else the first), with the per-step column
//    scan and argmin parallel across 1024 threads.  Identical fp64 operations in
//    identical order give scipy's assignment bit-for-bit, ties included.
//    No CPU fallback exists.
#include <climits>

#include "kernels.cuh"

namespace goat {
namespace {

template <class T>
__global__ void lap_cert_rows(const T *M, int64_t ld, int n, int maximize, int *cand, int *hits,
                              int *flag) {
    const int warps = blockDim.x / 32;
    const int lane = threadIdx.x & 31;
    for (int i = blockIdx.x * warps + threadIdx.x / 32; i < n; i += gridDim.x * warps) {
        const T *Mi = M + (int64_t)i * ld;
        double best = maximize ? -INFINITY : INFINITY;
        int idx = INT_MAX, cnt = 0;
        for (int j = lane; j < n; j += 32) {
            const double x = (double)Mi[j];
            const bool better = maximize ? (x > best) : (x < best);
            if (better) { best = x; idx = j; cnt = 1; }
            else if (x == best) { cnt += 1; idx = min(idx, j); }
        }
        for (int off = 16; off > 0; off >>= 1) {
            const double b2 = __shfl_xor_sync(0xffffffffu, best, off);
            const int i2 = __shfl_xor_sync(0xffffffffu, idx, off);
            const int c2 = __shfl_xor_sync(0xffffffffu, cnt, off);
            const bool better = maximize ? (b2 > best) : (b2 < best);
            if (better) { best = b2; idx = i2; cnt = c2; }
            else if (b2 == best) { cnt += c2; idx = min(idx, i2); }
        }
        if (lane == 0) {
            cand[i] = idx;
            if (cnt != 1) *flag = 0;
            else atomicAdd(&hits[idx], 1);
        }
    }
}

__global__ void lap_cert_cols(const int *hits, int n, int *flag) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        if (hits[j] != 1) *flag = 0;
}

struct Best {
    double v;
    int first;
    int lastfree;
};

__device__ __forceinline__ void best_merge(Best &a, const Best &b) {
    if (b.v < a.v) a = b;
    else if (b.v == a.v) {
        a.first = min(a.first, b.first);
        a.lastfree = max(a.lastfree, b.lastfree);
    }
}

constexpr int kLapThreads = 1024;

template <class T>
__global__ void __launch_bounds__(kLapThreads, 1)
    lap_sap_kernel(const T *M, int64_t ld, int n, double sign, LapWork w, int use_smem) {
    extern __shared__ __align__(16) unsigned char smem[];
    double *spc = w.spc, *v = w.v;
    int *path = w.path, *row4col = w.row4col, *rem = w.rem;
    unsigned char *SC = w.SC;
    if (use_smem) {
        spc = reinterpret_cast<double *>(smem);
        v = spc + n;
        path = reinterpret_cast<int *>(v + n);
        row4col = path + n;
        rem = row4col + n;
        SC = reinterpret_cast<unsigned char *>(rem + n);
    }
    double *u = w.u;
    int *col4row = w.col4row;
    unsigned char *SR = w.SR;
    __shared__ Best s_best[kLapThreads / 32];
    __shared__ int s_i, s_sink, s_nrem;
    __shared__ double s_minv;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (int j = tid; j < n; j += kLapThreads) {
        v[j] = 0.0; u[j] = 0.0; row4col[j] = -1; col4row[j] = -1; path[j] = -1;
    }
    __syncthreads();
    for (int cur = 0; cur < n; ++cur) {
        for (int it = tid; it < n; it += kLapThreads) {
            rem[it] = n - 1 - it; SR[it] = 0; SC[it] = 0; spc[it] = INFINITY;
        }
        if (tid == 0) { s_i = cur; s_sink = -1; s_nrem = n; s_minv = 0.0; }
        __syncthreads();
        for (;;) {
            const int i = s_i, nrem = s_nrem;
            const double minv = s_minv;
            const double ui = u[i];
            const T *Mi = M + (int64_t)i * ld;
            Best b{INFINITY, INT_MAX, -1};
            for (int it = tid; it < nrem; it += kLapThreads) {
                const int j = rem[it];
                // scipy: minVal + cost[i*nc+j] - u[i] - v[j], cost = -M when maximizing
                const double r = ((minv + sign * (double)Mi[j]) - ui) - v[j];
                double sj = spc[j];
                if (r < sj) { path[j] = i; spc[j] = r; sj = r; }
                if (sj < b.v) { b.v = sj; b.first = it; b.lastfree = (row4col[j] == -1) ? it : -1; }
                else if (sj == b.v && row4col[j] == -1) b.lastfree = it;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                Best o;
                o.v = __shfl_xor_sync(0xffffffffu, b.v, off);
                o.first = __shfl_xor_sync(0xffffffffu, b.first, off);
                o.lastfree = __shfl_xor_sync(0xffffffffu, b.lastfree, off);
                best_merge(b, o);
            }
            if (lane == 0) s_best[warp] = b;
            __syncthreads();
            if (tid == 0) {
                Best f = s_best[0];
                for (int q = 1; q < kLapThreads / 32; ++q) best_merge(f, s_best[q]);
                SR[i] = 1;
                if (!(f.v < INFINITY)) {
                    *w.status = -1;
                    s_sink = -2;
                } else {
                    const int index = f.lastfree >= 0 ? f.lastfree : f.first;
                    const int j = rem[index];
                    if (row4col[j] == -1) s_sink = j; else s_i = row4col[j];
                    SC[j] = 1;
                    rem[index] = rem[nrem - 1];
                    s_nrem = nrem - 1;
                    s_minv = f.v;
                }
            }
            __syncthreads();
            if (s_sink != -1) break;
        }
        if (s_sink == -2) return;
        const double minv = s_minv;
        // dual update (uses col4row before augmentation)
        for (int r = tid; r < n; r += kLapThreads) {
            if (SR[r] && r != cur) u[r] += minv - spc[col4row[r]];
            if (SC[r]) v[r] -= minv - spc[r];
        }
        __syncthreads();
        if (tid == 0) {
            u[cur] += minv;
            int j = s_sink;
            for (;;) {
                const int r = path[j];
                row4col[j] = r;
                const int t = col4row[r];
                col4row[r] = j;
                j = t;
                if (r == cur) break;
            }
        }
        __syncthreads();
    }
    if (tid == 0) *w.status = 0;
}

}  // namespace

template <class T>
void launch_lap_certificate(const T *M, int64_t ld, int n, int sense, int *cand, int *hits, int *flag,
                            cudaStream_t s) {
    GOAT_CUDA(cudaMemsetAsync(hits, 0, sizeof(int) * n, s));
    const int one = 1;
    GOAT_CUDA(cudaMemcpyAsync(flag, &one, sizeof(int), cudaMemcpyHostToDevice, s));
    const int wpb = 8;
    lap_cert_rows<T><<<std::min(ceil_div(n, wpb), 2048), 32 * wpb, 0, s>>>(M, ld, n, sense == GOAT_MAXIMIZE, cand,
                                                                            hits, flag); note_launch();
    lap_cert_cols<<<std::min(ceil_div(n, 256), 1024), 256, 0, s>>>(hits, n, flag); note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T>
void launch_lap_sap(const T *M, int64_t ld, int n, int sense, const LapWork &w, cudaStream_t s) {
    const size_t smem = (size_t)n * (8 + 8 + 4 + 4 + 4 + 1) + 16;
    int use_smem = smem <= 200 * 1024;
    if (use_smem)
        GOAT_CUDA(cudaFuncSetAttribute(lap_sap_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const double sign = (sense == GOAT_MAXIMIZE) ? -1.0 : 1.0;
    lap_sap_kernel<T><<<1, kLapThreads, use_smem ? smem : 0, s>>>(M, ld, n, sign, w, use_smem); note_launch();
    GOAT_CHECK_LAUNCH();
}

template void launch_lap_certificate<float>(const float *, int64_t, int, int, int *, int *, int *, cudaStream_t);
template void launch_lap_certificate<double>(const double *, int64_t, int, int, int *, int *, int *, cudaStream_t);
template void launch_lap_sap<float>(const float *, int64_t, int, int, const LapWork &, cudaStream_t);
template void launch_lap_sap<double>(const double *, int64_t, int, int, const LapWork &, cudaStream_t);

}  // namespace goat
