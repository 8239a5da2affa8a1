// LOT / Sinkhorn on B200: fused log-domain sweep kernels.
//
// Reference: sinkhorn.py:103-130 (lot), :60-85 (sinkhorn_knopp), :88-100
// (_sinkhorn_log).  Potentials f = log u, g = log v are carried in fp64; the
// per-element arithmetic runs in the handle's precision (fp32 uses exp2 on the
// SFU with log2(e)-scaled potentials, fp64 uses exp).
//
// One "pass" k reads every element of G exactly once from HBM/L2:
//   * row phase   f_k = -LSE_j(E_ij + g_{k-1,j})      (each CTA owns whole rows)
//     dev_{k-1}  = max_i |expm1(f_{k-1,i} - f_{k,i})| = max|u_{k-1} K v_{k-1} - 1|
//   * column phase, on the same registers: colpart[cta][j] = sum_i exp(E_ij + g_{k-1,j} + f_{k,i})
// A merge kernel turns the column partials into g_k = g_{k-1} - log(sum), and its
// last CTA applies the reference's stopping rule, so a converged loop turns every
// later pass into a no-op without a host round trip.  Pass 0 is the reference's
// marginal pre-check of K itself (sinkhorn.py:70-72); pass max_sweeps+1 is
// row-only and produces the deviation of the final iterate.  The returned
// iterate is exp(E + f_{s} + g_{s}) for the stopping sweep s -- the same u that
// produced the reported deviation (sinkhorn.py:84-85).
#include "kernels.cuh"

namespace goat {
namespace {

template <class T> struct VecT;
template <> struct VecT<float> { using V = float4; static constexpr int W = 4; };
template <> struct VecT<double> { using V = double2; static constexpr int W = 2; };

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Scaled exponential: fp32 works in log2 units, fp64 in natural units.
template <class T> struct SkMath;
template <> struct SkMath<float> {
    static constexpr double kScale = 1.4426950408889634;  // log2(e)
    __device__ static float ex(float x) { return ex2f(x); }
    __device__ static double lg(double x) { return log2(x); }
    __device__ static double exd(double x) { return exp2(x); }
};
template <> struct SkMath<double> {
    static constexpr double kScale = 1.0;
    __device__ static double ex(double x) { return exp(x); }
    __device__ static double lg(double x) { return log(x); }
    __device__ static double exd(double x) { return exp(x); }
};

template <class T> __device__ __forceinline__ T neg_inf();
template <> __device__ __forceinline__ float neg_inf<float>() { return -INFINITY; }
template <> __device__ __forceinline__ double neg_inf<double>() { return -INFINITY; }

// (m, s) log-sum-exp pair combine; -inf safe.
template <class T>
__device__ __forceinline__ void lse_combine(T &m, T &s, T m2, T s2) {
    T M = m > m2 ? m : m2;
    if (M == neg_inf<T>()) return;
    T a = (m == neg_inf<T>()) ? T(0) : s * SkMath<T>::ex(m - M);
    T b = (m2 == neg_inf<T>()) ? T(0) : s2 * SkMath<T>::ex(m2 - M);
    m = M;
    s = a + b;
}

template <class T, int CH, int R>
__global__ void __launch_bounds__(kThreads, 2) sk_pass_kernel(SkArgs a) {
    using V = typename VecT<T>::V;
    constexpr int VW = VecT<T>::W;
    constexpr int NW = kThreads / 32;
    __shared__ int s_k, s_done;
    __shared__ T s_m[NW][R], s_s[NW][R];
    __shared__ double s_lse[R];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        s_k = *(volatile int *)&a.st->k;
        s_done = *(volatile int *)&a.st->done;
    }
    __syncthreads();
    if (s_done) return;
    const int k = s_k;
    const int n = a.n;
    const bool pre = (k == 0);
    const bool rowonly = (k == a.st->max_sweeps + 1);
    // ring slots (selected, not indexed, so SkArgs stays in the constant bank)
    const double *gin = (k & 1) ? a.g[0] : a.g[1];  // slot of g_{k-1}
    const double *fprev = (k & 1) ? a.f[0] : a.f[1];
    double *fout = (k & 1) ? a.f[1] : a.f[0];
    const T *G = static_cast<const T *>(a.G);
    const double ks = SkMath<T>::kScale;
    const T coef = (T)(a.st->coef * ks);
    const T gmax = (T)a.st->gmax;

    // Per-thread columns: chunks q = tid + kThreads*c, columns q*VW .. q*VW+VW-1.
    T gl[CH][VW], acc[CH][VW];
#pragma unroll
    for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int e = 0; e < VW; ++e) {
            int col = (tid + kThreads * c) * VW + e;
            gl[c][e] = (col < n && !pre) ? (T)(gin[col] * ks) : T(0);
            acc[c][e] = T(0);
        }

    double devmax = 0.0;
    const int nbands = (n + R - 1) / R;
    for (int band = blockIdx.x; band < nbands; band += gridDim.x) {
        const int r0 = band * R;
        T x[R][CH][VW];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int q = tid + kThreads * c;
                const int row = r0 + r;
                V v;
                if (row < n && q * VW < n)
                    v = __ldg(reinterpret_cast<const V *>(G + (int64_t)row * a.ld + (int64_t)q * VW));
                else
                    memset(&v, 0, sizeof(V));
                const T *pv = reinterpret_cast<const T *>(&v);
#pragma unroll
                for (int e = 0; e < VW; ++e) x[r][c][e] = pv[e];
            }
        T m[R], s[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const bool rv = (r0 + r) < n;
            m[r] = neg_inf<T>();
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int e = 0; e < VW; ++e) {
                    const int col = (tid + kThreads * c) * VW + e;
                    // E_ij = coef * (gmax - G_ij), reference order (sinkhorn.py:125)
                    T arg = (rv && col < n) ? coef * (gmax - x[r][c][e]) + gl[c][e] : neg_inf<T>();
                    x[r][c][e] = arg;
                    m[r] = arg > m[r] ? arg : m[r];
                }
            s[r] = T(0);
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int e = 0; e < VW; ++e) {
                    T arg = x[r][c][e];
                    T y = (arg == neg_inf<T>()) ? T(0) : SkMath<T>::ex(arg - m[r]);
                    x[r][c][e] = y;
                    s[r] += y;
                }
        }
        // Block-wide (m, s) combine per row: warp shuffles, then smem across warps.
#pragma unroll
        for (int r = 0; r < R; ++r) {
            T mm = m[r], ss = s[r];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                T m2 = __shfl_xor_sync(0xffffffffu, mm, off);
                T s2 = __shfl_xor_sync(0xffffffffu, ss, off);
                lse_combine(mm, ss, m2, s2);
            }
            if (lane == 0) { s_m[warp][r] = mm; s_s[warp][r] = ss; }
        }
        __syncthreads();
        if (tid < R) {
            const int row = r0 + tid;
            double M = -INFINITY;
            for (int w = 0; w < NW; ++w) M = fmax(M, (double)s_m[w][tid]);
            double S = 0.0;
            if (M != -INFINITY)
                for (int w = 0; w < NW; ++w)
                    if ((double)s_m[w][tid] != -INFINITY)
                        S += (double)s_s[w][tid] * SkMath<T>::exd((double)s_m[w][tid] - M);
            const double lse = M + SkMath<T>::lg(S);  // scaled units
            s_lse[tid] = lse;
            if (row < n) {
                const double fnew = -lse / ks;
                double dev = 0.0;
                if (pre) dev = fabs(expm1(-fnew));                 // |rowsum(K) - 1|
                else if (k >= 2) dev = fabs(expm1(fprev[row] - fnew));  // |u K v - 1|
                if (!pre) fout[row] = fnew;
                devmax = fmax(devmax, dev);
            }
        }
        __syncthreads();
        if (!rowonly) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (m[r] == neg_inf<T>()) continue;
                // column contribution y = x * exp(m + f_col), f_col = 0 on the pre-check
                const double colf = pre ? 0.0 : -s_lse[r];
                const T sc = SkMath<T>::ex((T)((double)m[r] + colf));
#pragma unroll
                for (int c = 0; c < CH; ++c)
#pragma unroll
                    for (int e = 0; e < VW; ++e) acc[c][e] += x[r][c][e] * sc;
            }
        }
    }
    if (!rowonly) {
        T *cp = static_cast<T *>(a.colpart) + (int64_t)blockIdx.x * a.ldp;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int q = tid + kThreads * c;
            if (q * VW < n) {
                V v;
                T *pv = reinterpret_cast<T *>(&v);
#pragma unroll
                for (int e = 0; e < VW; ++e) pv[e] = acc[c][e];
                *reinterpret_cast<V *>(cp + (int64_t)q * VW) = v;
            }
        }
    }
    if (warp == 0) {
        for (int off = 16; off > 0; off >>= 1) devmax = fmax(devmax, __shfl_xor_sync(0xffffffffu, devmax, off));
        if (lane == 0) a.devpart[blockIdx.x] = devmax;
    }
}

// Exact column LSE for a column whose partial sum under/overflowed:
// g_j = -LSE_i(E_ij + f_i) over all rows (fp64).  Rare repair path.
template <class T>
__device__ double sk_exact_col(const SkArgs &a, int j, const double *f, bool pre) {
    const T *G = static_cast<const T *>(a.G);
    const double coef = a.st->coef, gmax = a.st->gmax;
    double M = -INFINITY;
    for (int i = 0; i < a.n; ++i) {
        double e = coef * (gmax - (double)G[(int64_t)i * a.ld + j]) + (pre ? 0.0 : f[i]);
        M = fmax(M, e);
    }
    double S = 0.0;
    for (int i = 0; i < a.n; ++i) {
        double e = coef * (gmax - (double)G[(int64_t)i * a.ld + j]) + (pre ? 0.0 : f[i]);
        S += exp(e - M);
    }
    return -(M + log(S));
}

template <class T>
__global__ void __launch_bounds__(kThreads) sk_merge_kernel(SkArgs a) {
    __shared__ int s_k, s_done, s_last;
    __shared__ double s_red[kThreads / 32];
    const int tid = threadIdx.x;
    if (tid == 0) {
        s_k = *(volatile int *)&a.st->k;
        s_done = *(volatile int *)&a.st->done;
    }
    __syncthreads();
    if (s_done) return;
    const int k = s_k, n = a.n;
    const int max_sweeps = a.st->max_sweeps;
    const double tol = a.st->tol;
    const bool pre = (k == 0);
    const bool rowonly = (k == max_sweeps + 1);
    const int j = blockIdx.x * kThreads + tid;
    double dloc = 0.0;
    if (j < n && !rowonly) {
        const T *cp = static_cast<const T *>(a.colpart);
        double S = 0.0;
        for (int b = 0; b < a.nblk; ++b) S += (double)cp[(int64_t)b * a.ldp + j];
        const double tiny = sizeof(T) == 4 ? 1e-30 : 1e-290;
        if (pre) {
            if (!(S > tiny)) S = exp(-sk_exact_col<T>(a, j, nullptr, true));
            dloc = fabs(S - 1.0);
        } else {
            const double gold = ((k & 1) ? a.g[0] : a.g[1])[j];
            double gnew = gold - log(S);
            if (!(S > tiny) || !isfinite(S)) {
                gnew = sk_exact_col<T>(a, j, (k & 1) ? a.f[1] : a.f[0], false);
                atomicAdd(&a.st->repaired, 1);
            }
            ((k & 1) ? a.g[1] : a.g[0])[j] = gnew;
        }
    }
    // block max of the column deviation (pre-check only)
    for (int off = 16; off > 0; off >>= 1) dloc = fmax(dloc, __shfl_xor_sync(0xffffffffu, dloc, off));
    if ((tid & 31) == 0) s_red[tid >> 5] = dloc;
    __syncthreads();
    if (tid == 0) {
        double d = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) d = fmax(d, s_red[w]);
        a.devcol[blockIdx.x] = d;
        __threadfence();
        int t = atomicAdd(&a.st->arrive, 1);
        s_last = (t == (int)gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last || tid != 0) return;
    __threadfence();
    // Last CTA: stopping rule of sinkhorn.py:70-72 / :82-85 (and :96-99 in log mode).
    double drow = 0.0, dcol = 0.0;
    for (int b = 0; b < a.nblk; ++b) drow = fmax(drow, __ldcg(&a.devpart[b]));
    for (int b = 0; b < (int)gridDim.x; ++b) dcol = fmax(dcol, __ldcg(&a.devcol[b]));
    SkState *st = a.st;
    st->arrive = 0;
    if (pre) {
        const double d0 = fmax(drow, dcol);
        st->last_dev = d0;
        if (d0 < tol) {  // K already balanced: return K itself, 0 sweeps
            st->done = 1; st->sweeps = 0; st->converged = 1; st->slot = 0; st->dev = d0;
        }
        st->k = 1;
        return;
    }
    if (k >= 2) {
        st->last_dev = drow;  // dev_{k-1}
        if (drow < tol) {
            st->done = 1; st->sweeps = k - 1; st->converged = 1; st->slot = (k - 1) & 1; st->dev = drow;
            return;
        }
        if (rowonly) {
            st->done = 1; st->sweeps = max_sweeps; st->converged = 0;
            st->slot = max_sweeps & 1; st->dev = drow;
            return;
        }
    }
    st->k = k + 1;
}

template <class T>
__global__ void __launch_bounds__(kThreads) sk_emit_kernel(SkArgs a, T *Q, int64_t ldq, const T *P,
                                                           int64_t ldp, const T *L, int64_t ldl,
                                                           double *part) {
    __shared__ double s_r[2][kThreads / 32];
    const int slot = a.st->slot;
    const double *f = slot ? a.f[1] : a.f[0], *g = slot ? a.g[1] : a.g[0];
    const T *G = static_cast<const T *>(a.G);
    const int n = a.n;
    double nrm = 0.0, lq = 0.0;
    const float ks = (float)SkMath<float>::kScale;
    const double coef = a.st->coef, gmax = a.st->gmax;
    const float coef2 = (float)(coef * SkMath<float>::kScale);
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const double fi = f[i];
        const T *Gi = G + (int64_t)i * a.ld;
        for (int j = threadIdx.x; j < n; j += kThreads) {
            T q;
            if (sizeof(T) == 8) {
                // exp(E + f + g), E in the reference's evaluation order
                const double e = coef * (gmax - (double)Gi[j]);
                q = (T)exp((e + fi) + g[j]);
            } else {
                const float e = coef2 * ((float)gmax - (float)Gi[j]);
                q = (T)ex2f(e + (float)((fi + g[j]) * ks));
            }
            Q[(int64_t)i * ldq + j] = q;
            if (P) { const double d = (double)q - (double)P[(int64_t)i * ldp + j]; nrm += d * d; }
            if (L) lq += (double)L[(int64_t)i * ldl + j] * (double)q;
        }
    }
    for (int off = 16; off > 0; off >>= 1) {
        nrm += __shfl_xor_sync(0xffffffffu, nrm, off);
        lq += __shfl_xor_sync(0xffffffffu, lq, off);
    }
    if ((threadIdx.x & 31) == 0) { s_r[0][threadIdx.x >> 5] = nrm; s_r[1][threadIdx.x >> 5] = lq; }
    __syncthreads();
    if (threadIdx.x == 0 && part) {
        double x = 0, y = 0;
        for (int w = 0; w < kThreads / 32; ++w) { x += s_r[0][w]; y += s_r[1][w]; }
        part[blockIdx.x * 4 + 0] = x;
        part[blockIdx.x * 4 + 1] = y;
    }
}

template <class T> constexpr int max_ch() { return 8; }
constexpr int rows_for(int ch) { return ch == 1 ? 8 : ch == 2 ? 4 : ch <= 4 ? 2 : 1; }

template <class T, int CH>
void launch_pass_ch(const SkArgs &a, const SkPlan &p, cudaStream_t s) {
    sk_pass_kernel<T, CH, rows_for(CH)><<<p.nblk, kThreads, 0, s>>>(a); note_launch();
}

}  // namespace

template <class T> SkPlan sk_plan(int n, int num_sms) {
    constexpr int VW = VecT<T>::W;
    SkPlan p;
    const int chunks = (n + VW - 1) / VW;
    p.ch = (chunks + kThreads - 1) / kThreads;
    if (p.ch > max_ch<T>())
        throw Error(GOAT_ENOTSUP, "sinkhorn: order " + std::to_string(n) +
                                      " exceeds the single-CTA row width of this build");
    p.rows = rows_for(p.ch);
    const int nbands = (n + p.rows - 1) / p.rows;
    p.nblk = std::max(1, std::min(nbands, num_sms));
    p.merge_blocks = (n + kThreads - 1) / kThreads;
    p.colpart_bytes = (size_t)p.nblk * round_up(n, 8) * sizeof(T);
    return p;
}

template <class T> void sk_launch_pass(const SkArgs &a, const SkPlan &p, cudaStream_t s) {
    switch (p.ch) {
        case 1: launch_pass_ch<T, 1>(a, p, s); break;
        case 2: launch_pass_ch<T, 2>(a, p, s); break;
        case 3: launch_pass_ch<T, 3>(a, p, s); break;
        case 4: launch_pass_ch<T, 4>(a, p, s); break;
        case 5: launch_pass_ch<T, 5>(a, p, s); break;
        case 6: launch_pass_ch<T, 6>(a, p, s); break;
        case 7: launch_pass_ch<T, 7>(a, p, s); break;
        case 8: launch_pass_ch<T, 8>(a, p, s); break;
        default: throw Error(GOAT_ENOTSUP, "sinkhorn: bad chunk count");
    }
    GOAT_CHECK_LAUNCH();
}

template <class T> void sk_launch_merge(const SkArgs &a, const SkPlan &p, cudaStream_t s) {
    sk_merge_kernel<T><<<p.merge_blocks, kThreads, 0, s>>>(a); note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T>
void sk_launch_emit(const SkArgs &a, T *Q, int64_t ldq, const T *P, int64_t ldp, const T *L,
                    int64_t ldl, double *part, int nblk, cudaStream_t s) {
    sk_emit_kernel<T><<<nblk, kThreads, 0, s>>>(a, Q, ldq, P, ldp, L, ldl, part); note_launch();
    GOAT_CHECK_LAUNCH();
}

template SkPlan sk_plan<float>(int, int);
template SkPlan sk_plan<double>(int, int);
template void sk_launch_pass<float>(const SkArgs &, const SkPlan &, cudaStream_t);
template void sk_launch_pass<double>(const SkArgs &, const SkPlan &, cudaStream_t);
template void sk_launch_merge<float>(const SkArgs &, const SkPlan &, cudaStream_t);
template void sk_launch_merge<double>(const SkArgs &, const SkPlan &, cudaStream_t);
template void sk_launch_emit<float>(const SkArgs &, float *, int64_t, const float *, int64_t,
                                    const float *, int64_t, double *, int, cudaStream_t);
template void sk_launch_emit<double>(const SkArgs &, double *, int64_t, const double *, int64_t,
                                     const double *, int64_t, double *, int, cudaStream_t);

}  // namespace goat
