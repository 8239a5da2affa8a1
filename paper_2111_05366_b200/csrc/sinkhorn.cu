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
// A merge step turns the column partials into g_k = g_{k-1} - log(sum) and applies
// the reference's stopping rule.  Pass 0 is the reference's marginal pre-check of
// K itself (sinkhorn.py:70-72); pass max_sweeps+1 is row-only and yields the
// deviation of the final iterate.  The returned iterate is exp(E + f_s + g_s) for
// the stopping sweep s -- the same u that produced the reported deviation
// (sinkhorn.py:84-85).
//
// Two drivers share the pass/merge bodies:
//   * sk_persistent_kernel: ONE cooperative launch runs every sweep; CTAs meet at
//     a software grid barrier after the pass (row results + column partials) and
//     after the merge (new g).  Every CTA evaluates the stopping rule from the
//     same device data, so they leave the loop together with no host round trip.
//   * sk_pass_kernel + sk_merge_kernel: one launch pair per sweep (fallback).
#include <algorithm>
#include <cstdlib>

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
    __device__ static double lgt(float x) { return (double)__log2f(x); }  // SFU log2
    __device__ static double exd(double x) { return exp2(x); }
    // |expm1(d)| at fp32 resolution (fp32 mode cannot resolve below ~1e-7 anyway)
    __device__ static double dev(double d) { return (double)fabsf(expm1f((float)d)); }
};
// fp64 exp for the sweep kernels: 2^(k/32) from a 32-entry table (two cache lines)
// times a degree-6 polynomial on |r| <= ln2/64; <= 1.5 ulp on [-700, 700] (max relative
// error 3.0e-16 against long double over 2e6 arguments), 12 fp64 operations with a
// 6-deep dependent chain instead of the library exp's ~17 with an 11-deep one.  The
// fp64 sweeps are exp-latency bound at 16 warps per SM (profiles/round2_ncu_fp64_sweep40k.md).
__device__ const double kExp2Tab[32] = {
    1.0, 1.0218971486541166, 1.0442737824274138, 1.0671404006768237, 1.0905077326652577, 1.1143867425958924,
    1.1387886347566916, 1.1637248587775775, 1.189207115002721, 1.215247359980469, 1.241857812073484,
    1.2690509571917332, 1.2968395546510096, 1.3252366431597413, 1.3542555469368927, 1.383909881963832,
    1.4142135623730951, 1.4451808069770467, 1.4768261459394993, 1.5091644275934228, 1.5422108254079407,
    1.5759808451078865, 1.6104903319492543, 1.645755478153965, 1.681792830507429, 1.718619298122478,
    1.7562521603732995, 1.7947090750031072, 1.8340080864093424, 1.8741676341103, 1.9152065613971474,
    1.9571441241754002};

__device__ __forceinline__ double exp_tab(double x) {
    if (!(fabs(x) < 700.0)) return exp(x);  // -inf, NaN, out of range: the library path
    const double t = fma(x, 46.16624130844683, 6755399441055744.0);  // 32/ln2; 1.5 * 2^52
    const int k = __double2loint(t);                                   // rint(x * 32 / ln2)
    const double kd = t - 6755399441055744.0;
    double r = fma(kd, -0.02166084898635745, x);   // ln2/32, high part (26 bits: the product is exact)
    r = fma(kd, -4.06140840434059e-10, r);         // low part
    double p = fma(r, 1.0 / 720.0, 1.0 / 120.0);
    p = fma(p, r, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    const double s = __ldg(kExp2Tab + (k & 31)) * p;
    // times 2^(k >> 5): straight into the exponent field (normal for |x| < 700)
    return __hiloint2double(__double2hiint(s) + ((k >> 5) << 20), __double2loint(s));
}

template <> struct SkMath<double> {
    static constexpr double kScale = 1.0;
    __device__ static double ex(double x) { return exp_tab(x); }
    __device__ static double lg(double x) { return log(x); }
    __device__ static double lgt(double x) { return log(x); }
    __device__ static double exd(double x) { return exp(x); }
    __device__ static double dev(double d) { return fabs(expm1(d)); }
};

// max without NaN handling (arguments are never NaN): one FMNMX
__device__ __forceinline__ float vmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double vmax(double a, double b) { return fmax(a, b); }

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

// Rows of this (possibly row-sharded) block; columns are always a.n.
__device__ __forceinline__ int rows_of(const SkArgs &a) { return a.m > 0 ? a.m : a.n; }

// Ring slots are selected, not indexed, so SkArgs stays in the parameter bank.
__device__ __forceinline__ double *fslot(const SkArgs &a, int s) { return (s & 1) ? a.f[1] : a.f[0]; }
__device__ __forceinline__ double *gslot(const SkArgs &a, int s) { return (s & 1) ? a.g[1] : a.g[0]; }

__device__ __forceinline__ void sk_stamp(const SkArgs &a, int k, int i) {
    if (a.trace && k == a.trace_k && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[blockIdx.x * 16 + i] = t;
    }
}

// stamp that waits for `dep` (diagnostics only)
__device__ __forceinline__ void sk_stamp_v(const SkArgs &a, int k, int i, double dep) {
    if (a.trace && k == a.trace_k && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) : "d"(dep));
        a.trace[blockIdx.x * 16 + i] = t;
    }
}

// ------------------------------------------------------------------ pass body
// Row bands are cyclic over row groups (grp, grp + ngrp, ...), so a group owns
// the same rows every pass.  With CL == 1 a group is one CTA that owns whole
// rows; with CL > 1 a group is a thread-block cluster whose CTA `rank` owns the
// column slice [c0, c1): each CTA reduces its slice of every row, the per-row
// (max, sum) pairs are exchanged through distributed shared memory (one cluster
// barrier per band) and every CTA combines them in rank order, so all CTAs of the
// cluster hold bit-identical row results.  Columns are owned per thread
// (16-byte chunks of the slice).
struct Slice {
    int c0, c1;     // this CTA's columns
    int grp, ngrp;  // row group (cluster) and number of groups
    int rank;       // rank in the cluster (0 when CL == 1)
};

__device__ __forceinline__ uint32_t dsmem_map(const void *p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(rank));
    return r;
}
// Remote (DSMEM) store of a pair that signals the receiver's mbarrier on arrival.
__device__ __forceinline__ void st_async_pair(uint32_t raddr, float a, float b, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(raddr),
                 "f"(a), "f"(b), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void st_async_pair(uint32_t raddr, double a, double b, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
                 "d"(a), "d"(b), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void xbar_init(uint64_t *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)));
}
__device__ __forceinline__ void xbar_arm(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
// CTA-scope acquire: the exchanged data lives in this CTA's shared memory and is
// published by the mbarrier's complete_tx.  (A cluster-scope acquire compiles to
// CCTL.IVALL -- an L1 invalidation on every completed wait -- which measured as
// the dominant stall of the wide-row kernels: every spill and stack reload then
// went to L2.)
__device__ __forceinline__ void xbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "XW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra XW_%=;\n"
        "}\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
        "r"(parity)
        : "memory");
}

// Per-CTA exchange area for cluster-split rows: slot [parity][rank][row] holds a
// (max, sum) pair written by peer `rank` with st.async; xbar[parity] counts the bytes.
template <class T, int R, int CL> struct __align__(16) RowXch {
    T pair[4][CL][R][2];
    uint64_t bar[4];
};

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Raw 16-byte loads of one band of R rows over this thread's chunks (zero outside).
template <class T, int CH, int R, int NT>
__device__ __forceinline__ void load_band_g(const SkArgs &a, const Slice &sl, int band, int nbands,
                                            typename VecT<T>::V (&dst)[R][CH]) {
    using V = typename VecT<T>::V;
    constexpr int VW = VecT<T>::W;
    const T *G = static_cast<const T *>(a.G);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int col = sl.c0 + ((int)threadIdx.x + NT * c) * VW;
            const int row = band * R + r;
            if (band < nbands && row < rows_of(a) && col < sl.c1)
                dst[r][c] = __ldg(reinterpret_cast<const V *>(G + (int64_t)row * a.ld + col));
            else
                memset(&dst[r][c], 0, sizeof(V));
        }
}

// RES: this CTA owns at most one band, held in registers (xres) for the whole
// solve -- G never changes between sweeps, so nothing is reloaded.
template <class T, int CH, int R, int CL, int NT, bool RES = false>
__device__ __forceinline__ void pass_body(const SkArgs &a, int k, int max_sweeps, double coef_d, double gmax_d,
                                          const Slice &sl, RowXch<T, R, CL> *xch, unsigned &xi,
                                          typename VecT<T>::V (&xres)[R][CH]) {
    using V = typename VecT<T>::V;
    constexpr int VW = VecT<T>::W;
    constexpr int NW = NT / 32;
    __shared__ T s_m[2][NW][R], s_s[2][NW][R];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = a.n;
    const bool pre = (k == 0);
    const bool rowonly = (k == max_sweeps + 1);
    const double *gin = gslot(a, k + 1);  // g_{k-1}
    const double *fprev = fslot(a, k + 1);
    double *fout = fslot(a, k);
    const double ks = SkMath<T>::kScale;
    const T coef = (T)(coef_d * ks);
    const T gmax = (T)gmax_d;
    const int c0 = sl.c0, c1 = sl.c1;
    const bool writer = (sl.rank == 0);  // one CTA per group writes f / deviation

    double devmax = 0.0;
    const int nbands = (rows_of(a) + R - 1) / R;
    // Raw 16-byte loads of one band; the next band is prefetched while the
    // current one is reduced, so the L2/HBM latency overlaps the row combine.
    V xv[R][CH];
    if constexpr (RES) {
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < CH; ++c) xv[r][c] = xres[r][c];
    } else {
        load_band_g<T, CH, R, NT>(a, sl, sl.grp, nbands, xv);
    }

    T gl[CH][VW], acc[CH][VW];
#pragma unroll
    for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int e = 0; e < VW; ++e) {
            const int col = c0 + (tid + NT * c) * VW + e;
            // Column offset g_j; columns outside the slice get -inf, so masking costs
            // nothing per element.  (E is formed as coef*(gmax - G) as in the
            // reference; folding coef*gmax into g cancels catastrophically.)
            const T gv = (!pre && col < c1) ? (T)(__ldcg(gin + col) * ks) : T(0);
            gl[c][e] = col < c1 ? gv : neg_inf<T>();
            acc[c][e] = T(0);
        }

    for (int band = sl.grp; band < nbands; band += sl.ngrp) {
        const int r0 = band * R;
        T x[R][CH][VW];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const T *pv = reinterpret_cast<const T *>(&xv[r][c]);
#pragma unroll
                for (int e = 0; e < VW; ++e) x[r][c][e] = pv[e];
            }
        if constexpr (!RES) load_band_g<T, CH, R, NT>(a, sl, band + sl.ngrp, nbands, xv);  // prefetch
        // f_{k-1} of row r0 + lane (warp 0 checks the deviation), fetched early
        double fprev_v = 0.0;
        if (writer && warp == 0 && lane < R && k >= 2 && r0 + lane < rows_of(a)) fprev_v = __ldcg(fprev + r0 + lane);
        T m[R], s[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            m[r] = neg_inf<T>();
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int e = 0; e < VW; ++e) {
                    const T arg = coef * (gmax - x[r][c][e]) + gl[c][e];  // E_ij + g_j (sinkhorn.py:125)
                    x[r][c][e] = arg;
                    m[r] = vmax(m[r], arg);
                }
        }
        sk_stamp_v(a, k, 8, (double)m[0]);
        // Warp max first (shuffle + max only), then exponentials against the warp
        // max and a plain sum butterfly: no SFU op on the shuffle chain.  Rows past
        // the end get m = -inf (skipped everywhere); exponentials use mx, which is
        // 0 for an all-masked warp so exp(-inf - mx) = 0 (no NaN).
        T mx[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const T m2 = __shfl_xor_sync(0xffffffffu, m[r], off);
                m[r] = m2 > m[r] ? m2 : m[r];
            }
            if (r0 + r >= n) m[r] = neg_inf<T>();
            mx[r] = (m[r] == neg_inf<T>()) ? T(0) : m[r];
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            T sp[VW];  // VW independent partial sums (short add chains)
#pragma unroll
            for (int e = 0; e < VW; ++e) sp[e] = T(0);
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int e = 0; e < VW; ++e) {
                    const T y = SkMath<T>::ex(x[r][c][e] - mx[r]);
                    x[r][c][e] = y;
                    sp[e] += y;
                }
            s[r] = T(0);
#pragma unroll
            for (int e = 0; e < VW; ++e) s[r] += sp[e];
            if (m[r] == neg_inf<T>()) s[r] = T(0);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) s[r] += __shfl_xor_sync(0xffffffffu, s[r], off);
        }
        sk_stamp_v(a, k, 9, (double)s[0]);
        // Per-warp pairs into a parity-double-buffered slot: one block barrier per
        // band; every warp then finishes all R rows itself (lane r <- row r) in
        // the same fixed order, so the results agree bit-for-bit across warps.
        const int par = ((band - sl.grp) / sl.ngrp) & 1;
        if (lane == 0) {
#pragma unroll
            for (int r = 0; r < R; ++r) { s_m[par][warp][r] = m[r]; s_s[par][warp][r] = s[r]; }
        }
        __syncthreads();
        // Cross-warp combine, lane-parallel: lane = (row rr, warp w) with NW lanes per
        // row; max butterfly, one exponential per lane, sum butterfly (fixed xor
        // trees: deterministic, identical in every warp).  Lane rr*NW holds row rr.
        T Mb = neg_inf<T>(), Sb = T(0);
        {
            constexpr int RL = 32 / NW;  // rows combined per warp pass
#pragma unroll
            for (int rb = 0; rb < R; rb += RL) {
                const int rr = rb + lane / NW, w = lane % NW;
                const bool ok = rr < R;
                const T mw = ok ? s_m[par][w][ok ? rr : 0] : neg_inf<T>();
                T M = mw;
#pragma unroll
                for (int off = NW / 2; off > 0; off >>= 1) {
                    const T m2 = __shfl_xor_sync(0xffffffffu, M, off);
                    M = m2 > M ? m2 : M;
                }
                T S = (mw != neg_inf<T>()) ? s_s[par][w][ok ? rr : 0] * SkMath<T>::ex(mw - M) : T(0);
#pragma unroll
                for (int off = NW / 2; off > 0; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
                // move row (rb + lane)'s result to lane (rb + lane) - rb ... i.e. lane r <- row r
#pragma unroll
                for (int q = 0; q < RL; ++q) {
                    const T Mq = __shfl_sync(0xffffffffu, M, q * NW);
                    const T Sq = __shfl_sync(0xffffffffu, S, q * NW);
                    if (lane == rb + q) { Mb = Mq; Sb = Sq; }
                }
            }
        }
        if constexpr (CL > 1) {
            // cluster combine without a cluster barrier: warp 0 pushes this CTA's
            // pairs into every peer's slot with st.async (mbarrier complete_tx);
            // each warp waits for the CL-1 remote pairs and combines all ranks in
            // rank order (its own pair from registers), identically in every CTA.
            const int xp = xi & 3;
            const uint32_t xph = (xi >> 2) & 1;
            if (warp == 0 && lane == 0) xbar_arm(&xch->bar[xp], (uint32_t)((CL - 1) * R * 2 * sizeof(T)));
            if (warp == 0 && lane < R) {
#pragma unroll
                for (int q = 0; q < CL; ++q)
                    if (q != sl.rank)
                        st_async_pair(dsmem_map(&xch->pair[xp][sl.rank][lane][0], q), Mb, Sb,
                                      dsmem_map(&xch->bar[xp], q));
            }
            if (lane < R) {
                xbar_wait(&xch->bar[xp], xph);
                T mq[CL], sq[CL];
#pragma unroll
                for (int q = 0; q < CL; ++q) {
                    mq[q] = (q == sl.rank) ? Mb : xch->pair[xp][q][lane][0];
                    sq[q] = (q == sl.rank) ? Sb : xch->pair[xp][q][lane][1];
                }
                Mb = neg_inf<T>();
#pragma unroll
                for (int q = 0; q < CL; ++q) Mb = mq[q] > Mb ? mq[q] : Mb;
                Sb = T(0);
#pragma unroll
                for (int q = 0; q < CL; ++q)
                    if (mq[q] != neg_inf<T>()) Sb += sq[q] * SkMath<T>::ex(mq[q] - Mb);
            }
            ++xi;
        }
        sk_stamp_v(a, k, 10, (double)Sb);
        double lse_l = 0.0;
        if (lane < R) {
            lse_l = (double)Mb + SkMath<T>::lgt(Sb);  // scaled units
            const int row = r0 + lane;
            if (writer && warp == 0 && row < rows_of(a)) {
                const double fnew = -lse_l * (1.0 / SkMath<T>::kScale);
                double dev = 0.0;
                if (pre) dev = SkMath<T>::dev(-fnew);                  // |rowsum(K) - 1|
                else if (k >= 2) dev = SkMath<T>::dev(fprev_v - fnew);  // |u K v - 1|
                if (!pre) __stcg(fout + row, fnew);
                devmax = fmax(devmax, dev);
            }
        }
        sk_stamp_v(a, k, 11, lse_l);
        double lse_r[R];
#pragma unroll
        for (int r = 0; r < R; ++r) lse_r[r] = __shfl_sync(0xffffffffu, lse_l, r);
        sk_stamp_v(a, k, 12, lse_r[0]);
        if (!rowonly) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (m[r] == neg_inf<T>()) continue;
                // column contribution y = x * exp(m + f_col), f_col = 0 on the pre-check
                const double colf = pre ? 0.0 : -lse_r[r];
                const T sc = SkMath<T>::ex((T)((double)mx[r] + colf));
#pragma unroll
                for (int c = 0; c < CH; ++c)
#pragma unroll
                    for (int e = 0; e < VW; ++e) acc[c][e] += x[r][c][e] * sc;
            }
        }
    }
    if (!rowonly) {
        T *cp = static_cast<T *>(a.colpart) + (int64_t)sl.grp * a.ldp;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int col = c0 + (tid + NT * c) * VW;
            if (col < c1) {
                V v;
                T *pv = reinterpret_cast<T *>(&v);
#pragma unroll
                for (int e = 0; e < VW; ++e) pv[e] = acc[c][e];
                __stcg(reinterpret_cast<V *>(cp + col), v);
            }
        }
    }
    sk_stamp_v(a, k, 14, (double)acc[0][0]);
    __shared__ double s_dev[NW];
    // rows are finished by lanes 0..R-1: reduce over the whole warp first
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) devmax = fmax(devmax, __shfl_xor_sync(0xffffffffu, devmax, off));
    if (lane == 0) s_dev[warp] = devmax;
    __syncthreads();
    if (tid == 0) {
        double d = 0.0;
        for (int w = 0; w < NW; ++w) d = fmax(d, s_dev[w]);
        __stcg(a.devpart + blockIdx.x, d);
        // max of non-negative doubles == max of their bit patterns: order-independent
        if (a.dslot) atomicMax(a.dslot + (k & 1), (unsigned long long)__double_as_longlong(d));
    }
    sk_stamp(a, k, 13);
}

// Clustered wide rows (CL > 1, one row per band): the cross-CTA row exchange is
// software-pipelined.  Iteration j reduces band j over this CTA's column slice and
// pushes the (max, sum) pair to every peer (st.async + mbarrier), then finishes band
// j-1 -- whose peer pairs have had a whole band to arrive -- with the row LSE, f,
// the deviation and the column contributions kept in registers from j-1.  A
// 4-slot ring keeps every slot a lagging peer may still read untouched.
template <class T, int CH, int CL, int NT>
__device__ __forceinline__ void pass_body_lag(const SkArgs &a, int k, int max_sweeps, double coef_d, double gmax_d,
                                              const Slice &sl, RowXch<T, 1, CL> *xch, unsigned &xi) {
    using V = typename VecT<T>::V;
    constexpr int VW = VecT<T>::W;
    constexpr int NW = NT / 32;
    __shared__ T s_m[2][NW], s_s[2][NW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool pre = (k == 0);
    const bool rowonly = (k == max_sweeps + 1);
    const double *gin = gslot(a, k + 1);
    const double *fprev = fslot(a, k + 1);
    double *fout = fslot(a, k);
    const T *G = static_cast<const T *>(a.G);
    const double ks = SkMath<T>::kScale;
    const T coef = (T)(coef_d * ks);
    const T gmax = (T)gmax_d;
    const int c0 = sl.c0, c1 = sl.c1;
    const bool writer = (sl.rank == 0);
    const int nbands = rows_of(a);

    V xv[CH];
    auto load_row = [&](int row, V (&dst)[CH]) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int col = c0 + (tid + NT * c) * VW;
            if (row < nbands && col < c1)
                dst[c] = __ldg(reinterpret_cast<const V *>(G + (int64_t)row * a.ld + col));
            else
                memset(&dst[c], 0, sizeof(V));
        }
    };
    load_row(sl.grp, xv);
    T gl[CH][VW], acc[CH][VW], xp[CH][VW];
#pragma unroll
    for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int e = 0; e < VW; ++e) {
            const int col = c0 + (tid + NT * c) * VW + e;
            const T gv = (!pre && col < c1) ? (T)(__ldcg(gin + col) * ks) : T(0);
            gl[c][e] = col < c1 ? gv : neg_inf<T>();
            acc[c][e] = T(0);
            xp[c][e] = T(0);
        }
    double devmax = 0.0;
    T mx_p = T(0), Mp = neg_inf<T>(), Sp = T(0);
    double fprev_p = 0.0;
    int row_p = -1;

    // finish row row_p (band of exchange index jp) from the peers' pairs
    auto finish = [&](unsigned jp) {
        double lse = 0.0;
        if (lane == 0) {
            const int xs = jp & 3;
            xbar_wait(&xch->bar[xs], (jp >> 2) & 1);
            T mq[CL], sq[CL];
#pragma unroll
            for (int q = 0; q < CL; ++q) {
                mq[q] = (q == sl.rank) ? Mp : xch->pair[xs][q][0][0];
                sq[q] = (q == sl.rank) ? Sp : xch->pair[xs][q][0][1];
            }
            T M = neg_inf<T>();
#pragma unroll
            for (int q = 0; q < CL; ++q) M = mq[q] > M ? mq[q] : M;
            T S = T(0);
#pragma unroll
            for (int q = 0; q < CL; ++q)
                if (mq[q] != neg_inf<T>()) S += sq[q] * SkMath<T>::ex(mq[q] - M);
            lse = (double)M + SkMath<T>::lgt(S);
            if (writer && warp == 0 && row_p < nbands) {
                const double fnew = -lse * (1.0 / SkMath<T>::kScale);
                double dev = 0.0;
                if (pre) dev = SkMath<T>::dev(-fnew);
                else if (k >= 2) dev = SkMath<T>::dev(fprev_p - fnew);
                if (!pre) __stcg(fout + row_p, fnew);
                devmax = fmax(devmax, dev);
            }
        }
        lse = __shfl_sync(0xffffffffu, lse, 0);
        if (!rowonly && row_p < nbands) {
            const double colf = pre ? 0.0 : -lse;
            const T sc = SkMath<T>::ex((T)((double)mx_p + colf));
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int e = 0; e < VW; ++e) acc[c][e] += xp[c][e] * sc;
        }
    };

    int it = 0;
    for (int row = sl.grp; row < nbands; row += sl.ngrp, ++it) {
        T x[CH][VW];
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const T *pv = reinterpret_cast<const T *>(&xv[c]);
#pragma unroll
            for (int e = 0; e < VW; ++e) x[c][e] = pv[e];
        }
        load_row(row + sl.ngrp, xv);  // prefetch
        double fpv = 0.0;
        if (writer && warp == 0 && lane == 0 && k >= 2) fpv = __ldcg(fprev + row);
        T m = neg_inf<T>();
#pragma unroll
        for (int c = 0; c < CH; ++c)
#pragma unroll
            for (int e = 0; e < VW; ++e) {
                const T arg = coef * (gmax - x[c][e]) + gl[c][e];
                x[c][e] = arg;
                m = vmax(m, arg);
            }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const T m2 = __shfl_xor_sync(0xffffffffu, m, off);
            m = m2 > m ? m2 : m;
        }
        const T mx = (m == neg_inf<T>()) ? T(0) : m;
        T sp[VW];  // VW independent partial sums (short add chains)
#pragma unroll
        for (int e = 0; e < VW; ++e) sp[e] = T(0);
#pragma unroll
        for (int c = 0; c < CH; ++c)
#pragma unroll
            for (int e = 0; e < VW; ++e) {
                const T y = SkMath<T>::ex(x[c][e] - mx);
                x[c][e] = y;
                sp[e] += y;
            }
        T sum = T(0);
#pragma unroll
        for (int e = 0; e < VW; ++e) sum += sp[e];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
        const int par = it & 1;
        if (lane == 0) { s_m[par][warp] = m; s_s[par][warp] = sum; }
        __syncthreads();
        // lane-parallel cross-warp combine (lane w holds warp w's pair); result in lane 0
        T Mb, Sb;
        {
            const T mw = lane < NW ? s_m[par][lane] : neg_inf<T>();
            T M = mw;
#pragma unroll
            for (int off = NW / 2; off > 0; off >>= 1) {
                const T m2 = __shfl_xor_sync(0xffffffffu, M, off);
                M = m2 > M ? m2 : M;
            }
            T S = (mw != neg_inf<T>()) ? s_s[par][lane] * SkMath<T>::ex(mw - M) : T(0);
#pragma unroll
            for (int off = NW / 2; off > 0; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
            Mb = M;
            Sb = S;
        }
        const unsigned j = xi;
        if (warp == 0 && lane == 0) {
            const int xs = j & 3;
            xbar_arm(&xch->bar[xs], (uint32_t)((CL - 1) * 2 * sizeof(T)));
#pragma unroll
            for (int q = 0; q < CL; ++q)
                if (q != sl.rank)
                    st_async_pair(dsmem_map(&xch->pair[xs][sl.rank][0][0], q), Mb, Sb, dsmem_map(&xch->bar[xs], q));
        }
        if (it > 0) finish(j - 1);
        // this band becomes the pending one
#pragma unroll
        for (int c = 0; c < CH; ++c)
#pragma unroll
            for (int e = 0; e < VW; ++e) xp[c][e] = x[c][e];
        mx_p = mx;
        Mp = Mb;
        Sp = Sb;
        fprev_p = fpv;
        row_p = row;
        ++xi;
    }
    if (it > 0) finish(xi - 1);
    if (!rowonly) {
        T *cp = static_cast<T *>(a.colpart) + (int64_t)sl.grp * a.ldp;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int col = c0 + (tid + NT * c) * VW;
            if (col < c1) {
                V v;
                T *pv = reinterpret_cast<T *>(&v);
#pragma unroll
                for (int e = 0; e < VW; ++e) pv[e] = acc[c][e];
                __stcg(reinterpret_cast<V *>(cp + col), v);
            }
        }
    }
    __shared__ double s_dev[NW];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) devmax = fmax(devmax, __shfl_xor_sync(0xffffffffu, devmax, off));
    if (lane == 0) s_dev[warp] = devmax;
    __syncthreads();
    if (tid == 0) {
        double d = 0.0;
        for (int w = 0; w < NW; ++w) d = fmax(d, s_dev[w]);
        __stcg(a.devpart + blockIdx.x, d);
        if (a.dslot) atomicMax(a.dslot + (k & 1), (unsigned long long)__double_as_longlong(d));
    }
}

// ------------------------------------------------------------------ TMA-staged wide rows
// Wide rows (one row per band, CL >= 1) stream through a ring of S shared-memory
// stages filled by 1-D bulk copies (cp.async.bulk, mbarrier complete_tx).  The
// ring runs ahead D = S-2 bands and wraps across sweeps (a CTA owns the same rows
// every sweep), so HBM requests stay in flight through the row reductions, the
// cluster exchange and the grid barriers.  No register prefetch copy: a thread
// holds only its chunk of the current band.  The exponentials of band j are
// written back in place and re-read by the lagged finish of band j (iteration
// j+1), so a stage is refilled only after the block barrier of iteration j+2.
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// The same copy with an L2 cache hint (policy from createpolicy): G is re-read
// every sweep, so when it fits in L2 an evict_last policy keeps it there.
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                              uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

struct WideRing {
    char *base;        // S stages of stage_bytes
    uint64_t *full;    // S mbarriers
    int S, stage_bytes;
    int nrows;         // rows this CTA processes per sweep
    uint32_t copy_bytes;
    unsigned issued;   // bands issued (thread 0)
    unsigned used;     // bands consumed (all threads)
};

template <class T>
__device__ __forceinline__ void ring_issue(const SkArgs &a, const Slice &sl, WideRing &rg) {
    if (a.single_pass && rg.issued >= (unsigned)rg.nrows) return;  // one sweep per launch
    const unsigned b = rg.issued++;
    const int row = sl.grp + (int)(b % (unsigned)rg.nrows) * sl.ngrp;
    const int s = (int)(b % (unsigned)rg.S);
    const T *src = static_cast<const T *>(a.G) + (int64_t)row * a.ld + sl.c0;
    xbar_arm(&rg.full[s], rg.copy_bytes);
    bulk_g2s(rg.base + (size_t)s * rg.stage_bytes, src, rg.copy_bytes, &rg.full[s]);
}

template <class T, int CH, int CL, int NT>
__device__ __forceinline__ void pass_body_tma(const SkArgs &a, int k, int max_sweeps, double coef_d, double gmax_d,
                                              const Slice &sl, RowXch<T, 1, CL> *xch, unsigned &xi, WideRing &rg) {
    using V = typename VecT<T>::V;
    constexpr int VW = VecT<T>::W;
    constexpr int NW = NT / 32;
    __shared__ T s_m[2][NW], s_s[2][NW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool pre = (k == 0);
    const bool rowonly = (k == max_sweeps + 1);
    const double *gin = gslot(a, k + 1);
    const double *fprev = fslot(a, k + 1);
    double *fout = fslot(a, k);
    const double ks = SkMath<T>::kScale;
    const T coef = (T)(coef_d * ks);
    const T gmax = (T)gmax_d;
    const int c0 = sl.c0, c1 = sl.c1;
    const bool writer = (sl.rank == 0);
    const int D = rg.S - 2;

    T gl[CH][VW], acc[CH][VW];
#pragma unroll
    for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int e = 0; e < VW; ++e) {
            const int col = c0 + (tid + NT * c) * VW + e;
            const T gv = (!pre && col < c1) ? (T)(__ldcg(gin + col) * ks) : T(0);
            gl[c][e] = col < c1 ? gv : neg_inf<T>();
            acc[c][e] = T(0);
        }
    double devmax = 0.0;
    T mx_p = T(0), Mp = neg_inf<T>(), Sp = T(0);
    double fprev_p = 0.0;
    int row_p = -1;
    unsigned band_p = 0;

    auto stage_of = [&](unsigned b) { return reinterpret_cast<V *>(rg.base + (size_t)(b % (unsigned)rg.S) * rg.stage_bytes); };

    auto finish = [&](unsigned jp) {
        double lse = 0.0;
        if (lane == 0) {
            T M = Mp, S = Sp;
            if constexpr (CL > 1) {
                const int xs = jp & 3;
                xbar_wait(&xch->bar[xs], (jp >> 2) & 1);
                T mq[CL], sq[CL];
#pragma unroll
                for (int q = 0; q < CL; ++q) {
                    mq[q] = (q == sl.rank) ? Mp : xch->pair[xs][q][0][0];
                    sq[q] = (q == sl.rank) ? Sp : xch->pair[xs][q][0][1];
                }
                M = neg_inf<T>();
#pragma unroll
                for (int q = 0; q < CL; ++q) M = mq[q] > M ? mq[q] : M;
                S = T(0);
#pragma unroll
                for (int q = 0; q < CL; ++q)
                    if (mq[q] != neg_inf<T>()) S += sq[q] * SkMath<T>::ex(mq[q] - M);
            }
            lse = (double)M + SkMath<T>::lgt(S);
            if (writer && warp == 0 && row_p < rows_of(a)) {
                const double fnew = -lse * (1.0 / SkMath<T>::kScale);
                double dev = 0.0;
                if (pre) dev = SkMath<T>::dev(-fnew);
                else if (k >= 2) dev = SkMath<T>::dev(fprev_p - fnew);
                if (!pre) __stcg(fout + row_p, fnew);
                devmax = fmax(devmax, dev);
            }
        }
        lse = __shfl_sync(0xffffffffu, lse, 0);
        if (!rowonly && row_p < rows_of(a)) {
            const double colf = pre ? 0.0 : -lse;
            const T sc = SkMath<T>::ex((T)((double)mx_p + colf));
            const V *st = stage_of(band_p);
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int col = c0 + (tid + NT * c) * VW;
                if (col < c1) {
                    const V yv = st[tid + NT * c];
                    const T *py = reinterpret_cast<const T *>(&yv);
#pragma unroll
                    for (int e = 0; e < VW; ++e) acc[c][e] += py[e] * sc;
                }
            }
        }
    };

    int it = 0;
    for (int row = sl.grp; row < rows_of(a); row += sl.ngrp, ++it) {
        const unsigned b = rg.used++;
        double fpv = 0.0;
        if (writer && warp == 0 && lane == 0 && k >= 2) fpv = __ldcg(fprev + row);
        xbar_wait(&rg.full[b % (unsigned)rg.S], (b / (unsigned)rg.S) & 1);
        V *st = stage_of(b);
        T x[CH][VW];
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int col = c0 + (tid + NT * c) * VW;
            V xv;
            if (col < c1) xv = st[tid + NT * c];
            else memset(&xv, 0, sizeof(V));
            const T *pv = reinterpret_cast<const T *>(&xv);
#pragma unroll
            for (int e = 0; e < VW; ++e) x[c][e] = pv[e];
        }
        T m = neg_inf<T>();
#pragma unroll
        for (int c = 0; c < CH; ++c)
#pragma unroll
            for (int e = 0; e < VW; ++e) {
                const T arg = coef * (gmax - x[c][e]) + gl[c][e];  // E_ij + g_j (sinkhorn.py:125)
                x[c][e] = arg;
                m = vmax(m, arg);
            }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const T m2 = __shfl_xor_sync(0xffffffffu, m, off);
            m = m2 > m ? m2 : m;
        }
        const T mx = (m == neg_inf<T>()) ? T(0) : m;
        T sp[VW];
#pragma unroll
        for (int e = 0; e < VW; ++e) sp[e] = T(0);
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int col = c0 + (tid + NT * c) * VW;
            V yv;
            T *py = reinterpret_cast<T *>(&yv);
#pragma unroll
            for (int e = 0; e < VW; ++e) {
                const T y = SkMath<T>::ex(x[c][e] - mx);
                py[e] = y;
                sp[e] += y;
            }
            if (!rowonly && col < c1) st[tid + NT * c] = yv;  // re-read by finish(b)
        }
        T sum = T(0);
#pragma unroll
        for (int e = 0; e < VW; ++e) sum += sp[e];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
        const int par = it & 1;
        if (lane == 0) { s_m[par][warp] = m; s_s[par][warp] = sum; }
        fence_proxy_async_smem();  // this thread's stage accesses precede later bulk refills
        __syncthreads();
        // stage of band b-2 is free: every thread has passed finish(b-2)
        if (tid == 0) ring_issue<T>(a, sl, rg);
        T Mb, Sb;
        {
            const T mw = lane < NW ? s_m[par][lane] : neg_inf<T>();
            T M = mw;
#pragma unroll
            for (int off = NW / 2; off > 0; off >>= 1) {
                const T m2 = __shfl_xor_sync(0xffffffffu, M, off);
                M = m2 > M ? m2 : M;
            }
            T S = (mw != neg_inf<T>()) ? s_s[par][lane] * SkMath<T>::ex(mw - M) : T(0);
#pragma unroll
            for (int off = NW / 2; off > 0; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
            Mb = M;
            Sb = S;
        }
        const unsigned j = xi;
        if constexpr (CL > 1) {
            if (warp == 0 && lane == 0) {
                const int xs = j & 3;
                xbar_arm(&xch->bar[xs], (uint32_t)((CL - 1) * 2 * sizeof(T)));
#pragma unroll
                for (int q = 0; q < CL; ++q)
                    if (q != sl.rank)
                        st_async_pair(dsmem_map(&xch->pair[xs][sl.rank][0][0], q), Mb, Sb, dsmem_map(&xch->bar[xs], q));
            }
        }
        if (it > 0) finish(j - 1);
        mx_p = mx;
        Mp = Mb;
        Sp = Sb;
        fprev_p = fpv;
        row_p = row;
        band_p = b;
        ++xi;
        (void)D;
    }
    if (it > 0) finish(xi - 1);
    if (!rowonly) {
        T *cp = static_cast<T *>(a.colpart) + (int64_t)sl.grp * a.ldp;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int col = c0 + (tid + NT * c) * VW;
            if (col < c1) {
                V v;
                T *pv = reinterpret_cast<T *>(&v);
#pragma unroll
                for (int e = 0; e < VW; ++e) pv[e] = acc[c][e];
                __stcg(reinterpret_cast<V *>(cp + col), v);
            }
        }
    }
    __shared__ double s_dev[NW];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) devmax = fmax(devmax, __shfl_xor_sync(0xffffffffu, devmax, off));
    if (lane == 0) s_dev[warp] = devmax;
    __syncthreads();
    if (tid == 0) {
        double d = 0.0;
        for (int w = 0; w < NW; ++w) d = fmax(d, s_dev[w]);
        __stcg(a.devpart + blockIdx.x, d);
        if (a.dslot) atomicMax(a.dslot + (k & 1), (unsigned long long)__double_as_longlong(d));
    }
}

// Exact column LSE for a column whose partial sum under/overflowed:
// g_j = -LSE_i(E_ij + f_i) over all rows (fp64).  Rare repair path.
template <class T>
__device__ __noinline__ double sk_exact_col(const T *G, int64_t ld, int n, int j, const double *f, bool pre, double coef,
                                            double gmax) {
    // (fields passed by value: a reference to the kernel's SkArgs would force a
    // per-thread stack copy of it)
    double M = -INFINITY;
    for (int i = 0; i < n; ++i) {
        const double e = coef * (gmax - (double)G[(int64_t)i * ld + j]) + (pre ? 0.0 : __ldcg(f + i));
        M = fmax(M, e);
    }
    double S = 0.0;
    for (int i = 0; i < n; ++i) {
        const double e = coef * (gmax - (double)G[(int64_t)i * ld + j]) + (pre ? 0.0 : __ldcg(f + i));
        S += exp(e - M);
    }
    return -(M + log(S));
}

// ------------------------------------------------------------------ merge body
// Columns [blk*256 + tid] strided by nblk*256.  On the pre-check writes this
// CTA's max |colsum - 1| to devcol[blk].
template <class T, int NT>
__device__ __forceinline__ void merge_body(const SkArgs &a, int k, double coef, double gmax, int blk, int nblk) {
    constexpr int NW = NT / 32;
    __shared__ double s_red[NW];
    const int tid = threadIdx.x, n = a.n, lane = tid & 31, warp = tid >> 5;
    const bool pre = (k == 0);
    const T *cp = static_cast<const T *>(a.colpart);
    const double tiny = sizeof(T) == 4 ? 1e-30 : 1e-290;
    const int np = a.nblk;
    double dloc = 0.0;
    // One warp per column: lanes split the partials (4 independent loads in
    // flight per lane), then a fixed xor tree -- deterministic.
    for (int j = blk * NW + warp; j < n; j += nblk * NW) {
        double S = 0.0;
        for (int b0 = 0; b0 < np; b0 += 128) {
            T v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int b = b0 + lane + 32 * u;
                v[u] = b < np ? __ldcg(cp + (int64_t)b * a.ldp + j) : T(0);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) S += (double)v[u];
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
        if (lane != 0) continue;
        if (pre) {
            // A column of K whose sum underflows the element type is at least 1 - tiny away
            // from 1: the pre-check only decides "already doubly stochastic?" (sinkhorn.py:70-72),
            // so its exact sum is not needed.  (Recomputing it in fp64, one lane per column,
            // cost ~0.5 s at n = 40000 on a hub-dominated gradient: most columns underflow.)
            if (!(S > tiny)) S = 0.0;
            dloc = fmax(dloc, fabs(S - 1.0));
        } else {
            const double gold = __ldcg(gslot(a, k + 1) + j);
            double gnew = gold - log(S);
            if (!(S > tiny) || !isfinite(S)) {
                gnew = sk_exact_col<T>(static_cast<const T *>(a.G), a.ld, a.n, j, fslot(a, k), false, coef, gmax);
                atomicAdd(&a.st->repaired, 1);
            }
            __stcg(gslot(a, k) + j, gnew);
        }
    }
    if (pre) {
        for (int off = 16; off > 0; off >>= 1) dloc = fmax(dloc, __shfl_xor_sync(0xffffffffu, dloc, off));
        if ((tid & 31) == 0) s_red[tid >> 5] = dloc;
        __syncthreads();
        if (tid == 0) {
            double d = 0.0;
            for (int w = 0; w < NT / 32; ++w) d = fmax(d, s_red[w]);
            __stcg(a.devcol + blk, d);
            if (a.dslot) atomicMax(a.dslot + 2, (unsigned long long)__double_as_longlong(d));
        }
    }
}

// Software grid barrier for a cooperative launch: arrival counter + generation.
// Counter and generation live on different 128-byte lines so the spinning
// readers do not contend with the arrivals.
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Monotone arrival counter (zeroed per launch): arrival is a release reduction,
// waiting is acquire polling until epoch * nblocks.  Measured 1.2 us at 148
// CTAs vs 2.0 us for a fence + generation-flag barrier (scripts/barrier_bench.cu).
__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned nblocks, unsigned &epoch) {
    ++epoch;
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(bar), "r"(1u) : "memory");
        const unsigned target = epoch * nblocks;
        while (ld_acquire(bar) < target) { }
    }
    __syncthreads();
}

// ------------------------------------------------------------------ drivers
template <class T, int CH, int R, int CL, int NT, bool RES, bool TMA>
__device__ __forceinline__ void sk_sweeps(const SkArgs &a, unsigned *bar, const Slice &sl, RowXch<T, R, CL> *xchp,
                                          unsigned &xi, int k0, int K, double tol, double coef, double gmax,
                                          typename VecT<T>::V (&xres)[R][CH], WideRing *rg) {
    const int blk = blockIdx.x, nblk = gridDim.x;
    const int nostop_k = a.st->nostop_k;
    unsigned epoch = 0;
    for (int k = k0;; ++k) {
        sk_stamp(a, k, 0);
        if constexpr (TMA) pass_body_tma<T, CH, CL, NT>(a, k, K, coef, gmax, sl, xchp, xi, *rg);
        else if constexpr (CL > 1 && R == 1) pass_body_lag<T, CH, CL, NT>(a, k, K, coef, gmax, sl, xchp, xi);
        else pass_body<T, CH, R, CL, NT, RES>(a, k, K, coef, gmax, sl, xchp, xi, xres);
        sk_stamp(a, k, 1);
        if (a.single_pass) {  // row-sharded driver: the caller reduces across ranks
            if constexpr (TMA) {
                if (threadIdx.x == 0)
                    for (unsigned b = rg->used; b < rg->issued; ++b)
                        xbar_wait(&rg->full[b % (unsigned)rg->S], (b / (unsigned)rg->S) & 1);
            }
            if constexpr (CL > 1) cluster_sync();
            return;
        }
        grid_barrier(bar, nblk, epoch);
        sk_stamp(a, k, 3);
        const double drow = __longlong_as_double((long long)__ldcg(a.dslot + (k & 1)));
        if (blk == 0 && threadIdx.x == 0) a.dslot[(k + 1) & 1] = 0ull;  // next sweep's slot
        int stop = 0, sweeps = 0, conv = 0, slot = 0;
        if (k >= 2) {
            if (drow < tol && k > nostop_k) { stop = 1; sweeps = k - 1; conv = 1; slot = (k - 1) & 1; }
            else if (k == K + 1) { stop = 1; sweeps = K; conv = 0; slot = K & 1; }
        }
        if (!stop) {
            merge_body<T, NT>(a, k, coef, gmax, blk, nblk);
            sk_stamp(a, k, 4);
            grid_barrier(bar, nblk, epoch);
            sk_stamp(a, k, 5);
            if (k == 0) {
                const double d0 = fmax(drow, __longlong_as_double((long long)__ldcg(a.dslot + 2)));
                if (d0 < tol) { stop = 1; sweeps = 0; conv = 1; slot = 0; }
                if (blk == 0 && threadIdx.x == 0) a.st->last_dev = d0;
                if (stop && blk == 0 && threadIdx.x == 0) a.st->dev = d0;
            }
        } else if (blk == 0 && threadIdx.x == 0) {
            a.st->dev = drow;
        }
        if (stop) {
            if (blk == 0 && threadIdx.x == 0) {
                a.st->done = 1; a.st->sweeps = sweeps; a.st->converged = conv; a.st->slot = slot;
                a.st->k = k + 1;
            }
            if constexpr (TMA) {
                // drain the bulk copies already issued for the next sweep
                if (threadIdx.x == 0)
                    for (unsigned b = rg->used; b < rg->issued; ++b)
                        xbar_wait(&rg->full[b % (unsigned)rg->S], (b / (unsigned)rg->S) & 1);
            }
            if constexpr (CL > 1) cluster_sync();
            return;
        }
    }
}

template <class T, int CH, int R, int CL, int NT, bool TMA = false>
__global__ void __launch_bounds__(NT, (NT > 256 ? 1 : 2)) sk_persistent_kernel(SkArgs a, unsigned *bar) {
    __shared__ int s_k, s_done;
    if (threadIdx.x == 0) { s_k = a.st->k; s_done = a.st->done | a.st->pending; }
    __syncthreads();
    if (a.single_pass && s_done) return;  // every CTA sees the same flags
    const int k0 = s_k;
    const int K = a.st->max_sweeps;
    const double tol = a.st->tol, coef = a.st->coef, gmax = a.st->gmax;
    const int blk = blockIdx.x, nblk = gridDim.x;
    Slice sl{0, a.n, blk, nblk, 0};
    if constexpr (CL > 1) {
        uint32_t rank, cid, ncl;
        asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        asm("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
        asm("mov.u32 %0, %%nclusterid.x;" : "=r"(ncl));
        sl.rank = (int)rank;
        sl.grp = (int)cid;
        sl.ngrp = (int)ncl;
        sl.c0 = min(a.n, (int)rank * a.slice_w);
        sl.c1 = min(a.n, sl.c0 + a.slice_w);
    }
    __shared__ RowXch<T, R, CL> xch;
    unsigned xi = 0;  // exchange counter (bands processed by this cluster so far)
    if constexpr (CL > 1) {
        if (threadIdx.x == 0) {
            for (int q = 0; q < 4; ++q) xbar_init(&xch.bar[q]);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        cluster_sync();  // every peer's barriers exist before the first st.async
    }
    using V = typename VecT<T>::V;
    V xres[R][CH];
    if constexpr (TMA) {
        static_assert(R == 1, "TMA ring streams one row per band");
        extern __shared__ __align__(128) char sk_ring[];
        __shared__ uint64_t full[8];
        WideRing rg;
        rg.base = sk_ring;
        rg.full = full;
        rg.S = a.stages;
        rg.stage_bytes = a.stage_bytes;
        rg.nrows = (rows_of(a) - sl.grp + sl.ngrp - 1) / sl.ngrp;
        rg.copy_bytes = (uint32_t)(((sl.c1 - sl.c0 + VecT<T>::W - 1) / VecT<T>::W) * sizeof(V));
        rg.issued = 0;
        rg.used = 0;
        if (threadIdx.x == 0) {
            for (int q = 0; q < rg.S; ++q) xbar_init(&full[q]);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            for (int q = 0; q < rg.S - 2; ++q) ring_issue<T>(a, sl, rg);
        }
        __syncthreads();
        sk_sweeps<T, CH, R, CL, NT, false, true>(a, bar, sl, &xch, xi, k0, K, tol, coef, gmax, xres, &rg);
        return;
    }
    if constexpr (CL == 1) {
        const int nbands = (rows_of(a) + R - 1) / R;
        if (a.resident && nbands <= nblk) {
            load_band_g<T, CH, R, NT>(a, sl, sl.grp, nbands, xres);
            sk_sweeps<T, CH, R, CL, NT, true, false>(a, bar, sl, &xch, xi, k0, K, tol, coef, gmax, xres, nullptr);
            return;
        }
    }
    sk_sweeps<T, CH, R, CL, NT, false, false>(a, bar, sl, &xch, xi, k0, K, tol, coef, gmax, xres, nullptr);
}

// ------------------------------------------------------------------ decoupled wide-row pipeline (fp32)
// Wide rows (one row per band) without a block barrier per band.  Row slices
// stream through a ring of S shared-memory stages (cp.async.bulk, full/empty
// mbarriers), and the three steps of a band are lagged so no warp waits on the
// latency of another step:
//   band b   : every warp reduces its columns of the row -> a (max, sum) pair
//              per warp, kept exponentials y_b in registers, arrives on wbar[b];
//   band b+1 : warp 0 combines the NW warp pairs (fixed tree) into the CTA pair
//              and sends it to every cluster rank (st.async + complete_tx);
//   band b+LAG: every warp combines the CL rank pairs in rank order -> row LSE ->
//              f_b, the deviation, and the column contributions acc += y_b * sc.
// LAG = 1 without a cluster (the CTA pair is local), 2 with one (the peers' pairs
// get a whole band to arrive).  Results are bit-identical to a lock-step order:
// every reduction tree is fixed.  A stage is refilled as soon as every warp has
// loaded it (empty barrier); the ring runs ahead across sweeps.
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_cta(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "MW_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra MW_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

template <int NW, int CL, int R> struct PipeSm {
    uint64_t full[8], empty[8], wbar[4], xbar[4];
    float xp[4][CL][R][2];  // per-rank CTA (max, sum) of every row of a band slot
};

struct PipeRing {
    char *base;
    int S, stage_bytes, row_bytes, nrows, nbands;
    uint32_t copy_bytes;
    unsigned issued;  // bands issued (thread 0)
    unsigned used;    // bands consumed (all threads)
};

// Thread 0: issue every band below `upto` whose stage has been released.  A band
// is R rows of this group (local rows b*R .. b*R+R-1), one bulk copy per row.
template <int NW, int CL, int R>
__device__ __forceinline__ void pipe_produce(const SkArgs &a, const Slice &sl, PipeRing &rg, PipeSm<NW, CL, R> &ps,
                                             unsigned upto) {
    while (rg.issued < upto) {
        if (a.single_pass && rg.issued >= (unsigned)rg.nbands) return;  // one sweep per launch
        const unsigned u = rg.issued;
        const int s = (int)(u % (unsigned)rg.S);
        if (u >= (unsigned)rg.S) mbar_wait_cta(&ps.empty[s], ((u / (unsigned)rg.S) - 1) & 1);
        const int lr0 = (int)(u % (unsigned)rg.nbands) * R;
        const int nv = min(R, rg.nrows - lr0);
        xbar_arm(&ps.full[s], rg.copy_bytes * (uint32_t)nv);
        for (int r = 0; r < nv; ++r) {
            const int row = sl.grp + (lr0 + r) * sl.ngrp;
            const float *src = static_cast<const float *>(a.G) + (int64_t)row * a.ld + sl.c0;
            void *dst = rg.base + (size_t)s * rg.stage_bytes + (size_t)r * rg.row_bytes;
            if (a.l2_last) bulk_g2s_hint(dst, src, rg.copy_bytes, &ps.full[s], l2_evict_last_policy());
            else bulk_g2s(dst, src, rg.copy_bytes, &ps.full[s]);
        }
        ++rg.issued;
    }
}

// Row shift of the exponentials.  MAXP (pre-check, sweep 1, single-pass
// launches, and any sweep redone after an out-of-range row): the warp/CTA/cluster
// row maximum, combined as (max, sum) pairs.  Otherwise the previous sweep's row
// LSE, -f_{k-1,i}: the exponent of every term is then bounded by the change of
// the row's LSE, no max reduction is needed, and the pairs reduce to plain sums.
// A row whose sum leaves [2^-40, 2^100] (early sweeps: g moved by > 40 log2
// units) sets the redo flag and the whole sweep is recomputed with MAXP.
constexpr int kPipeShiftRows = 2048;
constexpr float kShiftLo = 9.094947e-13f;   // 2^-40
constexpr float kShiftHi = 1.2676506e30f;   // 2^100

// Finish one row of a band: f_k of the row (writer), the pre-check deviation, and
// the column contributions acc += y * 2^(m_warp - lse) of this warp's exponentials.
#define PIPE_FINISH(LR, LSE, MWARP, YV)                                                         \
    do {                                                                                        \
        const double lse_ = (LSE);                                                              \
        if (writer) {                                                                           \
            const double fnew = -lse_ * (1.0 / SkMath<T>::kScale);                              \
            if (pre) devmax = fmax(devmax, SkMath<T>::dev(-fnew));                              \
            else __stcg(fout + sl.grp + (LR) * sl.ngrp, fnew);                                  \
        }                                                                                       \
        if (!rowonly && (MWARP) != neg_inf<T>()) {                                              \
            const T sc = SkMath<T>::ex((T)((double)(MWARP) + (pre ? 0.0 : -lse_)));             \
            _Pragma("unroll") for (int c = 0; c < CH; ++c)                                      \
                _Pragma("unroll") for (int e = 0; e < VW; ++e) acc[c][e] += (YV)[c][e] * sc;   \
        }                                                                                       \
    } while (0)

template <int CH, int CL, int NT, int R, bool MAXP>
__device__ __forceinline__ void pass_body_pipe(const SkArgs &a, int k, int max_sweeps, double coef_d, double gmax_d,
                                               const Slice &sl, PipeSm<NT / 32, CL, R> &ps, PipeRing &rg,
                                               unsigned *redo) {
    using T = float;
    using V = float4;
    constexpr int VW = 4;
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool pre = (k == 0);
    const bool rowonly = (k == max_sweeps + 1);
    const double *gin = gslot(a, k + 1);
    const double *fprev = fslot(a, k + 1);
    double *fout = fslot(a, k);
    const double ks = SkMath<T>::kScale;
    const T coef = (T)(coef_d * ks);
    const T gmax = (T)gmax_d;
    const int c0 = sl.c0, c1 = sl.c1;
    const bool writer = (sl.rank == 0) && warp == 0 && lane == 0;
    const int S = rg.S;

    // g of this thread's columns (scaled; -inf masks columns past the slice) lives
    // in shared memory after the ring: registers hold only the exponentials and
    // the column accumulators
    T acc[CH][VW];
    V *s_gl = reinterpret_cast<V *>(rg.base + (size_t)rg.S * rg.stage_bytes);
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        T gv[VW];
#pragma unroll
        for (int e = 0; e < VW; ++e) {
            const int col = c0 + (tid + NT * c) * VW + e;
            gv[e] = col < c1 ? ((!pre) ? (T)(__ldcg(gin + col) * ks) : T(0)) : neg_inf<T>();
            acc[c][e] = T(0);
        }
        s_gl[tid + NT * c] = make_float4(gv[0], gv[1], gv[2], gv[3]);  // read back by this thread only
    }
    // clusters: a band's exponentials wait in its stage for the lagged finish
    constexpr bool LAGGED = CL > 1;
    T mp[R];
#pragma unroll
    for (int r = 0; r < R; ++r) mp[r] = neg_inf<T>();
    double devmax = 0.0;  // pre-check only (writer thread)
    __shared__ T s_wp[2][NW][R][2];
    __shared__ float s_shift[MAXP ? 1 : kPipeShiftRows];
    bool bad = false;
    if constexpr (!MAXP) {
        for (int i = tid; i < rg.nrows; i += NT) s_shift[i] = (float)(-__ldcg(fprev + sl.grp + i * sl.ngrp) * ks);
        __syncthreads();
    }

    const int nrows = rg.nrows, nb = rg.nbands;
    const unsigned b0 = rg.used;
    for (int it = 0; it < nb + (LAGGED ? 1 : 0); ++it) {
        const unsigned b = b0 + (unsigned)it;
        // keep the ring full (never blocks in steady state: every warp passed the
        // block barrier of band b - 1); clusters release a stage one band later
        if (tid == 0) pipe_produce<NW, CL, R>(a, sl, rg, ps, b + (unsigned)S - (LAGGED ? 2u : 1u));
        T y[R][CH][VW];
        T m[R];
#pragma unroll
        for (int r = 0; r < R; ++r) m[r] = neg_inf<T>();
        if (it < nb) {
            const int s = (int)(b % (unsigned)S);
            mbar_wait_cta(&ps.full[s], (b / (unsigned)S) & 1);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const bool rv = it * R + r < nrows;
                const V *st = reinterpret_cast<const V *>(rg.base + (size_t)s * rg.stage_bytes + (size_t)r * rg.row_bytes);
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    const int col = c0 + (tid + NT * c) * VW;
                    V xv;
                    if (rv && col < c1) xv = st[tid + NT * c];
                    else xv = make_float4(0.f, 0.f, 0.f, 0.f);
                    y[r][c][0] = xv.x; y[r][c][1] = xv.y; y[r][c][2] = xv.z; y[r][c][3] = xv.w;
                }
            }
            if constexpr (!LAGGED) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&ps.empty[s]);
            }
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const V g4 = s_gl[tid + NT * c];
                const T gl[VW] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int e = 0; e < VW; ++e) {
                        const T arg = coef * (gmax - y[r][c][e]) + gl[e];  // E_ij + g_j (sinkhorn.py:125)
                        y[r][c][e] = arg;
                        if constexpr (MAXP) m[r] = vmax(m[r], arg);
                    }
            }
            if constexpr (MAXP) {
#pragma unroll
                for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                    for (int r = 0; r < R; ++r) m[r] = vmax(m[r], __shfl_xor_sync(0xffffffffu, m[r], off));
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r)  // the row's shift, identical in every warp and cluster rank
                    m[r] = (it * R + r < nrows) ? s_shift[it * R + r] : neg_inf<T>();
            }
            T sum[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const bool rv = it * R + r < nrows;
                const T mx = (m[r] == neg_inf<T>()) ? T(0) : m[r];
                T sp[VW];
#pragma unroll
                for (int e = 0; e < VW; ++e) sp[e] = T(0);
#pragma unroll
                for (int c = 0; c < CH; ++c)
#pragma unroll
                    for (int e = 0; e < VW; ++e) {
                        const T v = SkMath<T>::ex(y[r][c][e] - mx);
                        y[r][c][e] = v;
                        sp[e] += v;
                    }
                sum[r] = rv ? (sp[0] + sp[1]) + (sp[2] + sp[3]) : T(0);
                if (!rv) m[r] = neg_inf<T>();
            }
            if constexpr (LAGGED) {
                // the exponentials wait in the stage for the lagged finish
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    V *stw = reinterpret_cast<V *>(rg.base + (size_t)s * rg.stage_bytes + (size_t)r * rg.row_bytes);
#pragma unroll
                    for (int c = 0; c < CH; ++c) {
                        const int col = c0 + (tid + NT * c) * VW;
                        if (col < c1 && !rowonly)
                            stw[tid + NT * c] = make_float4(y[r][c][0], y[r][c][1], y[r][c][2], y[r][c][3]);
                    }
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                for (int r = 0; r < R; ++r) sum[r] += __shfl_xor_sync(0xffffffffu, sum[r], off);
            if (lane == 0) {
#pragma unroll
                for (int r = 0; r < R; ++r) { s_wp[b & 1][warp][r][0] = m[r]; s_wp[b & 1][warp][r][1] = sum[r]; }
            }
            __syncthreads();
            // every warp combines the NW warp pairs of each row (fixed tree: identical in all warps)
            T M[R], Sm[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if constexpr (MAXP) {
                    const T mv = lane < NW ? s_wp[b & 1][lane][r][0] : neg_inf<T>();
                    M[r] = mv;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) M[r] = vmax(M[r], __shfl_xor_sync(0xffffffffu, M[r], off));
                    Sm[r] = (mv != neg_inf<T>()) ? s_wp[b & 1][lane][r][1] * SkMath<T>::ex(mv - M[r]) : T(0);
                } else {
                    M[r] = m[r];
                    Sm[r] = lane < NW ? s_wp[b & 1][lane][r][1] : T(0);
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                for (int r = 0; r < R; ++r) Sm[r] += __shfl_xor_sync(0xffffffffu, Sm[r], off);
            if constexpr (!LAGGED) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (it * R + r >= nrows) continue;
                    if constexpr (!MAXP) bad |= !(Sm[r] >= kShiftLo && Sm[r] <= kShiftHi) || a.resident == 3;
                    PIPE_FINISH(it * R + r, (double)M[r] + SkMath<T>::lgt(Sm[r]), m[r], y[r]);
                }
            } else {
                // this CTA's pairs -> every rank of the cluster; finished next band
                const int xs = (int)(b & 3);
                if (warp == 0) {
                    if (lane == 0) xbar_arm(&ps.xbar[xs], (uint32_t)(CL * R * 2 * sizeof(T)));
                    __syncwarp();
                    if (lane < CL) {
#pragma unroll
                        for (int r = 0; r < R; ++r)
                            st_async_pair(dsmem_map(&ps.xp[xs][sl.rank][r][0], lane), M[r], Sm[r],
                                          dsmem_map(&ps.xbar[xs], lane));
                    }
                }
            }
        }
        if constexpr (LAGGED) {
            if (it >= 1) {
                const unsigned bf = b - 1;
                const int xs = (int)(bf & 3);
                T mq[R][CL], sq[R][CL];
                if (lane == 0) {
                    xbar_wait(&ps.xbar[xs], (bf >> 2) & 1);
#pragma unroll
                    for (int r = 0; r < R; ++r)
#pragma unroll
                        for (int q = 0; q < CL; ++q) { mq[r][q] = ps.xp[xs][q][r][0]; sq[r][q] = ps.xp[xs][q][r][1]; }
                }
                const int sf = (int)(bf % (unsigned)S);
#pragma unroll
                for (int r = 0; r < R; ++r) {
#pragma unroll
                    for (int q = 0; q < CL; ++q) {
                        mq[r][q] = __shfl_sync(0xffffffffu, mq[r][q], 0);
                        sq[r][q] = __shfl_sync(0xffffffffu, sq[r][q], 0);
                    }
                    const int lr = (it - 1) * R + r;
                    if (lr >= nrows) continue;
                    T M = neg_inf<T>(), Sm = T(0);
                    if constexpr (MAXP) {
#pragma unroll
                        for (int q = 0; q < CL; ++q) M = vmax(M, mq[r][q]);
#pragma unroll
                        for (int q = 0; q < CL; ++q)
                            if (mq[r][q] != neg_inf<T>()) Sm += sq[r][q] * SkMath<T>::ex(mq[r][q] - M);
                    } else {
                        M = mq[r][0];  // the common shift
#pragma unroll
                        for (int q = 0; q < CL; ++q) Sm += sq[r][q];
                        bad |= !(Sm >= kShiftLo && Sm <= kShiftHi) || a.resident == 3;
                    }
                    const V *stf = reinterpret_cast<const V *>(rg.base + (size_t)sf * rg.stage_bytes +
                                                               (size_t)r * rg.row_bytes);
                    T yl[CH][VW];
#pragma unroll
                    for (int c = 0; c < CH; ++c) {
                        const int col = c0 + (tid + NT * c) * VW;
                        const V yv = (col < c1 && !rowonly) ? stf[tid + NT * c] : make_float4(0.f, 0.f, 0.f, 0.f);
                        yl[c][0] = yv.x; yl[c][1] = yv.y; yl[c][2] = yv.z; yl[c][3] = yv.w;
                    }
                    PIPE_FINISH(lr, (double)M + SkMath<T>::lgt(Sm), mp[r], yl);
                }
                fence_proxy_async_smem();  // this thread's stage accesses precede the bulk refill
                __syncwarp();
                if (lane == 0) mbar_arrive(&ps.empty[sf]);
            }
#pragma unroll
            for (int r = 0; r < R; ++r) mp[r] = m[r];
        }
    }
    rg.used = b0 + (unsigned)nb;
    if (!rowonly) {
        T *cp = static_cast<T *>(a.colpart) + (int64_t)sl.grp * a.ldp;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int col = c0 + (tid + NT * c) * VW;
            if (col < c1) __stcg(reinterpret_cast<V *>(cp + col), make_float4(acc[c][0], acc[c][1], acc[c][2], acc[c][3]));
        }
    }
    if constexpr (!MAXP) {
        if (bad && tid == 0) atomicOr(redo, 1u);  // `bad` is uniform across the CTA
    }
    // dev_{k-1} = max over this group's rows of |expm1(f_{k-1} - f_k)| = |u K v - 1|
    __shared__ double s_dev[NW];
    if (sl.rank == 0 && k >= 2) {
        __syncthreads();  // the writer's f_k stores precede the reads below
        for (int i = tid; i < nrows; i += NT) {
            const int row = sl.grp + i * sl.ngrp;
            devmax = fmax(devmax, SkMath<T>::dev(__ldcg(fprev + row) - __ldcg(fout + row)));
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) devmax = fmax(devmax, __shfl_xor_sync(0xffffffffu, devmax, off));
    if (lane == 0) s_dev[warp] = devmax;
    __syncthreads();
    if (tid == 0) {
        double d = 0.0;
        for (int w = 0; w < NW; ++w) d = fmax(d, s_dev[w]);
        __stcg(a.devpart + blockIdx.x, d);
        if (a.dslot) atomicMax(a.dslot + (k & 1), (unsigned long long)__double_as_longlong(d));
    }
}

// GOAT_SK_RES (SkArgs::resident): 2 = max shift only, 3 = flag every fixed-shift sweep
// for a redo (tests of the redo path)
__device__ __forceinline__ bool env_shift_ok(const SkArgs &a) { return a.resident != 2; }

template <int CH, int CL, int NT, int R>
__global__ void __launch_bounds__(NT, NT <= 256 ? 2 : 1) sk_pipe_kernel(SkArgs a, unsigned *bar) {
    using T = float;
    constexpr int NW = NT / 32;
    __shared__ int s_k, s_done;
    if (threadIdx.x == 0) { s_k = a.st->k; s_done = a.st->done | a.st->pending; }
    __syncthreads();
    if (a.single_pass && s_done) return;
    const int k0 = s_k;
    const int K = a.st->max_sweeps;
    const double tol = a.st->tol, coef = a.st->coef, gmax = a.st->gmax;
    const int blk = blockIdx.x, nblk = gridDim.x;
    Slice sl{0, a.n, blk, nblk, 0};
    if constexpr (CL > 1) {
        uint32_t rank, cid, ncl;
        asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        asm("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
        asm("mov.u32 %0, %%nclusterid.x;" : "=r"(ncl));
        sl.rank = (int)rank;
        sl.grp = (int)cid;
        sl.ngrp = (int)ncl;
        sl.c0 = min(a.n, (int)rank * a.slice_w);
        sl.c1 = min(a.n, sl.c0 + a.slice_w);
    }
    __shared__ PipeSm<NW, CL, R> ps;
    extern __shared__ __align__(128) char sk_ring[];
    PipeRing rg;
    rg.base = sk_ring;
    rg.S = a.stages;
    rg.stage_bytes = a.stage_bytes;
    rg.row_bytes = a.stage_bytes / R;
    rg.nrows = (rows_of(a) - sl.grp + sl.ngrp - 1) / sl.ngrp;
    rg.nbands = (max(rg.nrows, 0) + R - 1) / R;
    rg.copy_bytes = (uint32_t)(((sl.c1 - sl.c0 + 3) / 4) * sizeof(float4));
    rg.issued = 0;
    rg.used = 0;
    if (threadIdx.x == 0) {
        for (int q = 0; q < rg.S; ++q) { mbar_init(&ps.full[q], 1); mbar_init(&ps.empty[q], NW); }
        for (int q = 0; q < 4; ++q) { mbar_init(&ps.wbar[q], NW); mbar_init(&ps.xbar[q], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if constexpr (CL > 1) cluster_sync();  // every peer's barriers exist before the first st.async
    else __syncthreads();
    if (rg.nrows <= 0) { rg.nrows = 0; rg.nbands = 0; }
    unsigned epoch = 0;
    auto drain = [&]() {  // no bulk copy may be in flight when the CTA exits
        if (threadIdx.x == 0)
            for (unsigned u = rg.used; u < rg.issued; ++u)
                mbar_wait_cta(&ps.full[u % (unsigned)rg.S], (u / (unsigned)rg.S) & 1);
        if constexpr (CL > 1) cluster_sync();
    };
    // redo flags (one per sweep parity) share the barrier scratch: bytes [256, 264)
    unsigned *redo = bar + 64;
    // single-pass launches (row-sharded driver) take the fixed shift too; a row that leaves
    // the window on any rank makes every rank repeat the sweep with the max shift (redo_next)
    const bool shift_ok = rg.nrows <= kPipeShiftRows && env_shift_ok(a) && !(a.single_pass && a.st->redo_next);
    for (int k = k0;; ++k) {
        bool maxp = !shift_ok || k <= 1;
        for (;;) {
            if (rg.nrows > 0) {
                if (maxp) pass_body_pipe<CH, CL, NT, R, true>(a, k, K, coef, gmax, sl, ps, rg, redo + (k & 1));
                else pass_body_pipe<CH, CL, NT, R, false>(a, k, K, coef, gmax, sl, ps, rg, redo + (k & 1));
            } else if (threadIdx.x == 0) {
                __stcg(a.devpart + blockIdx.x, 0.0);
            }
            if (a.single_pass) { drain(); return; }
            grid_barrier(bar, nblk, epoch);
            if (maxp || !__ldcg(redo + (k & 1))) break;
            // a row left the shift window: recompute the sweep with the max shift
            if (blk == 0 && threadIdx.x == 0) { a.dslot[k & 1] = 0ull; a.st->redone += 1; }
            grid_barrier(bar, nblk, epoch);
            maxp = true;
        }
        const double drow = __longlong_as_double((long long)__ldcg(a.dslot + (k & 1)));
        if (blk == 0 && threadIdx.x == 0) {
            a.dslot[(k + 1) & 1] = 0ull;  // next sweep's slots
            redo[(k + 1) & 1] = 0u;
        }
        int stop = 0, sweeps = 0, conv = 0, slot = 0;
        if (k >= 2) {
            if (drow < tol) { stop = 1; sweeps = k - 1; conv = 1; slot = (k - 1) & 1; }
            else if (k == K + 1) { stop = 1; sweeps = K; conv = 0; slot = K & 1; }
        }
        if (!stop) {
            merge_body<T, NT>(a, k, coef, gmax, blk, nblk);
            grid_barrier(bar, nblk, epoch);
            if (k == 0) {
                const double d0 = fmax(drow, __longlong_as_double((long long)__ldcg(a.dslot + 2)));
                if (d0 < tol) { stop = 1; sweeps = 0; conv = 1; slot = 0; }
                if (blk == 0 && threadIdx.x == 0) a.st->last_dev = d0;
                if (stop && blk == 0 && threadIdx.x == 0) a.st->dev = d0;
            }
        } else if (blk == 0 && threadIdx.x == 0) {
            a.st->dev = drow;
        }
        if (stop) {
            if (blk == 0 && threadIdx.x == 0) {
                a.st->done = 1; a.st->sweeps = sweeps; a.st->converged = conv; a.st->slot = slot;
                a.st->k = k + 1;
            }
            drain();
            return;
        }
    }
}

// ------------------------------------------------------------------ 2-CTA wide rows (fp32)
// 12288 < n <= 40960 (config 5: n = 40000).  A 2-CTA cluster owns a row group
// and CTA rank q the column slice q (<= 20480 columns), so the clusters pack all
// 148 SMs (4-CTA clusters strand 16).  Thread t owns the 16-byte chunks
// t + NT*c (c < CH) of the slice: the row's exponentials y and the sweep's
// column accumulators stay in registers, g of the slice in shared memory.  Row
// slices stream through a ring of S sub-row stages (CC chunks per thread each;
// cp.async.bulk with full/empty mbarriers).  Per row every warp releases its
// stages as soon as it has loaded them; after the row's named barrier thread 0
// refills every released stage, so up to S stages (~1.6 rows) stay in flight
// through the row's reduction and the cluster exchange.  Per row: one warp
// butterfly, one named barrier, one DSMEM pair exchange with the peer (st.async
// + mbarrier complete_tx), rank-order combine -- identical in both CTAs.  No
// exponentials are written back to shared memory.  Sweeps >= 2 use the previous
// row LSE as the shift (plain sums; out-of-window rows redo the sweep with the
// max shift), exactly as sk_pipe_kernel.
template <int NT, int CL> struct W2Sm {
    uint64_t full[16], empty[16], xbar[4];
    float xp[4][CL][2];            // [slot][rank][max, sum] of the exchanged CTA pairs
    float wp[2][NT / 32][2];       // per-warp (max, sum), parity double buffer
};

__device__ __forceinline__ void named_bar(int id, int nt) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nt) : "memory");
}

// Producer cursor (thread 0 only; kept in shared memory so it costs the compute
// threads no registers): chunks issued / to issue, next stage and its empty-barrier
// parity, the chunk's part and row, the row's source pointer -- advanced
// incrementally (no divisions on the issue path).
struct W2Prod {
    unsigned limit, issued;
    int ps, ppart, plr, width, hint;
    uint32_t pph;
    const float *prow, *row0;
    int64_t row_step;      // ngrp * ld
    uint64_t pol;          // L2 evict_first policy (G streams through once per sweep)
};

struct W2Ring {
    char *base;
    int S, CPR, nrows;
    int chunk_floats;      // columns per stage (NT * CC * 4)
    unsigned used;         // chunks consumed (every thread, uniform)
    int cs;                // consumer stage index
    uint32_t cph;          // consumer phase parity
    int nb;                // thread 0 also refills without blocking right after its row loads
    W2Prod *pr;
};

__device__ __forceinline__ bool mbar_test_cta(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// Thread 0: refill released stages, up to S chunks ahead of `used` (the chunks
// this thread has consumed).  block = false only tests the empty barriers (a
// stage some warp still reads is left for a later call).
template <int NT, int CL>
__device__ __forceinline__ void w2_issue(W2Ring &rg, W2Sm<NT, CL> &ws, unsigned used, bool block) {
    W2Prod &pr = *rg.pr;
    while (pr.issued < used + (unsigned)rg.S && pr.issued < pr.limit) {
        const int s = pr.ps;
        if (pr.issued >= (unsigned)rg.S) {
            if (block) mbar_wait_cta(&ws.empty[s], pr.pph);
            else if (!mbar_test_cta(&ws.empty[s], pr.pph)) return;
        }
        const int col0 = pr.ppart * rg.chunk_floats;
        const int cols = min(rg.chunk_floats, pr.width - col0);
        const uint32_t bytes = (uint32_t)(((cols + 3) / 4) * 16);
        char *dst = rg.base + (size_t)s * (size_t)rg.chunk_floats * 4;
        xbar_arm(&ws.full[s], bytes);
        if (pr.hint) bulk_g2s_hint(dst, pr.prow + col0, bytes, &ws.full[s], pr.pol);
        else bulk_g2s(dst, pr.prow + col0, bytes, &ws.full[s]);
        ++pr.issued;
        if (++pr.ps == rg.S) { pr.ps = 0; if (pr.issued > (unsigned)rg.S) pr.pph ^= 1u; }
        if (pr.issued == (unsigned)rg.S) pr.pph = 0;  // the first refill waits on phase 0
        if (++pr.ppart == rg.CPR) {
            pr.ppart = 0;
            if (++pr.plr == rg.nrows) { pr.plr = 0; pr.prow = pr.row0; }
            else pr.prow += pr.row_step;
        }
    }
}

// One row slice into registers: wait for all of the row's stages first, issue
// every shared-memory load, then release the stages together (the loads overlap;
// a per-stage wait/load/release chain serialised the warp that also refills).
template <int NT, int CL, int CH, int CC>
__device__ __forceinline__ void w2_load_row(W2Ring &rg, W2Sm<NT, CL> &ws, float (&y)[CH][4], int tid, int lane) {
    constexpr int CPR = CH / CC;
    int sidx[CPR];
    {
        int cs = rg.cs;
        uint32_t ph = rg.cph;
#pragma unroll
        for (int p = 0; p < CPR; ++p) {
            sidx[p] = cs;
            mbar_wait_cta(&ws.full[cs], ph);
            if (++cs == rg.S) { cs = 0; ph ^= 1u; }
        }
        rg.cs = cs;
        rg.cph = ph;
    }
#pragma unroll
    for (int p = 0; p < CPR; ++p) {
        const float4 *st = reinterpret_cast<const float4 *>(rg.base + (size_t)sidx[p] * rg.chunk_floats * 4);
#pragma unroll
        for (int q = 0; q < CC; ++q) {
            const float4 xv = st[tid + NT * q];
            y[p * CC + q][0] = xv.x; y[p * CC + q][1] = xv.y; y[p * CC + q][2] = xv.z; y[p * CC + q][3] = xv.w;
        }
    }
    __syncwarp();
    if (lane == 0) {
#pragma unroll
        for (int p = 0; p < CPR; ++p) mbar_arrive(&ws.empty[sidx[p]]);
    }
    rg.used += (unsigned)CPR;
    // refill whatever every warp has released so far (non-blocking)
    if (tid == 0 && rg.nb) w2_issue<NT, CL>(rg, ws, rg.used, false);
}

template <int NT, int CL, int CH, int CC, bool MAXP>
__device__ __forceinline__ void pass_body_wide(const SkArgs &a, int k, int max_sweeps, double coef_d, double gmax_d,
                                               const Slice &sl, W2Sm<NT, CL> &ws, W2Ring &rg, float4 *s_g,
                                               float *s_shift, unsigned &xi, unsigned *redo) {
    using T = float;
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool pre = (k == 0);
    const bool rowonly = (k == max_sweeps + 1);
    const double *gin = gslot(a, k + 1);
    const double *fprev = fslot(a, k + 1);
    double *fout = fslot(a, k);
    const double ks = SkMath<T>::kScale;
    const T coef = (T)(coef_d * ks);
    const T gmax = (T)gmax_d;
    const int c0 = sl.c0, c1 = sl.c1;
    const bool writer = (sl.rank == 0) && tid == 0;
    // g of this thread's chunks (scaled; -inf masks columns past the slice)
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        float gv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int col = c0 + (tid + NT * c) * 4 + e;
            gv[e] = col < c1 ? ((!pre) ? (T)(__ldcg(gin + col) * ks) : T(0)) : neg_inf<T>();
        }
        s_g[tid + NT * c] = make_float4(gv[0], gv[1], gv[2], gv[3]);  // read back by this thread only
    }
    if constexpr (!MAXP) {
        for (int i = tid; i < rg.nrows; i += NT) s_shift[i] = (float)(-__ldcg(fprev + sl.grp + i * sl.ngrp) * ks);
        named_bar(1, NT);
    }
    T acc[CH][4];
#pragma unroll
    for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[c][e] = T(0);
    double devmax = 0.0;
    bool bad = false;
    for (int lr = 0; lr < rg.nrows; ++lr) {
        // ---- this row's slice: CPR stages of CC chunks per thread
        T y[CH][4];
        w2_load_row<NT, CL, CH, CC>(rg, ws, y, tid, lane);
        // ---- E_ij + g_j (sinkhorn.py:125), shift, exponentials, warp pair
        T m;
        if constexpr (MAXP) {
            m = neg_inf<T>();
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const float4 g4 = s_g[tid + NT * c];
                const T gl[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const T arg = coef * (gmax - y[c][e]) + gl[e];
                    y[c][e] = arg;
                    m = vmax(m, arg);
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) m = vmax(m, __shfl_xor_sync(0xffffffffu, m, off));
        } else {
            m = s_shift[lr];  // the row's shift, identical in every warp and both ranks
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const float4 g4 = s_g[tid + NT * c];
                const T gl[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) y[c][e] = coef * (gmax - y[c][e]) + gl[e];
            }
        }
        const T mx = (m == neg_inf<T>()) ? T(0) : m;
        T sp[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
        for (int c = 0; c < CH; ++c)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const T v = SkMath<T>::ex(y[c][e] - mx);
                y[c][e] = v;
                sp[e] += v;
            }
        T sum = (sp[0] + sp[1]) + (sp[2] + sp[3]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
        const int par = (int)(xi & 1u);
        if (lane == 0) { ws.wp[par][warp][0] = m; ws.wp[par][warp][1] = sum; }
        named_bar(1, NT);
        // ---- CTA pair: every warp combines the NW warp pairs (fixed xor tree)
        T M, Sm;
        {
            const T mv = lane < NW ? ws.wp[par][lane][0] : neg_inf<T>();
            const T sv = lane < NW ? ws.wp[par][lane][1] : T(0);
            if constexpr (MAXP) {
                M = mv;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) M = vmax(M, __shfl_xor_sync(0xffffffffu, M, off));
                Sm = (mv != neg_inf<T>()) ? sv * SkMath<T>::ex(mv - M) : T(0);
            } else {
                M = m;
                Sm = sv;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) Sm += __shfl_xor_sync(0xffffffffu, Sm, off);
        }
        // ---- exchange with the CL-1 peer CTAs, combine in rank order
        const int xs = (int)(xi & 3u);
        const uint32_t xph = (xi >> 2) & 1u;
        if (tid == 0) xbar_arm(&ws.xbar[xs], (uint32_t)((CL - 1) * 2 * sizeof(T)));
        if (warp == 0 && lane < CL && lane != sl.rank)
            st_async_pair(dsmem_map(&ws.xp[xs][sl.rank][0], (uint32_t)lane), M, Sm,
                          dsmem_map(&ws.xbar[xs], (uint32_t)lane));
        // every warp passed the row barrier: all of this row's stages are free
        if (tid == 0) w2_issue<NT, CL>(rg, ws, rg.used, true);
        xbar_wait(&ws.xbar[xs], xph);
        T mq[CL], sq[CL];
#pragma unroll
        for (int q = 0; q < CL; ++q) {
            mq[q] = (q == sl.rank) ? M : ws.xp[xs][q][0];
            sq[q] = (q == sl.rank) ? Sm : ws.xp[xs][q][1];
        }
        T Mt, St = T(0);
        if constexpr (MAXP) {
            Mt = neg_inf<T>();
#pragma unroll
            for (int q = 0; q < CL; ++q) Mt = vmax(Mt, mq[q]);
#pragma unroll
            for (int q = 0; q < CL; ++q)
                if (mq[q] != neg_inf<T>()) St += sq[q] * SkMath<T>::ex(mq[q] - Mt);
        } else {
            Mt = mq[0];  // the common shift
#pragma unroll
            for (int q = 0; q < CL; ++q) St += sq[q];
            bad |= !(St >= kShiftLo && St <= kShiftHi) || a.resident == 3;
        }
        ++xi;
        const double lse = (double)Mt + SkMath<T>::lgt(St);  // scaled units
        if (writer) {
            const double fnew = -lse * (1.0 / ks);
            if (pre) devmax = fmax(devmax, SkMath<T>::dev(-fnew));
            else __stcg(fout + sl.grp + lr * sl.ngrp, fnew);
        }
        if (!rowonly && m != neg_inf<T>()) {
            // column contribution exp(E + g + f_k) = y * 2^(m - lse); the pre-check sums K
            const T sc = SkMath<T>::ex((T)((double)m + (pre ? 0.0 : -lse)));
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[c][e] += y[c][e] * sc;
        }
    }
    if (!rowonly) {
        T *cp = static_cast<T *>(a.colpart) + (int64_t)sl.grp * a.ldp;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int col = c0 + (tid + NT * c) * 4;
            if (col < c1) __stcg(reinterpret_cast<float4 *>(cp + col), make_float4(acc[c][0], acc[c][1], acc[c][2], acc[c][3]));
        }
    }
    if constexpr (!MAXP) {
        if (bad && tid == 0) atomicOr(redo, 1u);  // `bad` is uniform across the CTA
    }
    // dev_{k-1} = max over this group's rows of |expm1(f_{k-1} - f_k)| = |u K v - 1|
    __shared__ double s_dev[NW];
    __syncthreads();  // the writer's f_k stores precede the reads below
    if (sl.rank == 0 && k >= 2) {
        for (int i = tid; i < rg.nrows; i += NT) {
            const int row = sl.grp + i * sl.ngrp;
            devmax = fmax(devmax, SkMath<T>::dev(__ldcg(fprev + row) - __ldcg(fout + row)));
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) devmax = fmax(devmax, __shfl_xor_sync(0xffffffffu, devmax, off));
    if (lane == 0) s_dev[warp] = devmax;
    __syncthreads();
    if (tid == 0) {
        double d = 0.0;
        for (int w = 0; w < NW; ++w) d = fmax(d, s_dev[w]);
        __stcg(a.devpart + blockIdx.x, d);
        if (a.dslot) atomicMax(a.dslot + (k & 1), (unsigned long long)__double_as_longlong(d));
    }
}

// TMEM-lagged variant (TM) of the wide-row pass: as pass_body_wide, but a row's
// exponentials are parked in tensor memory (tcgen05.st, 32x32b: each thread its
// own TMEM lane) while the peer's pair of the row travels, and the row is
// finished one row later (tcgen05.ld back into registers, acc += y * sc) -- the
// cluster exchange latency hides behind the next row's loads and exponentials.
// TMEM holds two row slots per warp: (warp>>2)*2 + slot selects CH*4 columns of
// the warp's lane quadrant (warp & 3).
__device__ __forceinline__ void tm_st8(uint32_t taddr, const float *v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t taddr, float *v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <int NT, int CL, int CH, int CC, bool MAXP>
__device__ __forceinline__ void pass_body_tm(const SkArgs &a, int k, int max_sweeps, double coef_d, double gmax_d,
                                             const Slice &sl, W2Sm<NT, CL> &ws, W2Ring &rg, float4 *s_g,
                                             float *s_shift, unsigned &xi, unsigned *redo, uint32_t tbase) {
    using T = float;
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool pre = (k == 0);
    const bool rowonly = (k == max_sweeps + 1);
    const double *gin = gslot(a, k + 1);
    const double *fprev = fslot(a, k + 1);
    double *fout = fslot(a, k);
    const double ks = SkMath<T>::kScale;
    const T coef = (T)(coef_d * ks);
    const T gmax = (T)gmax_d;
    const int c0 = sl.c0, c1 = sl.c1;
    const bool writer = (sl.rank == 0) && tid == 0;
    const uint32_t tq = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
    // g of this thread's chunks (scaled; -inf masks columns past the slice) in TMEM
    // columns [(8 + (warp>>2)) * CH*4, ...) of the warp's lane quadrant
    const uint32_t tg = tq + (uint32_t)((8 + (warp >> 2)) * CH * 4);
    {
        float gv[CH][4];
#pragma unroll
        for (int c = 0; c < CH; ++c)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int col = c0 + (tid + NT * c) * 4 + e;
                gv[c][e] = col < c1 ? ((!pre) ? (T)(__ldcg(gin + col) * ks) : T(0)) : neg_inf<T>();
            }
#pragma unroll
        for (int c = 0; c < CH; c += 2) tm_st8(tg + (uint32_t)(c * 4), &gv[c][0]);
        tm_wait_st();
    }
    if constexpr (!MAXP) {
        for (int i = tid; i < rg.nrows; i += NT) s_shift[i] = (float)(-__ldcg(fprev + sl.grp + i * sl.ngrp) * ks);
        named_bar(1, NT);
    }
    T acc[CH][4];
#pragma unroll
    for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[c][e] = T(0);
    double devmax = 0.0;
    bool bad = false;
    const unsigned x0 = xi;
    T mprev = T(0), Mp = T(0), Sp = T(0);
#ifdef GOAT_SK_PHASE_TRACE
    // phase-cycle accounting of thread 0 for the traced sweep (GOAT_SK_TRACE=k, GOAT_SK_TRACE_RAW=1;
    // build with -DGOAT_SK_PHASE_TRACE)
    const bool tr = a.trace && k == a.trace_k && tid == 0;
    unsigned long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tl = tr ? clock64() : 0;
    auto tick = [&](int i) { if (tr) { const unsigned long long t = clock64(); tacc[i] += t - tl; tl = t; } };
#else
    auto tick = [](int) {};
#endif
    for (int it = 0; it <= rg.nrows; ++it) {
        T m = T(0), Mc = T(0), Sc = T(0);
        if (it < rg.nrows) {
            // ---- row it: loads, exponentials, this CTA's pair; exponentials -> TMEM
            T y[CH][4];
            tick(7);
            w2_load_row<NT, CL, CH, CC>(rg, ws, y, tid, lane);
            tick(1);
            // E_ij + g_j (sinkhorn.py:125), g streamed back from TMEM two chunks at a time
#pragma unroll
            for (int c = 0; c < CH; c += 2) {
                float gl[2][4];
                tm_ld8(tg + (uint32_t)(c * 4), &gl[0][0]);
                tm_wait_ld();
#pragma unroll
                for (int q = 0; q < 2; ++q)
#pragma unroll
                    for (int e = 0; e < 4; ++e) y[c + q][e] = coef * (gmax - y[c + q][e]) + gl[q][e];
            }
            if constexpr (MAXP) {
                m = neg_inf<T>();
#pragma unroll
                for (int c = 0; c < CH; ++c)
#pragma unroll
                    for (int e = 0; e < 4; ++e) m = vmax(m, y[c][e]);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) m = vmax(m, __shfl_xor_sync(0xffffffffu, m, off));
            } else {
                m = s_shift[it];
            }
            const T mx = (m == neg_inf<T>()) ? T(0) : m;
            T sp[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const T v = SkMath<T>::ex(y[c][e] - mx);
                    y[c][e] = v;
                    sp[e] += v;
                }
            // park the exponentials until the row is finished (next iteration)
            if (!rowonly) {
                const uint32_t tcol = tq + (uint32_t)(((warp >> 2) * 2 + (it & 1)) * CH * 4);
#pragma unroll
                for (int c = 0; c < CH; c += 2) tm_st8(tcol + (uint32_t)(c * 4), &y[c][0]);
            }
            T sum = (sp[0] + sp[1]) + (sp[2] + sp[3]);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
            const int par = it & 1;
            if (lane == 0) { ws.wp[par][warp][0] = m; ws.wp[par][warp][1] = sum; }
            tick(2);
            named_bar(1, NT);
            const T mv = lane < NW ? ws.wp[par][lane][0] : neg_inf<T>();
            tick(3);
            const T sv = lane < NW ? ws.wp[par][lane][1] : T(0);
            if constexpr (MAXP) {
                Mc = mv;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) Mc = vmax(Mc, __shfl_xor_sync(0xffffffffu, Mc, off));
                Sc = (mv != neg_inf<T>()) ? sv * SkMath<T>::ex(mv - Mc) : T(0);
            } else {
                Mc = m;
                Sc = sv;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) Sc += __shfl_xor_sync(0xffffffffu, Sc, off);
            const unsigned xr = x0 + (unsigned)it;
            if (tid == 0) xbar_arm(&ws.xbar[xr & 3u], (uint32_t)((CL - 1) * 2 * sizeof(T)));
            if (warp == 0 && lane < CL && lane != sl.rank)
                st_async_pair(dsmem_map(&ws.xp[xr & 3u][sl.rank][0], (uint32_t)lane), Mc, Sc,
                              dsmem_map(&ws.xbar[xr & 3u], (uint32_t)lane));
            // every warp passed the row barrier: all of this row's stages are free
            if (tid == 0) w2_issue<NT, CL>(rg, ws, rg.used, true);
            tick(4);
        }
        if (it >= 1) {
            // ---- finish row it-1 from every rank's pair (rank order)
            const int lr = it - 1;
            const unsigned xr = x0 + (unsigned)lr;
            xbar_wait(&ws.xbar[xr & 3u], (xr >> 2) & 1u);
            tick(5);
            T mq[CL], sq[CL];
#pragma unroll
            for (int q = 0; q < CL; ++q) {
                mq[q] = (q == sl.rank) ? Mp : ws.xp[xr & 3u][q][0];
                sq[q] = (q == sl.rank) ? Sp : ws.xp[xr & 3u][q][1];
            }
            T Mt, St = T(0);
            if constexpr (MAXP) {
                Mt = neg_inf<T>();
#pragma unroll
                for (int q = 0; q < CL; ++q) Mt = vmax(Mt, mq[q]);
#pragma unroll
                for (int q = 0; q < CL; ++q)
                    if (mq[q] != neg_inf<T>()) St += sq[q] * SkMath<T>::ex(mq[q] - Mt);
            } else {
                Mt = mq[0];  // the common shift
#pragma unroll
                for (int q = 0; q < CL; ++q) St += sq[q];
                bad |= !(St >= kShiftLo && St <= kShiftHi) || a.resident == 3;
            }
            const double lse = (double)Mt + SkMath<T>::lgt(St);  // scaled units
            if (writer) {
                const double fnew = -lse * (1.0 / ks);
                if (pre) devmax = fmax(devmax, SkMath<T>::dev(-fnew));
                else __stcg(fout + sl.grp + lr * sl.ngrp, fnew);
            }
            if (!rowonly) {
                // column contribution exp(E + g + f_k) = y * 2^(m - lse); the pre-check sums K
                T yl[CH][4];
                const uint32_t tcol = tq + (uint32_t)(((warp >> 2) * 2 + (lr & 1)) * CH * 4);
                tm_wait_st();
#pragma unroll
                for (int c = 0; c < CH; c += 2) tm_ld8(tcol + (uint32_t)(c * 4), &yl[c][0]);
                tm_wait_ld();
                const T sc = (mprev == neg_inf<T>()) ? T(0) : SkMath<T>::ex((T)((double)mprev + (pre ? 0.0 : -lse)));
#pragma unroll
                for (int c = 0; c < CH; ++c)
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[c][e] += yl[c][e] * sc;
            }
            tick(6);
        }
        mprev = m;
        Mp = Mc;
        Sp = Sc;
    }
    xi = x0 + (unsigned)rg.nrows;
#ifdef GOAT_SK_PHASE_TRACE
    if (tr) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a.trace[blockIdx.x * 16 + i] = tacc[i] + 1;
    }
#endif
    if (!rowonly) {
        T *cp = static_cast<T *>(a.colpart) + (int64_t)sl.grp * a.ldp;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int col = c0 + (tid + NT * c) * 4;
            if (col < c1) __stcg(reinterpret_cast<float4 *>(cp + col), make_float4(acc[c][0], acc[c][1], acc[c][2], acc[c][3]));
        }
    }
    if constexpr (!MAXP) {
        if (bad && tid == 0) atomicOr(redo, 1u);  // `bad` is uniform across the CTA
    }
    __shared__ double s_dev[NW];
    __syncthreads();  // the writer's f_k stores precede the reads below
    if (sl.rank == 0 && k >= 2) {
        for (int i = tid; i < rg.nrows; i += NT) {
            const int row = sl.grp + i * sl.ngrp;
            devmax = fmax(devmax, SkMath<T>::dev(__ldcg(fprev + row) - __ldcg(fout + row)));
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) devmax = fmax(devmax, __shfl_xor_sync(0xffffffffu, devmax, off));
    if (lane == 0) s_dev[warp] = devmax;
    __syncthreads();
    if (tid == 0) {
        double d = 0.0;
        for (int w = 0; w < NW; ++w) d = fmax(d, s_dev[w]);
        __stcg(a.devpart + blockIdx.x, d);
        if (a.dslot) atomicMax(a.dslot + (k & 1), (unsigned long long)__double_as_longlong(d));
    }
}

template <int NT, int CL, int CH, int CC, bool TM>
__global__ void __launch_bounds__(NT, (NT <= 256 ? 2 : 1)) sk_wide_kernel(SkArgs a, unsigned *bar) {
    __shared__ int s_k, s_done;
    if (threadIdx.x == 0) { s_k = a.st->k; s_done = a.st->done | a.st->pending; }
    __syncthreads();
    if (a.single_pass && s_done) return;
    const int k0 = s_k;
    const int K = a.st->max_sweeps;
    const double tol = a.st->tol, coef = a.st->coef, gmax = a.st->gmax;
    const int blk = blockIdx.x, nblk = gridDim.x;
    uint32_t rank, cid, ncl;
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    asm("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
    asm("mov.u32 %0, %%nclusterid.x;" : "=r"(ncl));
    Slice sl{0, a.n, (int)cid, (int)ncl, (int)rank};
    sl.c0 = min(a.n, (int)rank * a.slice_w);
    sl.c1 = min(a.n, sl.c0 + a.slice_w);
    __shared__ W2Sm<NT, CL> ws;
    extern __shared__ __align__(128) char sk_ring[];
    W2Ring rg;
    rg.S = a.stages;
    rg.CPR = CH / CC;
    rg.chunk_floats = NT * CC * 4;
    rg.base = sk_ring;
    float4 *s_g = reinterpret_cast<float4 *>(sk_ring + (size_t)rg.S * rg.chunk_floats * 4);
    float *s_shift = reinterpret_cast<float *>(s_g + (TM ? 0 : NT * CH));
    rg.nrows = max(0, (rows_of(a) - sl.grp + sl.ngrp - 1) / sl.ngrp);
    __shared__ W2Prod s_prod;
    rg.pr = &s_prod;
    rg.used = 0; rg.cs = 0; rg.cph = 0;
    rg.nb = (a.dbg & 128) ? 0 : 1;
    if (threadIdx.x == 0) {
        W2Prod &pr = s_prod;
        pr.width = sl.c1 - sl.c0;
        pr.limit = a.single_pass ? (unsigned)(rg.nrows * rg.CPR) : ~0u;
        pr.issued = 0;
        pr.ps = 0; pr.ppart = 0; pr.plr = 0; pr.pph = 0;
        pr.row0 = static_cast<const float *>(a.G) + (int64_t)sl.grp * a.ld + sl.c0;
        pr.prow = pr.row0;
        pr.row_step = (int64_t)sl.ngrp * a.ld;
        // bulk copies stream G through L2 once per sweep: evict_first unless GOAT_SK_DBG bit 64
        pr.hint = (a.dbg & 64) ? 0 : 1;
        pr.pol = 0;
        if (pr.hint) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pr.pol));
    }
    // the tail of a short last chunk is never written by the bulk copies: zero the
    // ring once so masked columns always read finite values
    for (int i = threadIdx.x; i < rg.S * NT * CC; i += NT)
        reinterpret_cast<float4 *>(sk_ring)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        for (int q = 0; q < rg.S; ++q) { mbar_init(&ws.full[q], 1); mbar_init(&ws.empty[q], NT / 32); }
        for (int q = 0; q < 4; ++q) mbar_init(&ws.xbar[q], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // TM: 512 TMEM columns (two parked rows per warp: 4 warps x 2 slots x CH*4 columns
    // per lane quadrant), allocated by warp 0
    __shared__ uint32_t s_tmem;
    if constexpr (TM) {
        if ((threadIdx.x >> 5) == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    cluster_sync();  // every peer's barriers exist before the first st.async
    uint32_t tbase = 0;
    if constexpr (TM) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tbase = s_tmem;
    }
    if (threadIdx.x == 0 && rg.nrows > 0) w2_issue<NT, CL>(rg, ws, 0u, true);
    unsigned epoch = 0, xi = 0;
    auto drain = [&]() {  // no bulk copy may be in flight when the CTA exits
        if (threadIdx.x == 0) {
            unsigned u = rg.used;
            int s = rg.cs;
            uint32_t ph = rg.cph;
            for (; u < s_prod.issued; ++u) {
                mbar_wait_cta(&ws.full[s], ph);
                if (++s == rg.S) { s = 0; ph ^= 1u; }
            }
        }
        if constexpr (TM) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        cluster_sync();
        if constexpr (TM) {
            if ((threadIdx.x >> 5) == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
            }
        }
    };
    unsigned *redo = bar + 64;
    const bool shift_ok = env_shift_ok(a) && !(a.single_pass && a.st->redo_next);
    for (int k = k0;; ++k) {
        bool maxp = !shift_ok || k <= 1;
        for (;;) {
            if (rg.nrows > 0) {
                if constexpr (TM) {
                    if (maxp) pass_body_tm<NT, CL, CH, CC, true>(a, k, K, coef, gmax, sl, ws, rg, s_g, s_shift, xi, redo + (k & 1), tbase);
                    else pass_body_tm<NT, CL, CH, CC, false>(a, k, K, coef, gmax, sl, ws, rg, s_g, s_shift, xi, redo + (k & 1), tbase);
                } else {
                    if (maxp) pass_body_wide<NT, CL, CH, CC, true>(a, k, K, coef, gmax, sl, ws, rg, s_g, s_shift, xi, redo + (k & 1));
                    else pass_body_wide<NT, CL, CH, CC, false>(a, k, K, coef, gmax, sl, ws, rg, s_g, s_shift, xi, redo + (k & 1));
                }
            } else if (threadIdx.x == 0) {
                __stcg(a.devpart + blockIdx.x, 0.0);
            }
            if (a.single_pass) { drain(); return; }
            grid_barrier(bar, nblk, epoch);
            if (maxp || !__ldcg(redo + (k & 1))) break;
            // a row left the shift window: recompute the sweep with the max shift
            if (blk == 0 && threadIdx.x == 0) { a.dslot[k & 1] = 0ull; a.st->redone += 1; }
            grid_barrier(bar, nblk, epoch);
            maxp = true;
        }
        const double drow = __longlong_as_double((long long)__ldcg(a.dslot + (k & 1)));
        if (blk == 0 && threadIdx.x == 0) {
            a.dslot[(k + 1) & 1] = 0ull;  // next sweep's slots
            redo[(k + 1) & 1] = 0u;
        }
        int stop = 0, sweeps = 0, conv = 0, slot = 0;
        if (k >= 2) {
            if (drow < tol) { stop = 1; sweeps = k - 1; conv = 1; slot = (k - 1) & 1; }
            else if (k == K + 1) { stop = 1; sweeps = K; conv = 0; slot = K & 1; }
        }
        if (!stop) {
            merge_body<float, NT>(a, k, coef, gmax, blk, nblk);
            grid_barrier(bar, nblk, epoch);
            if (k == 0) {
                const double d0 = fmax(drow, __longlong_as_double((long long)__ldcg(a.dslot + 2)));
                if (d0 < tol) { stop = 1; sweeps = 0; conv = 1; slot = 0; }
                if (blk == 0 && threadIdx.x == 0) a.st->last_dev = d0;
                if (stop && blk == 0 && threadIdx.x == 0) a.st->dev = d0;
            }
        } else if (blk == 0 && threadIdx.x == 0) {
            a.st->dev = drow;
        }
        if (stop) {
            if (blk == 0 && threadIdx.x == 0) {
                a.st->done = 1; a.st->sweeps = sweeps; a.st->converged = conv; a.st->slot = slot;
                a.st->k = k + 1;
            }
            drain();
            return;
        }
    }
}

template <int NT, int CL, int CH, bool TM, int CC = 2> void *wide2_fn() { return (void *)sk_wide_kernel<NT, CL, CH, CC, TM>; }
void *wide2_for(int nt, int cl, int ch, bool tm = false, int cc = 2) {
    // TM: a half row in two bulk copies per row (cc = ch / 2), or 16 KB stages (cc = 2)
    if (tm && nt == 512 && cl == 2 && cc * 2 == ch) {
        switch (ch) {
            case 4: return wide2_fn<512, 2, 4, true, 2>();
            case 6: return wide2_fn<512, 2, 6, true, 3>();
            case 8: return wide2_fn<512, 2, 8, true, 4>();
            case 10: return wide2_fn<512, 2, 10, true, 5>();
        }
    }
    if (tm && nt == 512 && cl == 2 && cc == 2) {
        switch (ch) {
            case 6: return wide2_fn<512, 2, 6, true>();
            case 8: return wide2_fn<512, 2, 8, true>();
            case 10: return wide2_fn<512, 2, 10, true>();
        }
    }
#define GOAT_W2(NT_, CL_)                                       \
    if (!tm && nt == NT_ && cl == CL_) {                        \
        switch (ch) {                                           \
            case 4: return wide2_fn<NT_, CL_, 4, false>();      \
            case 6: return wide2_fn<NT_, CL_, 6, false>();      \
            case 8: return wide2_fn<NT_, CL_, 8, false>();      \
            case 10: return wide2_fn<NT_, CL_, 10, false>();    \
        }                                                       \
    }
    GOAT_W2(512, 2)
    GOAT_W2(256, 4)
#undef GOAT_W2
    throw Error(GOAT_ENOTSUP, "sinkhorn: no wide-row kernel for threads=" + std::to_string(nt) + " cluster=" +
                                  std::to_string(cl) + " chunks=" + std::to_string(ch));
}

// ------------------------------------------------------------------ row-sharded sweep
// Column sums of this block's pass (fixed CTA order, fp64) and its max row deviation.
template <class T>
__global__ void __launch_bounds__(kThreads) sk_shard_colsum_kernel(SkArgs a, int pass_blocks, double *send,
                                                                   const unsigned *redo) {
    if (*(volatile int *)&a.st->done || *(volatile int *)&a.st->pending) return;
    const int n = a.n, np = a.nblk;
    const T *cp = static_cast<const T *>(a.colpart);
    for (int j = blockIdx.x * kThreads + threadIdx.x; j < n; j += gridDim.x * kThreads) {
        double S = 0.0;
        for (int b = 0; b < np; ++b) S += (double)__ldcg(cp + (int64_t)b * a.ldp + j);
        send[j] = S;
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        double d = 0.0;
        for (int b = threadIdx.x; b < pass_blocks; b += 32) d = fmax(d, __ldcg(a.devpart + b));
        for (int off = 16; off > 0; off >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, off));
        // a fixed-shift pass that left the window on this rank: its column sums are void, and
        // an infinite deviation tells every rank's merge to repeat the sweep with the max shift
        if (threadIdx.x == 0) send[n] = __ldcg(redo + (*(volatile int *)&a.st->k & 1)) ? INFINITY : d;
    }
}

// The gathered [world][n+1] rows merged in rank order (identical on every rank), then
// the stopping rule of sk_sweeps and g_k = g_{k-1} - log(colsum).
// A column sum that under/overflows (fp32: every entry below the ex2 range) is
// flagged in bad[] and the sweep is left pending: sk_shard_repair_pass/merge then
// compute those columns' exact fp64 LSE across all ranks, as sk_exact_col does
// on one GPU, and finish the sweep.
constexpr int kShardMergeThreads = 1024;
__device__ __forceinline__ void shard_finish(SkState *st, int k, int stop, int sweeps, int conv, int slot) {
    if (stop) { st->done = 1; st->sweeps = sweeps; st->converged = conv; st->slot = slot; }
    st->pending = 0;
    st->k = k + 1;
}

__device__ __forceinline__ double block_max_1024(double v, double *s_red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    __syncthreads();
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    double r = 0.0;
    for (int w = 0; w < kShardMergeThreads / 32; ++w) r = fmax(r, s_red[w]);
    return r;
}

// Several CTAs split the columns (a single CTA took 84 us per sweep at n = 40000 -- half of a
// rank's pass time at 8 GPUs); each leaves its (max column deviation, flagged-column count) in
// devcol[2 * blk ..] and the LAST CTA to finish -- st->arrive counts them -- applies the
// stopping rule and advances the loop state, so no CTA reads the state after it was advanced.
// Every quantity is a max or an integer sum: the result does not depend on which CTA is last.
__global__ void __launch_bounds__(kShardMergeThreads) sk_shard_merge_kernel(SkArgs a, const double *recv, int world,
                                                                            double tiny, unsigned char *bad) {
    __shared__ double s_red[kShardMergeThreads / 32];
    __shared__ int s_bad, s_last;
    SkState *st = a.st;
    if (*(volatile int *)&st->done || *(volatile int *)&st->pending) return;  // no CTA of this launch writes them before all have read
    const int tid = threadIdx.x;
    const int k = *(volatile int *)&st->k, K = st->max_sweeps, n = a.n;
    const int64_t ld1 = (int64_t)n + 1;
    const double tol = st->tol;
    const bool pre = (k == 0);
    if (tid == 0) s_bad = 0;
    double drow = 0.0;
    for (int r = 0; r < world; ++r) drow = fmax(drow, recv[r * ld1 + n]);
    // some rank's fixed-shift pass left the window (colsum kernel): repeat sweep k with the max shift
    const bool redo = isinf(drow) && !st->redo_next;
    int stop = 0, sweeps = 0, conv = 0, slot = 0;
    if (k >= 2 && !redo) {
        if (drow < tol && k > st->nostop_k) { stop = 1; sweeps = k - 1; conv = 1; slot = (k - 1) & 1; }
        else if (k == K + 1) { stop = 1; sweeps = K; conv = 0; slot = K & 1; }
    }
    __syncthreads();
    double dcol = 0.0;
    int nbad = 0;
    if (!stop && !redo) {
        const double *gold = gslot(a, k + 1);
        double *gnew = gslot(a, k);
        for (int j = blockIdx.x * kShardMergeThreads + tid; j < n; j += gridDim.x * kShardMergeThreads) {
            double S = 0.0;
            for (int r = 0; r < world; ++r) S += recv[r * ld1 + j];
            bool b = !(S > tiny) || !isfinite(S);
            if (pre && b) {  // an underflowed column of K is ~1 away from 1: no exact sum needed (merge_body)
                dcol = fmax(dcol, 1.0);
                bad[j] = 0;
                continue;
            }
            bad[j] = b;
            nbad += b;
            if (b) continue;
            if (pre) dcol = fmax(dcol, fabs(S - 1.0));
            else gnew[j] = gold[j] - log(S);
        }
    }
    if (nbad) atomicAdd(&s_bad, nbad);
    dcol = block_max_1024(dcol, s_red);  // includes the barrier that publishes s_bad
    if (tid == 0) {
        __stcg(a.devcol + 2 * blockIdx.x, dcol);
        __stcg(a.devcol + 2 * blockIdx.x + 1, (double)s_bad);
        __threadfence();
        s_last = (atomicAdd(&st->arrive, 1) == (int)gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last || tid != 0) return;
    __threadfence();
    st->arrive = 0;
    if (redo) {
        st->redo_next = 1;
        st->redone += 1;
        return;  // k unchanged: the next pass repeats it
    }
    st->redo_next = 0;
    if (stop) {
        st->dev = drow;
        shard_finish(st, k, stop, sweeps, conv, slot);
        return;
    }
    double dc = 0.0, nb = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) {
        dc = fmax(dc, __ldcg(a.devcol + 2 * b));
        nb += __ldcg(a.devcol + 2 * b + 1);
    }
    if (nb > 0.0) {  // the repair round finishes this sweep
        st->repaired += (int)nb;
        st->dcol = dc;
        st->last_dev = drow;
        st->pending = 1;
        return;
    }
    if (pre) {
        const double d0 = fmax(drow, dc);
        if (d0 < tol) { stop = 1; sweeps = 0; conv = 1; slot = 0; st->dev = d0; }
        st->last_dev = d0;
    }
    shard_finish(st, k, stop, sweeps, conv, slot);
}

// Exact column LSE pairs over this block's rows for the flagged columns (fp64):
// pair[2j] = max_i arg_ij, pair[2j+1] = sum_i exp(arg_ij - max), arg = E_ij (+ f_k,i).
template <class T>
__global__ void __launch_bounds__(kThreads) sk_shard_repair_pass_kernel(SkArgs a, const unsigned char *bad,
                                                                        double *pair) {
    if (!*(volatile int *)&a.st->pending) return;
    const int n = a.n, m = rows_of(a), k = a.st->k;
    const bool pre = (k == 0);
    const double coef = a.st->coef, gmax = a.st->gmax;
    const double *f = fslot(a, k);
    const T *G = static_cast<const T *>(a.G);
    for (int j = blockIdx.x * kThreads + threadIdx.x; j < n; j += gridDim.x * kThreads) {
        double M = -INFINITY, S = 0.0;
        if (bad[j]) {
            for (int i = 0; i < m; ++i) M = fmax(M, coef * (gmax - (double)G[(int64_t)i * a.ld + j]) + (pre ? 0.0 : f[i]));
            for (int i = 0; i < m; ++i)
                S += exp(coef * (gmax - (double)G[(int64_t)i * a.ld + j]) + (pre ? 0.0 : f[i]) - M);
        }
        pair[2 * j] = M;
        pair[2 * j + 1] = S;
    }
}

// Rank-order combine of the gathered pairs [world][2n]; finishes the pending sweep.
__global__ void __launch_bounds__(kShardMergeThreads) sk_shard_repair_merge_kernel(SkArgs a, const double *recv,
                                                                                   int world, const unsigned char *bad) {
    __shared__ double s_red[kShardMergeThreads / 32];
    SkState *st = a.st;
    if (!*(volatile int *)&st->pending) return;
    const int tid = threadIdx.x, k = st->k, n = a.n;
    const bool pre = (k == 0);
    double *gnew = gslot(a, k);
    double dcol = 0.0;
    for (int j = tid; j < n; j += kShardMergeThreads) {
        if (!bad[j]) continue;
        double M = -INFINITY;
        for (int r = 0; r < world; ++r) M = fmax(M, recv[(int64_t)r * 2 * n + 2 * j]);
        double S = 0.0;
        for (int r = 0; r < world; ++r) {
            const double mr = recv[(int64_t)r * 2 * n + 2 * j];
            if (mr != -INFINITY) S += recv[(int64_t)r * 2 * n + 2 * j + 1] * exp(mr - M);
        }
        const double lse = M + log(S);
        if (pre) dcol = fmax(dcol, fabs(exp(lse) - 1.0));
        else gnew[j] = -lse;
    }
    dcol = block_max_1024(dcol, s_red);
    if (tid != 0) return;
    int stop = 0, sweeps = 0, conv = 0, slot = 0;
    if (pre) {
        const double d0 = fmax(st->last_dev, fmax(st->dcol, dcol));
        if (d0 < st->tol) { stop = 1; sweeps = 0; conv = 1; slot = 0; st->dev = d0; }
        st->last_dev = d0;
    }
    shard_finish(st, k, stop, sweeps, conv, slot);
}

template <class T, int CH, int R>
__global__ void __launch_bounds__(kThreads, 2) sk_pass_kernel(SkArgs a) {
    __shared__ int s_k, s_done;
    if (threadIdx.x == 0) {
        s_k = *(volatile int *)&a.st->k;
        s_done = *(volatile int *)&a.st->done;
    }
    __syncthreads();
    if (s_done) return;
    const Slice sl{0, a.n, (int)blockIdx.x, (int)gridDim.x, 0};
    unsigned xi = 0;
    typename VecT<T>::V unused[R][CH];
    pass_body<T, CH, R, 1, kThreads>(a, s_k, a.st->max_sweeps, a.st->coef, a.st->gmax, sl, nullptr, xi, unused);
}

template <class T>
__global__ void __launch_bounds__(kThreads) sk_merge_kernel(SkArgs a) {
    __shared__ int s_k, s_done, s_last;
    const int tid = threadIdx.x;
    if (tid == 0) {
        s_k = *(volatile int *)&a.st->k;
        s_done = *(volatile int *)&a.st->done;
    }
    __syncthreads();
    if (s_done) return;
    const int k = s_k;
    const int K = a.st->max_sweeps;
    const double tol = a.st->tol;
    const bool pre = (k == 0);
    if (k != K + 1) merge_body<T, kThreads>(a, k, a.st->coef, a.st->gmax, blockIdx.x, gridDim.x);
    if (tid == 0) {
        if (!pre) __stcg(a.devcol + blockIdx.x, 0.0);
        __threadfence();
        const int t = atomicAdd(&a.st->arrive, 1);
        s_last = (t == (int)gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last || tid != 0) return;
    __threadfence();
    // Last CTA: stopping rule of sinkhorn.py:70-72 / :82-85 (and :96-99 in log mode).
    double drow = 0.0, dcol = 0.0;  // single thread here
    for (int b = 0; b < a.nblk; ++b) drow = fmax(drow, __ldcg(a.devpart + b));
    for (int b = 0; b < (int)gridDim.x; ++b) dcol = fmax(dcol, __ldcg(a.devcol + b));
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
        if (drow < tol && k > st->nostop_k) {
            st->done = 1; st->sweeps = k - 1; st->converged = 1; st->slot = (k - 1) & 1; st->dev = drow;
            return;
        }
        if (k == K + 1) {
            st->done = 1; st->sweeps = K; st->converged = 0; st->slot = K & 1; st->dev = drow;
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
    const double *f = fslot(a, slot), *g = gslot(a, slot);
    const T *G = static_cast<const T *>(a.G);
    const int n = a.n;
    double nrm = 0.0, lq = 0.0;
    const double coef = a.st->coef, gmax = a.st->gmax;
    const float ks = (float)SkMath<float>::kScale;
    const float coef2 = (float)(coef * SkMath<float>::kScale);
    for (int i = blockIdx.x; i < rows_of(a); i += gridDim.x) {
        const double fi = __ldcg(f + i);
        const T *Gi = G + (int64_t)i * a.ld;
        for (int j = threadIdx.x; j < n; j += kThreads) {
            T q;
            if (sizeof(T) == 8) {
                // exp(E + f + g), E in the reference's evaluation order
                const double e = coef * (gmax - (double)Gi[j]);
                q = (T)exp((e + fi) + __ldcg(g + j));
            } else {
                const float e = coef2 * ((float)gmax - (float)Gi[j]);
                q = (T)ex2f(e + (float)((fi + __ldcg(g + j)) * ks));
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

constexpr int kMaxCh = 8;
constexpr int rows_for(int ch) { return ch == 1 ? 8 : ch == 2 ? 4 : ch <= 4 ? 2 : 1; }
// Wide rows (n > 8192 fp32 / 4096 fp64) run 512-thread CTAs, one per SM:
// half the chunks per thread, 16 warps to hide the reduction chains.
constexpr int kWideThreads = 512;
constexpr int rows_for(int ch, int nt) { return nt == kThreads ? rows_for(ch) : 1; }

template <class T, int CH, int CL, int NT, bool TMA = false> void *persistent_fn() {
    return (void *)sk_persistent_kernel<T, CH, rows_for(CH, NT), CL, NT, TMA>;
}

template <class T> void *persistent_for(int ch, int cl, int nt, bool tma = false) {
    if (nt == kThreads && cl == 1) {
        switch (ch) {
            case 1: return persistent_fn<T, 1, 1, kThreads>();
            case 2: return persistent_fn<T, 2, 1, kThreads>();
            case 3: return persistent_fn<T, 3, 1, kThreads>();
            case 4: return persistent_fn<T, 4, 1, kThreads>();
            case 5: return persistent_fn<T, 5, 1, kThreads>();
            case 6: return persistent_fn<T, 6, 1, kThreads>();
            case 7: return persistent_fn<T, 7, 1, kThreads>();
            case 8: return persistent_fn<T, 8, 1, kThreads>();
        }
    }
#define GOAT_CL(C)                                                                                       \
    if (nt == kWideThreads && cl == C) {                                                                 \
        switch (ch) {                                                                                    \
            case 3: return tma ? persistent_fn<T, 3, C, kWideThreads, true>() : persistent_fn<T, 3, C, kWideThreads>(); \
            case 4: return tma ? persistent_fn<T, 4, C, kWideThreads, true>() : persistent_fn<T, 4, C, kWideThreads>(); \
            case 5: return tma ? persistent_fn<T, 5, C, kWideThreads, true>() : persistent_fn<T, 5, C, kWideThreads>(); \
            case 6: return tma ? persistent_fn<T, 6, C, kWideThreads, true>() : persistent_fn<T, 6, C, kWideThreads>(); \
            case 7: return tma ? persistent_fn<T, 7, C, kWideThreads, true>() : persistent_fn<T, 7, C, kWideThreads>(); \
            case 8: return tma ? persistent_fn<T, 8, C, kWideThreads, true>() : persistent_fn<T, 8, C, kWideThreads>(); \
        }                                                                                                \
    }
    GOAT_CL(1)
    GOAT_CL(2)
    GOAT_CL(4)
    GOAT_CL(8)
#undef GOAT_CL
    throw Error(GOAT_ENOTSUP, "sinkhorn: no kernel for chunks=" + std::to_string(ch) + " cluster=" +
                                  std::to_string(cl) + " threads=" + std::to_string(nt));
}

int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

cudaLaunchConfig_t persistent_config(const SkPlan &p, cudaStream_t s, cudaLaunchAttribute (&attrs)[2]) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.nblk);
    cfg.blockDim = dim3(p.nt);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = s;
    attrs[0].id = cudaLaunchAttributeCooperative;
    // GOAT_SK_NOCOOP=1 drops the cooperative flag (profilers cannot replay it);
    // the grid is still sized to the co-resident maximum.
    // Under ncu (it sets NV_NSIGHT_INJECTION_TRANSPORT_TYPE) a cooperative cluster launch is
    // refused at replay; the grid is co-resident-sized either way.
    static const bool profiled = getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") != nullptr;
    attrs[0].val.cooperative = (env_int("GOAT_SK_NOCOOP", 0) || profiled) ? 0 : 1;
    attrs[1].id = cudaLaunchAttributeClusterDimension;
    const int cdim = p.cl;
    attrs[1].val.clusterDim.x = cdim;
    attrs[1].val.clusterDim.y = 1;
    attrs[1].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = cdim > 1 ? 2 : 1;
    return cfg;
}



// ------------------------------------------------------------------ small-n tile kernel
// n <= ~2500 (fp32): the LOT is latency bound (a sweep of the lock-step kernel
// is ~3.5 us of pass plus two grid barriers and a distributed merge, at n = 64
// as at n = 1000).  Here a thread-block cluster of CL CTAs owns a group of rows,
// CTA rank q the column slice q, and the G tile stays in shared memory for the
// whole LOT.  One warp covers a row's slice, so a row's (max, sum) pair needs
// only a warp butterfly; the CL pairs of a row meet through DSMEM (st.async +
// mbarrier) and every CTA combines them in rank order.  After the single grid
// barrier of a sweep every CTA merges the column partials of ITS OWN slice
// (fixed order over the row groups): the same-rank CTAs of every cluster compute
// the same g slice redundantly, so there is no second barrier and no reload of g.
constexpr int kTileThreads = 512;
constexpr int kTileWarps = kTileThreads / 32;

template <class T, int CL, int CPL, int RPW>
__global__ void __launch_bounds__(kTileThreads, 1) sk_tile_kernel(SkArgs a, unsigned *bar, int rows_g) {
    constexpr int SW = 32 * CPL;  // slice width held per CTA (columns, padded)
    constexpr int NW = kTileWarps;
    extern __shared__ __align__(16) unsigned char tsm[];
    T *tile = reinterpret_cast<T *>(tsm);                                 // [rows_g][SW]
    T *wpart = tile + (size_t)rows_g * SW;                                // [NW][SW]
    double *gsl = reinterpret_cast<double *>(wpart + (size_t)NW * SW);   // [SW] g (natural units)
    T *gst = reinterpret_cast<T *>(gsl + SW);                              // [SW] g scaled (-inf: masked)
    double *fpr = reinterpret_cast<double *>(gst + SW + (SW & 1));        // [rows_g] f_{k-1} of the group's rows
    T *xp = reinterpret_cast<T *>(fpr + rows_g);                          // [2][CL][rows_g][2]
    __shared__ uint64_t xbar[2];
    __shared__ double s_red[NW];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t rank = 0, cid = blockIdx.x, ncl = gridDim.x;
    if constexpr (CL > 1) {
        asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        asm("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
        asm("mov.u32 %0, %%nclusterid.x;" : "=r"(ncl));
    }
    const int n = a.n, grp = (int)cid, ngrp = (int)ncl;
    const int c0 = min(n, (int)rank * a.slice_w), c1 = min(n, c0 + a.slice_w);
    const int r0 = grp * rows_g, nr = max(0, min(rows_g, n - r0));  // rows [r0, r0 + nr)
    const int K = a.st->max_sweeps;
    const double tol = a.st->tol, coef_d = a.st->coef, gmax_d = a.st->gmax;
    const double ks = SkMath<T>::kScale;
    const T coef = (T)(coef_d * ks), gmax = (T)gmax_d;
    const int k0 = a.st->k, nostop_k = a.st->nostop_k;
    const T *G = static_cast<const T *>(a.G);
    // tile, g slice (from slot k0+1), barriers
    for (int idx = tid; idx < rows_g * SW; idx += kTileThreads) {
        const int r = idx / SW, c = idx % SW;
        tile[idx] = (r < nr && c0 + c < c1) ? G[(int64_t)(r0 + r) * a.ld + c0 + c] : T(0);
    }
    for (int c = tid; c < SW; c += kTileThreads) {
        const bool ok = c0 + c < c1;
        // g_{k0-1}: zero before sweep 1 (the pre-check uses no g; slot 1 may hold a
        // previous LOT's potentials)
        const double gv = (ok && k0 >= 1) ? __ldcg(gslot(a, k0 + 1) + c0 + c) : 0.0;
        gsl[c] = gv;
        gst[c] = ok ? (T)(gv * ks) : neg_inf<T>();
    }
    // a LOT resumed at pass k0 >= 2 (the fp64 finish of an fp32 handle): f_{k0-1}
    for (int r = tid; r < rows_g; r += kTileThreads)
        fpr[r] = (k0 >= 2 && r < nr) ? __ldcg(fslot(a, k0 + 1) + r0 + r) : 0.0;
    if (tid == 0) {
        xbar_init(&xbar[0]);
        xbar_init(&xbar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if constexpr (CL > 1) cluster_sync();
    else __syncthreads();

    const bool writer = rank == 0 && lane == 0;
    unsigned epoch = 0;
    int par = 0;
    for (int k = k0;; ++k, par ^= 1) {
        const bool pre = (k == 0), rowonly = (k == K + 1);
        double *fout = fslot(a, k);
        sk_stamp(a, k, 0);
        if (tid == 0) xbar_arm(&xbar[par], (uint32_t)(CL * nr * 2 * sizeof(T)));
        // ---- rows: warp w owns rows w, w + NW, ...
        T y[RPW][CPL], mw[RPW];
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            const int r = warp + NW * i;
            mw[i] = neg_inf<T>();
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const T arg = (r < nr) ? coef * (gmax - tile[r * SW + lane + 32 * q]) + gst[lane + 32 * q]
                                       : neg_inf<T>();  // E_ij + g_j (sinkhorn.py:125)
                y[i][q] = arg;
                mw[i] = vmax(mw[i], arg);
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
            for (int i = 0; i < RPW; ++i) mw[i] = vmax(mw[i], __shfl_xor_sync(0xffffffffu, mw[i], off));
        T sw[RPW];
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            const T mx = (mw[i] == neg_inf<T>()) ? T(0) : mw[i];
            T sp = T(0);
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                y[i][q] = SkMath<T>::ex(y[i][q] - mx);
                sp += y[i][q];
            }
            sw[i] = sp;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
            for (int i = 0; i < RPW; ++i) sw[i] += __shfl_xor_sync(0xffffffffu, sw[i], off);
        // this CTA's pair of each row -> every rank (incl. itself)
        if (lane < CL) {
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const int r = warp + NW * i;
                if (r < nr) {
                    T *slot = xp + (((size_t)par * CL + rank) * rows_g + r) * 2;
                    if constexpr (CL > 1)
                        st_async_pair(dsmem_map(slot, (uint32_t)lane), mw[i], sw[i], dsmem_map(&xbar[par], (uint32_t)lane));
                    else
                        st_async_pair((uint32_t)__cvta_generic_to_shared(slot), mw[i], sw[i],
                                      (uint32_t)__cvta_generic_to_shared(&xbar[par]));
                }
            }
        }
        sk_stamp_v(a, k, 1, (double)sw[0]);
        xbar_wait(&xbar[par], (uint32_t)((k - k0) >> 1) & 1u);
        sk_stamp(a, k, 2);
        double devmax = 0.0;
        T sc[RPW];
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            const int r = warp + NW * i;
            sc[i] = T(0);
            if (r >= nr) continue;
            T M = neg_inf<T>();
#pragma unroll
            for (int q = 0; q < CL; ++q) M = vmax(M, xp[(((size_t)par * CL + q) * rows_g + r) * 2]);
            T S = T(0);
#pragma unroll
            for (int q = 0; q < CL; ++q) {
                const T mq = xp[(((size_t)par * CL + q) * rows_g + r) * 2];
                if (mq != neg_inf<T>()) S += xp[(((size_t)par * CL + q) * rows_g + r) * 2 + 1] * SkMath<T>::ex(mq - M);
            }
            const double lse = (double)M + SkMath<T>::lgt(S);  // scaled units
            const double fnew = -lse * (1.0 / ks);
            if (writer) {
                double dev = 0.0;
                if (pre) dev = SkMath<T>::dev(-fnew);                  // |rowsum(K) - 1|
                else if (k >= 2) dev = SkMath<T>::dev(fpr[r] - fnew);  // |u K v - 1|
                if (!pre) { __stcg(fout + r0 + r, fnew); fpr[r] = fnew; }
                devmax = fmax(devmax, dev);
            }
            if (!rowonly && mw[i] != neg_inf<T>())
                sc[i] = SkMath<T>::ex((T)((double)mw[i] + (pre ? 0.0 : -lse)));
        }
        if (!rowonly) {
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                T cp = T(0);
#pragma unroll
                for (int i = 0; i < RPW; ++i) cp += y[i][q] * sc[i];
                wpart[warp * SW + lane + 32 * q] = cp;
            }
        }
        if (lane == 0) s_red[warp] = devmax;
        sk_stamp(a, k, 3);
        __syncthreads();
        sk_stamp(a, k, 4);
        if (!rowonly) {
            // double-buffered by sweep parity: a CTA of another cluster may still be
            // merging this group's sweep-(k-1) partials (there is one grid barrier per
            // sweep); the k-2 buffer is free since every CTA passed barrier k-1 after
            // its merge of sweep k-2.
            T *cp = static_cast<T *>(a.colpart) + ((int64_t)(k & 1) * ngrp + grp) * a.ldp;
            for (int c = tid; c < SW; c += kTileThreads) {
                if (c0 + c >= c1) continue;
                T v = T(0);
#pragma unroll
                for (int w = 0; w < NW; ++w) v += wpart[w * SW + c];
                __stcg(cp + c0 + c, v);
            }
        }
        if (tid == 0) {
            double d = 0.0;
            for (int w = 0; w < NW; ++w) d = fmax(d, s_red[w]);
            // three rotating slots [3 + k % 3]: with one barrier per sweep a slot is
            // cleared a full sweep before its next use (see below)
            if (d > 0.0) atomicMax(a.dslot + 3 + (k % 3), (unsigned long long)__double_as_longlong(d));
        }
        sk_stamp(a, k, 5);
        grid_barrier(bar, gridDim.x, epoch);
        sk_stamp(a, k, 6);
        const double drow = __longlong_as_double((long long)__ldcg(a.dslot + 3 + (k % 3)));
        int stop = 0, sweeps = 0, conv = 0, slot = 0;
        if (k >= 2) {
            if (drow < tol && k > nostop_k) { stop = 1; sweeps = k - 1; conv = 1; slot = (k - 1) & 1; }
            else if (k == K + 1) { stop = 1; sweeps = K; conv = 0; slot = K & 1; }
        }
        if (stop) {
            if (blockIdx.x == 0 && tid == 0) {
                a.st->dev = drow;
                a.st->done = 1; a.st->sweeps = sweeps; a.st->converged = conv; a.st->slot = slot;
                a.st->k = k + 1;
            }
            break;
        }
        // ---- merge of this CTA's columns (fixed order over the row groups, fp64).
        // (Measured: this plain loop beats batching all partial loads or splitting a
        // column's groups over two threads -- profiles/round1_sk_tile.md.)
        const T *cpa = static_cast<const T *>(a.colpart) + (int64_t)(k & 1) * ngrp * a.ldp;
        const double tiny = sizeof(T) == 4 ? 1e-30 : 1e-290;
        double dloc = 0.0;
        for (int c = tid; c < SW; c += kTileThreads) {
            const int j = c0 + c;
            if (j >= c1) continue;
            double Ssum = 0.0;
            for (int g = 0; g < ngrp; ++g) Ssum += (double)__ldcg(cpa + (int64_t)g * a.ldp + j);
            if (pre) {
                if (!(Ssum > tiny)) Ssum = 0.0;  // underflowed column of K: deviation ~1 (see merge_body)
                dloc = fmax(dloc, fabs(Ssum - 1.0));
            } else {
                double gnew = gsl[c] - log(Ssum);
                if (!(Ssum > tiny) || !isfinite(Ssum)) gnew = sk_exact_col<T>(G, a.ld, n, j, fout, false, coef_d, gmax_d);
                gsl[c] = gnew;
                gst[c] = (T)(gnew * ks);
                if (grp == 0) __stcg(gslot(a, k) + j, gnew);
            }
        }
        if (blockIdx.x == 0 && tid == 0) a.dslot[3 + ((k + 2) % 3)] = 0ull;
        if (pre) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) dloc = fmax(dloc, __shfl_xor_sync(0xffffffffu, dloc, off));
            if (lane == 0) s_red[warp] = dloc;
            __syncthreads();
            if (tid == 0) {
                double d = 0.0;
                for (int w = 0; w < NW; ++w) d = fmax(d, s_red[w]);
                atomicMax(a.dslot + 2, (unsigned long long)__double_as_longlong(d));
            }
            grid_barrier(bar, gridDim.x, epoch);  // pre-check only: the column deviation is global
            const double d0 = fmax(drow, __longlong_as_double((long long)__ldcg(a.dslot + 2)));
            if (blockIdx.x == 0 && tid == 0) a.st->last_dev = d0;
            if (d0 < tol) {
                if (blockIdx.x == 0 && tid == 0) {
                    a.st->dev = d0;
                    a.st->done = 1; a.st->sweeps = 0; a.st->converged = 1; a.st->slot = 0;
                    a.st->k = k + 1;
                }
                break;
            }
        }
        sk_stamp(a, k, 7);
        __syncthreads();  // the new g slice before the next pass
        sk_stamp(a, k, 8);
    }
    if constexpr (CL > 1) cluster_sync();  // no CTA leaves while peers may still write into it
}

}  // namespace

template <int CH, int CL, int R> void *pipe_fn() { return (void *)sk_pipe_kernel<CH, CL, kWideThreads, R>; }
template <int CH, int CL> void *pipe_fn256() { return (void *)sk_pipe_kernel<CH, CL, 256, 1>; }

void *pipe_for(int ch, int cl, int nt, int rows) {
    // two 256-thread CTAs per SM (GOAT_SK_PIPE_NT=256)
    if (nt == 256 && rows == 1) {
        if (cl == 4 && ch == 5) return pipe_fn256<5, 4>();
        if (cl == 8 && ch == 5) return pipe_fn256<5, 8>();
        if (cl == 8 && ch == 4) return pipe_fn256<4, 8>();
        if (cl == 8 && ch == 3) return pipe_fn256<3, 8>();
    }
#define GOAT_PCL(C)                                                 \
    if (nt == kWideThreads && cl == C && rows == 1) {               \
        switch (ch) {                                               \
            case 3: return pipe_fn<3, C, 1>();                      \
            case 4: return pipe_fn<4, C, 1>();                      \
            case 5: return pipe_fn<5, C, 1>();                      \
            case 6: return pipe_fn<6, C, 1>();                      \
            case 7: return pipe_fn<7, C, 1>();                      \
        }                                                           \
    }                                                               \
    if (nt == kWideThreads && cl == C && rows == 2) {               \
        switch (ch) {                                               \
            case 3: return pipe_fn<3, C, 2>();                      \
            case 4: return pipe_fn<4, C, 2>();                      \
            case 5: return pipe_fn<5, C, 2>();                      \
        }                                                           \
    }
    // 3 rows per band for whole rows of <= 6144 columns (GOAT_SK_PIPE_R1=3)
    if (nt == kWideThreads && cl == 1 && ch == 3 && rows == 3) return pipe_fn<3, 1, 3>();
    GOAT_PCL(1)
    GOAT_PCL(2)
    GOAT_PCL(4)
    GOAT_PCL(8)
#undef GOAT_PCL
    throw Error(GOAT_ENOTSUP, "sinkhorn: no pipelined kernel for chunks=" + std::to_string(ch) + " cluster=" +
                                  std::to_string(cl) + " rows=" + std::to_string(rows));
}

// Wide fp32 rows: the decoupled bulk-copy pipeline (sk_pipe_kernel), one
// 512-thread CTA per SM, clusters of 2/4/8 once a row exceeds 6 chunks/thread.
bool pipe_plan(int n, int mrows, SkPlan &p) {
    constexpr int VW = 4;
    p.nt = kWideThreads;
    if (env_int("GOAT_SK_PIPE_NT", 512) == 256) {
        // experimental: 2 CTAs per SM, 8-CTA clusters, ~108 KB of ring per CTA
        const int cl = env_int("GOAT_SK_PIPE_CL", 8);
        p.nt = 256; p.cl = cl; p.rows = 1; p.pipe = true;
        p.slice_w = (int)round_up(ceil_div(n, cl), 8 * VW);
        p.ch = std::max(3, ceil_div(ceil_div(p.slice_w, VW), p.nt));
        if (!((cl == 4 && p.ch == 5) || (cl == 8 && p.ch >= 3 && p.ch <= 5))) return false;
        p.stage_bytes = (int)round_up((size_t)p.slice_w * sizeof(float), 128);
        const size_t glb = (size_t)p.nt * p.ch * 16;
        p.stages = std::min(8, (int)((104 * 1024 - glb) / p.stage_bytes));
        if (p.stages < 4) return false;
        p.smem = (size_t)p.stages * p.stage_bytes + glb;
        (void)mrows;
        return true;
    }
    p.cl = 1;
    p.slice_w = (int)round_up(n, 8 * VW);
    p.ch = std::max(3, ceil_div(ceil_div(n, VW), p.nt));
    if (p.ch > env_int("GOAT_SK_PIPE_CH1", 6)) {
        // Clustered rows: the pipelined kernel keeps a band's exponentials in its
        // stage until the lagged cluster finish.  It measured faster than the
        // lock-step cluster kernel where both split rows the same way with <= 6
        // chunks per thread (n = 20000: 0.487 vs 0.521 ms, n = 40000: 2.155 vs
        // 2.339 ms); where the lock-step kernel can hold 7-8 chunks per thread
        // instead (n = 16384 unsplit, n = 65536 in 4 slices) it keeps the bigger
        // bands and wins (profiles/round1_sk_pipe.md).  GOAT_SK_PIPE=2 forces it.
        int lcl = 1, lch = ceil_div(ceil_div(n, VW), kWideThreads);
        while (lch > kMaxCh && lcl < 8) {
            lcl *= 2;
            lch = ceil_div(ceil_div((int)round_up(ceil_div(n, lcl), 8 * VW), VW), kWideThreads);
        }
        if (env_int("GOAT_SK_PIPE", 1) != 2 && (lcl == 1 || lch > 6)) return false;
        // the same split as the lock-step kernel, unless GOAT_SK_PIPE_CL forces one
        // (3- and 6-CTA clusters measured slower: fewer co-resident SMs).  The
        // lagged finish holds two stages, so at least four must fit beside g.
        const int maxch = std::min(7, env_int("GOAT_SK_PIPE_CH", 7));
        const int force = env_int("GOAT_SK_PIPE_CL", 0);
        bool found = false;
        const int R = std::max(1, std::min(2, env_int("GOAT_SK_PIPE_R", 1)));
        for (int cl : {2, 4, 8}) {
            if (force ? cl != force : (cl != lcl && env_int("GOAT_SK_PIPE", 1) != 2 && R == 1)) continue;
            const int sw = (int)round_up(ceil_div(n, cl), 8 * VW);
            const int ch = std::max(3, ceil_div(ceil_div(sw, VW), p.nt));
            const size_t stage = R * round_up((size_t)sw * sizeof(float), 128), glb = (size_t)p.nt * ch * 16;
            if (ch > (R == 1 ? maxch : 5) || (220 * 1024 - glb) / stage < 4) continue;
            p.cl = cl; p.slice_w = sw; p.ch = ch; p.rows = R;
            found = true;
            break;
        }
        if (!found) return false;
    }
    if (p.cl == 1)  // rows per band, whole-row CTAs: 2 for short rows (4096 < n <= 6144)
        p.rows = std::max(1, std::min(ceil_div(ceil_div(n, VW), p.nt) <= 3 ? 3 : 2, env_int("GOAT_SK_PIPE_R1", (n > 4096 && n <= 6144) ? 2 : 1)));
    p.pipe = true;
    // ring stages (R row slices each) + one more slice for g (scaled)
    p.stage_bytes = p.rows * (int)round_up((size_t)p.slice_w * sizeof(float), 128);
    const size_t gl_bytes = (size_t)p.nt * p.ch * 16;  // every thread's chunks, masked ones included
    p.stages = std::min(8, (int)((220 * 1024 - gl_bytes) / p.stage_bytes));
    if (const int st = env_int("GOAT_SK_STAGES", 0)) p.stages = std::min(p.stages, std::max(3, st));
    if (p.stages < 3) return false;
    p.smem = (size_t)p.stages * p.stage_bytes + gl_bytes;
    (void)mrows;
    return true;
}

template <class T, int CL, int CPL, int RPW> void *tile_fn() { return (void *)sk_tile_kernel<T, CL, CPL, RPW>; }

template <class T> void *tile_for(int cl, int cpl, int rpw) {
#define GOAT_TL(C, P)                                          \
    if (cl == C && cpl == P) {                                 \
        switch (rpw) {                                         \
            case 1: return tile_fn<T, C, P, 1>();              \
            case 2: return tile_fn<T, C, P, 2>();              \
            case 3: return tile_fn<T, C, P, 3>();              \
            case 4: return tile_fn<T, C, P, 4>();              \
        }                                                      \
    }
    GOAT_TL(2, 1) GOAT_TL(2, 2) GOAT_TL(2, 4) GOAT_TL(2, 8)
    GOAT_TL(4, 1) GOAT_TL(4, 2) GOAT_TL(4, 4) GOAT_TL(4, 8) GOAT_TL(4, 16)
    GOAT_TL(8, 2) GOAT_TL(8, 4) GOAT_TL(8, 8)
#undef GOAT_TL
    return nullptr;
}

template <class T> size_t tile_smem(int rows_g, int sw, int cl) {
    return (size_t)rows_g * sw * sizeof(T) + (size_t)kTileWarps * sw * sizeof(T) + (size_t)sw * 8 +
           (size_t)sw * sizeof(T) + (size_t)rows_g * 8 + (size_t)2 * cl * rows_g * 2 * sizeof(T);
}

template <class T> bool tile_plan_width(int n, int num_sms, SkPlan &p, int cl, int cpl) {
    const int sw = 32 * cpl;
    int ncl = 0;
    {
        // co-resident clusters with the largest shared-memory footprint this n can need
        int rows_guess = (int)round_up(ceil_div(n, std::max(1, num_sms / cl)), 2);
        void *fn = tile_for<T>(cl, cpl, std::min(4, ceil_div(rows_guess, kTileWarps)));
        if (!fn) return false;
        const size_t smem = tile_smem<T>(rows_guess, sw, cl);
        if (smem > 200 * 1024) return false;
        GOAT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cl * num_sms);
        cfg.blockDim = dim3(kTileThreads);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at;
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = cl; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
        cfg.attrs = &at;
        cfg.numAttrs = 1;
        GOAT_CUDA(cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg));
    }
    if (ncl < 1) return false;
    int ngrp = std::max(1, std::min(ncl, n / 2));
    // Row groups: below n = 256 the merge of a column's partials dominates the
    // sweep and fewer, taller groups win (measured n = 96: 8 groups 4.1 vs 5.1 us
    // fp64, 3.3 vs 4.3 us fp32; n = 200: 8 groups fp32 4.0 vs 4.8, 16 groups fp64
    // 5.5 vs 5.9); from n = 296 every co-resident cluster is best
    // (profiles/round1_sk_tile_grp.json).  GOAT_SK_TILE_GRP overrides the cap.
    const int grp_cap = env_int("GOAT_SK_TILE_GRP", n < 256 ? ((sizeof(T) == 8 && n > 128) ? 16 : 8) : 0);
    if (grp_cap > 0) ngrp = std::max(1, std::min(ngrp, grp_cap));
    const int rows_g = (int)round_up(ceil_div(n, ngrp), 2);
    const int rpw = ceil_div(rows_g, kTileWarps);
    if (rpw > 4) return false;
    void *fn = tile_for<T>(cl, cpl, rpw);
    if (!fn) return false;
    p.smem = tile_smem<T>(rows_g, sw, cl);
    if (p.smem > 200 * 1024) return false;
    GOAT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
    p.tile = true;
    p.persistent = true;
    p.cl = cl;
    p.nt = kTileThreads;
    p.ch = cpl;
    p.rows = rpw;
    p.tile_rows = rows_g;
    p.slice_w = (int)round_up(ceil_div(n, cl), 8);
    p.ngrp = (n + rows_g - 1) / rows_g;
    p.nblk = p.ngrp * cl;
    p.merge_blocks = 1;
    // two parity buffers of ngrp rows (sk_tile_kernel double-buffers the partials)
    p.colpart_bytes = (size_t)std::max(2 * p.ngrp, num_sms * 2) * round_up(n, 8) * sizeof(T);
    return true;
}

// Small n (whole-LOT-resident tiles, see sk_tile_kernel): clusters of 4 CTAs
// split the columns; row groups = co-resident clusters.
template <class T> bool tile_plan(int n, int num_sms, SkPlan &p) {
    if (env_int("GOAT_SK_TILE", 1) == 0) return false;
    // measured: 2 CTAs at n = 64 (3.7 vs 5.7 us), 4 from n = 500 (4.1 vs 6.2 us)
    const int cl = env_int("GOAT_SK_TILE_CL", n < 256 ? 2 : 4);
    if (cl != 2 && cl != 4 && cl != 8) return false;
    const int sw = (int)round_up(ceil_div(n, cl), 32);
    const int cpl = sw / 32;
    if ((cpl != 1 && cpl != 2 && cpl != 4 && cpl != 8 && !(cl == 4 && cpl == 16)) || (cl == 8 && cpl < 2)) {
        // round the slice up to the next instantiated width
        int c = 1;
        while (c < cpl) c *= 2;
        if (c > (cl == 4 ? 16 : 8) || (cl == 8 && c < 2)) return false;
        return tile_plan_width<T>(n, num_sms, p, cl, c);
    }
    return tile_plan_width<T>(n, num_sms, p, cl, cpl);
}

// Wide fp32 rows, 12288 < n <= 40960 (sk_wide_kernel): a cluster splits each
// row into CL slices of <= 10 chunks per thread held in registers; g of the
// slice and an S-stage ring of sub-row stages in shared memory.  Shapes: one
// 512-thread CTA per SM in 2-CTA clusters, or two 256-thread CTAs per SM in
// 4-CTA clusters (GOAT_SK_WIDE_CL=2|4).
bool wide2_plan(int n, int mrows, int num_sms, SkPlan &p) {
    const int mode = env_int("GOAT_SK_WIDE", 1);
    if (mode == 0) return false;
    // measured faster than the previous kernels from n ~ 22000 (n = 25000: 0.715 vs
    // 0.799 ms, 32768: 0.937 vs 1.20, 40000: 1.29 vs 2.12; n = 20000: 0.535 vs 0.479);
    // GOAT_SK_WIDE=2 forces it for any n up to 40960
    if (mode != 2 && (n <= 22000 || n > 40960)) return false;
    if (n > 40960) return false;
    constexpr int VW = 4;
    // mode 1 (default): rows parked in TMEM for a lagged finish (TM, 2-CTA clusters);
    // 4: lock-step finish (GOAT_SK_WIDE_CL=4 for two 256-thread CTAs per SM in 4-CTA clusters)
    const bool tm = mode != 4;
    const int CL = (!tm && env_int("GOAT_SK_WIDE_CL", 2) == 4) ? 4 : 2;
    const int NT = CL == 2 ? 512 : 256;
    const int per_sm = CL == 2 ? 1 : 2;
    const int sw = (int)round_up(ceil_div(n, CL), 8 * VW);
    int ch = ceil_div(ceil_div(sw, VW), NT);
    ch = (int)round_up(std::max(ch, 4), 2);
    if (ch > 10) return false;
    // TM: two stages per row and a ring of two rows (measured at n = 40000: 40 KB
    // stages, S = 4 -> 1.40 ms/sweep; 16 KB stages 1.65-1.87; S = 5 -> 1.95);
    // GOAT_SK_WIDE_CC=2 selects 16 KB stages
    const int CC = (tm && env_int("GOAT_SK_WIDE_CC", 0) != 2) ? ch / 2 : 2;
    p = SkPlan{};
    p.nt = NT; p.cl = CL; p.ch = ch; p.rows = 1; p.slice_w = sw; p.wide2 = true; p.wide_tm = tm; p.persistent = true;
    p.stage_bytes = NT * CC * 16;
    void *const kfn = wide2_for(NT, CL, ch, tm, CC);
    p.rows = CC;  // chunks per stage (the launcher selects the kernel by it)
    // the ring takes what g and the shift table leave of this CTA's share of shared memory
    const size_t gl = tm ? 0 : (size_t)NT * ch * 16;  // TM keeps g in tensor memory
    const size_t budget = (228 * 1024) / per_sm - 3 * 1024;
    const int rows_max = ceil_div(mrows, std::max(1, per_sm * num_sms / CL));
    const size_t shift = round_up((size_t)(rows_max + 64) * 4, 128);
    if (gl + shift >= budget) return false;
    int S = (int)((budget - gl - shift) / p.stage_bytes);
    S = std::min(16, S);
    if (tm && CC * 2 == ch) S = std::min(S, 4);
    if (const int st = env_int("GOAT_SK_STAGES", 0)) S = std::min(S, std::max(3, st));
    if (S < 2 * (ch / CC) && S < 6) return false;
    p.stages = S;
    p.smem = (size_t)S * p.stage_bytes + gl + shift;
    GOAT_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
    cudaLaunchAttribute attrs[2];
    SkPlan q = p;
    q.nblk = CL * num_sms;
    cudaLaunchConfig_t cfg = persistent_config(q, nullptr, attrs);
    cudaLaunchAttribute cattr = attrs[1];
    cfg.attrs = &cattr;
    cfg.numAttrs = 1;
    int ncl = 0;
    GOAT_CUDA(cudaOccupancyMaxActiveClusters(&ncl, kfn, &cfg));
    if (ncl < 1) return false;
    int ngrp = std::max(1, std::min(mrows, ncl));
    if (const int force = env_int("GOAT_SK_BLOCKS", 0)) ngrp = std::max(1, std::min({force / CL, mrows, ncl}));
    if (ceil_div(mrows, ngrp) + 64 > (int)(shift / 4)) return false;
    p.ngrp = ngrp;
    p.nblk = CL * ngrp;
    p.merge_blocks = std::max(1, std::min((n + 7) / 8, 4 * num_sms));
    p.colpart_bytes = (size_t)std::max(p.nblk, num_sms * 2) * round_up(n, 8) * sizeof(float);
    return true;
}

template <class T> SkPlan sk_plan(int n, int num_sms, int mrows, bool sharded) {
    if (mrows < 0) mrows = n;
    constexpr int VW = VecT<T>::W;
    SkPlan p;
    if (!sharded && mrows == n) {
        SkPlan tp;  // committed only if complete
        if (tile_plan<T>(n, num_sms, tp)) return tp;
    }
    // fp32 rows of more than 6144 columns take the bulk-copy pipeline (measured at
    // n = 8192: 0.084 vs 0.104 ms; at n = 5000 the register kernel wins, 0.043 vs
    // 0.050); GOAT_SK_PIPE=3 forces it for any n, 0 disables it
    if (sizeof(T) == 4) {
        SkPlan wp;  // committed only if complete
        if (wide2_plan(n, mrows, num_sms, wp)) return wp;
    }
    SkPlan pp;  // a pipe plan is committed only if it is complete
    // (and 4096 < n <= 6144 with 2-row bands: n = 5000 0.0395 vs 0.0425 ms)
    if (sizeof(T) == 4 && (ceil_div(ceil_div(n, VW), kThreads) > 6 || (n > 4096 && n <= 6144) ||
                           env_int("GOAT_SK_PIPE", 1) == 3) &&
        env_int("GOAT_SK_PIPE", 1) && pipe_plan(n, mrows, pp) && (p = pp, true)) {
        void *const kfn = pipe_for(p.ch, p.cl, p.nt, p.rows);
        GOAT_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
        if (p.cl > 1) GOAT_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        p.persistent = true;
        int groups = 0;
        if (p.cl == 1) {
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)kfn, p.nt, p.smem);
            groups = std::max(1, occ) * num_sms;
        } else {
            cudaLaunchAttribute attrs[2];
            SkPlan q = p;
            q.nblk = p.cl * num_sms;
            cudaLaunchConfig_t cfg = persistent_config(q, nullptr, attrs);
            cudaLaunchAttribute cattr = attrs[1];
            cfg.attrs = &cattr;
            cfg.numAttrs = 1;
            int ncl = 0;
            GOAT_CUDA(cudaOccupancyMaxActiveClusters(&ncl, kfn, &cfg));
            groups = std::max(1, ncl);
        }
        int ngrp = std::max(1, std::min(mrows, groups));
        if (const int force = env_int("GOAT_SK_BLOCKS", 0)) ngrp = std::max(1, std::min({force / p.cl, mrows, groups}));
        p.ngrp = ngrp;
        p.nblk = ngrp * p.cl;
        p.merge_blocks = std::max(1, std::min((n + 7) / 8, 4 * num_sms));
        p.colpart_bytes = (size_t)std::max(p.nblk, num_sms * 2) * round_up(n, 8) * sizeof(T);
        return p;
    }
    // Row width per CTA: whole rows when they fit kMaxCh chunks per thread,
    // else a cluster of cl CTAs splits each row into column slices.
    p.cl = 1;
    p.nt = kThreads;
    p.slice_w = (int)round_up(n, 8 * VW);
    p.ch = ceil_div(ceil_div(n, VW), kThreads);
    const int maxch = std::max(3, std::min(kMaxCh, env_int("GOAT_SK_MAXCH", kMaxCh)));
    bool wide = false;
    if (p.ch > kMaxCh) {
        // wide rows: 512-thread CTAs (or two 256-thread CTAs per SM), then
        // clusters of 2/4/8 splitting the row
        wide = true;
        p.nt = kWideThreads;
        p.ch = std::max(3, ceil_div(ceil_div(n, VW), p.nt));
        while (p.ch > maxch && p.cl < 8) {
            p.cl *= 2;
            p.slice_w = (int)round_up(ceil_div(n, p.cl), 8 * VW);
            p.ch = std::max(3, ceil_div(ceil_div(p.slice_w, VW), p.nt));
        }
    }
    if (p.ch > kMaxCh)
        throw Error(GOAT_ENOTSUP, "sinkhorn: order " + std::to_string(n) + " exceeds 8-CTA clusters of this build");
    p.rows = wide ? 1 : rows_for(p.ch, p.nt);
    const int nbands = (mrows + p.rows - 1) / p.rows;
    // Cluster-split wide rows stream through the bulk-copy ring (measured: +30%
    // at n = 20000-40000); unsplit wide rows keep the register prefetch, which
    // measured faster at n = 10000 (profiles/round1_sk_tune.md).
    if (wide && p.cl > 1 && env_int("GOAT_SK_TMA", 1)) {
        // as many row-slice stages as ~200 KB of shared memory holds
        p.stage_bytes = (int)round_up((size_t)p.slice_w * sizeof(T), 128);
        p.stages = std::max(3, std::min(8, 200 * 1024 / p.stage_bytes));
        if (const int st = env_int("GOAT_SK_STAGES", 0)) p.stages = std::max(3, std::min(8, st));
        p.smem = (size_t)p.stages * p.stage_bytes;
        GOAT_CUDA(cudaFuncSetAttribute(persistent_for<T>(p.ch, p.cl, p.nt, true),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
    }
    void *const kfn = persistent_for<T>(p.ch, p.cl, p.nt, p.stages > 0);
    p.persistent = env_int("GOAT_SK_PERSISTENT", 1) != 0 || p.nt != kThreads;
    // Co-resident groups (CTAs, or clusters of cl CTAs) for the cooperative launch.
    int groups = 0;
    if (p.cl == 1) {
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)kfn, p.nt, p.smem);
        groups = std::max(1, occ) * num_sms;  // measured: all co-resident CTAs is fastest (n <= 5000)
    } else {
        cudaLaunchAttribute attrs[2];
        SkPlan q = p;
        q.nblk = p.cl * num_sms;
        cudaLaunchConfig_t cfg = persistent_config(q, nullptr, attrs);
        cfg.numAttrs = 0;  // occupancy query takes the cluster shape, not the cooperative flag
        cudaLaunchAttribute cattr = attrs[1];
        cfg.attrs = &cattr;
        cfg.numAttrs = 1;
        int ncl = 0;
        GOAT_CUDA(cudaOccupancyMaxActiveClusters(&ncl, kfn, &cfg));
        groups = std::max(1, ncl);
    }
    int ngrp = std::max(1, std::min(nbands, groups));
    if (const int force = env_int("GOAT_SK_BLOCKS", 0)) ngrp = std::max(1, std::min({force / p.cl, nbands, groups}));
    if (!p.persistent) ngrp = std::max(1, std::min(nbands, num_sms));
    p.ngrp = ngrp;
    p.nblk = ngrp * p.cl;
    p.merge_blocks = std::max(1, std::min((n + 7) / 8, 4 * num_sms));  // one warp per column
    p.colpart_bytes = (size_t)std::max(p.nblk, num_sms * 2) * round_up(n, 8) * sizeof(T);
    return p;
}

template <class T, int CH>
void launch_pass_ch(const SkArgs &a, const SkPlan &p, cudaStream_t s) {
    sk_pass_kernel<T, CH, rows_for(CH)><<<p.nblk, kThreads, 0, s>>>(a);
    note_launch();
}

template <class T> void sk_launch_pass(const SkArgs &a, const SkPlan &p, cudaStream_t s) {
    if (p.cl != 1 || p.nt != kThreads) throw Error(GOAT_ENOTSUP, "sinkhorn: wide rows need the persistent driver");
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

template <class T> void sk_launch_persistent(const SkArgs &a, const SkPlan &p, unsigned *bar, cudaStream_t s) {
    // bar: [0] arrivals, [32] generation, bytes [512, 544) the dev-max slots
    GOAT_CUDA(cudaMemsetAsync(bar, 0, 1024, s));
    SkArgs args = a;
    args.dslot = reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(bar) + 512);
    args.nblk = p.ngrp;  // column-partial rows = row groups
    args.slice_w = p.slice_w;
    args.resident = env_int("GOAT_SK_RES", 1);
    // G re-read by the bulk-copy ring stays in L2 when it fits (GOAT_SK_L2HINT)
    args.l2_last = p.pipe && env_int("GOAT_SK_L2HINT", 0) &&
                   (double)a.n * a.ld * sizeof(T) <= env_int("GOAT_SK_L2HINT_MB", 112) * 1048576.0;
    args.stages = p.stages;
    args.stage_bytes = p.stage_bytes;
    args.dbg = env_int("GOAT_SK_DBG", 0);
    void *params[] = {&args, &bar};
    cudaLaunchAttribute attrs[2];
    cudaLaunchConfig_t cfg = persistent_config(p, s, attrs);
    if (p.tile && args.single_pass) throw Error(GOAT_ENOTSUP, "sinkhorn: the tile plan has no single-pass mode");
    void *fn = p.tile    ? tile_for<T>(p.cl, p.ch, p.rows)
               : p.wide2 ? wide2_for(p.nt, p.cl, p.ch, p.wide_tm, p.rows)
               : p.pipe  ? pipe_for(p.ch, p.cl, p.nt, p.rows)
                         : persistent_for<T>(p.ch, p.cl, p.nt, p.stages > 0);
    int rows_g = p.tile_rows;
    void *tparams[] = {&args, &bar, &rows_g};
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, p.tile ? tparams : params);
    if (e != cudaSuccess && attrs[0].val.cooperative) {
        // a profiler that replays kernels rejects cooperative cluster launches; the
        // grid is sized to the co-resident maximum, so launch it plainly
        (void)cudaGetLastError();
        attrs[0].val.cooperative = 0;
        e = cudaLaunchKernelExC(&cfg, fn, p.tile ? tparams : params);
    }
    GOAT_CUDA(e);
    note_launch();
}

template <class T>
void sk_launch_shard_pass(const SkArgs &a, const SkPlan &p, unsigned *bar, double *send, cudaStream_t s) {
    if (!p.persistent) throw Error(GOAT_ENOTSUP, "sharded sinkhorn needs the persistent pass kernel");
    SkArgs args = a;
    args.single_pass = 1;
    sk_launch_persistent<T>(args, p, bar, s);
    args.nblk = p.ngrp;
    sk_shard_colsum_kernel<T><<<std::max(1, std::min(ceil_div(a.n, kThreads), 4 * 148)), kThreads, 0, s>>>(
        args, p.nblk, send, bar + 64);
    note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T>
void sk_launch_shard_merge(const SkArgs &a, const double *recv, int world, unsigned char *bad, cudaStream_t s) {
    const double tiny = sizeof(T) == 4 ? 1e-30 : 1e-290;
    const int blocks = std::max(1, std::min(64, ceil_div(a.n, kShardMergeThreads)));
    sk_shard_merge_kernel<<<blocks, kShardMergeThreads, 0, s>>>(a, recv, world, tiny, bad);
    note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T> void sk_launch_shard_repair_pass(const SkArgs &a, const unsigned char *bad, double *pair,
                                                    cudaStream_t s) {
    sk_shard_repair_pass_kernel<T><<<std::max(1, std::min(ceil_div(a.n, kThreads), 4 * 148)), kThreads, 0, s>>>(
        a, bad, pair);
    note_launch();
    GOAT_CHECK_LAUNCH();
}

void sk_launch_shard_repair_merge(const SkArgs &a, const double *recv, int world, const unsigned char *bad,
                                  cudaStream_t s) {
    sk_shard_repair_merge_kernel<<<1, kShardMergeThreads, 0, s>>>(a, recv, world, bad);
    note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T>
void sk_launch_emit(const SkArgs &a, T *Q, int64_t ldq, const T *P, int64_t ldp, const T *L,
                    int64_t ldl, double *part, int nblk, cudaStream_t s) {
    sk_emit_kernel<T><<<nblk, kThreads, 0, s>>>(a, Q, ldq, P, ldp, L, ldl, part); note_launch();
    GOAT_CHECK_LAUNCH();
}

template SkPlan sk_plan<float>(int, int, int, bool);
template SkPlan sk_plan<double>(int, int, int, bool);
template void sk_launch_shard_pass<float>(const SkArgs &, const SkPlan &, unsigned *, double *, cudaStream_t);
template void sk_launch_shard_pass<double>(const SkArgs &, const SkPlan &, unsigned *, double *, cudaStream_t);
template void sk_launch_shard_merge<float>(const SkArgs &, const double *, int, unsigned char *, cudaStream_t);
template void sk_launch_shard_merge<double>(const SkArgs &, const double *, int, unsigned char *, cudaStream_t);
template void sk_launch_shard_repair_pass<float>(const SkArgs &, const unsigned char *, double *, cudaStream_t);
template void sk_launch_shard_repair_pass<double>(const SkArgs &, const unsigned char *, double *, cudaStream_t);
template void sk_launch_pass<float>(const SkArgs &, const SkPlan &, cudaStream_t);
template void sk_launch_pass<double>(const SkArgs &, const SkPlan &, cudaStream_t);
template void sk_launch_merge<float>(const SkArgs &, const SkPlan &, cudaStream_t);
template void sk_launch_merge<double>(const SkArgs &, const SkPlan &, cudaStream_t);
template void sk_launch_persistent<float>(const SkArgs &, const SkPlan &, unsigned *, cudaStream_t);
template void sk_launch_persistent<double>(const SkArgs &, const SkPlan &, unsigned *, cudaStream_t);
template void sk_launch_emit<float>(const SkArgs &, float *, int64_t, const float *, int64_t,
                                    const float *, int64_t, double *, int, cudaStream_t);
template void sk_launch_emit<double>(const SkArgs &, double *, int64_t, const double *, int64_t,
                                     const double *, int64_t, double *, int, cudaStream_t);

}  // namespace goat
