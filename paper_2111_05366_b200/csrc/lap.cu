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
#include <algorithm>
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
    lap_sap_kernel(const T *M, int64_t ld, int n, double sign, LapWork w, int use_smem, int warm) {
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

    if (warm) {
        // warm start (auction repair): tight partial assignment + feasible duals given
        for (int j = tid; j < n; j += kLapThreads) {
            v[j] = w.v[j]; row4col[j] = w.row4col[j]; path[j] = -1;
        }
    } else {
        for (int j = tid; j < n; j += kLapThreads) {
            v[j] = 0.0; u[j] = 0.0; row4col[j] = -1; col4row[j] = -1; path[j] = -1;
        }
    }
    __syncthreads();
    for (int cur = 0; cur < n; ++cur) {
        if (warm && col4row[cur] != -1) continue;  // already assigned (uniform: global, synced)
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


// ------------------------------------------------------------------ auction
// Forward auction with epsilon scaling (Bertsekas) for large n, as the fast
// front end of the exact solver: warps bid for unassigned rows (best and
// second-best of val_ij - p_j over all columns), columns take the highest bid
// (atomicMax on the bit pattern of non-negative doubles, ties to the lowest
// row), prices rise to the winning bid.  One cooperative launch runs every
// phase; the result is eps-optimal, and lap_auction_repair + the warm-started
// augmenting-path kernel turn it into a certified exact optimum.
struct AucArgs {
    int n;
    int64_t ld;
    double sign;           // val = sign * M  (+1 maximize, -1 minimize)
    double eps0, eps_min, theta;
    double *price;         // [n]
    int *row_col;          // [n] column of row (-1)
    int *col_row;          // [n] row of column (-1)
    unsigned long long *bid_val;  // [n] highest bid on column (bits), 0 = none
    int *bid_row;          // [n] winning row (INT_MAX = none)
    int *row_bid;          // [n] column this row bid on this round (-1)
    double *row_bid_v;     // [n]
    unsigned *bar;         // grid barrier counter (zeroed)
    int *counters;         // [0] assigned columns, [1] rounds (diagnostic), [2] status
    int *list;             // [n] unassigned rows of the round
    double *part_w;        // [2 * CTAs] (best, second) of a CTA's share of a row (few-bidder rounds)
    int *part_j;           // [CTAs] its best column
    int max_rounds;
    int tail;              // a phase ends once at most `tail` rows are unassigned
    int keep;              // later phases keep the rows that satisfy eps-CS
    int stall;             // a phase also ends after `stall` rounds without a new minimum of unassigned rows (0 = never)
};

__device__ __forceinline__ unsigned ld_acq(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void gbar(unsigned *bar, unsigned nb, unsigned &epoch) {
    ++epoch;
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(bar), "r"(1u) : "memory");
        while (ld_acq(bar) < epoch * nb) { }
    }
    __syncthreads();
}

// Row scans of the auction: 16-byte loads of the cost row and of the price vector
// (VW = 4 floats / 2 doubles per lane per step, two steps in flight).  Lanes walk
// ascending column indices, so a strict '>' keeps the lowest index among equal
// profits within a lane; callers combine lanes with the (value, index) rule.
template <class T>
__device__ __forceinline__ void row_profits(const T *Mi, const double *price, double sign, int n, int q,
                                            double (&v)[16 / sizeof(T)]) {
    constexpr int VW = 16 / sizeof(T);
    const int j0 = q * VW;
    T x[VW];
    *reinterpret_cast<uint4 *>(x) = *reinterpret_cast<const uint4 *>(Mi + j0);  // rows are padded to 32 bytes
    if (j0 + VW <= n) {
#pragma unroll
        for (int e = 0; e < VW; e += 2) {
            const double2 p = __ldcg(reinterpret_cast<const double2 *>(price + j0 + e));
            v[e] = sign * (double)x[e] - p.x;
            v[e + 1] = sign * (double)x[e + 1] - p.y;
        }
    } else {
#pragma unroll
        for (int e = 0; e < VW; ++e) v[e] = (j0 + e < n) ? sign * (double)x[e] - __ldcg(price + j0 + e) : -INFINITY;
    }
}

template <class T>
__device__ __forceinline__ void scan_top2(const T *Mi, const double *price, double sign, int n, int start, int stride,
                                          double &w1, double &w2, int &j1) {
    constexpr int VW = 16 / sizeof(T);
    const int nv = (n + VW - 1) / VW;
#pragma unroll 2
    for (int q = start; q < nv; q += stride) {
        double v[VW];
        row_profits<T>(Mi, price, sign, n, q, v);
#pragma unroll
        for (int e = 0; e < VW; ++e) {
            if (v[e] > w1) { w2 = w1; w1 = v[e]; j1 = q * VW + e; }
            else if (v[e] > w2) w2 = v[e];
        }
    }
}

// R rows per warp: the price vector is loaded once per column step and shared by the
// R row loads (the price reads are 2/3 of the L2->SM traffic of a one-row scan).
template <class T, int R>
__device__ __forceinline__ void scan_top2_rows(const T *const (&Mi)[R], const double *price, double sign, int n,
                                               int start, int stride, double (&w1)[R], double (&w2)[R], int (&j1)[R]) {
    constexpr int VW = 16 / sizeof(T);
    const int nv = (n + VW - 1) / VW;
    for (int q = start; q < nv; q += stride) {
        const int j0 = q * VW;
        double p[VW];
        if (j0 + VW <= n) {
#pragma unroll
            for (int e = 0; e < VW; e += 2) {
                const double2 pp = __ldcg(reinterpret_cast<const double2 *>(price + j0 + e));
                p[e] = pp.x;
                p[e + 1] = pp.y;
            }
        } else {
#pragma unroll
            for (int e = 0; e < VW; ++e) p[e] = (j0 + e < n) ? __ldcg(price + j0 + e) : INFINITY;  // profit -inf
        }
        T x[R][VW];
#pragma unroll
        for (int k = 0; k < R; ++k) *reinterpret_cast<uint4 *>(x[k]) = *reinterpret_cast<const uint4 *>(Mi[k] + j0);
#pragma unroll
        for (int k = 0; k < R; ++k)
#pragma unroll
            for (int e = 0; e < VW; ++e) {
                const double v = sign * (double)x[k][e] - p[e];
                if (v > w1[k]) { w2[k] = w1[k]; w1[k] = v; j1[k] = j0 + e; }
                else if (v > w2[k]) w2[k] = v;
            }
    }
}

// Named barrier of a warp group inside a CTA (ids 1-4 as immediates, so the kernel
// reserves 5 barriers instead of all 16).
__device__ __forceinline__ void group_bar(int grp, int threads) {
    switch (grp) {
        case 0: asm volatile("bar.sync 1, %0;" ::"r"(threads) : "memory"); break;
        case 1: asm volatile("bar.sync 2, %0;" ::"r"(threads) : "memory"); break;
        case 2: asm volatile("bar.sync 3, %0;" ::"r"(threads) : "memory"); break;
        default: asm volatile("bar.sync 4, %0;" ::"r"(threads) : "memory"); break;
    }
}

// (best, second, lowest index of the best) of two partial scans
__device__ __forceinline__ void top2_merge(double &w1, double &w2, int &j1, double b1, double b2, int bj) {
    if (b1 > w1 || (b1 == w1 && bj < j1)) { w2 = fmax(b2, w1); w1 = b1; j1 = bj; }
    else w2 = fmax(w2, b1);
}
__device__ __forceinline__ void top2_warp(double &w1, double &w2, int &j1) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double b1 = __shfl_xor_sync(0xffffffffu, w1, off);
        const double b2 = __shfl_xor_sync(0xffffffffu, w2, off);
        const int bj = __shfl_xor_sync(0xffffffffu, j1, off);
        top2_merge(w1, w2, j1, b1, b2, bj);
    }
}

template <class T>
__device__ __forceinline__ double scan_best(const T *Mi, const double *price, double sign, int n, int start, int stride) {
    constexpr int VW = 16 / sizeof(T);
    const int nv = (n + VW - 1) / VW;
    double best = -INFINITY;
#pragma unroll 2
    for (int q = start; q < nv; q += stride) {
        double v[VW];
        row_profits<T>(Mi, price, sign, n, q, v);
#pragma unroll
        for (int e = 0; e < VW; ++e) best = fmax(best, v[e]);
    }
    return best;
}

template <class T>
__global__ void __launch_bounds__(256, 3) lap_auction_kernel(const T *M, AucArgs a) {
    const int n = a.n, lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int gt = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    unsigned epoch = 0;
    __shared__ int s_done;
    int rounds = 0, phases = 0;
    unsigned scans = 0;  // diagnostics: bidder rows scanned by this thread
    for (double eps = a.eps0;; eps = fmax(eps / a.theta, a.eps_min)) {
        ++phases;
        // new phase, prices kept.  First phase: empty assignment.  Later phases keep
        // every row that already satisfies eps-complementary slackness for the new
        // eps (its column within eps of its best profit) and free only the others,
        // so a phase re-bids the violators instead of all n rows.
        // Every CTA has read counters[0] for the previous phase's stop test
        // before it is reset (a slow CTA would otherwise see 0 and keep bidding).
        if (rounds > 0) gbar(a.bar, gridDim.x, epoch);
        if (rounds == 0 || a.keep == 0) {
            for (int j = gt; j < n; j += nt) { a.row_col[j] = -1; a.col_row[j] = -1; }
            if (gt == 0) a.counters[0] = 0;
        } else {
            if (gt == 0) a.counters[0] = 0;
            gbar(a.bar, gridDim.x, epoch);
            for (int i = gw; i < n; i += nwarps) {
                const int j0 = __ldcg(a.row_col + i);
                if (j0 < 0) continue;
                const T *Mi = M + (int64_t)i * a.ld;
                double best = scan_best<T>(Mi, a.price, a.sign, n, lane, 32);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, off));
                if (lane == 0) {
                    if (a.sign * (double)Mi[j0] - __ldcg(a.price + j0) >= best - eps) {
                        atomicAdd(a.counters, 1);
                    } else {
                        a.row_col[i] = -1;
                        a.col_row[j0] = -1;
                    }
                }
            }
        }
        for (int j = gt; j < n; j += nt) { a.bid_val[j] = 0ull; a.bid_row[j] = INT_MAX; a.row_bid[j] = -1; }
        gbar(a.bar, gridDim.x, epoch);
        int best_un = INT_MAX, since = 0;  // thread 0 of every CTA tracks the same counters: uniform
        for (;;) {
            // (A) bids of unassigned rows: (best, second best, lowest index of the best) of
            // val_ij - p_j over the row, whatever the work split.  The split follows the
            // number of bidders so every round streams rows at full width: at most one
            // bidder per CTA -> a CTA per row; more -> the bidders are compacted into a
            // list and taken by groups of 4 / 2 warps, a warp per row, or 2 / 4 rows per
            // warp (one load of the price vector serves the rows of a warp).
            auto post_bid = [&](int i, double w1, double w2, int j1) {
                const double gap = (w2 == -INFINITY) ? 0.0 : (w1 - w2);
                const double bid = __ldcg(a.price + j1) + gap + eps;
                a.row_bid[i] = j1;
                a.row_bid_v[i] = bid;
                atomicMax(a.bid_val + j1, (unsigned long long)__double_as_longlong(bid));
                ++scans;
            };
            __shared__ double s_w1[8], s_w2[8];
            __shared__ int s_j1[8];
            const int wib = threadIdx.x >> 5;
            // diagnostics (GOAT_LAP_VERBOSE): rounds and time of phase (A) per work split
            unsigned long long t_a0 = 0;
            int regime = 0;
            if (gt == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_a0));
            if (n - __ldcg(a.counters) <= (int)gridDim.x / 2) {
                // few bidders (the long tail of a phase: 6820 of config 5's 8082 rounds):
                // P = CTAs / bidders CTAs share each row, column-interleaved, and meet
                // through a per-CTA partial in global scratch (one extra grid barrier) --
                // a lone CTA streaming a 160 KB row took 86 us per round.
                for (int i = gt; i < n; i += nt)
                    if (__ldcg(a.row_col + i) == -1) a.list[atomicAdd(a.counters + 6, 1)] = i;
                gbar(a.bar, gridDim.x, epoch);
                const int nb = __ldcg(a.counters + 6);
                const int P = max(1, min(16, (int)gridDim.x / max(nb, 1)));
                const int idx = blockIdx.x / P, part = blockIdx.x - idx * P;
                if (idx < nb) {
                    const int i = __ldcg(a.list + idx);
                    const T *Mi = M + (int64_t)i * a.ld;
                    double w1 = -INFINITY, w2 = -INFINITY;
                    int j1 = INT_MAX;
                    scan_top2<T>(Mi, a.price, a.sign, n, part * (int)blockDim.x + threadIdx.x, P * (int)blockDim.x, w1, w2, j1);
                    top2_warp(w1, w2, j1);
                    if (lane == 0) { s_w1[wib] = w1; s_w2[wib] = w2; s_j1[wib] = j1; }
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        for (int q = 1; q < (int)(blockDim.x >> 5); ++q) top2_merge(w1, w2, j1, s_w1[q], s_w2[q], s_j1[q]);
                        a.part_w[2 * blockIdx.x] = w1;
                        a.part_w[2 * blockIdx.x + 1] = w2;
                        a.part_j[blockIdx.x] = j1;
                    }
                }
                gbar(a.bar, gridDim.x, epoch);
                if (idx < nb && part == 0 && threadIdx.x == 0) {
                    double w1 = -INFINITY, w2 = -INFINITY;
                    int j1 = INT_MAX;
                    for (int q = 0; q < P; ++q) {  // fixed order: deterministic
                        const int b = blockIdx.x + q;
                        top2_merge(w1, w2, j1, __ldcg(a.part_w + 2 * b), __ldcg(a.part_w + 2 * b + 1), __ldcg(a.part_j + b));
                    }
                    post_bid(__ldcg(a.list + idx), w1, w2, j1);
                }
            } else {
                // compact the bidders (the list order varies between runs; each row's bid
                // does not depend on it)
                for (int i = gt; i < n; i += nt)
                    if (__ldcg(a.row_col + i) == -1) a.list[atomicAdd(a.counters + 6, 1)] = i;
                gbar(a.bar, gridDim.x, epoch);
                const int nb = __ldcg(a.counters + 6);
                regime = nb * 4 <= nwarps ? 1 : nb * 2 <= nwarps ? 2 : nb < nwarps + nwarps / 2 ? 3 : nb < 3 * nwarps ? 4 : 5;
                if (nb * 2 <= nwarps) {
                    // GW warps of a CTA per row
                    const int GW = (nb * 4 <= nwarps) ? 4 : 2;
                    const int gpc = 8 / GW, grp = wib / GW, tig = threadIdx.x - grp * GW * 32;
                    for (int idx = blockIdx.x * gpc + grp; idx < nb; idx += (int)gridDim.x * gpc) {
                        const int i = __ldcg(a.list + idx);
                        const T *Mi = M + (int64_t)i * a.ld;
                        double w1 = -INFINITY, w2 = -INFINITY;
                        int j1 = INT_MAX;
                        scan_top2<T>(Mi, a.price, a.sign, n, tig, GW * 32, w1, w2, j1);
                        top2_warp(w1, w2, j1);
                        if (lane == 0) { s_w1[wib] = w1; s_w2[wib] = w2; s_j1[wib] = j1; }
                        group_bar(grp, GW * 32);
                        if (tig == 0) {
                            for (int q = 1; q < GW; ++q) top2_merge(w1, w2, j1, s_w1[wib + q], s_w2[wib + q], s_j1[wib + q]);
                            post_bid(i, w1, w2, j1);
                        }
                        group_bar(grp, GW * 32);
                    }
                } else if (nb < nwarps + nwarps / 2) {
                    for (int idx = gw; idx < nb; idx += nwarps) {
                        const int i = __ldcg(a.list + idx);
                        double w1 = -INFINITY, w2 = -INFINITY;
                        int j1 = INT_MAX;
                        scan_top2<T>(M + (int64_t)i * a.ld, a.price, a.sign, n, lane, 32, w1, w2, j1);
                        top2_warp(w1, w2, j1);
                        if (lane == 0) post_bid(i, w1, w2, j1);
                    }
                } else if (nb < 3 * nwarps) {
                    constexpr int R = 2;
                    for (int base = gw * R; base < nb; base += nwarps * R) {
                        int rows[R];
                        const T *Mi[R];
                        double w1[R], w2[R];
                        int j1[R];
#pragma unroll
                        for (int k = 0; k < R; ++k) {
                            rows[k] = __ldcg(a.list + min(base + k, nb - 1));
                            Mi[k] = M + (int64_t)rows[k] * a.ld;
                            w1[k] = w2[k] = -INFINITY;
                            j1[k] = INT_MAX;
                        }
                        scan_top2_rows<T, R>(Mi, a.price, a.sign, n, lane, 32, w1, w2, j1);
#pragma unroll
                        for (int k = 0; k < R; ++k) {
                            top2_warp(w1[k], w2[k], j1[k]);
                            if (lane == 0 && base + k < nb) post_bid(rows[k], w1[k], w2[k], j1[k]);
                        }
                    }
                } else {
                    // most of the scan volume (config 5: 617 rounds, ~25 000 bidders each):
                    // 4 rows per warp, and the CTA walks the columns in tiles whose prices
                    // are staged once in shared memory for its 32 row scans (the fp64 price
                    // reads were 2/3 of a row scan's L2->SM traffic, 1/3 with 4 rows per warp)
                    constexpr int R = 4, TC = 2048, VW = 16 / sizeof(T);
                    __shared__ __align__(16) double s_price[2][TC];
                    const int passes = ((nb + R - 1) / R + nwarps - 1) / nwarps;  // uniform over the grid
                    for (int ps = 0; ps < passes; ++ps) {
                        const int base = (ps * nwarps + gw) * R;
                        const bool active = base < nb;
                        int rows[R];
                        const T *Mi[R];
                        double w1[R], w2[R];
                        int j1[R];
#pragma unroll
                        for (int k = 0; k < R; ++k) {
                            rows[k] = __ldcg(a.list + min(base + k, nb - 1));
                            Mi[k] = M + (int64_t)rows[k] * a.ld;
                            w1[k] = w2[k] = -INFINITY;
                            j1[k] = INT_MAX;
                        }
                        for (int t0 = 0, buf = 0; t0 < n; t0 += TC, buf ^= 1) {
                            // the other buffer was last read two tiles ago: every warp has passed
                            // the barrier of the previous tile since
                            for (int c = threadIdx.x; c < TC; c += blockDim.x)
                                s_price[buf][c] = (t0 + c < n) ? __ldcg(a.price + t0 + c) : INFINITY;  // profit -inf
                            __syncthreads();
                            if (!active) continue;
#pragma unroll 2
                            for (int q = lane; q < TC / VW; q += 32) {
                                const int j0 = t0 + q * VW;
                                if (j0 >= n) break;
                                double p[VW];
#pragma unroll
                                for (int e = 0; e < VW; e += 2) {
                                    const double2 pp = *reinterpret_cast<const double2 *>(&s_price[buf][q * VW + e]);
                                    p[e] = pp.x;
                                    p[e + 1] = pp.y;
                                }
                                T x[R][VW];
#pragma unroll
                                for (int k = 0; k < R; ++k)
                                    *reinterpret_cast<uint4 *>(x[k]) = *reinterpret_cast<const uint4 *>(Mi[k] + j0);
#pragma unroll
                                for (int k = 0; k < R; ++k)
#pragma unroll
                                    for (int e = 0; e < VW; ++e) {
                                        const double v = a.sign * (double)x[k][e] - p[e];
                                        if (v > w1[k]) { w2[k] = w1[k]; w1[k] = v; j1[k] = j0 + e; }
                                        else if (v > w2[k]) w2[k] = v;
                                    }
                            }
                        }
#pragma unroll
                        for (int k = 0; k < R; ++k) {
                            top2_warp(w1[k], w2[k], j1[k]);
                            if (lane == 0 && base + k < nb) post_bid(rows[k], w1[k], w2[k], j1[k]);
                        }
                        __syncthreads();  // the price buffers are rewritten by the next pass
                    }
                }
            }
            gbar(a.bar, gridDim.x, epoch);
            if (gt == 0) {
                unsigned long long t_a1;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_a1));
                a.counters[8 + regime] += 1;
                reinterpret_cast<unsigned long long *>(a.counters + 16)[regime] += t_a1 - t_a0;
            }
            // (B) ties on the winning bid go to the lowest row
            for (int i = gt; i < n; i += nt) {
                const int j = __ldcg(a.row_bid + i);
                if (j >= 0 && (unsigned long long)__double_as_longlong(__ldcg(a.row_bid_v + i)) == __ldcg(a.bid_val + j))
                    atomicMin(a.bid_row + j, i);
            }
            gbar(a.bar, gridDim.x, epoch);
            // (C) columns take their winner; evicted owners become unassigned
            for (int j = gt; j < n; j += nt) {
                const unsigned long long bv = __ldcg(a.bid_val + j);
                if (bv == 0ull) continue;
                const int w = __ldcg(a.bid_row + j);
                const int old = __ldcg(a.col_row + j);
                if (old >= 0) a.row_col[old] = -1;
                else atomicAdd(a.counters, 1);
                a.col_row[j] = w;
                a.row_col[w] = j;
                a.price[j] = __longlong_as_double((long long)bv);
                a.bid_val[j] = 0ull;
                a.bid_row[j] = INT_MAX;
            }
            for (int i = gt; i < n; i += nt) a.row_bid[i] = -1;
            if (gt == 0) a.counters[6] = 0;  // next round's bidder list
            gbar(a.bar, gridDim.x, epoch);
            ++rounds;
            // The last few bidders of a phase fight long price wars on near-tied
            // columns; the exact repair assigns them far cheaper, so a phase stops
            // at `tail` unassigned rows (the next phase restarts from the prices).
            // Exact ties (0/1-graph gradients, integer costs) make the last bidders trade a
            // column back and forth in eps-sized steps: a phase that has not reached a new
            // minimum of unassigned rows for `stall` rounds hands them to the repair too.
            if (threadIdx.x == 0) {
                const int un = n - __ldcg(a.counters);
                if (un < best_un) { best_un = un; since = 0; } else ++since;
                s_done = un <= a.tail || rounds >= a.max_rounds || (a.stall > 0 && since >= a.stall);
            }
            __syncthreads();
            if (s_done) break;
        }
        if (eps <= a.eps_min || rounds >= a.max_rounds) break;
    }
    if (gt == 0) { a.counters[1] = rounds; a.counters[2] = (rounds >= a.max_rounds) ? 1 : 0; a.counters[5] = phases; }
    if (scans) atomicAdd(reinterpret_cast<unsigned *>(a.counters) + 4, scans);
}

// Exact-repair preparation: duals from the auction prices in the minimisation
// form of the augmenting-path solver (cost c = -val, v_j = -p_j,
// u_i = min_j c_ij - v_j); rows whose column is not an exact argmin are freed.
template <class T>
__global__ void lap_auction_repair(const T *M, AucArgs a, double *u, double *v, int *row4col, int *col4row, int *nfree) {
    const int n = a.n, lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int i = gw; i < n; i += nwarps) {
        const T *Mi = M + (int64_t)i * a.ld;
        double best = scan_best<T>(Mi, a.price, a.sign, n, lane, 32);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, off));
        if (lane == 0) {
            u[i] = -best;
            const int j = a.row_col[i];
            const bool tight = j >= 0 && (a.sign * (double)Mi[j] - a.price[j]) == best;
            col4row[i] = tight ? j : -1;
            if (!tight) atomicAdd(nfree, 1);
        }
    }
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        v[j] = -a.price[j];
        const int r = a.col_row[j];
        const bool keep = r >= 0 && a.row_col[r] == j;
        row4col[j] = keep ? r : -1;
    }
}


// Warm-start tightening before the repair: a row is kept by the repair only if
// its auction column attains max_j(val_ij - p_j) exactly.  Bidding leaves the
// last bidder eps below its second-best column, so many rows miss by < eps.
// Lowering the price of row i's column by that gap (delta_i) makes the row tight;
// other rows' maxima may move, so a few Jacobi rounds are run.  Any price vector
// gives feasible duals (u_i is recomputed as the row max), so exactness is
// untouched -- this only shrinks the set of rows the repair must re-assign.
template <class T>
__global__ void lap_tighten_rows(const T *M, AucArgs a, double *delta) {
    const int n = a.n, lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int i = gw; i < n; i += nwarps) {
        const int j0 = a.row_col[i];
        if (j0 < 0) { if (lane == 0) delta[i] = 0.0; continue; }
        const T *Mi = M + (int64_t)i * a.ld;
        double best = scan_best<T>(Mi, a.price, a.sign, n, lane, 32);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, off));
        if (lane == 0) delta[i] = best - (a.sign * (double)Mi[j0] - a.price[j0]);
    }
}

__global__ void lap_tighten_cols(AucArgs a, const double *delta) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x) {
        const int j = a.row_col[i];
        if (j >= 0 && delta[i] > 0.0) a.price[j] -= delta[i];
    }
}

// Drop columns whose row was freed (second pass: col4row is final).
__global__ void lap_auction_unlink(int n, const int *col4row, int *row4col) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int r = row4col[j];
        if (r >= 0 && col4row[r] != j) row4col[j] = -1;
    }
}


// ------------------------------------------------------------------ cluster repair
// Warm-started augmenting paths for large n on a thread-block cluster.  The
// single-CTA solver above keeps all per-column state in global memory once n
// outgrows shared memory, so every Dijkstra step streams ~25 bytes per column
// through one SM.  Here CL CTAs split the columns into contiguous slices held in
// shared memory (spc, v, path, row4col, and ucol = u of the row matched to the
// column); a step reads only each CTA's slice of the frontier rows, and its minimum
// is an exchange through distributed shared memory plus cluster barriers.  Ties:
// smallest reduced cost, then a free column (the lowest index).  Dual updates and
// the augmentation are those of the single-CTA solver, so the result is an exact
// optimum (scipy's value; on ties possibly another optimal permutation).
__device__ __forceinline__ unsigned cl_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <class P> __device__ __forceinline__ P *cl_map(P *p, unsigned rank) {
    // generic address of the same shared-memory object in CTA `rank`
    void *r;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(p), "r"(rank));
    return static_cast<P *>(r);
}

constexpr int kLapClThreads = 1024;

// One CTA's view of the next distance level of the search.
struct LapLevel {
    double v;   // smallest tentative distance among its unscanned columns (INFINITY: none)
    int count;  // unscanned columns at that distance
    int freej;  // lowest free column among them (INT_MAX: none)
    int pad;
};

// The search settles a whole DISTANCE LEVEL per step: every unscanned column whose
// tentative distance equals the current minimum is scanned at once (label setting
// stays valid for equal keys since reduced costs are >= 0), and the rows matched to
// them form the next frontier, relaxed together.  On the 0/1-graph gradients this
// solver sees, > 90 % of the single-column steps sat at an unchanged distance
// (config 5: 631 276 steps for 122 rows, 580 062 of them ties), so levels cut the
// cluster barriers 5.5x (114 221 levels).  The frontier (row, u) list lives in global
// scratch (w.rem, w.spc), written in a fixed order -- CTA rank, then thread, then
// column -- so path choices among equal distances are deterministic.
template <class T, int CL>
__global__ void __launch_bounds__(kLapClThreads, 1)
    lap_cluster_sap_kernel(const T *M, int64_t ld, int n, double sign, LapWork w, int W) {
    extern __shared__ __align__(16) unsigned char smem[];
    double *spc = reinterpret_cast<double *>(smem);
    double *v = spc + W;
    double *ucol = v + W;
    int *path = reinterpret_cast<int *>(ucol + W);
    int *r4c = path + W;
    unsigned char *SC = reinterpret_cast<unsigned char *>(r4c + W);
    constexpr int NW = kLapClThreads / 32;
    __shared__ LapLevel lvl[2][CL];
    __shared__ double s_wmin[NW];
    __shared__ int s_wcnt[NW], s_wfree[NW];
    const unsigned rank = cl_rank();
    const int c0 = (int)rank * W, c1 = min(n, c0 + W), wloc = max(0, c1 - c0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int *col4row = w.col4row;
    int *frow = w.rem;     // frontier rows of the current level
    double *fu = w.spc;    // their duals
    for (int jl = tid; jl < wloc; jl += kLapClThreads) {
        const int j = c0 + jl;
        v[jl] = w.v[j];
        const int r = w.row4col[j];
        r4c[jl] = r;
        ucol[jl] = r >= 0 ? w.u[r] : 0.0;
    }
    cl_sync();
    int par = 0;
    int d_rows = 0, d_levels = 0, d_cols = 0;  // diagnostics (GOAT_LAP_VERBOSE): free rows, levels, columns scanned
    for (int cur = 0; cur < n; ++cur) {
        if (__ldcg(col4row + cur) != -1) continue;  // matched (uniform: published by the last cluster barrier)
        ++d_rows;
        for (int jl = tid; jl < wloc; jl += kLapClThreads) { SC[jl] = 0; spc[jl] = INFINITY; }
        __syncthreads();
        const double ucur = __ldcg(w.u + cur);
        double minv = 0.0;
        int sink = -1, nf = 1;
        bool first = true;  // the first frontier is the free row itself
        for (;;) {
            // (1) relax this CTA's unscanned columns from every frontier row.  A thread's
            // columns (up to 4 at a time) are relaxed together, frontier rows outermost, so
            // the cost loads of one row -- cold HBM reads, the longest link of a level --
            // are independent and overlap: config 5's repair 734 -> 592 ms.  (A column-outer
            // loop paid one load latency per column: the 8-CTA cluster, with twice the
            // columns per thread, measured 951 ms.  Batching four frontier rows as well,
            // 16 loads in flight, measured slower: 862 ms.)
            double tmin = INFINITY;
            for (int jb = tid; jb < wloc; jb += 4 * kLapClThreads) {
                int jl[4];
                bool act[4];
                double vj[4], sj[4];
                int pj[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    jl[c] = jb + c * kLapClThreads;
                    act[c] = jl[c] < wloc && !SC[jl[c]];
                    vj[c] = act[c] ? v[jl[c]] : 0.0;
                    sj[c] = act[c] ? spc[jl[c]] : INFINITY;
                    pj[c] = -1;
                }
                for (int q = 0; q < nf; ++q) {
                    const int i = first ? cur : __ldcg(frow + q);
                    const double ui = first ? ucur : __ldcg(fu + q);
                    const T *Mi = M + (int64_t)i * ld + c0;
                    T m[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) m[c] = act[c] ? Mi[jl[c]] : T(0);
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const double r = ((minv + sign * (double)m[c]) - ui) - vj[c];
                        if (act[c] && r < sj[c]) { sj[c] = r; pj[c] = i; }
                    }
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (!act[c]) continue;
                    if (pj[c] >= 0) { spc[jl[c]] = sj[c]; path[jl[c]] = pj[c]; }
                    tmin = fmin(tmin, sj[c]);
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) tmin = fmin(tmin, __shfl_xor_sync(0xffffffffu, tmin, off));
            if (lane == 0) s_wmin[warp] = tmin;
            __syncthreads();
            double bmin = INFINITY;
#pragma unroll
            for (int q = 0; q < NW; ++q) bmin = fmin(bmin, s_wmin[q]);
            // (2) this CTA's columns at its minimum: count, lowest free one
            int cnt = 0, fj = INT_MAX;
            if (bmin < INFINITY) {
                for (int jl = tid; jl < wloc; jl += kLapClThreads) {
                    if (SC[jl] || spc[jl] != bmin) continue;
                    ++cnt;
                    if (r4c[jl] == -1) fj = min(fj, c0 + jl);
                }
            }
            int incl = cnt;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += t;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) fj = min(fj, __shfl_xor_sync(0xffffffffu, fj, off));
            if (lane == 31) s_wcnt[warp] = incl;
            if (lane == 0) s_wfree[warp] = fj;
            __syncthreads();
            int woff = 0, bcount = 0, bfree = INT_MAX;
#pragma unroll
            for (int q = 0; q < NW; ++q) {
                if (q < warp) woff += s_wcnt[q];
                bcount += s_wcnt[q];
                bfree = min(bfree, s_wfree[q]);
            }
            if (tid < CL) *cl_map(&lvl[par][rank], (unsigned)tid) = LapLevel{bmin, bcount, bfree, 0};
            cl_sync();
            // (3) the global level: distance, a free column to stop at, list offsets
            double d = INFINITY;
#pragma unroll
            for (int q = 0; q < CL; ++q) d = fmin(d, lvl[par][q].v);
            if (!(d < INFINITY)) {
                if (rank == 0 && tid == 0) *w.status = -1;
                return;  // infeasible (uniform across the cluster)
            }
            int gfree = INT_MAX, base = 0, total = 0;
#pragma unroll
            for (int q = 0; q < CL; ++q) {
                if (lvl[par][q].v != d) continue;
                gfree = min(gfree, lvl[par][q].freej);
                if (q < (int)rank) base += lvl[par][q].count;
                total += lvl[par][q].count;
            }
            par ^= 1;
            minv = d;
            ++d_levels;
            if (gfree != INT_MAX) {
                sink = gfree;
                if (sink >= c0 && sink < c1 && tid == 0) SC[sink - c0] = 1;
                break;
            }
            // (4) scan every column of the level; their rows are the next frontier.  (Measured:
            // writing each CTA's candidates speculatively before the barrier, to save the
            // second barrier, is slower -- 18 vs 12 us per level -- every CTA then flushes
            // global writes each level; carrying up to two (row, u) entries per CTA inline in
            // the level exchange and skipping the list and its barrier for such levels is
            // slower too, 882 vs 734 ms on config 5's repair.)
            if (bmin == d && cnt) {
                int idx = base + woff + (incl - cnt);
                for (int jl = tid; jl < wloc; jl += kLapClThreads) {
                    if (SC[jl] || spc[jl] != d) continue;
                    frow[idx] = r4c[jl];
                    fu[idx] = ucol[jl];
                    ++idx;
                    SC[jl] = 1;
                }
                __threadfence();
            }
            nf = total;
            d_cols += total;
            first = false;
            cl_sync();  // the frontier list is complete and visible to every CTA
        }
        __syncthreads();
        // dual update (matcher order of the single-CTA solver): scanned columns
        for (int jl = tid; jl < wloc; jl += kLapClThreads) {
            if (!SC[jl]) continue;
            const double dd = minv - spc[jl];
            v[jl] -= dd;
            if (c0 + jl != sink) ucol[jl] += dd;  // u of the visited row matched to the column
        }
        cl_sync();
        if (rank == 0 && tid == 0) {
            // augment along the path: sink <- ... <- cur (ucol moves with its row)
            const double unew = ucur + minv;
            int j = sink;
            for (;;) {
                const unsigned oj = (unsigned)(j / W);
                const int r = *cl_map(&path[j - (int)oj * W], oj);
                const int t = __ldcg(col4row + r);
                double ur = unew;
                if (r != cur) {
                    const unsigned ot = (unsigned)(t / W);
                    ur = *cl_map(&ucol[t - (int)ot * W], ot);
                }
                *cl_map(&r4c[j - (int)oj * W], oj) = r;
                *cl_map(&ucol[j - (int)oj * W], oj) = ur;
                col4row[r] = j;
                if (r == cur) break;
                j = t;
            }
        }
        cl_sync();
    }
    for (int jl = tid; jl < wloc; jl += kLapClThreads) {
        w.row4col[c0 + jl] = r4c[jl];
        w.v[c0 + jl] = v[jl];
    }
    if (rank == 0 && tid == 0) { *w.status = 0; w.status[1] = d_rows; w.status[2] = d_levels; w.status[3] = d_cols; }
}

}  // namespace

template <class T>
int launch_lap_auction(const T *M, int64_t ld, int n, int sense, double range, const LapWork &w,
                       const AuctionWork &aw, int num_sms, cudaStream_t s) {
    AucArgs a{};
    a.n = n; a.ld = ld; a.sign = (sense == GOAT_MAXIMIZE) ? 1.0 : -1.0;
    a.eps0 = std::max(range, 1e-300) / 4.0;
    // GOAT_LAP_EPS_END (final eps = range * 10^-x / n) and GOAT_LAP_THETA (eps
    // divisor per phase) trade auction rounds against rows left for the exact repair
    const char *ee = getenv("GOAT_LAP_EPS_END");
    const char *th = getenv("GOAT_LAP_THETA");
    a.eps_min = std::max(range, 1e-300) * pow(10.0, -(ee ? atof(ee) : 7.0)) / std::max(n, 1);
    a.theta = th ? std::max(2.0, atof(th)) : 8.0;
    a.price = aw.price; a.row_col = aw.row_col; a.col_row = aw.col_row; a.bid_val = aw.bid_val;
    a.bid_row = aw.bid_row; a.row_bid = aw.row_bid; a.row_bid_v = aw.row_bid_v; a.bar = aw.bar;
    a.counters = aw.counters; a.max_rounds = 200000;
    a.list = w.rem;  // free until the repair
    a.part_w = aw.part_w;
    a.part_j = aw.part_j;
    const char *te = getenv("GOAT_LAP_TAIL");  // divisor: tail = n / div (0 = complete every phase)
    // measured (profiles/round1_lap_tail_scan.log): ending a phase at n/128 free rows
    // cuts the auction's bidding-war tail at n <= 8192 (c4 LAP 44 -> 29 ms, c3 75 ->
    // 63 ms, the exact repair absorbs the extra rows); n/2048 beyond it, where a row left
    // to the cluster repair costs ~5 ms (n = 40000, profiles/round2_lap_scan.log:
    // n/512 -> 1634 + 1339 ms, n/1024 -> 1657 + 1164, n/2048 -> 1796 + 711, n/4096 -> 2396 + 540)
    // (the switch follows the repair solver: one CTA while its state fits shared memory,
    // the same test launch_lap_sap makes, else the cluster solver)
    const bool one_cta_repair = (size_t)n * (8 + 8 + 4 + 4 + 4 + 1) + 16 <= 200 * 1024;
    const int div = te ? atoi(te) : (one_cta_repair ? 128 : 2048);
    a.tail = div > 0 ? n / div : 0;
    const char *se = getenv("GOAT_LAP_STALL");
    a.stall = se ? atoi(se) : 0;
    const char *ke = getenv("GOAT_LAP_KEEP");
    a.keep = ke ? atoi(ke) : 0;  // measured: rounds 6556 -> 6482 at n = 40000, no gain; opt-in
    GOAT_CUDA(cudaMemsetAsync(aw.price, 0, sizeof(double) * n, s));
    GOAT_CUDA(cudaMemsetAsync(aw.bar, 0, 256, s));
    GOAT_CUDA(cudaMemsetAsync(aw.counters, 0, 128, s));
    int occ = 0;
    GOAT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lap_auction_kernel<T>, 256, 0));
    const int grid = std::min(kAucMaxCtas, std::max(1, occ) * num_sms);
    void *params[] = {(void *)&M, &a};
    const bool verbose = getenv("GOAT_LAP_VERBOSE") != nullptr;
    cudaEvent_t ev[3];
    if (verbose) { for (auto &e : ev) cudaEventCreate(&e); cudaEventRecord(ev[0], s); }
    GOAT_CUDA(cudaLaunchCooperativeKernel((const void *)lap_auction_kernel<T>, dim3(grid), dim3(256), params, 0, s));
    note_launch();
    if (verbose) cudaEventRecord(ev[1], s);
    const char *tr = getenv("GOAT_LAP_TIGHTEN");  // Jacobi rounds (0 = off)
    const int rounds = tr ? atoi(tr) : 16;  // measured: freed rows 15815 -> 170 at n = 40000, repair 4.3 -> 3.4 s
    for (int r = 0; r < rounds; ++r) {
        lap_tighten_rows<T><<<num_sms * 4, 256, 0, s>>>(M, a, aw.row_bid_v);  // row_bid_v: free n-vector now
        lap_tighten_cols<<<std::max(1, std::min(ceil_div(n, 256), num_sms * 4)), 256, 0, s>>>(a, aw.row_bid_v);
        note_launch(2);
    }
    lap_auction_repair<T><<<num_sms * 4, 256, 0, s>>>(M, a, w.u, w.v, w.row4col, w.col4row, aw.counters + 3); note_launch();
    lap_auction_unlink<<<std::max(1, std::min(ceil_div(n, 256), num_sms * 4)), 256, 0, s>>>(n, w.col4row, w.row4col); note_launch();
    GOAT_CHECK_LAUNCH();
    if (verbose) {
        cudaEventRecord(ev[2], s);
        cudaEventSynchronize(ev[2]);
        float t_auc = 0, t_tight = 0;
        cudaEventElapsedTime(&t_auc, ev[0], ev[1]);
        cudaEventElapsedTime(&t_tight, ev[1], ev[2]);
        int cnt[32];
        cudaMemcpy(cnt, aw.counters, 128, cudaMemcpyDeviceToHost);
        const unsigned long long *tns = reinterpret_cast<const unsigned long long *>(cnt + 16);
        const char *names[6] = {"cta/row", "4 warps/row", "2 warps/row", "warp/row", "2 rows/warp", "4 rows/warp"};
        for (int r = 0; r < 6; ++r)
            if (cnt[8 + r]) fprintf(stderr, "lap   bidding by %-12s %6d rounds %8.1f ms\n", names[r], cnt[8 + r], tns[r] * 1e-6);
        fprintf(stderr, "lap n=%d auction kernel %.1f ms (%d phases, %d rounds, %u bidder-row scans = %.1f GB), %d tighten "
                        "rounds + duals %.1f ms (tail %d, eps_min %.3g)\n", n, t_auc, cnt[5], cnt[1], (unsigned)cnt[4],
                (double)(unsigned)cnt[4] * n * sizeof(T) / 1e9, rounds, t_tight, a.tail, a.eps_min);
        for (auto &e : ev) cudaEventDestroy(e);
    }
    return 0;
}

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

template <class T, int CL>
bool try_cluster_sap(const T *M, int64_t ld, int n, double sign, const LapWork &w, cudaStream_t s) {
    const int W = (int)round_up(ceil_div(n, CL), 8);
    const size_t smem = (size_t)W * (8 + 8 + 8 + 4 + 4 + 1) + 16;
    if (smem > 200 * 1024) return false;
    auto fn = lap_cluster_sap_kernel<T, CL>;
    GOAT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (CL > 8) GOAT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(CL);
    cfg.blockDim = dim3(kLapClThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) != cudaSuccess || ncl < 1) {
        cudaGetLastError();
        return false;
    }
    GOAT_CUDA(cudaLaunchKernelEx(&cfg, fn, M, ld, n, sign, w, W));
    note_launch();
    return true;
}

template <class T>
void launch_lap_sap(const T *M, int64_t ld, int n, int sense, const LapWork &w, cudaStream_t s, int warm) {
    const size_t smem = (size_t)n * (8 + 8 + 4 + 4 + 4 + 1) + 16;
    const char *lce = getenv("GOAT_LAP_CLUSTER");  // 0: never, 2: always (tests), else when smem overflows
    const int lc = lce ? atoi(lce) : 1;
    if (warm && lc != 0 && (smem > 200 * 1024 || lc == 2)) {
        // warm repair too large for one CTA's shared memory: the cluster solver
        const double sign = (sense == GOAT_MAXIMIZE) ? -1.0 : 1.0;
        // GOAT_LAP_CL=8 prefers the 8-CTA cluster (measurement: config 5's repair 951 vs 734 ms
        // with 16 CTAs -- twice the columns per thread, each a dependent load per frontier row)
        const char *cle = getenv("GOAT_LAP_CL");
        const bool prefer8 = cle && atoi(cle) == 8;
        if ((prefer8 && try_cluster_sap<T, 8>(M, ld, n, sign, w, s)) || try_cluster_sap<T, 16>(M, ld, n, sign, w, s) ||
            try_cluster_sap<T, 8>(M, ld, n, sign, w, s)) {
            GOAT_CHECK_LAUNCH();
            return;
        }
    }
    // warm repair that fits one CTA: GOAT_LAP_LEVELS=1 runs the level-wise solver on a
    // cluster of one instead of the single-column solver below.  Off by default: without
    // exact ties a level is one column and costs two barriers more (c3 final LAP, n = 5000:
    // 35.6 vs 19.6 ms; c4, n = 2000: 27.0 vs 27.3 ms -- profiles/round2_lap_levels_one_cta.log).
    const char *lve = getenv("GOAT_LAP_LEVELS");
    if (warm && lve && atoi(lve) == 1) {
        const double sign1 = (sense == GOAT_MAXIMIZE) ? -1.0 : 1.0;
        if (try_cluster_sap<T, 1>(M, ld, n, sign1, w, s)) {
            GOAT_CHECK_LAUNCH();
            return;
        }
    }
    int use_smem = smem <= 200 * 1024;
    if (use_smem)
        GOAT_CUDA(cudaFuncSetAttribute(lap_sap_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const double sign = (sense == GOAT_MAXIMIZE) ? -1.0 : 1.0;
    lap_sap_kernel<T><<<1, kLapThreads, use_smem ? smem : 0, s>>>(M, ld, n, sign, w, use_smem, warm); note_launch();
    GOAT_CHECK_LAUNCH();
}

template int launch_lap_auction<float>(const float *, int64_t, int, int, double, const LapWork &, const AuctionWork &, int,
                                       cudaStream_t);
template int launch_lap_auction<double>(const double *, int64_t, int, int, double, const LapWork &,
                                        const AuctionWork &, int, cudaStream_t);
template void launch_lap_certificate<float>(const float *, int64_t, int, int, int *, int *, int *, cudaStream_t);
template void launch_lap_certificate<double>(const double *, int64_t, int, int, int *, int *, int *, cudaStream_t);
template void launch_lap_sap<float>(const float *, int64_t, int, int, const LapWork &, cudaStream_t, int);
template void launch_lap_sap<double>(const double *, int64_t, int, int, const LapWork &, cudaStream_t, int);

}  // namespace goat
