// Sparse (CSR) adjacency for the GOAT gradient on B200.
//
// Reference: gradient(A, B, P) = A P B^T + A^T P B (matcher.py:100-107) with
// dense float64 operands.  For sparse graphs (BASELINE config 5: n = 40000,
// p = 0.01, ~1.6e7 nonzeros per graph) the products are row-gather SpMMs:
//   step 1  X^T = (A Q)^T                 (and (A^T Q)^T when directed)
//   step 2  G   = (B X^T [+ B^T X2^T])^T   = A Q B^T + A^T Q B
// Every SpMM is   out = alpha * (sum_t S_t D_t)^T,  S_t CSR, D_t dense n x ld:
// a CTA computes a 32-row x 256-column tile of sum_t S_t D_t with one warp per
// 4 rows (a lane owns 8 consecutive columns; the nonzeros of a row are fetched
// 32 at a time and broadcast by shuffles; 4 row gathers are kept in flight),
// then writes the tile transposed through shared memory (coalesced 32-element
// segments).  Tiles are ordered column-block-major so the gathered slice
// D[:, j0:j0+256] (n x 1 KB fp32) stays L2-resident while every row tile of
// that block runs.  Accumulation is fp32/fp64 FMA in CSR order: deterministic.
//
// Also here: CSR canonical checks, transposes (CUB radix sort on (col, row)
// keys), symmetry, degree vectors for the barycenter gradient, and the
// integer-exact objective sum_{(i,j) in A} A_ij B_{p(i) p(j)} (core.py:120-124).
#include <cub/device/device_radix_sort.cuh>

#include "kernels.cuh"

namespace goat {
namespace {

constexpr int kSpRows = 32;     // rows of a tile
constexpr int kSpCols = 256;    // columns of a tile (8 per lane)
constexpr int kSpThreads = 256; // 8 warps x 4 rows

template <class T> struct SpVec;
template <> struct SpVec<float> { using V = float4; static constexpr int W = 4; };
template <> struct SpVec<double> { using V = double2; static constexpr int W = 2; };

template <class T, int NTERMS>
struct SpmmArgs {
    int rows;       // rows of every S_t (= columns of out)
    int cols;       // columns of every D_t (= rows of out)
    int64_t ld;     // leading dimension of D_t
    int64_t ldo;    // leading dimension of out
    const int64_t *rowptr[2];
    const int *col[2];
    const T *val[2];
    const T *D[2];
    T *out;
    double alpha;
    int nrt;  // row tiles
};

template <class T>
__device__ __forceinline__ void gather_add(T (&acc)[8], const T *drow, int jl, T v) {
    using V = typename SpVec<T>::V;
    constexpr int W = SpVec<T>::W;
#pragma unroll
    for (int u = 0; u < 8 / W; ++u) {
        const V d = __ldg(reinterpret_cast<const V *>(drow + jl) + u);
        const T *pd = reinterpret_cast<const T *>(&d);
#pragma unroll
        for (int e = 0; e < W; ++e) acc[u * W + e] = fma(v, pd[e], acc[u * W + e]);
    }
}

template <class T, int NTERMS>
__global__ void __launch_bounds__(kSpThreads) spmm_t_kernel(SpmmArgs<T, NTERMS> p) {
    extern __shared__ __align__(16) unsigned char sp_smem[];
    T *tile = reinterpret_cast<T *>(sp_smem);  // [kSpCols][kSpRows + 1]
    const int cb = blockIdx.x / p.nrt, rt = blockIdx.x % p.nrt;
    const int i0 = rt * kSpRows, j0 = cb * kSpCols;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int jl = j0 + lane * 8;
    const bool jok = jl < p.cols;  // ld >= round_up(cols, 8): a started 8-chunk is in bounds
#pragma unroll 1
    for (int r = 0; r < 4; ++r) {
        const int li = warp * 4 + r;
        const int i = i0 + li;
        T acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = T(0);
        if (i < p.rows) {
#pragma unroll
            for (int t = 0; t < NTERMS; ++t) {
                const int64_t q0 = p.rowptr[t][i], q1 = p.rowptr[t][i + 1];
                const T *D = p.D[t];
                for (int64_t qb = q0; qb < q1; qb += 32) {
                    const int cnt = (int)min((int64_t)32, q1 - qb);
                    const int myc = lane < cnt ? __ldg(p.col[t] + qb + lane) : 0;
                    const T myv = lane < cnt ? (p.val[t] ? __ldg(p.val[t] + qb + lane) : T(1)) : T(0);
                    int q = 0;
                    for (; q + 4 <= cnt; q += 4) {
                        int c[4];
                        T v[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            c[u] = __shfl_sync(0xffffffffu, myc, q + u);
                            v[u] = __shfl_sync(0xffffffffu, myv, q + u);
                        }
                        if (jok) {
#pragma unroll
                            for (int u = 0; u < 4; ++u) gather_add<T>(acc, D + (int64_t)c[u] * p.ld, jl, v[u]);
                        }
                    }
                    for (; q < cnt; ++q) {
                        const int c = __shfl_sync(0xffffffffu, myc, q);
                        const T v = __shfl_sync(0xffffffffu, myv, q);
                        if (jok) gather_add<T>(acc, D + (int64_t)c * p.ld, jl, v);
                    }
                }
            }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) tile[(lane * 8 + e) * (kSpRows + 1) + li] = acc[e];
    }
    __syncthreads();
    // transposed store: out[j][i0 .. i0+32)
    const T alpha = (T)p.alpha;
    for (int c = warp; c < kSpCols; c += kSpThreads / 32) {
        const int j = j0 + c;
        const int i = i0 + lane;
        if (j < p.cols && i < p.rows) p.out[(int64_t)j * p.ldo + i] = alpha * tile[c * (kSpRows + 1) + lane];
    }
}

// ---------------------------------------------------------------- CSR utilities
// flag[0] <- 0 if some row is not strictly increasing or a column is out of range
__global__ void csr_check_kernel(const int64_t *rowptr, const int *col, int rows, int n, int64_t nnz, int *flag) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && (rowptr[0] != 0 || rowptr[rows] != nnz)) *flag = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) {
        const int64_t a = rowptr[i], b = rowptr[i + 1];
        if (a > b || a < 0 || b > nnz) { *flag = 0; continue; }
        int prev = -1;
        for (int64_t q = a; q < b; ++q) {
            const int c = col[q];
            if (c <= prev || c >= n) { *flag = 0; break; }
            prev = c;
        }
    }
}

template <class T> __global__ void finite_kernel(const T *v, int64_t nnz, int *flag) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite((double)v[q])) *flag = 0;
}

// keys[q] = col * n + row, idx[q] = q
__global__ void csr_keys_kernel(const int64_t *rowptr, const int *col, int n, int64_t *keys, int *idx) {
    for (int i = blockIdx.x; i < n; i += gridDim.x)
        for (int64_t q = rowptr[i] + threadIdx.x; q < rowptr[i + 1]; q += blockDim.x) {
            keys[q] = (int64_t)col[q] * n + i;
            idx[q] = (int)q;
        }
}

template <class T>
__global__ void csr_from_keys_kernel(const int64_t *keys, const int *idx, const T *val, int n, int64_t nnz,
                                     int *colT, T *valT) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x) {
        colT[q] = (int)(keys[q] % n);
        if (val) valT[q] = val[idx[q]];
    }
}

// rowptrT[c] = first q with keys[q] >= c * n
__global__ void csr_rowptr_kernel(const int64_t *keys, int64_t nnz, int n, int64_t *rowptrT) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c <= n; c += gridDim.x * blockDim.x) {
        const int64_t key = (int64_t)c * n;
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        rowptrT[c] = lo;
    }
}

template <class T>
__global__ void csr_equal_kernel(const int64_t *ra, const int *ca, const T *va, const int64_t *rb, const int *cb,
                                 const T *vb, int n, int64_t nnz, int *flag) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, str = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i <= n; i += str)
        if (ra[i] != rb[i]) *flag = 0;
    for (int64_t q = tid; q < nnz; q += str) {
        if (ca[q] != cb[q]) *flag = 0;
        if (va && vb && va[q] != vb[q]) *flag = 0;
    }
}

// rs[i] = sum of row i (fp64, CSR order)
template <class T> __global__ void csr_rowsum_kernel(const int64_t *rowptr, const T *val, int n, double *rs) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double s = 0.0;
        const int64_t a = rowptr[i], b = rowptr[i + 1];
        if (val) for (int64_t q = a; q < b; ++q) s += (double)val[q];
        else s = (double)(b - a);
        rs[i] = s;
    }
}

// part[row] = sum_{q in row i of A} a_q * B[p(i), p(col_q)]  (fp64, CSR order); a warp per row
template <class T>
__global__ void csr_qap_rows_kernel(const int64_t *ra, const int *ca, const T *va, const int64_t *rb, const int *cb,
                                    const T *vb, const int *perm, int n, double *rowsum) {
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int i = w; i < n; i += nw) {
        const int pi = perm[i];
        const int64_t b0 = rb[pi], b1 = rb[pi + 1];
        double s = 0.0;
        for (int64_t q = ra[i] + lane; q < ra[i + 1]; q += 32) {
            const int pj = perm[ca[q]];
            int64_t lo = b0, hi = b1;  // binary search pj in row pi of B
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (cb[mid] < pj) lo = mid + 1;
                else hi = mid;
            }
            if (lo < b1 && cb[lo] == pj)
                s += (va ? (double)va[q] : 1.0) * (vb ? (double)vb[lo] : 1.0);
        }
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) rowsum[i] = s;
    }
}

// one block: fixed-order sum of v[0..n) -> out
__global__ void fixed_sum_kernel(const double *v, int n, double *out) {
    __shared__ double s[kThreads];
    double t = 0.0;
    for (int i = threadIdx.x; i < n; i += kThreads) t += v[i];
    s[threadIdx.x] = t;
    __syncthreads();
    for (int st = kThreads / 2; st > 0; st >>= 1) {
        if ((int)threadIdx.x < st) s[threadIdx.x] += s[threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = s[0];
}

}  // namespace

template <class T>
void launch_spmm_t(int rows, int cols, int64_t ld, int64_t ldo, int nterms, const DevCsr<T> *S, const T *const *D,
                   double alpha, T *out, cudaStream_t s) {
    require(nterms == 1 || nterms == 2, "spmm: 1 or 2 terms");
    require(ld >= round_up(cols, 8) && ldo >= rows, "spmm: leading dimension");
    const int nrt = ceil_div(rows, kSpRows), ncb = ceil_div(cols, kSpCols);
    const size_t smem = (size_t)kSpCols * (kSpRows + 1) * sizeof(T);
    const int64_t grid = (int64_t)nrt * ncb;
    require(grid < (1ll << 31), "spmm: order too large");
    auto fill = [&](auto &p) {
        p.rows = rows; p.cols = cols; p.ld = ld; p.ldo = ldo; p.out = out; p.alpha = alpha; p.nrt = nrt;
        for (int t = 0; t < nterms; ++t) {
            p.rowptr[t] = S[t].rowptr; p.col[t] = S[t].col; p.val[t] = S[t].val; p.D[t] = D[t];
        }
    };
    if (nterms == 1) {
        SpmmArgs<T, 1> p{};
        fill(p);
        GOAT_CUDA(cudaFuncSetAttribute(spmm_t_kernel<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        spmm_t_kernel<T, 1><<<(unsigned)grid, kSpThreads, smem, s>>>(p);
    } else {
        SpmmArgs<T, 2> p{};
        fill(p);
        GOAT_CUDA(cudaFuncSetAttribute(spmm_t_kernel<T, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        spmm_t_kernel<T, 2><<<(unsigned)grid, kSpThreads, smem, s>>>(p);
    }
    note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T> void launch_csr_check(const DevCsr<T> &a, int rows, int n, int *flag, cudaStream_t s) {
    csr_check_kernel<<<std::max(1, std::min(ceil_div(rows, kThreads), 1184)), kThreads, 0, s>>>(a.rowptr, a.col, rows,
                                                                                                 n, a.nnz, flag);
    note_launch();
    if (a.val && a.nnz) {
        finite_kernel<T><<<1184, kThreads, 0, s>>>(a.val, a.nnz, flag);
        note_launch();
    }
    GOAT_CHECK_LAUNCH();
}

size_t csr_transpose_scratch(int64_t nnz) {
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const int64_t *)nullptr, (int64_t *)nullptr,
                                    (const int *)nullptr, (int *)nullptr, (int64_t)std::max<int64_t>(nnz, 1));
    return round_up(tmp, 256) + (size_t)std::max<int64_t>(nnz, 1) * (2 * 8 + 2 * 4) + 1024;
}

template <class T>
void launch_csr_transpose(const DevCsr<T> &a, int n, int64_t *rowptrT, int *colT, T *valT, void *scratch,
                          size_t scratch_bytes, cudaStream_t s) {
    const int64_t nnz = a.nnz;
    if (nnz == 0) {
        GOAT_CUDA(cudaMemsetAsync(rowptrT, 0, (size_t)(n + 1) * 8, s));
        return;
    }
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const int64_t *)nullptr, (int64_t *)nullptr, (const int *)nullptr,
                                    (int *)nullptr, nnz);
    char *base = static_cast<char *>(scratch);
    char *sort_tmp = base;
    int64_t *k0 = reinterpret_cast<int64_t *>(base + round_up(tmp, 256));
    int64_t *k1 = k0 + nnz;
    int *i0 = reinterpret_cast<int *>(k1 + nnz);
    int *i1 = i0 + nnz;
    require((size_t)(reinterpret_cast<char *>(i1 + nnz) - base) <= scratch_bytes, "csr transpose: scratch too small");
    csr_keys_kernel<<<std::min(n, 4096), 128, 0, s>>>(a.rowptr, a.col, n, k0, i0);
    note_launch();
    int bits = 1;
    while (bits < 63 && ((int64_t)1 << bits) < (int64_t)n * n) ++bits;
    GOAT_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp, tmp, k0, k1, i0, i1, nnz, 0, bits, s));
    note_launch();
    csr_from_keys_kernel<T><<<1184, kThreads, 0, s>>>(k1, i1, a.val, n, nnz, colT, valT);
    csr_rowptr_kernel<<<std::max(1, std::min(ceil_div(n + 1, kThreads), 1184)), kThreads, 0, s>>>(k1, nnz, n, rowptrT);
    note_launch(2);
    GOAT_CHECK_LAUNCH();
}

template <class T> void launch_csr_equal(const DevCsr<T> &a, const DevCsr<T> &b, int n, int *flag, cudaStream_t s) {
    if (a.nnz != b.nnz) {
        const int zero = 0;
        GOAT_CUDA(cudaMemcpyAsync(flag, &zero, sizeof(int), cudaMemcpyHostToDevice, s));
        return;
    }
    csr_equal_kernel<T><<<1184, kThreads, 0, s>>>(a.rowptr, a.col, a.val, b.rowptr, b.col, b.val, n, a.nnz, flag);
    note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T> void launch_csr_rowsum(const DevCsr<T> &a, int n, double *rs, cudaStream_t s) {
    csr_rowsum_kernel<T><<<std::max(1, std::min(ceil_div(n, kThreads), 1184)), kThreads, 0, s>>>(a.rowptr, a.val, n, rs);
    note_launch();
    GOAT_CHECK_LAUNCH();
}

template <class T>
void launch_csr_qap_perm(const DevCsr<T> &a, const DevCsr<T> &b, const int *perm, int n, double *rowsum, double *out,
                         cudaStream_t s) {
    csr_qap_rows_kernel<T><<<std::max(1, std::min(ceil_div(n, 8), 4736)), kThreads, 0, s>>>(
        a.rowptr, a.col, a.val, b.rowptr, b.col, b.val, perm, n, rowsum);
    fixed_sum_kernel<<<1, kThreads, 0, s>>>(rowsum, n, out);
    note_launch(2);
    GOAT_CHECK_LAUNCH();
}

#define GOAT_SP_INST(T)                                                                                          \
    template void launch_spmm_t<T>(int, int, int64_t, int64_t, int, const DevCsr<T> *, const T *const *, double, \
                                   T *, cudaStream_t);                                                           \
    template void launch_csr_check<T>(const DevCsr<T> &, int, int, int *, cudaStream_t);                         \
    template void launch_csr_transpose<T>(const DevCsr<T> &, int, int64_t *, int *, T *, void *, size_t,        \
                                          cudaStream_t);                                                         \
    template void launch_csr_equal<T>(const DevCsr<T> &, const DevCsr<T> &, int, int *, cudaStream_t);          \
    template void launch_csr_rowsum<T>(const DevCsr<T> &, int, double *, cudaStream_t);                          \
    template void launch_csr_qap_perm<T>(const DevCsr<T> &, const DevCsr<T> &, const int *, int, double *,      \
                                         double *, cudaStream_t);
GOAT_SP_INST(float)
GOAT_SP_INST(double)
#undef GOAT_SP_INST

}  // namespace goat
