// tcgen05 / TMEM / TMA GEMM for the gradient products (matcher.py:107), sm_100a.
//
//   C[M x N] = alpha * sum_t  A_t[M x K] . B_t[N x K]^T        (fp32 accumulate in TMEM)
//
// Every operand is a bf16 "plane", K-major (row-major with K contiguous), loaded
// by TMA with 128-byte swizzle.  A sum over terms t is a K-concatenation: the
// producer streams (term, k-block) pairs into one accumulator.  That is how the
// fp32 iterate is carried exactly enough on bf16 tensor cores: X = X_hi + X_mid +
// X_lo (three bf16 planes, 24 mantissa bits) while 0/1 or integer adjacency is a
// single exact plane, so A X^T = sum_p A X_p^T.
//
// CTA tile 128 x 256 x 64, 4-stage smem ring (48 KB/stage), one elected thread
// issues tcgen05.mma (M=128, N=256, K=16) into a 256-column TMEM accumulator;
// TMA (warp 0) and MMA (warp 1) synchronise through mbarriers; tcgen05.commit
// releases smem stages.  Epilogue: 4 warps tcgen05.ld their 32 TMEM lanes and
// either store fp32 C or split C straight into the bf16 planes of the next GEMM.
#include <cuda.h>
#include <cuda_bf16.h>

#include <mutex>

#include "gemm_tc.cuh"

namespace goat {
namespace {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_BYTES = BN * BK * 2;  // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int kEpiWarps = 8;
constexpr int TC_THREADS = 64 + 32 * kEpiWarps;  // TMA, MMA, 8 epilogue warps
constexpr int TMEM_COLS = 512;                    // two 256-column chunk accumulators
constexpr size_t TC_SMEM = (size_t)STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// UMMA shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row atoms
// 1024 B apart (SBO), LBO unused (=1), descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// Instruction descriptor: kind::f16, A = B = BF16, D = F32, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Warp roles: warp 0 = TMA producer, warp 1 = MMA issuer (+ TMEM owner),
// warps 2..9 = promotion/epilogue.  The MMA accumulates `chunk` k-steps into one
// of two 256-column TMEM buffers; epilogue warp w drains TMEM lane group w%4,
// column half (w-2)/4, of each finished chunk into 128 fp32 registers with
// round-to-nearest adds while the MMA fills the other buffer.  This bounds the
// tensor core's truncating fp32 accumulation to `chunk` steps (promotion).
__global__ void __launch_bounds__(TC_THREADS, 1) tc_gemm_kernel(const __grid_constant__ TcGemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem;
    uint8_t *sB = smem + STAGES * A_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE_BYTES);
    uint64_t *empty = full + STAGES;
    uint64_t *cfull = empty + STAGES;  // [2] MMA -> epilogue: chunk accumulated
    uint64_t *cempty = cfull + 2;      // [2] epilogue -> MMA: chunk drained
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(cempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
        for (int b = 0; b < 2; ++b) { mbar_init(cfull + b, 1); mbar_init(cempty + b, kEpiWarps); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int t = 0; t < p.nterms; ++t) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.terms[t].a)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.terms[t].b)) : "memory");
        }
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    // split-K slice of this CTA: steps [i0, i0 + total) of the flattened (term, k-block) sequence
    const int i0 = blockIdx.z * p.kpb;
    const int total = max(0, min(p.nterms * p.kblocks, i0 + p.kpb) - i0);
    const int C = max(1, p.chunk);
    const int nchunks = (total + C - 1) / C;

    if (warp == 0) {
        if (lane == 0) {  // TMA producer
            for (int it = 0; it < total; ++it) {
                const int s = it % STAGES;
                if (it >= STAGES) mbar_wait(empty + s, ((it / STAGES) & 1) ^ 1);
                const int t = (i0 + it) / p.kblocks, kb = (i0 + it) % p.kblocks;
                mbar_expect_tx(full + s, STAGE_BYTES);
                tma_load_2d(sA + s * A_BYTES, &p.terms[t].a, kb * BK, p.terms[t].a_row0 + m0, full + s);
                tma_load_2d(sB + s * B_BYTES, &p.terms[t].b, kb * BK, p.terms[t].b_row0 + n0, full + s);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            constexpr uint32_t idesc = idesc_bf16(BM, BN);
            for (int it = 0; it < total; ++it) {
                const int c = it / C, b = c & 1;
                const bool first = (it % C) == 0;
                if (first && c >= 2) mbar_wait(cempty + b, ((c >> 1) - 1) & 1);
                const int s = it % STAGES;
                mbar_wait(full + s, (it / STAGES) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t a0 = smem_u32(sA + s * A_BYTES), b0 = smem_u32(sB + s * B_BYTES);
                const uint32_t d = tmem + (uint32_t)(b * BN);
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)  // 16 bf16 = 32 bytes along K inside the swizzle atom
                    umma_bf16(d, sdesc(a0 + 32 * k), sdesc(b0 + 32 * k), idesc, (!first || k > 0) ? 1u : 0u);
                umma_commit(empty + s);  // frees the stage once these MMAs have read it
                if ((it % C) == C - 1 || it == total - 1) umma_commit(cfull + b);
            }
        }
        __syncwarp();
    } else {
        // Promotion + epilogue
        const int lg = warp & 3, half = (warp - 2) >> 2;
        float acc[128];
#pragma unroll
        for (int j = 0; j < 128; ++j) acc[j] = 0.f;
        const uint32_t tbase = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(half * 128);
        for (int c = 0; c < nchunks; ++c) {
            const int b = c & 1;
            mbar_wait(cfull + b, (c >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                uint32_t r[16];
                tmem_ld16(tbase + (uint32_t)(b * BN + j * 16), r);
#pragma unroll
                for (int q = 0; q < 16; ++q) acc[j * 16 + q] += __uint_as_float(r[q]);
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(cempty + b);
        }
        const int row = m0 + lg * 32 + lane;
        if (row < p.M) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int col0 = n0 + half * 128 + j * 16;
                if (col0 >= p.N) continue;
                float v[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) v[q] = p.alpha * acc[j * 16 + q];
                const bool full16 = col0 + 16 <= p.N;
                if (p.mode == 0) {
                    float *dst = p.C + blockIdx.z * p.slice_stride + (int64_t)row * p.ldc + col0;
                    if (full16) {
#pragma unroll
                        for (int q = 0; q < 16; q += 4)
                            *reinterpret_cast<float4 *>(dst + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
                    } else {
                        for (int q = 0; q < 16 && col0 + q < p.N; ++q) dst[q] = v[q];
                    }
                } else {
                    // split fp32 -> bf16 planes: hi = rn(v), mid = rn(v - hi), lo = rn(v - hi - mid)
                    for (int pl = 0; pl < p.nplanes; ++pl) {
                        __nv_bfloat16 *dst = p.planes + pl * p.plane_stride + (int64_t)row * p.ldpl + col0;
                        uint32_t w[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const __nv_bfloat16 lo = __float2bfloat16_rn(v[2 * q]);
                            const __nv_bfloat16 hi = __float2bfloat16_rn(v[2 * q + 1]);
                            v[2 * q] -= __bfloat162float(lo);
                            v[2 * q + 1] -= __bfloat162float(hi);
                            w[q] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
                        }
                        if (full16) {
                            *reinterpret_cast<uint4 *>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
                            *reinterpret_cast<uint4 *>(dst + 8) = make_uint4(w[4], w[5], w[6], w[7]);
                        } else {
                            for (int q = 0; q < 16 && col0 + q < p.N; ++q)
                                dst[q] = __ushort_as_bfloat16((unsigned short)(w[q >> 1] >> (16 * (q & 1))));
                        }
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// Split-K reduction in a fixed slice order (round-to-nearest fp32 adds), then
// either fp32 out (scaled) or the bf16 plane split of the next GEMM's operand.
__global__ void slice_reduce_kernel(const float *S, int64_t slice_stride, int nslices, int rows, int cols,
                                    int64_t ld, float alpha, float *out, __nv_bfloat16 *planes,
                                    int64_t plane_stride, int nplanes) {
    for (int i = blockIdx.x; i < rows; i += gridDim.x)
        for (int j = threadIdx.x; j < ld; j += blockDim.x) {
            const int64_t o = (int64_t)i * ld + j;
            float v = 0.f;
            if (j < cols)
                for (int z = 0; z < nslices; ++z) v += S[z * slice_stride + o];
            v *= alpha;
            if (out) {
                if (j < cols) out[o] = v;
            } else {
                for (int pl = 0; pl < nplanes; ++pl) {
                    const __nv_bfloat16 b = __float2bfloat16_rn(v);
                    planes[pl * plane_stride + o] = b;
                    v -= __bfloat162float(b);
                }
            }
        }
}

// fp32 -> bf16 planes (same split as the epilogue) for a row-major n x n matrix.
__global__ void split_planes_kernel(const float *X, int64_t ldx, int rows, int cols, __nv_bfloat16 *planes,
                                    int64_t ldp, int64_t plane_stride, int nplanes) {
    for (int i = blockIdx.x; i < rows; i += gridDim.x)
        for (int j = threadIdx.x; j < ldp; j += blockDim.x) {
            float v = j < cols ? X[(int64_t)i * ldx + j] : 0.f;
            for (int pl = 0; pl < nplanes; ++pl) {
                const __nv_bfloat16 b = __float2bfloat16_rn(v);
                planes[pl * plane_stride + (int64_t)i * ldp + j] = b;
                v -= __bfloat162float(b);
            }
        }
}

// Transposed split: planes[j][i] from X[i][j] (bf16 planes of X^T), 32x32 smem tiles.
__global__ void split_planes_t_kernel(const float *X, int64_t ldx, int n, __nv_bfloat16 *planes, int64_t ldp,
                                      int64_t plane_stride, int nplanes) {
    __shared__ float tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int i = by + k, j = bx + threadIdx.x;
        tile[k][threadIdx.x] = (i < n && j < n) ? X[(int64_t)i * ldx + j] : 0.f;
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int j = bx + k, i = by + threadIdx.x;  // out[j][i] = X[i][j]
        if (j >= n || i >= ldp) continue;
        float v = tile[threadIdx.x][k];
        for (int pl = 0; pl < nplanes; ++pl) {
            const __nv_bfloat16 b = __float2bfloat16_rn(v);
            planes[pl * plane_stride + (int64_t)j * ldp + i] = b;
            v -= __bfloat162float(b);
        }
    }
}

// 1 if every entry is exactly representable in bf16 (so one plane is exact).
__global__ void bf16_exact_kernel(const float *X, int64_t ldx, int n, int rows, int *flag) {
    for (int i = blockIdx.x; i < rows; i += gridDim.x)
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            const float v = X[(int64_t)i * ldx + j];
            if (__bfloat162float(__float2bfloat16_rn(v)) != v) *flag = 0;
        }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw Error(GOAT_ECUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

}  // namespace

void tc_make_map(CUtensorMap *map, const void *base, int64_t rows, int64_t cols, int64_t ld_elems, int box_rows) {
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld_elems * 2)};
    cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(GOAT_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

int tc_box_rows_a() { return BM; }
int tc_box_rows_b() { return BN; }

void tc_gemm(const TcGemmParams &p, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        GOAT_CUDA(cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC_SMEM));
        attr = true;
    }
    if (p.nterms < 1 || p.nterms > kTcMaxTerms) throw Error(GOAT_EINVAL, "tc_gemm: bad term count");
    if (p.kslices < 1 || (p.kslices > 1 && p.mode != 0)) throw Error(GOAT_EINVAL, "tc_gemm: bad k-slicing");
    dim3 grid(ceil_div(p.N, BN), ceil_div(p.M, BM), p.kslices);
    tc_gemm_kernel<<<grid, TC_THREADS, TC_SMEM, s>>>(p);
    note_launch();
    GOAT_CHECK_LAUNCH();
}

void tc_slice_reduce(const float *S, int64_t slice_stride, int nslices, int rows, int cols, int64_t ld, float alpha,
                     float *out, __nv_bfloat16 *planes, int64_t plane_stride, int nplanes, cudaStream_t s) {
    slice_reduce_kernel<<<std::min(rows, 4096), 256, 0, s>>>(S, slice_stride, nslices, rows, cols, ld, alpha, out,
                                                              planes, plane_stride, nplanes);
    note_launch();
    GOAT_CHECK_LAUNCH();
}

int tc_block_m() { return BM; }
int tc_block_n() { return BN; }
int tc_block_k() { return BK; }

void tc_split_planes(const float *X, int64_t ldx, int rows, int cols, __nv_bfloat16 *planes, int64_t ldp,
                     int64_t plane_stride, int nplanes, cudaStream_t s) {
    split_planes_kernel<<<std::min(rows, 4096), 256, 0, s>>>(X, ldx, rows, cols, planes, ldp, plane_stride, nplanes);
    note_launch();
    GOAT_CHECK_LAUNCH();
}

void tc_split_planes_t(const float *X, int64_t ldx, int n, __nv_bfloat16 *planes, int64_t ldp, int64_t plane_stride,
                       int nplanes, cudaStream_t s) {
    dim3 grid(ceil_div(n, 32), ceil_div(n, 32));
    split_planes_t_kernel<<<grid, dim3(32, 8), 0, s>>>(X, ldx, n, planes, ldp, plane_stride, nplanes);
    note_launch();
    GOAT_CHECK_LAUNCH();
}

bool tc_bf16_exact(const float *X, int64_t ldx, int n, int *dflag, cudaStream_t s, int rows) {
    const int one = 1;
    if (rows < 0) rows = n;
    GOAT_CUDA(cudaMemcpyAsync(dflag, &one, sizeof(int), cudaMemcpyHostToDevice, s));
    bf16_exact_kernel<<<std::max(1, std::min(rows, 2048)), 256, 0, s>>>(X, ldx, n, rows, dflag);
    note_launch();
    int r = 0;
    GOAT_CUDA(cudaMemcpyAsync(&r, dflag, sizeof(int), cudaMemcpyDeviceToHost, s));
    GOAT_CUDA(cudaStreamSynchronize(s));
    return r != 0;
}

}  // namespace goat
