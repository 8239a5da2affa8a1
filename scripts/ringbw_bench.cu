// Microbenchmark: HBM read rate of the wide-row LOT streaming pattern without the
// Sinkhorn arithmetic.  Persistent grid (one CTA per SM), each CTA streams its
// rows (row-cyclic) through a ring of S shared-memory stages filled by
// cp.async.bulk (SPLIT copies per stage), every warp reads its 16-byte chunks
// and releases the stage on an empty mbarrier.  MODE 1 = register double
// buffering with plain 16-byte loads (no ring), for comparison.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ringbw scripts/ringbw_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t *b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void marrive(uint64_t *b) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mexpect(uint64_t *b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t *b, uint32_t par) {
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}

template <int NT, int CH, int WORK>
__global__ void __launch_bounds__(NT, 1) ring_kernel(const float *G, int rows, int64_t ld, int width, int S, int split, float *out) {
    extern __shared__ __align__(128) char ring[];
    __shared__ uint64_t full[8], empty[8], wbar[4], xbar[4];
    constexpr int NW = NT / 32;
    __shared__ float wp[4][NW][2], xp[4][2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float yp[CH][4];
    float mp = 0.f;
    const int nrows = (rows - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const uint32_t bytes = (uint32_t)width * 4;
    const int stage = (int)((bytes + 127) / 128 * 128);
    if (tid == 0) {
        for (int s = 0; s < S; ++s) { minit(&full[s], 1); minit(&empty[s], NW); }
        for (int s = 0; s < 4; ++s) { minit(&wbar[s], NW); minit(&xbar[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned issued = 0;
    auto produce = [&](unsigned upto) {
        while (issued < upto && issued < (unsigned)nrows) {
            const unsigned u = issued;
            const int s = u % S;
            if (u >= (unsigned)S) mwait(&empty[s], ((u / S) - 1) & 1);
            const float *src = G + (int64_t)(blockIdx.x + u * gridDim.x) * ld;
            mexpect(&full[s], bytes);
            const uint32_t part = (bytes / split + 15) / 16 * 16;
            for (uint32_t o = 0; o < bytes; o += part) bulk(ring + (size_t)s * stage + o, reinterpret_cast<const char *>(src) + o, min(part, bytes - o), &full[s]);
            ++issued;
        }
    };
    float acc = 0.f;
    float ac[CH][4], gl[CH][4];
    for (int c = 0; c < CH; ++c) for (int e = 0; e < 4; ++e) { ac[c][e] = 0.f; gl[c][e] = 0.01f * (c + e); }
    for (int it = 0; it < nrows; ++it) {
        if (tid == 0) produce(it + S - 1);
        const int s = it % S;
        mwait(&full[s], (it / S) & 1);
        const float4 *st = reinterpret_cast<const float4 *>(ring + (size_t)s * stage);
        if (WORK == 0) {
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int q = tid + NT * c;
                if (q * 4 < width) { float4 v = st[q]; acc += (v.x + v.y) + (v.z + v.w); }
            }
            __syncwarp();
            if (lane == 0) marrive(&empty[s]);
        } else if (WORK >= 4) {
            // coupled: per-warp pairs -> rotating combiner (next iteration) -> finish with lag 1
            const unsigned b = it;
            if (WORK == 4 && it >= 1 && warp == (int)((b - 1) % NW)) {
                const int xs = (b - 1) & 3;
                if (lane == 0) mwait(&wbar[xs], ((b - 1) >> 2) & 1);
                __syncwarp();
                const float mv = lane < NW ? wp[xs][lane][0] : -INFINITY;
                float M = mv;
                for (int off = 16; off; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
                float Sm = mv != -INFINITY ? wp[xs][lane][1] * exp2f(mv - M) : 0.f;
                for (int off = 16; off; off >>= 1) Sm += __shfl_xor_sync(0xffffffffu, Sm, off);
                if (lane == 0) { xp[xs][0] = M; xp[xs][1] = Sm; marrive(&xbar[xs]); }
            }
            float x[CH][4];
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int q = tid + NT * c;
                float4 v = q * 4 < width ? st[q] : make_float4(0, 0, 0, 0);
                x[c][0] = v.x; x[c][1] = v.y; x[c][2] = v.z; x[c][3] = v.w;
            }
            __syncwarp();
            if (lane == 0) marrive(&empty[s]);
            float m = -INFINITY;
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int e = 0; e < 4; ++e) { x[c][e] = -1.44f * (100.f - x[c][e]) + gl[c][e]; if (WORK != 6) m = fmaxf(m, x[c][e]); }
            if (WORK != 6) { for (int off = 16; off; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off)); } else m = -60.f;
            float spv[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int e = 0; e < 4; ++e) { x[c][e] = exp2f(x[c][e] - m); spv[e] += x[c][e]; }
            float sp = (spv[0] + spv[1]) + (spv[2] + spv[3]);
            for (int off = 16; off; off >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, off);
            if (WORK == 4) {
                if (lane == 0) { wp[b & 3][warp][0] = m; wp[b & 3][warp][1] = sp; marrive(&wbar[b & 3]); }
                if (it >= 1) {
                    const int xs = (b - 1) & 3;
                    float M, Sm;
                    if (lane == 0) { mwait(&xbar[xs], ((b - 1) >> 2) & 1); M = xp[xs][0]; Sm = xp[xs][1]; }
                    M = __shfl_sync(0xffffffffu, M, 0);
                    Sm = __shfl_sync(0xffffffffu, Sm, 0);
                    const float sc = exp2f(mp - M) / Sm;
#pragma unroll
                    for (int c = 0; c < CH; ++c)
#pragma unroll
                        for (int e = 0; e < 4; ++e) ac[c][e] += yp[c][e] * sc;
                }
            } else {  // lock-step: block combine right away
                if (lane == 0) { wp[b & 1][warp][0] = m; wp[b & 1][warp][1] = sp; }
                __syncthreads();
                float M, Sm;
                if (WORK == 6) {
                    Sm = lane < NW ? wp[b & 1][lane][1] : 0.f;
                    for (int off = 16; off; off >>= 1) Sm += __shfl_xor_sync(0xffffffffu, Sm, off);
                    M = m;
                } else {
                    const float mv = lane < NW ? wp[b & 1][lane][0] : -INFINITY;
                    M = mv;
                    for (int off = 16; off; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
                    Sm = mv != -INFINITY ? wp[b & 1][lane][1] * exp2f(mv - M) : 0.f;
                    for (int off = 16; off; off >>= 1) Sm += __shfl_xor_sync(0xffffffffu, Sm, off);
                }
                const float sc = exp2f(m - M) / Sm;
#pragma unroll
                for (int c = 0; c < CH; ++c)
#pragma unroll
                    for (int e = 0; e < 4; ++e) ac[c][e] += x[c][e] * sc;
            }
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int e = 0; e < 4; ++e) yp[c][e] = x[c][e];
            mp = m;
        } else {
            float x[CH][4];
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int q = tid + NT * c;
                float4 v = q * 4 < width ? st[q] : make_float4(0, 0, 0, 0);
                x[c][0] = v.x; x[c][1] = v.y; x[c][2] = v.z; x[c][3] = v.w;
            }
            __syncwarp();
            if (lane == 0) marrive(&empty[s]);
            float m = -INFINITY;
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int e = 0; e < 4; ++e) { x[c][e] = -1.44f * (100.f - x[c][e]) + gl[c][e]; if (WORK != 3) m = fmaxf(m, x[c][e]); }
            if (WORK != 3) for (int off = 16; off; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
            else m = -50.f;
            float spv[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int e = 0; e < 4; ++e) { x[c][e] = exp2f(x[c][e] - m); spv[e] += x[c][e]; }
            float sp = (spv[0] + spv[1]) + (spv[2] + spv[3]);
            for (int off = 16; off; off >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, off);
            const float sc = WORK == 2 ? __frcp_rn(sp) : 1.0f / sp;
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int e = 0; e < 4; ++e) ac[c][e] += x[c][e] * sc;
        }
    }
    for (int c = 0; c < CH; ++c) for (int e = 0; e < 4; ++e) acc += ac[c][e];
    if (acc == 1234.5f) out[tid] = acc;
}

template <int NT, int CH>
__global__ void __launch_bounds__(NT, 1) reg_kernel(const float *G, int rows, int64_t ld, int width, float *out) {
    float4 xv[CH];
    auto load = [&](int row) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int col = (threadIdx.x + NT * c) * 4;
            xv[c] = (row < rows && col < width) ? __ldg(reinterpret_cast<const float4 *>(G + (int64_t)row * ld + col)) : make_float4(0, 0, 0, 0);
        }
    };
    float acc = 0.f;
    load(blockIdx.x);
    for (int row = blockIdx.x; row < rows; row += gridDim.x) {
        float4 x[CH];
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = xv[c];
        load(row + gridDim.x);
#pragma unroll
        for (int c = 0; c < CH; ++c) acc += (x[c].x + x[c].y) + (x[c].z + x[c].w);
    }
    if (acc == 1234.5f) out[threadIdx.x] = acc;
}

int main() {
    const int n = 40000;
    const int64_t ld = 40000;
    float *G, *out;
    cudaMalloc(&G, (size_t)n * ld * 4);
    cudaMalloc(&out, 4096);
    {
        float *h = (float *)malloc((size_t)ld * 4 * 64);
        for (int64_t i = 0; i < ld * 64; ++i) h[i] = (float)((i * 2654435761u) % 100000) * 1e-3f;
        for (int r = 0; r < n; r += 64) cudaMemcpy(G + (size_t)r * ld, h, (size_t)ld * 4 * 64, cudaMemcpyHostToDevice);
        free(h);
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto run_ring = [&](int width, int S, int split, int grid_mult, int work = 0, int nt = 512) {
        // rows of `width` floats: the matrix viewed as (n*ld/width) rows
        const int rows = (int)((int64_t)n * ld / width);
        const size_t smem = (size_t)S * ((width * 4 + 127) / 128 * 128);
        auto k = nt == 256 ? (work == 5 ? ring_kernel<256, 5, 5> : ring_kernel<256, 5, 6>) : work == 0 ? ring_kernel<512, 5, 0> : work == 1 ? ring_kernel<512, 5, 1> : work == 3 ? ring_kernel<512, 5, 3> : work == 4 ? ring_kernel<512, 5, 4> : work == 5 ? ring_kernel<512, 5, 5> : ring_kernel<512, 5, 6>;
        if (width > 10240) { printf("width too large\n"); return; }
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int grid = sms * grid_mult;
        for (int w = 0; w < 2; ++w) k<<<grid, nt, smem>>>(G, rows, width, width, S, split, out);
        cudaEventRecord(e0);
        const int reps = 5;
        for (int r = 0; r < reps; ++r) k<<<grid, nt, smem>>>(G, rows, width, width, S, split, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        printf("ring work=%d width=%5d (%5.1f KB) S=%d split=%d grid=%d: %.1f GB/s %s\n", work, width, width * 4 / 1024.0, S, split, grid,
               (double)rows * width * 4 * reps / (ms * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
    };
    auto run_reg = [&](int width) {
        const int rows = (int)((int64_t)n * ld / width);
        auto k = reg_kernel<512, 5>;
        for (int w = 0; w < 2; ++w) k<<<sms, 512>>>(G, rows, width, width, out);
        cudaEventRecord(e0);
        const int reps = 5;
        for (int r = 0; r < reps; ++r) k<<<sms, 512>>>(G, rows, width, width, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("reg  width=%5d (%5.1f KB): %.1f GB/s\n", width, width * 4 / 1024.0, (double)rows * width * 4 * reps / (ms * 1e-3) / 1e9);
    };
    run_ring(10000, 4, 1, 1);
    run_ring(10000, 4, 1, 1, 1);
    run_ring(10000, 4, 1, 1, 3);
    run_ring(10000, 4, 1, 1, 4);
    run_ring(10000, 4, 1, 1, 5);
    run_ring(10000, 4, 1, 1, 6);
    run_ring(5000, 4, 1, 2, 5, 256);
    run_ring(5000, 4, 1, 2, 6, 256);
    run_ring(5000, 5, 1, 2, 5, 256);
    run_reg(10000);
    run_reg(5000);
    return 0;
}
