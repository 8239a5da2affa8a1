// Microbenchmark: HBM read bandwidth of the LOT access pattern (persistent CTAs,
// row-cyclic, each thread CH 16-byte chunks per row), with increasing per-row work.
#include <cstdio>
#include <cuda_runtime.h>
template <int NT, int CH, int MODE>
__global__ void __launch_bounds__(NT, 1) rowbw(const float *G, int n, int ld, float *out) {
    __shared__ float sm[NT / 32];
    float acc = 0.f, tot = 0.f;
    float4 xv[CH];
    auto load = [&](int row) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            int col = (threadIdx.x + NT * c) * 4;
            xv[c] = (row < n && col < n) ? __ldg(reinterpret_cast<const float4 *>(G + (size_t)row * ld + col)) : make_float4(0, 0, 0, 0);
        }
    };
    load(blockIdx.x);
    for (int row = blockIdx.x; row < n; row += gridDim.x) {
        float4 x[CH];
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = xv[c];
        load(row + gridDim.x);
        float s = 0.f;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (MODE == 0) s += x[c].x + x[c].y + x[c].z + x[c].w;
            else s += exp2f(x[c].x) + exp2f(x[c].y) + exp2f(x[c].z) + exp2f(x[c].w);
        }
        if (MODE >= 2) {  // per-row block reduction
            for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
            __syncthreads();
            float b = 0.f;
            if ((threadIdx.x & 31) < NT / 32) b = sm[threadIdx.x & 31];
            for (int off = 16; off; off >>= 1) b += __shfl_xor_sync(0xffffffffu, b, off);
            s = b;
            if (MODE == 3) __syncthreads();
        }
        acc += s;
        tot += acc * 1e-30f;
    }
    out[blockIdx.x * NT + threadIdx.x] = tot;
}
template <int NT, int CH, int MODE> void run(const float *G, int n, float *o, const char *name, int occ) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    rowbw<NT, CH, MODE><<<148 * occ, NT>>>(G, n, n, o);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) rowbw<NT, CH, MODE><<<148 * occ, NT>>>(G, n, n, o);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    printf("%-28s n=%d NT=%d CH=%d occ=%d: %.3f ms  %.0f GB/s (%s)\n", name, n, NT, CH, occ, ms, (double)n * n * 4 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    int n = 20000;  // 1.6 GB, CH = 20000/4/512 ~ 10 -> use 1024 threads CH=5
    float *G, *o; cudaMalloc(&G, (size_t)n * n * 4); cudaMalloc(&o, 1 << 24); cudaMemset(G, 0, (size_t)n * n * 4);
    run<1024, 5, 0>(G, n, o, "load+sum", 1);
    run<1024, 5, 1>(G, n, o, "load+exp2", 1);
    run<1024, 5, 2>(G, n, o, "load+exp2+blockreduce", 1);
    run<1024, 5, 3>(G, n, o, "load+exp2+blockreduce+2sync", 1);
    n = 10000;
    run<512, 5, 0>(G, n, o, "load+sum", 1);
    run<512, 5, 1>(G, n, o, "load+exp2", 1);
    run<512, 5, 2>(G, n, o, "load+exp2+blockreduce", 1);
    run<256, 5, 2>(G, 5000, o, "load+exp2+blockreduce", 2);
    run<512, 5, 2>(G, n, o, "load+exp2+blockreduce x2occ", 2);
}
