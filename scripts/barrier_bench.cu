// Microbenchmark: software grid barrier variants used by the persistent LOT kernel.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void red_release(unsigned *p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
// (a) generation barrier with __threadfence (current)
__device__ __forceinline__ void bar_a(unsigned *bar, unsigned nb, unsigned) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned *cnt = bar, *gen = bar + 32;
        const unsigned g = ld_acquire(gen);
        __threadfence();
        if (atomicAdd(cnt, 1u) == nb - 1) { atomicExch(cnt, 0u); __threadfence(); atomicAdd(gen, 1u); }
        else { while (ld_acquire(gen) == g) { } }
    }
    __syncthreads();
}
// (b) monotone counter: red.release arrival, ld.acquire poll until epoch*nb
__device__ __forceinline__ void bar_b(unsigned *bar, unsigned nb, unsigned epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        red_release(bar, 1u);
        const unsigned target = epoch * nb;
        while (ld_acquire(bar) < target) { }
    }
    __syncthreads();
}
template <int V> __global__ void bar_kernel(unsigned *bar, int iters) {
    for (int i = 0; i < iters; ++i) {
        if (V == 0) bar_a(bar, gridDim.x, i + 1);
        else if (V == 1) bar_b(bar, gridDim.x, i + 1);
        else cg::this_grid().sync();
    }
}
template <int V> void run(const char *name, unsigned *bar) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int nb : {16, 148, 296}) {
        int iters = 2000;
        void *args[] = {&bar, &iters};
        cudaMemset(bar, 0, 1024);
        cudaLaunchCooperativeKernel((void *)bar_kernel<V>, nb, 256, args, 0, 0);
        cudaMemset(bar, 0, 1024);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void *)bar_kernel<V>, nb, 256, args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("%s nb=%d: %.3f us (%s)\n", name, nb, ms * 1000 / iters, cudaGetErrorString(cudaGetLastError()));
    }
}
int main() {
    unsigned *bar; cudaMalloc(&bar, 1024);
    run<0>("gen+threadfence", bar);
    run<1>("red.release+ld.acquire", bar);
    run<2>("cg::grid.sync", bar);
}
