// tcgen05 GEMM interface (gemm_tc.cu).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace goat {

constexpr int kTcMaxTerms = 12;

// One K-concatenated term: A-operand plane rows [a_row0, a_row0 + M), B-operand
// plane rows [b_row0, b_row0 + N), both K-major bf16 with K = GEMM K.
struct alignas(64) TcTerm {
    CUtensorMap a;
    CUtensorMap b;
    int a_row0;
    int b_row0;
};

struct TcGemmParams {
    TcTerm terms[kTcMaxTerms];
    int nterms;
    int M, N, K, kblocks;
    int kslices;           // split-K: CTA z covers steps [z*kpb, (z+1)*kpb) of the
    int kpb;               //   flattened (term, k-block) sequence
    int chunk;             // k-steps per TMEM chunk before promotion into fp32 registers
    int64_t slice_stride;  // elements between slice outputs (mode 0)
    float alpha;
    int mode;  // 0: fp32 C (slice z at C + z*slice_stride); 1: bf16 planes (kslices == 1 only)
    float *C;
    int64_t ldc;
    __nv_bfloat16 *planes;
    int64_t ldpl;
    int64_t plane_stride;  // elements between planes
    int nplanes;
};

// Tensor map over a bf16 row-major [rows x cols] matrix with leading dim ld_elems,
// box = 64 (K) x box_rows, 128-byte swizzle.
void tc_make_map(CUtensorMap *map, const void *base, int64_t rows, int64_t cols, int64_t ld_elems, int box_rows);
int tc_box_rows_a();
int tc_box_rows_b();
void tc_gemm(const TcGemmParams &p, cudaStream_t s);
// out (fp32, scaled) or planes (bf16 split) = alpha * sum_z S[z]
void tc_slice_reduce(const float *S, int64_t slice_stride, int nslices, int rows, int cols, int64_t ld, float alpha,
                     float *out, __nv_bfloat16 *planes, int64_t plane_stride, int nplanes, cudaStream_t s);
int tc_block_m();
int tc_block_n();
int tc_block_k();
void tc_split_planes(const float *X, int64_t ldx, int rows, int cols, __nv_bfloat16 *planes, int64_t ldp,
                     int64_t plane_stride, int nplanes, cudaStream_t s);
void tc_split_planes_t(const float *X, int64_t ldx, int n, __nv_bfloat16 *planes, int64_t ldp, int64_t plane_stride,
                       int nplanes, cudaStream_t s);
bool tc_bf16_exact(const float *X, int64_t ldx, int n, int *dflag, cudaStream_t s, int rows = -1);

}  // namespace goat
