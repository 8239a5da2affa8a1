// Shared helpers for libgoat (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "goat.h"

namespace goat {

// A failure inside the library: carries a GOAT_E* code to the C-ABI edge.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define GOAT_CUDA(call)                                                                  \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess) {                                                         \
            int code_ = (e_ == cudaErrorMemoryAllocation) ? GOAT_EOOM : GOAT_ECUDA;      \
            throw ::goat::Error(code_, std::string(#call) + ": " + cudaGetErrorString(e_)); \
        }                                                                                \
    } while (0)

#define GOAT_CHECK_LAUNCH() GOAT_CUDA(cudaGetLastError())

inline void require(bool ok, const std::string &msg) {
    if (!ok) throw Error(GOAT_EINVAL, msg);
}

constexpr int kThreads = 256;

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// Device buffer (owning, raw bytes).
struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    void ensure(size_t b) {
        if (b <= bytes) return;
        release();
        GOAT_CUDA(cudaMalloc(&p, b));
        bytes = b;
    }
    template <class T> T *as() const { return static_cast<T *>(p); }
};

// Sinkhorn device-side loop state (one per handle).
struct SkState {
    int k;          // next pass index (0 = marginal pre-check)
    int done;
    int sweeps;
    int converged;
    int slot;       // potentials slot holding the returned (f, g)
    int arrive;     // last-block-done counter for the merge kernel
    int repaired;   // columns recomputed by the exact LSE repair (diagnostic)
    int pending;    // row-sharded driver: a column repair round is due before sweep k can finish
    double dev;     // returned deviation
    double last_dev;
    // per-LOT parameters (device-resident so a captured sweep graph is reusable)
    double gmax;    // shift: max G (maximize) / min G (minimize)
    double coef;    // E = coef * (gmax - G): -lam/scale (maximize), +lam/scale (minimize)
    double tol;
    int max_sweeps;
    int log_mode;
    double dcol;    // row-sharded pre-check: column deviation of the columns that needed no repair
    int redone;     // wide fp32 rows: sweeps recomputed with the max shift (diagnostic)
    int nostop_k;   // a resumed LOT: the convergence test may not fire at passes <= nostop_k (0 = none)
    int redo_next;  // row-sharded driver: the next pass repeats sweep k with the max shift (a row left the fixed-shift window on some rank)
};

// Count of kernels this library launched (reported as gpu_launches).
long &launch_count();
inline void note_launch(int k = 1) { launch_count() += k; }

}  // namespace goat
