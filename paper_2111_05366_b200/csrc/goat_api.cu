// libgoat C ABI: handle management and the Frank-Wolfe (GOAT) orchestration.
//
// goat_fw_core replaces _fw_core (matcher.py:177-212).  Per outer iteration the
// reference does 10 n^3 dgemm-class products (gradient 4, line search 4,
// objective 2).  Here the gradient is carried by linearity
//     G(P_{k+1}) = a G(P_k) + (1-a) G(Q_k)                     (matcher.py:197)
// so only G(Q_k) = A Q B^T + A^T Q B is new (2 products when A, B are
// symmetric, 4 otherwise), and the line-search coefficients and the logged
// objective come from dot products against it:
//     t1 = <G(Q), P> = s_PQ + s_QP,   s_QQ = <G(Q), Q> / 2,   s_PP = f(P)
//     c2 = s_PP - t1 + s_QQ,          c1 = t1 - 2 s_QQ (+ <L, P - Q>)
//     f(aP + (1-a)Q) = a^2 s_PP + a(1-a) t1 + (1-a)^2 s_QQ (+ a<L,P> + (1-a)<L,Q>)
// (identities of matcher.py:110-122 and :170-174, all accumulated in fp64).
#include <nvtx3/nvToolsExt.h>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <vector>

#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace goat {

long &launch_count() {
    static thread_local long c = 0;
    return c;
}

static thread_local std::string g_last_error;

struct Handle {
    int device = 0;
    int precision = GOAT_FP64;
    int gemm = GOAT_GEMM_AUTO;
    int split = 3;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    // workspace (sized for the largest order seen)
    int64_t cap_n = 0;    // vectors / scratch sized for this order
    int64_t cap_mat = 0;  // n x n workspace sized for this order
    DevBuf A, B, P, Q, G, GQ, T1, L, Gl, M;     // element = precision
    DevBuf A64, B64, G64, stage;                     // fp64 inputs (objective) + upload staging
    DevBuf f[2], g[2], colpart, devpart, devcol, state, red, scal, vec, ivec;
    DevBuf lap_d[3], lap_i[4], lap_b[2], lap_misc, bar;
    DevBuf auc_d[2], auc_i[4], auc_u64, auc_misc;  // auction LAP state
    // tcgen05 path: bf16 planes of A, A^T, the first-GEMM operand ([B] or [B; B^T]),
    // the iterate X and the intermediate Y^T.
    DevBuf tcA, tcAt, tcB, tcX, tcY, tcS;
    int tc_na = 0, tc_nb = 0;  // planes of A / B (1 when exact in bf16)
    // row-sharded primitives (goat_shard_*): this rank's block of rows
    struct Shard {
        int64_t n = 0, m = 0;
        bool sym = false, tc = false, ready = false, fill = false;
        DevBuf A, AT, B, X;       // A rows, A^T rows (m x ld), B (n x ld), GEMM intermediate
        DevBuf pA, pB, pQT, pX;   // tcgen05 planes: [A_r; A^T_r], [B; B^T], Q^T, [X; X2]
        int na = 0, nb = 0;
        SkPlan plan;
        DevBuf bad;               // per-column repair flags of the current sweep
        bool csr = false;         // gradient by SpMM on CSR rows (goat_shard_setup_csr)
        // fp32 handles: the LOT finishes in fp64 arithmetic below the fp32 deviation floor
        // (goat_shard_lot_refine; same rule as run_lot)
        double user_tol = 0.0;
        bool phase64 = false;
        SkPlan plan64;
        DevBuf G64;
    } sh;
    // sparse (CSR) adjacency: A, A^T, B, B^T (goat_fw_core_csr*); values null = 0/1
    struct Csr {
        DevBuf rowptr, col, val;
        int64_t nnz = 0;
        bool has_val = false;
    } csA, csAT, csB, csBT;
    Csr shA, shAT, shB, shBT;  // row-sharded CSR: this rank's rows of A, A^T; B, B^T
    DevBuf csScratch;
    bool csr_sym = false;
    int64_t cap_ab = 0;  // dense A, B sized for this order
    double *h_scal = nullptr;                   // pinned host scalars
    int lap_stats[4] = {0, 0, 0, 0};            // last auction: assigned, rounds, capped, freed
    SkState *h_state = nullptr;                 // pinned
    ~Handle() {
        if (h_scal) cudaFreeHost(h_scal);
        if (h_state) cudaFreeHost(h_state);
        if (own_stream) cudaStreamDestroy(own_stream);
    }
};

namespace {


inline int64_t ld_for(int64_t n) { return round_up(std::max<int64_t>(n, 1), 8); }

// Below this order the scipy-visiting-order solver runs from scratch (its
// assignments match scipy even under ties); above it the auction front end.
constexpr int kAuctionMinN = 256;

// matrices = false: vectors, reduction scratch and LAP state only (the row-sharded
// primitives keep their own blocks; a full n x n buffer per rank would defeat sharding).
// dense = false: the CSR path, which never holds A or B as n x n matrices.
void ensure_workspace(Handle &h, int64_t n, bool matrices = true, bool dense = true) {
    GOAT_CUDA(cudaSetDevice(h.device));
    const int64_t ld = ld_for(n);
    const size_t es = h.precision == GOAT_FP32 ? 4 : 8;
    const size_t mat = (size_t)n * ld * es;
    if (matrices && n > h.cap_mat) {
        for (DevBuf *b : {&h.P, &h.Q, &h.G, &h.GQ, &h.T1, &h.M}) b->ensure(mat);
        h.cap_mat = n;
    }
    if (matrices && dense && n > h.cap_ab) {
        for (DevBuf *b : {&h.A, &h.B}) b->ensure(mat);
        h.cap_ab = n;
    }
    if (n <= h.cap_n) return;
    const size_t vec = (size_t)ld * 8;
    for (int s = 0; s < 2; ++s) { h.f[s].ensure(vec); h.g[s].ensure(vec); }
    h.vec.ensure(vec * 4);
    h.ivec.ensure((size_t)ld * 4 * 4);
    h.devpart.ensure(4096 * 8);
    h.devcol.ensure((size_t)std::max<int64_t>(4096, ld / kThreads + 2) * 8);
    h.bar.ensure(1024);
    h.state.ensure(sizeof(SkState));
    h.red.ensure(kRedBlocks * 8 * 8);
    h.scal.ensure(64 * 8);
    const size_t cp = h.precision == GOAT_FP32 ? sk_plan<float>((int)n, h.num_sms).colpart_bytes
                                               : sk_plan<double>((int)n, h.num_sms).colpart_bytes;
    h.colpart.ensure(cp);
    for (int s = 0; s < 3; ++s) h.lap_d[s].ensure(vec);
    for (int s = 0; s < 4; ++s) h.lap_i[s].ensure((size_t)ld * 4);
    for (int s = 0; s < 2; ++s) h.lap_b[s].ensure((size_t)ld);
    h.lap_misc.ensure(64);
    h.cap_n = n;
}

void ensure_f64_inputs(Handle &h, int64_t n) {
    const size_t mat = (size_t)n * ld_for(n) * 8;
    h.A64.ensure(mat);
    h.B64.ensure(mat);
    h.stage.ensure(mat);
}

struct Ctx {
    Handle &h;
    int n;
    int64_t ld;
    cudaStream_t s;
    bool sym = false;
    bool tc = false;  // gradient on tcgen05 (fp32 mode)
    bool csr = false; // gradient by SpMM on the handle's CSR adjacency
    Ctx(Handle &hh, int nn) : h(hh), n(nn), ld(ld_for(nn)), s(hh.stream) {}
};

// ------------------------------------------------------------------ tcgen05 gradient
// Terms (p, q) of a split product sum_p X_p . sum_q Y_q kept when p + q < max(nx, ny):
// drops only products of two low-order planes (below fp32 rounding).
int add_terms(TcGemmParams &g, const __nv_bfloat16 *a, int na, int64_t a_stride, int a_rows, int a_row0,
              const __nv_bfloat16 *b, int nb, int64_t b_stride, int b_rows, int b_row0, int64_t ld, int K) {
    const int lim = std::max(na, nb);
    for (int p = 0; p < na; ++p)
        for (int q = 0; q < nb; ++q) {
            if (p + q >= lim) continue;
            if (g.nterms >= kTcMaxTerms) throw Error(GOAT_ENOTSUP, "tcgen05: too many split terms");
            TcTerm &t = g.terms[g.nterms++];
            tc_make_map(&t.a, a + p * a_stride, a_rows, K, ld, tc_box_rows_a());
            tc_make_map(&t.b, b + q * b_stride, b_rows, K, ld, tc_box_rows_b());
            t.a_row0 = a_row0;
            t.b_row0 = b_row0;
        }
    return g.nterms;
}

// Per-solve preparation: exactness of A, B in bf16 and their planes.
void tc_prepare(Ctx &c, const float *A, const float *B) {
    Handle &h = c.h;
    const int n = c.n;
    const int64_t ld = c.ld, mat = (int64_t)n * ld;
    int *flag = h.ivec.as<int>();
    h.tc_na = tc_bf16_exact(A, ld, n, flag, c.s) ? 1 : h.split;
    h.tc_nb = tc_bf16_exact(B, ld, n, flag, c.s) ? 1 : h.split;
    const int S = h.split;
    h.tcA.ensure(mat * 2 * h.tc_na);
    h.tcX.ensure(mat * 2 * S);
    const int yrows = c.sym ? n : 2 * n;
    h.tcY.ensure((int64_t)yrows * ld * 2 * S);
    h.tcB.ensure((int64_t)yrows * ld * 2 * h.tc_nb);
    auto *pa = h.tcA.as<__nv_bfloat16>();
    auto *pb = h.tcB.as<__nv_bfloat16>();
    tc_split_planes(A, ld, n, n, pa, ld, mat, h.tc_na, c.s);
    if (c.sym) {
        tc_split_planes(B, ld, n, n, pb, ld, mat, h.tc_nb, c.s);  // B^T = B
    } else {
        h.tcAt.ensure(mat * 2 * h.tc_na);
        tc_split_planes_t(A, ld, n, h.tcAt.as<__nv_bfloat16>(), ld, mat, h.tc_na, c.s);
        // first-GEMM A operand, per plane: rows [0,n) = B, rows [n,2n) = B^T
        tc_split_planes(B, ld, n, n, pb, ld, 2 * mat, h.tc_nb, c.s);
        tc_split_planes_t(B, ld, n, pb + mat, ld, 2 * mat, h.tc_nb, c.s);
    }
}

// Split-K: the tensor core's fp32 accumulation error grows with the number of
// chained MMAs; accuracy comes from in-kernel promotion (chunk k-steps per TMEM
// chain), and split-K slices (reduced in fixed order) only fill the SMs when
// there are few output tiles.
void tc_set_slices(const Handle &h, TcGemmParams &g, int rows, int cols, int64_t ld, int kblocks) {
    const int steps = g.nterms * kblocks;
    const int tiles = ceil_div(cols, tc_block_n()) * ceil_div(rows, tc_block_m());
    int sl = std::min(8, ceil_div(2 * h.num_sms, tiles));
    if (const char *e = getenv("GOAT_TC_KSLICES")) sl = std::max(1, atoi(e));
    const int64_t cap = (int64_t)1 << 31;
    while (sl > 1 && (int64_t)sl * rows * ld * 4 > cap) --sl;
    sl = std::max(1, std::min(sl, steps));
    g.kpb = ceil_div(steps, sl);
    g.kslices = ceil_div(steps, g.kpb);
    const char *ce = getenv("GOAT_TC_CHUNK");
    g.chunk = ce ? std::max(1, atoi(ce)) : 4;  // measured: 2-6e-7 of max|G|, speed flat in chunk
}

// Run a prepared product: mode-1 output (bf16 planes) or fp32 C = alpha * sum of terms,
// through split-K slices when set_slices chose them.
void tc_run(Handle &h, TcGemmParams &g, int rows, int cols, int64_t ld, float alpha, float *C,
            __nv_bfloat16 *planes, int64_t plane_stride, int nplanes, cudaStream_t s) {
    const int64_t out_stride = (int64_t)rows * ld;
    if (g.kslices == 1) {
        g.alpha = alpha;
        if (planes) {
            g.mode = 1; g.planes = planes; g.ldpl = ld; g.plane_stride = plane_stride; g.nplanes = nplanes;
            g.C = nullptr; g.ldc = 0; g.slice_stride = 0;
        } else {
            g.mode = 0; g.C = C; g.ldc = ld; g.slice_stride = 0; g.planes = nullptr; g.nplanes = 0;
        }
        tc_gemm(g, s);
        return;
    }
    h.tcS.ensure((size_t)g.kslices * out_stride * 4);
    g.mode = 0; g.alpha = 1.f; g.C = h.tcS.as<float>(); g.ldc = ld; g.slice_stride = out_stride;
    g.planes = nullptr; g.nplanes = 0;
    tc_gemm(g, s);
    tc_slice_reduce(h.tcS.as<float>(), out_stride, g.kslices, rows, cols, ld, alpha, planes ? nullptr : C, planes,
                    plane_stride, planes ? nplanes : 0, s);
}

// out = A X B^T + A^T X B on tensor cores:
//   Y^T = [B; B^T] X^T   (M = n or 2n)        -> bf16 planes of Y^T
//   G   = A Y1 + A^T Y2  (K-concatenated)     -> fp32
void tc_gradient(Ctx &c, const float *X, float *out) {
    Handle &h = c.h;
    const int n = c.n, S = h.split;
    const int64_t ld = c.ld, mat = (int64_t)n * ld;
    const int yrows = c.sym ? n : 2 * n;
    auto *px = h.tcX.as<__nv_bfloat16>();
    auto *py = h.tcY.as<__nv_bfloat16>();
    tc_split_planes(X, ld, n, n, px, ld, mat, S, c.s);
    const int64_t ystride = (int64_t)yrows * ld;
    const int kblocks = ceil_div(n, tc_block_k());
    auto set_slices = [&](TcGemmParams &g, int rows) { tc_set_slices(h, g, rows, n, ld, kblocks); };
    static thread_local TcGemmParams g1, g2;
    // Y^T = [B; B^T] X^T
    g1.nterms = 0;
    add_terms(g1, h.tcB.as<__nv_bfloat16>(), h.tc_nb, ystride, yrows, 0, px, S, mat, n, 0, ld, n);
    g1.M = yrows; g1.N = n; g1.K = n; g1.kblocks = kblocks; g1.alpha = 1.f;
    set_slices(g1, yrows);
    if (g1.kslices == 1) {
        g1.mode = 1; g1.planes = py; g1.ldpl = ld; g1.plane_stride = ystride; g1.nplanes = S;
        g1.C = nullptr; g1.ldc = 0; g1.slice_stride = 0;
        tc_gemm(g1, c.s);
    } else {
        h.tcS.ensure((size_t)g1.kslices * ystride * 4);
        g1.mode = 0; g1.C = h.tcS.as<float>(); g1.ldc = ld; g1.slice_stride = ystride;
        g1.planes = nullptr; g1.nplanes = 0;
        tc_gemm(g1, c.s);
        tc_slice_reduce(h.tcS.as<float>(), ystride, g1.kslices, yrows, n, ld, 1.f, nullptr, py, ystride, S, c.s);
    }
    // G = A Y1 (+ A^T Y2)
    g2.nterms = 0;
    add_terms(g2, h.tcA.as<__nv_bfloat16>(), h.tc_na, mat, n, 0, py, S, ystride, yrows, 0, ld, n);
    if (!c.sym)
        add_terms(g2, h.tcAt.as<__nv_bfloat16>(), h.tc_na, mat, n, 0, py, S, ystride, yrows, n, ld, n);
    const float alpha = c.sym ? 2.f : 1.f;
    g2.M = n; g2.N = n; g2.K = n; g2.kblocks = kblocks;
    set_slices(g2, n);
    g2.mode = 0; g2.planes = nullptr; g2.nplanes = 0; g2.ldc = ld;
    if (g2.kslices == 1) {
        g2.alpha = alpha; g2.C = out; g2.slice_stride = 0;
        tc_gemm(g2, c.s);
    } else {
        h.tcS.ensure((size_t)g2.kslices * mat * 4);
        g2.alpha = 1.f; g2.C = h.tcS.as<float>(); g2.slice_stride = mat;
        tc_gemm(g2, c.s);
        tc_slice_reduce(h.tcS.as<float>(), mat, g2.kslices, n, n, ld, alpha, out, nullptr, 0, 0, c.s);
    }
}

// Upload a host fp64 matrix (leading dim lds) into dst (precision T, ld).
template <class T>
void upload(Ctx &c, const double *src, int64_t lds, T *dst, double *stage64, int *nonfinite = nullptr) {
    GOAT_CUDA(cudaMemcpy2DAsync(stage64, c.ld * 8, src, lds * 8, (size_t)c.n * 8, c.n,
                                cudaMemcpyHostToDevice, c.s));
    launch_convert<T>(stage64, c.ld, dst, c.ld, c.n, 1.0, c.s, nonfinite);  // also zeroes the padding
}

// core.py:23-26: a non-finite entry is a ValueError (GOAT_EINVAL), checked on the
// device while the inputs are converted (flags: [0] A, [1] B, [2] L, [3] P0).
void require_finite(Ctx &c, int *flags_dev, int count) {
    int f[4] = {0, 0, 0, 0};
    GOAT_CUDA(cudaMemcpyAsync(f, flags_dev, sizeof(int) * count, cudaMemcpyDeviceToHost, c.s));
    GOAT_CUDA(cudaStreamSynchronize(c.s));
    static const char *names[4] = {"A", "B", "L", "init"};
    for (int q = 0; q < count; ++q)
        if (f[q]) throw Error(GOAT_EINVAL, std::string(names[q]) + " contains non-finite entries");
}

template <class T> void download(Ctx &c, const T *src, double *dst, int64_t ldd, double *stage64) {
    launch_convert_to_f64<T>(src, c.ld, stage64, c.ld, c.n, c.s);
    GOAT_CUDA(cudaMemcpy2DAsync(dst, ldd * 8, stage64, c.ld * 8, (size_t)c.n * 8, c.n,
                                cudaMemcpyDeviceToHost, c.s));
    GOAT_CUDA(cudaStreamSynchronize(c.s));
}

void sync(Ctx &c) { GOAT_CUDA(cudaStreamSynchronize(c.s)); }

// ------------------------------------------------------------------ gradient
// out = A X B^T + A^T X B (matcher.py:107); symmetric inputs: 2 A X B.
template <class T> DevCsr<T> csr_view(const Handle::Csr &m) {
    DevCsr<T> v;
    v.rowptr = m.rowptr.as<int64_t>();
    v.col = m.col.as<int>();
    v.val = m.has_val ? m.val.as<T>() : nullptr;
    v.nnz = m.nnz;
    return v;
}

// CSR gradient (spmm.cu): X1^T = (A X)^T [, X2^T = (A^T X)^T], then
// out = (B X1^T [+ B^T X2^T])^T = A X B^T + A^T X B; symmetric: 2 (B X1^T)^T.
template <class T> void csr_gradient(Ctx &c, const T *X, T *out, T *tmp) {
    Handle &h = c.h;
    const DevCsr<T> a = csr_view<T>(h.csA), at = csr_view<T>(h.csAT);
    const DevCsr<T> b = csr_view<T>(h.csB), bt = csr_view<T>(h.csBT);
    T *x1t = tmp, *x2t = h.M.as<T>();
    const T *d1[1] = {X};
    launch_spmm_t<T>(c.n, c.n, c.ld, c.ld, 1, &a, d1, 1.0, x1t, c.s);
    if (c.sym) {
        const T *d2[1] = {x1t};
        launch_spmm_t<T>(c.n, c.n, c.ld, c.ld, 1, &b, d2, 2.0, out, c.s);
    } else {
        launch_spmm_t<T>(c.n, c.n, c.ld, c.ld, 1, &at, d1, 1.0, x2t, c.s);
        const DevCsr<T> s2[2] = {b, bt};
        const T *d2[2] = {x1t, x2t};
        launch_spmm_t<T>(c.n, c.n, c.ld, c.ld, 2, s2, d2, 1.0, out, c.s);
    }
}

template <class T>
void gradient(Ctx &c, const T *A, const T *B, const T *X, T *out, T *tmp) {
    const int n = c.n;
    const int64_t ld = c.ld;
    if (c.csr) {
        csr_gradient<T>(c, X, out, tmp);
        return;
    }
    if constexpr (std::is_same<T, float>::value) {
        if (c.tc) {
            tc_gradient(c, X, out);
            return;
        }
    }
    if (c.sym) {
        gemm_simt<T>(n, n, n, 1.0, X, ld, 0, B, ld, 0, 0.0, tmp, ld, c.s);
        gemm_simt<T>(n, n, n, 2.0, A, ld, 0, tmp, ld, 0, 0.0, out, ld, c.s);
    } else {
        gemm_simt<T>(n, n, n, 1.0, X, ld, 0, B, ld, 1, 0.0, tmp, ld, c.s);  // X B^T
        gemm_simt<T>(n, n, n, 1.0, A, ld, 0, tmp, ld, 0, 0.0, out, ld, c.s);  // A (X B^T)
        gemm_simt<T>(n, n, n, 1.0, X, ld, 0, B, ld, 0, 0.0, tmp, ld, c.s);  // X B
        gemm_simt<T>(n, n, n, 1.0, A, ld, 1, tmp, ld, 0, 1.0, out, ld, c.s);  // + A^T (X B)
    }
}

// Engine choice: fp32 runs the gradient on tcgen05 unless GOAT_GEMM_SIMT was asked for.
template <class T> void setup_gemm(Ctx &c, const T *A, const T *B) {
    if constexpr (std::is_same<T, float>::value) {
        c.tc = c.h.gemm != GOAT_GEMM_SIMT;
        if (c.tc) tc_prepare(c, A, B);
    }
}

template <class T> bool is_symmetric(Ctx &c, const T *X) {
    int *flag = c.h.ivec.as<int>();
    const int one = 1;
    GOAT_CUDA(cudaMemcpyAsync(flag, &one, sizeof(int), cudaMemcpyHostToDevice, c.s));
    launch_is_symmetric<T>(X, c.ld, c.n, flag, c.s);
    int r = 0;
    GOAT_CUDA(cudaMemcpyAsync(&r, flag, sizeof(int), cudaMemcpyDeviceToHost, c.s));
    sync(c);
    return r != 0;
}

// ------------------------------------------------------------------ LOT
struct LotOut {
    int sweeps = 0, converged = 0;
    double dev = 0.0;
    double nrm = 0.0;  // sum (Q - P)^2 (when P given)
    double lq = 0.0;   // <L, Q> (when L given)
    bool used_kernel = true;
    int fp64_from = -1;  // fp32 handles: sweeps done in fp32 before the fp64 finish (-1: none)
};

// Sweeps in fp32 arithmetic stop at this marginal deviation; below it an fp32
// handle finishes the LOT in fp64 arithmetic (run_lot).  GOAT_SK_FP64_FINISH=0
// keeps the pure-fp32 loop (measurement only: it cannot meet tol < floor).
constexpr double kFp32DevFloorDefault = 1e-4;
// GOAT_SK_FP32_FLOOR overrides it (measurement: lower floors keep more sweeps in fp32
// but approach the ~1e-6 noise of the fp32 deviation itself)
inline double fp32_dev_floor() {
    static const double v = [] {
        const char *e = getenv("GOAT_SK_FP32_FLOOR");
        const double x = e ? atof(e) : 0.0;
        return x > 0.0 ? x : kFp32DevFloorDefault;
    }();
    return v;
}
inline bool fp64_finish_enabled() {
    const char *e = getenv("GOAT_SK_FP64_FINISH");
    return !(e && atoi(e) == 0);
}

// Runs the sweep loop from the device state (SkState.k .. stop) and leaves the
// final state in h.h_state.
template <class U>
void run_sweeps(Ctx &c, const SkArgs &a, const SkPlan &plan, int max_sweeps) {
    Handle &h = c.h;
    if (plan.persistent) {
        sk_launch_persistent<U>(a, plan, h.bar.as<unsigned>(), c.s);
    } else {
        const int max_passes = max_sweeps + 2;
        const int poll = 8;
        for (int p = 0; p < max_passes; ++p) {
            sk_launch_pass<U>(a, plan, c.s);
            sk_launch_merge<U>(a, plan, c.s);
            if ((p + 1) % poll == 0 || p + 1 == max_passes) {
                GOAT_CUDA(cudaMemcpyAsync(h.h_state, a.st, sizeof(SkState), cudaMemcpyDeviceToHost, c.s));
                sync(c);
                if (h.h_state->done) break;
            }
        }
    }
    GOAT_CUDA(cudaMemcpyAsync(h.h_state, a.st, sizeof(SkState), cudaMemcpyDeviceToHost, c.s));
    sync(c);
    if (!h.h_state->done) throw Error(GOAT_ECUDA, "sinkhorn loop did not terminate");
}

// mode: 0 = lot(M) (sinkhorn.py:103-130); 1 = sinkhorn_knopp on K = exp(-Gin)
template <class T>
LotOut run_lot(Ctx &c, const T *Gin, int sense, double lam, int max_sweeps, double tol, T *Q,
               const T *P, const T *L, int mode) {
    Handle &h = c.h;
    const int n = c.n;
    LotOut out;
    double gmax = 0.0, coef = 1.0;
    int log_mode = 0;
    if (mode == 0) {
        double *mm = h.scal.as<double>();
        launch_minmax<T>(Gin, c.ld, n, h.red.as<double>(), mm, c.s);
        GOAT_CUDA(cudaMemcpyAsync(h.h_scal, mm, 2 * sizeof(double), cudaMemcpyDeviceToHost, c.s));
        sync(c);
        const double lo = h.h_scal[0], hi = h.h_scal[1];
        const double scale = hi - lo;  // == shifted.max() (sinkhorn.py:115-119)
        if (scale == 0.0) {            // sinkhorn.py:121-124: exact barycenter, 0 sweeps
            launch_fill<T>(Q, c.ld, n, 1.0 / n, c.s);
            out.sweeps = 0; out.converged = 1; out.dev = 0.0;
            out.used_kernel = false;
            return out;
        }
        const bool maximize = (sense == GOAT_MAXIMIZE);
        gmax = maximize ? hi : lo;
        coef = maximize ? -lam / scale : lam / scale;
        // sinkhorn.py:127: K.min() = exp(-lam/scale * scale) underflows -> log-domain path
        log_mode = !(std::exp((-lam / scale) * scale) > 0.0);
    } else {
        gmax = 0.0;  // E = 1 * (0 - (-log K)) = log K
        coef = 1.0;
    }
    SkPlan plan = sk_plan<T>(n, h.num_sms);
    SkArgs a{};
    a.G = Gin; a.ld = c.ld; a.n = n;
    a.f[0] = h.f[0].as<double>(); a.f[1] = h.f[1].as<double>();
    a.g[0] = h.g[0].as<double>(); a.g[1] = h.g[1].as<double>();
    a.colpart = h.colpart.p; a.ldp = ld_for(n);
    a.devpart = h.devpart.as<double>(); a.devcol = h.devcol.as<double>();
    a.st = h.state.as<SkState>(); a.nblk = plan.nblk;
    GOAT_CUDA(cudaMemsetAsync(a.f[0], 0, c.ld * 8, c.s));
    GOAT_CUDA(cudaMemsetAsync(a.g[0], 0, c.ld * 8, c.s));
    // fp32 arithmetic resolves the marginal deviation |u K v - 1| only down to
    // ~1e-5 (exponent rounding at |E + f + g| ~ 1e2), so a tolerance below
    // fp32_dev_floor() (the default 1e-8, sinkhorn.py:32) can never fire and every LOT
    // would run max_sweeps.  fp32 handles therefore sweep in fp32 down to the
    // floor and finish in fp64 arithmetic on the same (exactly widened) fp32 G
    // from the same potentials, which restores the reference's stopping rule.
    const bool finish64 = sizeof(T) == 4 && tol < fp32_dev_floor() && fp64_finish_enabled();
    SkState st0{};
    st0.k = log_mode ? 1 : 0;
    st0.gmax = gmax; st0.coef = coef; st0.tol = finish64 ? fp32_dev_floor() : tol;
    st0.max_sweeps = max_sweeps; st0.log_mode = log_mode;
    *h.h_state = st0;
    GOAT_CUDA(cudaMemcpyAsync(a.st, h.h_state, sizeof(SkState), cudaMemcpyHostToDevice, c.s));
    run_sweeps<T>(c, a, plan, max_sweeps);
    if constexpr (sizeof(T) == 4) if (finish64 && h.h_state->converged) {
        // Stopped at the floor at pass k = sweeps + 1 (which produced f_k and
        // dev_{k-1} in fp32).  The fp64 loop re-enters one pass earlier: pass k-1
        // recomputes f_{k-1} and g_{k-1} in fp64 from g_{k-2} (still in its ring
        // slot: pass k never merged), so the first deviation it may act on, dev_{k-1}
        // at pass k, compares two fp64 row sums.  The re-entry pass itself cannot
        // stop (its f_{k-2} slot was overwritten).  sweeps == 0: the marginal
        // pre-check fired, redone from scratch.
        const int swept = h.h_state->sweeps;
        h.G64.ensure((size_t)n * c.ld * sizeof(double));
        launch_convert_to_f64<T>(Gin, c.ld, h.G64.as<double>(), c.ld, n, c.s);
        SkPlan plan64 = sk_plan<double>(n, h.num_sms);
        h.colpart.ensure(plan64.colpart_bytes);
        SkArgs a64 = a;
        a64.G = h.G64.p; a64.colpart = h.colpart.p; a64.nblk = plan64.nblk;
        a.colpart = h.colpart.p;
        SkState st1 = st0;
        st1.tol = tol;
        if (swept > 0) { st1.k = swept; st1.nostop_k = swept; }
        else {
            GOAT_CUDA(cudaMemsetAsync(a.f[0], 0, c.ld * 8, c.s));
            GOAT_CUDA(cudaMemsetAsync(a.g[0], 0, c.ld * 8, c.s));
        }
        *h.h_state = st1;
        GOAT_CUDA(cudaMemcpyAsync(a.st, h.h_state, sizeof(SkState), cudaMemcpyHostToDevice, c.s));
        run_sweeps<double>(c, a64, plan64, max_sweeps);
        out.fp64_from = swept;
    }
    out.sweeps = h.h_state->sweeps;
    out.converged = h.h_state->converged;
    out.dev = h.h_state->dev;
    if (getenv("GOAT_SK_VERBOSE")) {
        fprintf(stderr, "lot n=%d sweeps %d converged %d dev %.3g fp64_from %d redone %d repaired %d\n", n, out.sweeps,
                out.converged, out.dev, out.fp64_from, h.h_state->redone, h.h_state->repaired);
        if (getenv("GOAT_SK_RETIME")) {
            // diagnostics: the handle-precision sweep kernel timed alone on THIS cost matrix
            // (50 sweeps that cannot converge), then the loop state is restored
            const SkState keep = *h.h_state;
            SkState st = st0;
            st.tol = 1e-300; st.max_sweeps = 50;
            *h.h_state = st;
            GOAT_CUDA(cudaMemcpyAsync(a.st, h.h_state, sizeof(SkState), cudaMemcpyHostToDevice, c.s));
            std::vector<double> fsave((size_t)c.ld * 4);
            for (int q = 0; q < 2; ++q) {
                GOAT_CUDA(cudaMemcpyAsync(fsave.data() + (size_t)q * c.ld, a.f[q], c.ld * 8, cudaMemcpyDeviceToHost, c.s));
                GOAT_CUDA(cudaMemcpyAsync(fsave.data() + (size_t)(2 + q) * c.ld, a.g[q], c.ld * 8, cudaMemcpyDeviceToHost, c.s));
            }
            sync(c);
            GOAT_CUDA(cudaMemsetAsync(a.f[0], 0, c.ld * 8, c.s));
            GOAT_CUDA(cudaMemsetAsync(a.g[0], 0, c.ld * 8, c.s));
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0, c.s);
            run_sweeps<T>(c, a, plan, 50);
            cudaEventRecord(e1, c.s);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            fprintf(stderr, "lot n=%d retimed: %.3f ms per pass over 52 passes (redone %d repaired %d)\n", n, ms / 52.0,
                    h.h_state->redone, h.h_state->repaired);
            for (int q = 0; q < 2; ++q) {
                GOAT_CUDA(cudaMemcpyAsync(a.f[q], fsave.data() + (size_t)q * c.ld, c.ld * 8, cudaMemcpyHostToDevice, c.s));
                GOAT_CUDA(cudaMemcpyAsync(a.g[q], fsave.data() + (size_t)(2 + q) * c.ld, c.ld * 8, cudaMemcpyHostToDevice, c.s));
            }
            *h.h_state = keep;
            GOAT_CUDA(cudaMemcpyAsync(a.st, h.h_state, sizeof(SkState), cudaMemcpyHostToDevice, c.s));
            sync(c);
        }
    }
    double *part = h.red.as<double>();
    const int eb = kRedBlocks;
    sk_launch_emit<T>(a, Q, c.ld, P, c.ld, L, c.ld, part, eb, c.s);
    if (P || L) {
        // reuse the 5-wide finisher on [nrm, lq, *, *] rows of width 4 -> do it on host
        std::vector<double> hp((size_t)eb * 4);
        GOAT_CUDA(cudaMemcpyAsync(hp.data(), part, eb * 4 * 8, cudaMemcpyDeviceToHost, c.s));
        sync(c);
        double nrm = 0, lq = 0;
        for (int b = 0; b < eb; ++b) { nrm += hp[b * 4]; lq += hp[b * 4 + 1]; }
        out.nrm = nrm;
        out.lq = lq;
    }
    return out;
}

// Phase timer (CUDA events on the handle's stream); a named timer also opens an
// NVTX range (header-only nvtx3: visible to Nsight tools, free otherwise).
struct Timer {
    cudaEvent_t a, b;
    cudaStream_t s;
    bool range = false;
    explicit Timer(cudaStream_t st, const char *name = nullptr) : s(st) {
        if (name) { nvtxRangePushA(name); range = true; }
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
    }
    double stop() {
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        return ms;
    }
    ~Timer() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        if (range) nvtxRangePop();
    }
};

// ------------------------------------------------------------------ LAP
template <class T>
int run_lap(Ctx &c, const T *M, int sense, int *perm_dev, std::vector<int> &perm_host) {
    Handle &h = c.h;
    const int n = c.n;
    int *cand = perm_dev;
    int *hits = h.lap_i[3].as<int>();
    int *flag = h.lap_misc.as<int>();
    launch_lap_certificate<T>(M, c.ld, n, sense, cand, hits, flag, c.s);
    int certified = 0;
    GOAT_CUDA(cudaMemcpyAsync(&certified, flag, sizeof(int), cudaMemcpyDeviceToHost, c.s));
    sync(c);
    if (!certified) {
        LapWork w{};
        w.u = h.lap_d[0].as<double>(); w.v = h.lap_d[1].as<double>(); w.spc = h.lap_d[2].as<double>();
        w.path = h.lap_i[0].as<int>(); w.row4col = h.lap_i[1].as<int>();
        w.col4row = perm_dev; w.rem = h.lap_i[2].as<int>();
        w.SR = h.lap_b[0].as<unsigned char>(); w.SC = h.lap_b[1].as<unsigned char>();
        w.status = flag + 4;
        int warm = 0;
        const char *ae = getenv("GOAT_LAP_AUCTION");
        if (n >= kAuctionMinN && !(ae && atoi(ae) == 0)) {
            // eps-scaling auction, then certified repair by warm-started augmenting paths
            double *mm = h.scal.as<double>() + 48;
            launch_minmax<T>(M, c.ld, n, h.red.as<double>(), mm, c.s);
            double lohi[2];
            GOAT_CUDA(cudaMemcpyAsync(lohi, mm, 16, cudaMemcpyDeviceToHost, c.s));
            sync(c);
            const size_t vb = (size_t)n * 8, ib = (size_t)n * 4;
            for (int q = 0; q < 2; ++q) h.auc_d[q].ensure(vb);
            for (int q = 0; q < 4; ++q) h.auc_i[q].ensure(ib);
            h.auc_u64.ensure(vb);
            h.auc_misc.ensure(512 + (size_t)kAucMaxCtas * 24);
            AuctionWork aw{};
            aw.price = h.auc_d[0].as<double>(); aw.row_bid_v = h.auc_d[1].as<double>();
            aw.row_col = h.auc_i[0].as<int>(); aw.col_row = h.auc_i[1].as<int>();
            aw.bid_row = h.auc_i[2].as<int>(); aw.row_bid = h.auc_i[3].as<int>();
            aw.bid_val = h.auc_u64.as<unsigned long long>();
            aw.counters = h.auc_misc.as<int>();
            aw.bar = reinterpret_cast<unsigned *>(h.auc_misc.as<char>() + 256);
            aw.part_w = reinterpret_cast<double *>(h.auc_misc.as<char>() + 512);
            aw.part_j = reinterpret_cast<int *>(h.auc_misc.as<char>() + 512 + (size_t)kAucMaxCtas * 16);
            launch_lap_auction<T>(M, c.ld, n, sense, lohi[1] - lohi[0], w, aw, h.num_sms, c.s);
            GOAT_CUDA(cudaMemcpyAsync(h.lap_stats, aw.counters, 16, cudaMemcpyDeviceToHost, c.s));
            warm = 1;
        }
        const bool verbose = getenv("GOAT_LAP_VERBOSE") != nullptr;
        if (verbose) {
            sync(c);
            fprintf(stderr, "lap n=%d auction: assigned %d rounds %d capped %d freed %d\n", n, h.lap_stats[0],
                    h.lap_stats[1], h.lap_stats[2], h.lap_stats[3]);
        }
        Timer tsap(c.s);
        GOAT_CUDA(cudaMemsetAsync(w.status, 0, 4 * sizeof(int), c.s));
        launch_lap_sap<T>(M, c.ld, n, sense, w, c.s, warm);
        int status4[4] = {0, 0, 0, 0};
        GOAT_CUDA(cudaMemcpyAsync(status4, w.status, 4 * sizeof(int), cudaMemcpyDeviceToHost, c.s));
        sync(c);
        const int status = status4[0];
        if (verbose)
            fprintf(stderr, "lap n=%d augmenting-path repair: %.1f ms (cluster solver: %d rows, %d distance levels, %d "
                            "columns scanned)\n", n, tsap.stop(), status4[1], status4[2], status4[3]);
        if (status != 0) throw Error(GOAT_EINVAL, "cost matrix is infeasible");
    }
    perm_host.resize(n);
    GOAT_CUDA(cudaMemcpyAsync(perm_host.data(), perm_dev, n * sizeof(int), cudaMemcpyDeviceToHost, c.s));
    sync(c);
    return certified;
}

double alpha_opt(double c2, double c1, int sense) {
    // matcher.py:125-135
    if (c2 != 0.0) {
        const double crit = -c1 / (2.0 * c2);
        const bool ok = (sense == GOAT_MAXIMIZE) ? (c2 < 0) : (c2 > 0);
        if (ok && 0.0 <= crit && crit <= 1.0) return crit;
    }
    const double end = c2 + c1;
    if (sense == GOAT_MAXIMIZE) return end >= 0.0 ? 1.0 : 0.0;
    return end <= 0.0 ? 1.0 : 0.0;
}


// Core loop on device-resident inputs in the workspace (A, B, optional L, P = P0).
template <class T>
void fw_loop(Ctx &c, bool have_L, bool p0_bary, const goat_options &o, goat_fw_result *res) {
    Handle &h = c.h;
    const int n = c.n;
    const int64_t ld = c.ld;
    T *A = h.A.as<T>(), *B = h.B.as<T>();
    T *P = h.P.as<T>(), *Q = h.Q.as<T>(), *G = h.G.as<T>(), *GQ = h.GQ.as<T>(), *T1 = h.T1.as<T>();
    T *L = have_L ? h.L.as<T>() : nullptr;
    T *Gl = have_L ? h.Gl.as<T>() : nullptr;
    double *dots = h.scal.as<double>() + 16;
    double *hd = h.h_scal + 16;
    double t_grad = 0, t_lot = 0, t_ls = 0, t_lap = 0;

    if (c.csr) {
        c.sym = h.csr_sym;
    } else {
        c.sym = is_symmetric<T>(c, A) && is_symmetric<T>(c, B);
        setup_gemm<T>(c, A, B);
    }
    {
        Timer tm(c.s, "goat.gradient");
        if (p0_bary) {
            launch_fill<T>(P, ld, n, 1.0 / n, c.s);  // core.py:89-93
            if (c.csr) {
                // degree vectors [A 1 | A^T 1 | B 1 | B^T 1] straight from the CSR rows
                double *v = h.vec.as<double>();
                launch_csr_rowsum<T>(csr_view<T>(h.csA), n, v, c.s);
                launch_csr_rowsum<T>(csr_view<T>(h.csAT), n, v + n, c.s);
                launch_csr_rowsum<T>(csr_view<T>(h.csB), n, v + 2 * n, c.s);
                launch_csr_rowsum<T>(csr_view<T>(h.csBT), n, v + 3 * n, c.s);
                launch_bary_grad_vec<T>(v, G, ld, n, c.s);
            } else {
                launch_bary_grad<T>(A, ld, B, ld, G, ld, n, h.vec.as<double>(), c.s);
            }
        } else {
            gradient<T>(c, A, B, P, G, T1);
        }
        t_grad += tm.stop();
    }
    // f(P0) (matcher.py:184): <G(P0), P0>/2 + <L, P0>
    launch_fw_dots<T>(G, G, P, P, L, ld, n, h.red.as<double>(), dots, c.s);
    GOAT_CUDA(cudaMemcpyAsync(hd, dots, 6 * 8, cudaMemcpyDeviceToHost, c.s));
    sync(c);
    res->hist_obj[0] = 0.5 * hd[2] + (have_L ? hd[5] : 0.0);
    res->hist_alpha[0] = NAN;
    int iterations = 0, converged = 0;
    for (int i = 1; i <= o.max_iters; ++i) {
        const T *Gin = G;
        if (have_L) { launch_add<T>(G, L, Gl, ld, n, c.s); Gin = Gl; }
        LotOut lo;
        {
            Timer tm(c.s, "goat.lot");
            if (o.step_solver == GOAT_STEP_LOT) {
                lo = run_lot<T>(c, Gin, o.sense, o.lam, o.max_sweeps, o.sk_tol, Q, nullptr, nullptr, 0);
            } else {
                // FAQ step (matcher.py:191-192): Q = permutation_matrix(LAP(G))
                std::vector<int> ph;
                run_lap<T>(c, Gin, o.sense, h.ivec.as<int>(), ph);
                launch_perm_matrix<T>(h.ivec.as<int>(), Q, ld, n, c.s);
                lo.sweeps = 0; lo.converged = 1;
            }
            const double t_this = tm.stop();
            t_lot += t_this;
            if (res->lot_ms) res->lot_ms[i - 1] = t_this;
        }
        if (res->lot_sweeps) res->lot_sweeps[i - 1] = lo.sweeps;
        if (res->lot_converged) res->lot_converged[i - 1] = lo.converged;
        if (res->lot_dev) res->lot_dev[i - 1] = lo.dev;
        if (res->lot_fp64_from) res->lot_fp64_from[i - 1] = lo.fp64_from;
        {
            Timer tm(c.s, "goat.gradient");
            gradient<T>(c, A, B, Q, GQ, T1);
            t_grad += tm.stop();
        }
        Timer tm(c.s, "goat.line_search");
        launch_fw_dots<T>(G, GQ, P, Q, L, ld, n, h.red.as<double>(), dots, c.s);
        GOAT_CUDA(cudaMemcpyAsync(hd, dots, 6 * 8, cudaMemcpyDeviceToHost, c.s));
        sync(c);
        // g(a) = f(Q + a D) = f(Q) + c1 a + c2 a^2, D = P - Q (matcher.py:110-122)
        const double c1 = hd[0] + (have_L ? hd[4] : 0.0);
        const double c2 = 0.5 * hd[1];
        const double fQ = 0.5 * hd[2] + (have_L ? hd[5] : 0.0);
        const double nrm = hd[3];
        const double al = alpha_opt(c2, c1, o.sense);
        const double bl = 1.0 - al;
        res->hist_obj[i] = fQ + al * c1 + al * al * c2;  // f(aP + (1-a)Q)
        res->hist_alpha[i] = al;
        const double step = std::fabs(bl) * std::sqrt(nrm);  // ||P_new - P||_F
        if (al == 0.0) {
            std::swap(h.P.p, h.Q.p);
            std::swap(h.G.p, h.GQ.p);
            P = h.P.as<T>(); Q = h.Q.as<T>(); G = h.G.as<T>(); GQ = h.GQ.as<T>();
        } else if (al != 1.0) {
            launch_axpby<T>(bl, Q, al, P, ld, n, c.s);   // P <- a P + (1-a) Q
            launch_axpby<T>(bl, GQ, al, G, ld, n, c.s);  // G <- a G + (1-a) G(Q)
        }
        iterations = i;
        t_ls += tm.stop();
        if (step < o.fw_tol) { converged = 1; break; }
    }
    // final projection (matcher.py:205-211)
    const T *Gin = G;
    if (have_L) { launch_add<T>(G, L, Gl, ld, n, c.s); Gin = Gl; }
    std::vector<int> ph;
    Timer tm(c.s, "goat.lap");
    res->lap_certified = run_lap<T>(c, Gin, o.sense, h.ivec.as<int>(), ph);
    t_lap += tm.stop();
    for (int r = 0; r < n; ++r) res->assignment[r] = ph[r];
    res->iterations = iterations;
    res->converged = converged;
    res->time_ms[0] = t_grad; res->time_ms[1] = t_lot; res->time_ms[2] = t_ls; res->time_ms[3] = t_lap;
}

template <class T>
void objective_on_device(Ctx &c, bool have64) {
    Handle &h = c.h;
    if (!have64) {
        ensure_f64_inputs(h, c.n);
        launch_convert_to_f64<T>(h.A.as<T>(), c.ld, h.A64.as<double>(), c.ld, c.n, c.s);
        launch_convert_to_f64<T>(h.B.as<T>(), c.ld, h.B64.as<double>(), c.ld, c.n, c.s);
    }
}

void validate_opts(const goat_options *o) {
    require(o != nullptr, "options must not be NULL");
    require(o->max_iters >= 1, "max_iters must be at least 1");
    require(o->fw_tol > 0, "fw_tol must be positive");
    require(o->lam > 0, "lam must be positive");
    require(o->max_sweeps >= 1, "max_sweeps must be at least 1");
    require(o->sk_tol > 0, "tol must be positive");
    require(o->sense == GOAT_MINIMIZE || o->sense == GOAT_MAXIMIZE, "bad objective sense");
    require(o->step_solver == GOAT_STEP_LOT || o->step_solver == GOAT_STEP_EXACT_LAP, "bad step_solver");
}

template <class T>
void fw_core_host(Handle &h, int64_t n, const double *A, int64_t lda, const double *B, int64_t ldb,
                  const double *L, int64_t ldl, const double *P0, int64_t ldp, const goat_options *o,
                  goat_fw_result *res) {
    auto t0 = std::chrono::steady_clock::now();
    ensure_workspace(h, n);
    ensure_f64_inputs(h, n);
    if (L) { h.L.ensure(h.A.bytes); h.Gl.ensure(h.A.bytes); }
    Ctx c(h, (int)n);
    Timer setup(c.s);
    int *fin = h.lap_misc.as<int>() + 8;  // 4 non-finite flags
    GOAT_CUDA(cudaMemsetAsync(fin, 0, 4 * sizeof(int), c.s));
    upload<T>(c, A, lda, h.A.as<T>(), h.A64.as<double>(), fin);
    upload<T>(c, B, ldb, h.B.as<T>(), h.B64.as<double>(), fin + 1);
    if (L) upload<T>(c, L, ldl, h.L.as<T>(), h.stage.as<double>(), fin + 2);
    if (P0) upload<T>(c, P0, ldp, h.P.as<T>(), h.stage.as<double>(), fin + 3);
    require_finite(c, fin, 4);
    res->time_ms[4] = setup.stop();
    fw_loop<T>(c, L != nullptr, P0 == nullptr, *o, res);
    // objective on the inputs (core.py:120-124), fp64, fixed order
    int *perm = h.ivec.as<int>();
    std::vector<int> ph(n);
    for (int64_t r = 0; r < n; ++r) ph[r] = (int)res->assignment[r];
    GOAT_CUDA(cudaMemcpyAsync(perm, ph.data(), n * 4, cudaMemcpyHostToDevice, c.s));
    launch_qap_perm(h.A64.as<double>(), c.ld, h.B64.as<double>(), c.ld, perm, (int)n, h.red.as<double>(),
                    h.scal.as<double>() + 40, c.s);
    GOAT_CUDA(cudaMemcpyAsync(h.h_scal + 40, h.scal.as<double>() + 40, 8, cudaMemcpyDeviceToHost, c.s));
    sync(c);
    res->objective = h.h_scal[40];
    res->time_ms[5] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

template <class T>
void fw_core_dev(Handle &h, int64_t n, const T *A, int64_t lda, const T *B, int64_t ldb, const T *L,
                 int64_t ldl, const T *P0, int64_t ldp, const goat_options *o, goat_fw_result *res) {
    auto t0 = std::chrono::steady_clock::now();
    ensure_workspace(h, n);
    if (L) { h.L.ensure(h.A.bytes); h.Gl.ensure(h.A.bytes); }
    Ctx c(h, (int)n);
    const size_t es = sizeof(T);
    auto cp = [&](const T *src, int64_t lds, T *dst) {
        GOAT_CUDA(cudaMemcpy2DAsync(dst, c.ld * es, src, lds * es, n * es, n, cudaMemcpyDeviceToDevice, c.s));
    };
    GOAT_CUDA(cudaMemsetAsync(h.A.p, 0, h.A.bytes, c.s));
    GOAT_CUDA(cudaMemsetAsync(h.B.p, 0, h.B.bytes, c.s));
    cp(A, lda, h.A.as<T>());
    cp(B, ldb, h.B.as<T>());
    if (L) cp(L, ldl, h.L.as<T>());
    if (P0) cp(P0, ldp, h.P.as<T>());
    res->time_ms[4] = 0;
    fw_loop<T>(c, L != nullptr, P0 == nullptr, *o, res);
    ensure_f64_inputs(h, n);
    objective_on_device<T>(c, false);
    int *perm = h.ivec.as<int>();
    std::vector<int> ph(n);
    for (int64_t r = 0; r < n; ++r) ph[r] = (int)res->assignment[r];
    GOAT_CUDA(cudaMemcpyAsync(perm, ph.data(), n * 4, cudaMemcpyHostToDevice, c.s));
    launch_qap_perm(h.A64.as<double>(), c.ld, h.B64.as<double>(), c.ld, perm, (int)n, h.red.as<double>(),
                    h.scal.as<double>() + 40, c.s);
    GOAT_CUDA(cudaMemcpyAsync(h.h_scal + 40, h.scal.as<double>() + 40, 8, cudaMemcpyDeviceToHost, c.s));
    sync(c);
    res->objective = h.h_scal[40];
    res->time_ms[5] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

template <class F> int guarded(F &&f) {
    try {
        f();
        return GOAT_OK;
    } catch (const Error &e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception &e) {
        g_last_error = e.what();
        return GOAT_ECUDA;
    }
}

void check_order(int64_t n) {
    require(n >= 1, "order must be positive");
    require(n <= (int64_t)1 << 30, "order too large");
}

template <class F> void dispatch(Handle &h, F &&f) {
    if (h.precision == GOAT_FP32) f((float *)nullptr);
    else f((double *)nullptr);
}

// ------------------------------------------------------------------ row-sharded primitives
// One rank owns rows [r0, r0 + m) of the n x n iterates (the caller's row block;
// every block buffer is m x ld, ld = ld_for(n)).  The gradient of a block is
//     G_r = (A_r Q) B^T + (A^T_r Q) B          (symmetric: 2 (A_r Q) B)
// which needs the whole Q (the caller all-gathers it) and B, both replicated;
// A_r and A^T_r are the block's rows of A and A^T.  Both chains are two
// row-local products of m x n x n, so the work divides by the rank count.
__global__ void assign_sum_kernel(const float *Mf, const double *Md, int64_t ld, const int *perm, int n,
                                  double *out) {
    __shared__ double s_r[32];
    double v = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        v += Mf ? (double)Mf[(int64_t)i * ld + perm[i]] : Md[(int64_t)i * ld + perm[i]];
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31) == 0) s_r[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_r[w];
        *out = t;
    }
}

void shard_tc_prepare(Handle &h) {
    auto &S = h.sh;
    const int n = (int)S.n, m = (int)S.m;
    const int64_t ld = ld_for(n), mat = (int64_t)n * ld;
    cudaStream_t s = h.stream;
    int *flag = h.ivec.as<int>();
    const float *A = S.A.as<float>(), *AT = S.AT.as<float>(), *B = S.B.as<float>();
    const bool a_exact = tc_bf16_exact(A, ld, n, flag, s, m) && (S.sym || tc_bf16_exact(AT, ld, n, flag, s, m));
    S.na = a_exact ? 1 : h.split;
    S.nb = tc_bf16_exact(B, ld, n, flag, s) ? 1 : h.split;
    const int arows = S.sym ? m : 2 * m, brows = S.sym ? n : 2 * n;
    const int64_t astride = (int64_t)arows * ld, bstride = (int64_t)brows * ld;
    S.pA.ensure((size_t)astride * 2 * S.na);
    S.pB.ensure((size_t)bstride * 2 * S.nb);
    S.pQT.ensure((size_t)mat * 2 * h.split);
    S.pX.ensure((size_t)astride * 2 * h.split);
    auto *pa = S.pA.as<__nv_bfloat16>();
    auto *pb = S.pB.as<__nv_bfloat16>();
    tc_split_planes(A, ld, m, n, pa, ld, astride, S.na, s);
    if (!S.sym) tc_split_planes(AT, ld, m, n, pa + (int64_t)m * ld, ld, astride, S.na, s);
    tc_split_planes(B, ld, n, n, pb, ld, bstride, S.nb, s);
    if (!S.sym) tc_split_planes_t(B, ld, n, pb + mat, ld, bstride, S.nb, s);
}

template <class T> DevCsr<T> csr_view(const Handle::Csr &m);

template <class T> void shard_gradient(Handle &h, const T *Q, T *out) {
    auto &S = h.sh;
    const int n = (int)S.n, m = (int)S.m;
    const int64_t ld = ld_for(n), mat = (int64_t)n * ld;
    cudaStream_t s = h.stream;
    if (S.csr) {
        // X1^T = (A_r Q)^T [, X2^T = (A^T_r Q)^T]  (n x m), then
        // G_r = (B X1^T [+ B^T X2^T])^T  (m x n) = A_r Q B^T + A^T_r Q B
        const int64_t ldm = ld_for(m);
        T *x1t = S.X.as<T>(), *x2t = x1t + (int64_t)n * ldm;
        const DevCsr<T> a = csr_view<T>(h.shA), at = csr_view<T>(h.shAT);
        const DevCsr<T> b = csr_view<T>(h.shB), bt = csr_view<T>(h.shBT);
        const T *d1[1] = {Q};
        launch_spmm_t<T>(m, n, ld, ldm, 1, &a, d1, 1.0, x1t, s);
        if (S.sym) {
            const T *d2[1] = {x1t};
            launch_spmm_t<T>(n, m, ldm, ld, 1, &b, d2, 2.0, out, s);
        } else {
            launch_spmm_t<T>(m, n, ld, ldm, 1, &at, d1, 1.0, x2t, s);
            const DevCsr<T> s2[2] = {b, bt};
            const T *d2[2] = {x1t, x2t};
            launch_spmm_t<T>(n, m, ldm, ld, 2, s2, d2, 1.0, out, s);
        }
        return;
    }
    if constexpr (std::is_same<T, float>::value) {
        if (S.tc) {
            const int SP = h.split;
            const int arows = S.sym ? m : 2 * m, brows = S.sym ? n : 2 * n;
            const int64_t astride = (int64_t)arows * ld, bstride = (int64_t)brows * ld;
            const int kblocks = ceil_div(n, tc_block_k());
            auto *pqt = S.pQT.as<__nv_bfloat16>();
            auto *px = S.pX.as<__nv_bfloat16>();
            tc_split_planes_t(Q, ld, n, pqt, ld, mat, SP, s);  // K-major operand of A_r Q
            static thread_local TcGemmParams g1, g2;
            // [X; X2] = [A_r; A^T_r] Q   -> bf16 planes
            g1.nterms = 0;
            add_terms(g1, S.pA.as<__nv_bfloat16>(), S.na, astride, arows, 0, pqt, SP, mat, n, 0, ld, n);
            g1.M = arows; g1.N = n; g1.K = n; g1.kblocks = kblocks;
            tc_set_slices(h, g1, arows, n, ld, kblocks);
            tc_run(h, g1, arows, n, ld, 1.f, nullptr, px, astride, SP, s);
            // G_r = X B^T + X2 B   (symmetric: 2 X B)
            g2.nterms = 0;
            add_terms(g2, px, SP, astride, arows, 0, S.pB.as<__nv_bfloat16>(), S.nb, bstride, brows, 0, ld, n);
            if (!S.sym) add_terms(g2, px, SP, astride, arows, m, S.pB.as<__nv_bfloat16>(), S.nb, bstride, brows, n, ld, n);
            g2.M = m; g2.N = n; g2.K = n; g2.kblocks = kblocks;
            tc_set_slices(h, g2, m, n, ld, kblocks);
            tc_run(h, g2, m, n, ld, S.sym ? 2.f : 1.f, out, nullptr, 0, 0, s);
            return;
        }
    }
    T *X = S.X.as<T>();
    const T *A = S.A.as<T>(), *AT = S.AT.as<T>(), *B = S.B.as<T>();
    gemm_simt<T>(m, n, n, 1.0, A, ld, 0, Q, ld, 0, 0.0, X, ld, s);                          // A_r Q
    gemm_simt<T>(m, n, n, S.sym ? 2.0 : 1.0, X, ld, 0, B, ld, S.sym ? 0 : 1, 0.0, out, ld, s);  // (A_r Q) B^T
    if (!S.sym) {
        gemm_simt<T>(m, n, n, 1.0, AT, ld, 0, Q, ld, 0, 0.0, X, ld, s);   // A^T_r Q
        gemm_simt<T>(m, n, n, 1.0, X, ld, 0, B, ld, 0, 1.0, out, ld, s);  // + (A^T_r Q) B
    }
}


// ------------------------------------------------------------------ CSR adjacency
// Copies one CSR graph to the handle (host or device source; host values are
// float64 and converted to the handle's precision), checks it (sorted rows,
// columns in range, finite values), and builds its transpose.
template <class T>
void csr_load(Handle &h, int n, const goat_csr &src, bool device_src, Handle::Csr &dst, Handle::Csr &dstT,
              cudaStream_t s) {
    const int64_t nnz = src.nnz;
    require(nnz >= 0 && src.rowptr && (nnz == 0 || src.colidx), "csr: NULL rowptr/colidx");
    const auto kind = device_src ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    for (Handle::Csr *m : {&dst, &dstT}) {
        m->rowptr.ensure((size_t)(n + 1) * 8);
        m->col.ensure((size_t)std::max<int64_t>(nnz, 1) * 4);
        m->nnz = nnz;
        m->has_val = src.values != nullptr;
        if (m->has_val) m->val.ensure((size_t)std::max<int64_t>(nnz, 1) * sizeof(T));
    }
    if (!device_src) {
        require(src.rowptr[0] == 0 && src.rowptr[n] == nnz, "csr: rowptr[0] must be 0 and rowptr[n] = nnz");
    }
    GOAT_CUDA(cudaMemcpyAsync(dst.rowptr.p, src.rowptr, (size_t)(n + 1) * 8, kind, s));
    if (nnz) GOAT_CUDA(cudaMemcpyAsync(dst.col.p, src.colidx, (size_t)nnz * 4, kind, s));
    if (dst.has_val && nnz) {
        if (device_src || sizeof(T) == 8) {
            GOAT_CUDA(cudaMemcpyAsync(dst.val.p, src.values, (size_t)nnz * sizeof(T), kind, s));
        } else {
            std::vector<T> tmp((size_t)nnz);
            const double *v = static_cast<const double *>(src.values);
            for (int64_t q = 0; q < nnz; ++q) tmp[q] = (T)v[q];
            GOAT_CUDA(cudaMemcpyAsync(dst.val.p, tmp.data(), (size_t)nnz * sizeof(T), cudaMemcpyHostToDevice, s));
            GOAT_CUDA(cudaStreamSynchronize(s));  // tmp goes out of scope
        }
    }
    int *flag = h.ivec.as<int>();
    const int one = 1;
    GOAT_CUDA(cudaMemcpyAsync(flag, &one, sizeof(int), cudaMemcpyHostToDevice, s));
    launch_csr_check<T>(csr_view<T>(dst), n, n, flag, s);
    int ok = 0;
    GOAT_CUDA(cudaMemcpyAsync(&ok, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    GOAT_CUDA(cudaStreamSynchronize(s));
    require(ok == 1, "csr: rows must hold strictly increasing column indices in [0, n) and finite values");
    const size_t need = csr_transpose_scratch(nnz);
    h.csScratch.ensure(need);
    launch_csr_transpose<T>(csr_view<T>(dst), n, dstT.rowptr.as<int64_t>(), dstT.col.as<int>(),
                            dstT.has_val ? dstT.val.as<T>() : nullptr, h.csScratch.p, h.csScratch.bytes, s);
}

template <class T> bool csr_equal(Handle &h, int n, const Handle::Csr &a, const Handle::Csr &b, cudaStream_t s) {
    int *flag = h.ivec.as<int>();
    const int one = 1;
    GOAT_CUDA(cudaMemcpyAsync(flag, &one, sizeof(int), cudaMemcpyHostToDevice, s));
    launch_csr_equal<T>(csr_view<T>(a), csr_view<T>(b), n, flag, s);
    int r = 0;
    GOAT_CUDA(cudaMemcpyAsync(&r, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    GOAT_CUDA(cudaStreamSynchronize(s));
    return r == 1;
}

template <class T> void csr_setup(Handle &h, int n, const goat_csr &A, const goat_csr &B, bool device_src) {
    ensure_workspace(h, n, true, false);
    cudaStream_t s = h.stream;
    csr_load<T>(h, n, A, device_src, h.csA, h.csAT, s);
    csr_load<T>(h, n, B, device_src, h.csB, h.csBT, s);
    h.csr_sym = csr_equal<T>(h, n, h.csA, h.csAT, s) && csr_equal<T>(h, n, h.csB, h.csBT, s);
    // SpMM writes only columns [0, n) of each row: keep the padding of every n x n buffer zero
    for (DevBuf *b : {&h.P, &h.Q, &h.G, &h.GQ, &h.T1, &h.M}) GOAT_CUDA(cudaMemsetAsync(b->p, 0, b->bytes, s));
}

template <class T>
void fw_core_csr(Handle &h, int64_t n, const goat_csr &A, const goat_csr &B, bool device_src, const void *L,
                 int64_t ldl, const void *P0, int64_t ldp, const goat_options *o, goat_fw_result *res) {
    auto t0 = std::chrono::steady_clock::now();
    Ctx c(h, (int)n);
    Timer setup(c.s);
    csr_setup<T>(h, (int)n, A, B, device_src);
    c.csr = true;
    const size_t es = sizeof(T);
    if (L) { h.L.ensure(h.P.bytes); h.Gl.ensure(h.P.bytes); GOAT_CUDA(cudaMemsetAsync(h.L.p, 0, h.L.bytes, c.s)); }
    if (device_src) {
        auto cp = [&](const void *src, int64_t lds, T *dst) {
            GOAT_CUDA(cudaMemcpy2DAsync(dst, c.ld * es, src, lds * es, n * es, n, cudaMemcpyDeviceToDevice, c.s));
        };
        if (L) cp(L, ldl, h.L.as<T>());
        if (P0) cp(P0, ldp, h.P.as<T>());
    } else if (L || P0) {
        h.stage.ensure((size_t)n * c.ld * 8);
        if (L) upload<T>(c, static_cast<const double *>(L), ldl, h.L.as<T>(), h.stage.as<double>());
        if (P0) upload<T>(c, static_cast<const double *>(P0), ldp, h.P.as<T>(), h.stage.as<double>());
    }
    res->time_ms[4] = setup.stop();
    fw_loop<T>(c, L != nullptr, P0 == nullptr, *o, res);
    // objective on the inputs (core.py:120-124): sum over A's entries of A_ij B_{p(i)p(j)}
    int *perm = h.ivec.as<int>();
    std::vector<int> ph(n);
    for (int64_t r = 0; r < n; ++r) ph[r] = (int)res->assignment[r];
    GOAT_CUDA(cudaMemcpyAsync(perm, ph.data(), n * 4, cudaMemcpyHostToDevice, c.s));
    launch_csr_qap_perm<T>(csr_view<T>(h.csA), csr_view<T>(h.csB), perm, (int)n, h.vec.as<double>(),
                           h.scal.as<double>() + 40, c.s);
    GOAT_CUDA(cudaMemcpyAsync(h.h_scal + 40, h.scal.as<double>() + 40, 8, cudaMemcpyDeviceToHost, c.s));
    sync(c);
    res->objective = h.h_scal[40];
    res->time_ms[5] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}


// ------------------------------------------------------------------ seeded core
// matcher.py:245-269: with m seeds the free block is matched with the constant
// linear term L = A21 B21^T + A12^T B12 (matcher.py:267).  The reference forms L
// on the host (an nf x nf product of inner size m); here the seed blocks cross the
// boundary and L is formed on the device by two GEMMs.
template <class T>
void upload_rect(Ctx &c, const double *src, int64_t lds, int rows, int cols, T *dst, int64_t ldd) {
    std::vector<T> tmp((size_t)rows * ldd, T(0));
    for (int r = 0; r < rows; ++r)
        for (int q = 0; q < cols; ++q) tmp[(size_t)r * ldd + q] = (T)src[(int64_t)r * lds + q];
    GOAT_CUDA(cudaMemcpyAsync(dst, tmp.data(), tmp.size() * sizeof(T), cudaMemcpyHostToDevice, c.s));
    GOAT_CUDA(cudaStreamSynchronize(c.s));  // tmp goes out of scope
}

template <class T>
void fw_core_seeded(Handle &h, int64_t nf, int64_t m, const double *A22, int64_t lda22, const double *B22,
                    int64_t ldb22, const double *A21, int64_t lda21, const double *A12, int64_t lda12,
                    const double *B21, int64_t ldb21, const double *B12, int64_t ldb12, const double *P0,
                    int64_t ldp, const goat_options *o, goat_fw_result *res) {
    auto t0 = std::chrono::steady_clock::now();
    ensure_workspace(h, nf);
    ensure_f64_inputs(h, nf);
    h.L.ensure(h.A.bytes);
    h.Gl.ensure(h.A.bytes);
    Ctx c(h, (int)nf);
    Timer setup(c.s);
    upload<T>(c, A22, lda22, h.A.as<T>(), h.A64.as<double>());
    upload<T>(c, B22, ldb22, h.B.as<T>(), h.B64.as<double>());
    if (P0) upload<T>(c, P0, ldp, h.P.as<T>(), h.stage.as<double>());
    // seed blocks: [A21 | B21] (nf x m) and [A12 | B12] (m x nf), leading dim ldm / c.ld
    const int64_t ldm = round_up(std::max<int64_t>(m, 1), 8);
    DevBuf blk;
    blk.ensure(((size_t)2 * nf * ldm + (size_t)2 * m * c.ld) * sizeof(T));
    T *a21 = blk.as<T>(), *b21 = a21 + nf * ldm, *a12 = b21 + nf * ldm, *b12 = a12 + m * c.ld;
    upload_rect<T>(c, A21, lda21, (int)nf, (int)m, a21, ldm);
    upload_rect<T>(c, B21, ldb21, (int)nf, (int)m, b21, ldm);
    upload_rect<T>(c, A12, lda12, (int)m, (int)nf, a12, c.ld);
    upload_rect<T>(c, B12, ldb12, (int)m, (int)nf, b12, c.ld);
    T *L = h.L.as<T>();
    GOAT_CUDA(cudaMemsetAsync(L, 0, h.L.bytes, c.s));
    gemm_simt<T>((int)nf, (int)nf, (int)m, 1.0, a21, ldm, 0, b21, ldm, 1, 0.0, L, c.ld, c.s);  // A21 B21^T
    gemm_simt<T>((int)nf, (int)nf, (int)m, 1.0, a12, c.ld, 1, b12, c.ld, 0, 1.0, L, c.ld, c.s);  // + A12^T B12
    res->time_ms[4] = setup.stop();
    fw_loop<T>(c, true, P0 == nullptr, *o, res);
    // objective on the free block (the caller adds the seed terms, matcher.py:283)
    int *perm = h.ivec.as<int>();
    std::vector<int> ph(nf);
    for (int64_t r = 0; r < nf; ++r) ph[r] = (int)res->assignment[r];
    GOAT_CUDA(cudaMemcpyAsync(perm, ph.data(), nf * 4, cudaMemcpyHostToDevice, c.s));
    launch_qap_perm(h.A64.as<double>(), c.ld, h.B64.as<double>(), c.ld, perm, (int)nf, h.red.as<double>(),
                    h.scal.as<double>() + 40, c.s);
    GOAT_CUDA(cudaMemcpyAsync(h.h_scal + 40, h.scal.as<double>() + 40, 8, cudaMemcpyDeviceToHost, c.s));
    sync(c);
    res->objective = h.h_scal[40];
    res->time_ms[5] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

template <class T> SkArgs shard_sk_args(Handle &h, const void *G) {
    auto &S = h.sh;
    SkArgs a{};
    a.G = G; a.ld = ld_for(S.n); a.n = (int)S.n; a.m = (int)S.m;
    a.f[0] = h.f[0].as<double>(); a.f[1] = h.f[1].as<double>();
    a.g[0] = h.g[0].as<double>(); a.g[1] = h.g[1].as<double>();
    a.colpart = h.colpart.p; a.ldp = ld_for(S.n);
    a.devpart = h.devpart.as<double>(); a.devcol = h.devcol.as<double>();
    a.st = h.state.as<SkState>(); a.nblk = S.plan.nblk;
    return a;
}

}  // namespace
}  // namespace goat

using namespace goat;

struct goat_handle : goat::Handle {};

extern "C" {

const char *goat_last_error(void) { return g_last_error.c_str(); }

const char *goat_version(void) { return "goat 0.1 sm_100a (fused log-domain sinkhorn, device LSAP)"; }

int goat_create(goat_handle **out, const goat_config *cfg) {
    return guarded([&] {
        require(out != nullptr, "out must not be NULL");
        goat_config def{0, GOAT_FP64, GOAT_GEMM_AUTO, 3};
        const goat_config &c = cfg ? *cfg : def;
        require(c.precision == GOAT_FP32 || c.precision == GOAT_FP64, "precision must be GOAT_FP32 or GOAT_FP64");
        int count = 0;
        GOAT_CUDA(cudaGetDeviceCount(&count));
        require(c.device >= 0 && c.device < count, "device ordinal out of range");
        auto *h = new goat_handle();
        h->device = c.device;
        h->precision = c.precision;
        h->gemm = c.gemm;
        h->split = c.split_terms ? c.split_terms : 3;
        try {
            GOAT_CUDA(cudaSetDevice(c.device));
            GOAT_CUDA(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, c.device));
            GOAT_CUDA(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
            h->stream = h->own_stream;
            GOAT_CUDA(cudaMallocHost(&h->h_scal, 64 * sizeof(double)));
            GOAT_CUDA(cudaMallocHost(&h->h_state, sizeof(SkState)));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int goat_destroy(goat_handle *h) {
    return guarded([&] {
        if (!h) return;
        cudaSetDevice(h->device);
        cudaStreamSynchronize(h->stream);
        delete h;
    });
}

int goat_reserve(goat_handle *h, int64_t n) {
    return guarded([&] {
        require(h != nullptr, "handle must not be NULL");
        check_order(n);
        ensure_workspace(*h, n);
    });
}

int goat_fw_core(goat_handle *h, int64_t n, const double *A, int64_t lda, const double *B, int64_t ldb,
                 const double *L, int64_t ldl, const double *P0, int64_t ldp, const goat_options *opts,
                 goat_fw_result *res) {
    return guarded([&] {
        require(h && A && B && res && res->assignment && res->hist_obj && res->hist_alpha, "NULL argument");
        check_order(n);
        validate_opts(opts);
        require(lda >= n && ldb >= n && (!L || ldl >= n) && (!P0 || ldp >= n), "leading dimension < n");
        launch_count() = 0;
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            fw_core_host<T>(*h, n, A, lda, B, ldb, L, ldl, P0, ldp, opts, res);
        });
        res->gpu_launches = (int32_t)launch_count();
    });
}

int goat_fw_core_device(goat_handle *h, int64_t n, const void *dA, int64_t lda, const void *dB, int64_t ldb,
                        const void *dL, int64_t ldl, const void *dP0, int64_t ldp, const goat_options *opts,
                        goat_fw_result *res) {
    return guarded([&] {
        require(h && dA && dB && res && res->assignment && res->hist_obj && res->hist_alpha, "NULL argument");
        check_order(n);
        validate_opts(opts);
        require(lda >= n && ldb >= n && (!dL || ldl >= n) && (!dP0 || ldp >= n), "leading dimension < n");
        launch_count() = 0;
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            fw_core_dev<T>(*h, n, (const T *)dA, lda, (const T *)dB, ldb, (const T *)dL, ldl, (const T *)dP0, ldp,
                           opts, res);
        });
        res->gpu_launches = (int32_t)launch_count();
    });
}

int goat_gradient(goat_handle *h, int64_t n, const double *A, int64_t lda, const double *B, int64_t ldb,
                  const double *P, int64_t ldp, double *G, int64_t ldg) {
    return guarded([&] {
        require(h && A && B && P && G, "NULL argument");
        check_order(n);
        ensure_workspace(*h, n);
        ensure_f64_inputs(*h, n);
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            Ctx c(*h, (int)n);
            double *stage = h->stage.as<double>();
            upload<T>(c, A, lda, h->A.as<T>(), stage);
            upload<T>(c, B, ldb, h->B.as<T>(), stage);
            upload<T>(c, P, ldp, h->P.as<T>(), stage);
            c.sym = is_symmetric<T>(c, h->A.as<T>()) && is_symmetric<T>(c, h->B.as<T>());
            setup_gemm<T>(c, h->A.as<T>(), h->B.as<T>());
            gradient<T>(c, h->A.as<T>(), h->B.as<T>(), h->P.as<T>(), h->G.as<T>(), h->T1.as<T>());
            download<T>(c, h->G.as<T>(), G, ldg, stage);
        });
    });
}

static int lot_common(goat_handle *h, int64_t n, const double *M, int64_t ldm, int32_t sense, double lam,
                      int32_t max_sweeps, double tol, double *Q, int64_t ldq, int32_t *converged,
                      int32_t *sweeps, double *deviation, int mode) {
    return guarded([&] {
        require(h && M && Q, "NULL argument");
        check_order(n);
        require(sense == GOAT_MINIMIZE || sense == GOAT_MAXIMIZE, "sense must be minimize or maximize");
        require(lam > 0 && max_sweeps >= 1 && tol > 0, "invalid Sinkhorn parameters");
        ensure_workspace(*h, n);
        ensure_f64_inputs(*h, n);
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            Ctx c(*h, (int)n);
            double *stage = h->stage.as<double>();
            upload<T>(c, M, ldm, h->M.as<T>(), stage);
            const T *Gin = h->M.as<T>();
            if (mode == 1) {
                int *bad = h->ivec.as<int>();
                GOAT_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), c.s));
                launch_neglog<T>(h->M.as<T>(), c.ld, h->G.as<T>(), c.ld, (int)n, bad, c.s);
                int hb = 0;
                GOAT_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, c.s));
                sync(c);
                require(!hb, "sinkhorn_knopp requires strictly positive entries");
                Gin = h->G.as<T>();
            }
            LotOut lo = run_lot<T>(c, Gin, sense, lam, max_sweeps, tol, h->Q.as<T>(), nullptr, nullptr, mode);
            if (converged) *converged = lo.converged;
            if (sweeps) *sweeps = lo.sweeps;
            if (deviation) *deviation = lo.dev;
            if (mode == 1 && lo.sweeps == 0) {  // sinkhorn.py:71-72 returns K itself
                for (int64_t r = 0; r < n; ++r) std::memcpy(Q + r * ldq, M + r * ldm, n * 8);
            } else {
                download<T>(c, h->Q.as<T>(), Q, ldq, stage);
            }
        });
    });
}

int goat_lot(goat_handle *h, int64_t n, const double *M, int64_t ldm, int32_t sense, double lam,
             int32_t max_sweeps, double tol, double *Q, int64_t ldq, int32_t *converged, int32_t *sweeps,
             double *deviation) {
    return lot_common(h, n, M, ldm, sense, lam, max_sweeps, tol, Q, ldq, converged, sweeps, deviation, 0);
}

int goat_lot_device(goat_handle *h, int64_t n, const void *dM, int64_t ldm, int32_t sense, double lam,
                    int32_t max_sweeps, double tol, void *dQ, int64_t ldq, int32_t *converged, int32_t *sweeps,
                    double *deviation) {
    return guarded([&] {
        require(h && dM && dQ, "NULL argument");
        check_order(n);
        require(sense == GOAT_MINIMIZE || sense == GOAT_MAXIMIZE, "sense must be minimize or maximize");
        require(lam > 0 && max_sweeps >= 1 && tol > 0, "invalid Sinkhorn parameters");
        require(ldm == ld_for(n) && ldq == ld_for(n), "lot_device: leading dimensions must be round_up(n, 8)");
        require(((uintptr_t)dM & 15) == 0 && ((uintptr_t)dQ & 15) == 0, "lot_device: buffers must be 16-byte aligned");
        ensure_workspace(*h, n, false);
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            Ctx c(*h, (int)n);
            LotOut lo = run_lot<T>(c, static_cast<const T *>(dM), sense, lam, max_sweeps, tol, static_cast<T *>(dQ),
                                   nullptr, nullptr, 0);
            if (converged) *converged = lo.converged;
            if (sweeps) *sweeps = lo.sweeps;
            if (deviation) *deviation = lo.dev;
        });
    });
}

int goat_sinkhorn_knopp(goat_handle *h, int64_t n, const double *K, int64_t ldk, int32_t max_sweeps, double tol,
                        double *Q, int64_t ldq, int32_t *converged, int32_t *sweeps, double *deviation) {
    return lot_common(h, n, K, ldk, GOAT_MAXIMIZE, 1.0, max_sweeps, tol, Q, ldq, converged, sweeps, deviation, 1);
}

int goat_line_search_coeffs(goat_handle *h, int64_t n, const double *A, int64_t lda, const double *B,
                            int64_t ldb, const double *L, int64_t ldl, const double *P, int64_t ldp,
                            const double *Q, int64_t ldq, double *c2, double *c1) {
    return guarded([&] {
        require(h && A && B && P && Q && c2 && c1, "NULL argument");
        check_order(n);
        ensure_workspace(*h, n);
        ensure_f64_inputs(*h, n);
        if (L) h->L.ensure(h->A.bytes);
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            Ctx c(*h, (int)n);
            double *stage = h->stage.as<double>();
            upload<T>(c, A, lda, h->A.as<T>(), stage);
            upload<T>(c, B, ldb, h->B.as<T>(), stage);
            upload<T>(c, P, ldp, h->P.as<T>(), stage);
            upload<T>(c, Q, ldq, h->Q.as<T>(), stage);
            T *Ld = nullptr;
            if (L) { upload<T>(c, L, ldl, h->L.as<T>(), stage); Ld = h->L.as<T>(); }
            c.sym = is_symmetric<T>(c, h->A.as<T>()) && is_symmetric<T>(c, h->B.as<T>());
            setup_gemm<T>(c, h->A.as<T>(), h->B.as<T>());
            gradient<T>(c, h->A.as<T>(), h->B.as<T>(), h->P.as<T>(), h->G.as<T>(), h->T1.as<T>());
            gradient<T>(c, h->A.as<T>(), h->B.as<T>(), h->Q.as<T>(), h->GQ.as<T>(), h->T1.as<T>());
            double *d = h->scal.as<double>() + 16;
            launch_fw_dots<T>(h->G.as<T>(), h->GQ.as<T>(), h->P.as<T>(), h->Q.as<T>(), Ld, c.ld, (int)n,
                              h->red.as<double>(), d, c.s);
            GOAT_CUDA(cudaMemcpyAsync(h->h_scal + 16, d, 6 * 8, cudaMemcpyDeviceToHost, c.s));
            sync(c);
            *c2 = 0.5 * h->h_scal[17];
            *c1 = h->h_scal[16] + (L ? h->h_scal[20] : 0.0);
        });
    });
}

int goat_set_stream(goat_handle *h, void *stream) {
    return guarded([&] {
        require(h != nullptr, "handle must not be NULL");
        h->stream = stream ? static_cast<cudaStream_t>(stream) : h->own_stream;
    });
}

int goat_bench_sweep(goat_handle *h, int64_t n, const void *dG, int64_t ld, int32_t reps, double *ms_per_sweep) {
    return guarded([&] {
        require(h && dG && ms_per_sweep && reps >= 1, "bad argument");
        require(ld >= n && ld % 8 == 0 && ((uintptr_t)dG & 15) == 0, "bench_sweep: ld must be a multiple of 8, G 16-byte aligned");
        check_order(n);
        ensure_workspace(*h, n);
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            Ctx c(*h, (int)n);
            SkPlan plan = sk_plan<T>((int)n, h->num_sms);
            SkArgs a{};
            a.G = dG; a.ld = ld; a.n = (int)n;
            a.f[0] = h->f[0].as<double>(); a.f[1] = h->f[1].as<double>();
            a.g[0] = h->g[0].as<double>(); a.g[1] = h->g[1].as<double>();
            a.colpart = h->colpart.p; a.ldp = ld_for(n);
            a.devpart = h->devpart.as<double>(); a.devcol = h->devcol.as<double>();
            a.st = h->state.as<SkState>(); a.nblk = plan.nblk;
            GOAT_CUDA(cudaMemsetAsync(h->f[0].p, 0, c.ld * 8, c.s));
            GOAT_CUDA(cudaMemsetAsync(h->f[1].p, 0, c.ld * 8, c.s));
            GOAT_CUDA(cudaMemsetAsync(h->g[0].p, 0, c.ld * 8, c.s));
            GOAT_CUDA(cudaMemsetAsync(h->g[1].p, 0, c.ld * 8, c.s));
            // A LOT that cannot converge (tol ~ 0): pre-check + `reps` sweeps +
            // the row-only pass, exactly the in-situ work of the production loop.
            SkState st{};
            st.k = 0;
            // E = -(100 - G) in [-100, 0] for G in [0, 100): the lam = 100 unit-range
            // Gibbs exponent of the production loop (sinkhorn.py:125).
            st.gmax = 100.0; st.coef = -1.0; st.tol = 1e-300; st.max_sweeps = reps;
            *h->h_state = st;
            auto run = [&] {
                GOAT_CUDA(cudaMemcpyAsync(a.st, h->h_state, sizeof(SkState), cudaMemcpyHostToDevice, c.s));
                if (plan.persistent) {
                    sk_launch_persistent<T>(a, plan, h->bar.as<unsigned>(), c.s);
                } else {
                    for (int r = 0; r < reps + 2; ++r) {
                        sk_launch_pass<T>(a, plan, c.s);
                        sk_launch_merge<T>(a, plan, c.s);
                    }
                }
            };
            run();  // warm
            if (const char *tk = getenv("GOAT_SK_TRACE")) {
                // diagnostics: per-CTA phase stamps of one sweep, summarised on stderr
                const int nb = plan.nblk;
                DevBuf tb;
                tb.ensure((size_t)nb * 16 * sizeof(unsigned long long));
                GOAT_CUDA(cudaMemsetAsync(tb.p, 0, (size_t)nb * 128, c.s));
                a.trace = tb.as<unsigned long long>();
                a.trace_k = atoi(tk);
                run();
                GOAT_CUDA(cudaStreamSynchronize(c.s));
                std::vector<unsigned long long> t((size_t)nb * 16);
                GOAT_CUDA(cudaMemcpy(t.data(), tb.p, t.size() * 8, cudaMemcpyDeviceToHost));
                unsigned long long t0 = ~0ull;
                for (int b = 0; b < nb; ++b) if (t[b * 16]) t0 = std::min(t0, t[b * 16]);
                if (getenv("GOAT_SK_TRACE_RAW")) t0 = 0;  // accumulated phase cycles, not stamps
                fprintf(stderr, "sk_trace n=%d nblk=%d cl=%d stages=%d (ns after first pass start): stamp min/median/max\n", (int)n, nb, plan.cl, plan.stages);
                for (int i = 0; i < 16; ++i) {
                    std::vector<double> v;
                    for (int b = 0; b < nb; ++b) if (t[b * 16 + i]) v.push_back((double)(t[b * 16 + i] - t0));
                    if (v.empty()) continue;
                    std::sort(v.begin(), v.end());
                    fprintf(stderr, "  stamp %d: %8.0f %8.0f %8.0f\n", i, v.front(), v[v.size() / 2], v.back());
                }
                a.trace = nullptr;
                a.trace_k = -1;
            }
            cudaEvent_t e0, e1;
            GOAT_CUDA(cudaEventCreate(&e0));
            GOAT_CUDA(cudaEventCreate(&e1));
            GOAT_CUDA(cudaEventRecord(e0, c.s));
            run();
            GOAT_CUDA(cudaEventRecord(e1, c.s));
            GOAT_CUDA(cudaEventSynchronize(e1));
            float ms = 0;
            GOAT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            *ms_per_sweep = ms / (reps + 2);
            if (getenv("GOAT_SK_VERBOSE")) {
                GOAT_CUDA(cudaMemcpy(h->h_state, a.st, sizeof(SkState), cudaMemcpyDeviceToHost));
                fprintf(stderr, "bench_sweep n=%d cl=%d ch=%d pipe=%d stages=%d sweeps=%d redone=%d\n", (int)n, plan.cl,
                        plan.ch, (int)plan.pipe, plan.stages, h->h_state->sweeps, h->h_state->redone);
            }
        });
    });
}

int goat_bench_gradient(goat_handle *h, int64_t n, const void *dA, const void *dB, const void *dX, int32_t reps,
                        double *ms, int32_t *products, int32_t *terms) {
    return guarded([&] {
        require(h && dA && dB && dX && ms && reps >= 1, "bad argument");
        check_order(n);
        ensure_workspace(*h, n);
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            Ctx c(*h, (int)n);
            const size_t es = sizeof(T);
            auto cp = [&](const void *src, T *dst) {
                GOAT_CUDA(cudaMemcpy2DAsync(dst, c.ld * es, src, n * es, n * es, n, cudaMemcpyDeviceToDevice, c.s));
            };
            GOAT_CUDA(cudaMemsetAsync(h->A.p, 0, h->A.bytes, c.s));
            GOAT_CUDA(cudaMemsetAsync(h->B.p, 0, h->B.bytes, c.s));
            GOAT_CUDA(cudaMemsetAsync(h->P.p, 0, h->P.bytes, c.s));
            cp(dA, h->A.as<T>());
            cp(dB, h->B.as<T>());
            cp(dX, h->P.as<T>());
            c.sym = is_symmetric<T>(c, h->A.as<T>()) && is_symmetric<T>(c, h->B.as<T>());
            setup_gemm<T>(c, h->A.as<T>(), h->B.as<T>());
            gradient<T>(c, h->A.as<T>(), h->B.as<T>(), h->P.as<T>(), h->G.as<T>(), h->T1.as<T>());  // warm
            cudaEvent_t e0, e1;
            GOAT_CUDA(cudaEventCreate(&e0));
            GOAT_CUDA(cudaEventCreate(&e1));
            GOAT_CUDA(cudaEventRecord(e0, c.s));
            for (int r = 0; r < reps; ++r)
                gradient<T>(c, h->A.as<T>(), h->B.as<T>(), h->P.as<T>(), h->G.as<T>(), h->T1.as<T>());
            GOAT_CUDA(cudaEventRecord(e1, c.s));
            GOAT_CUDA(cudaEventSynchronize(e1));
            float t = 0;
            GOAT_CUDA(cudaEventElapsedTime(&t, e0, e1));
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            *ms = t / reps;
            if (products) *products = c.sym ? 2 : 4;
            if (terms) *terms = c.tc ? std::max(h->tc_na, h->split) : 0;
        });
    });
}

int goat_lap(goat_handle *h, int64_t n, const double *M, int64_t ldm, int32_t sense, int64_t *assignment,
             double *objective, int32_t *certified) {
    return guarded([&] {
        require(h && M && assignment, "NULL argument");
        check_order(n);
        require(sense == GOAT_MINIMIZE || sense == GOAT_MAXIMIZE, "sense must be minimize or maximize");
        ensure_workspace(*h, n);
        ensure_f64_inputs(*h, n);
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            Ctx c(*h, (int)n);
            upload<T>(c, M, ldm, h->M.as<T>(), h->stage.as<double>());
            std::vector<int> ph;
            const int cert = run_lap<T>(c, h->M.as<T>(), sense, h->ivec.as<int>(), ph);
            if (certified) *certified = cert;
            double obj = 0.0;
            for (int64_t r = 0; r < n; ++r) {
                assignment[r] = ph[r];
                obj += M[r * ldm + ph[r]];
            }
            if (objective) *objective = obj;
        });
    });
}

int goat_qap_objective_perm(goat_handle *h, int64_t n, const double *A, int64_t lda, const double *B,
                            int64_t ldb, const int64_t *perm, double *objective) {
    return guarded([&] {
        require(h && A && B && perm && objective, "NULL argument");
        check_order(n);
        ensure_workspace(*h, n);
        ensure_f64_inputs(*h, n);
        std::vector<int> ph(n);
        std::vector<char> seen(n, 0);
        for (int64_t r = 0; r < n; ++r) {
            require(perm[r] >= 0 && perm[r] < n && !seen[perm[r]], "permutation is not a bijection");
            seen[perm[r]] = 1;
            ph[r] = (int)perm[r];
        }
        Ctx c(*h, (int)n);
        GOAT_CUDA(cudaMemcpy2DAsync(h->A64.p, c.ld * 8, A, lda * 8, n * 8, n, cudaMemcpyHostToDevice, c.s));
        GOAT_CUDA(cudaMemcpy2DAsync(h->B64.p, c.ld * 8, B, ldb * 8, n * 8, n, cudaMemcpyHostToDevice, c.s));
        int *pd = h->ivec.as<int>();
        GOAT_CUDA(cudaMemcpyAsync(pd, ph.data(), n * 4, cudaMemcpyHostToDevice, c.s));
        launch_qap_perm(h->A64.as<double>(), c.ld, h->B64.as<double>(), c.ld, pd, (int)n, h->red.as<double>(),
                        h->scal.as<double>() + 40, c.s);
        GOAT_CUDA(cudaMemcpyAsync(h->h_scal + 40, h->scal.as<double>() + 40, 8, cudaMemcpyDeviceToHost, c.s));
        sync(c);
        *objective = h->h_scal[40];
    });
}


// ------------------------------------------------------------------ row-sharded C ABI
static goat::Handle::Shard &shard_of(goat_handle *h) {
    require(h && h->sh.ready, "goat_shard_setup has not been called on this handle");
    return h->sh;
}

int goat_shard_setup(goat_handle *h, int64_t n, int64_t m, const void *dA_rows, const void *dAT_rows,
                     const void *dB, int64_t ld) {
    return guarded([&] {
        require(h && dA_rows && dB, "NULL argument");
        check_order(n);
        require(m >= 1 && m <= n, "block rows must be in [1, n]");
        require(ld >= n, "leading dimension < n");
        ensure_workspace(*h, n, false);
        auto &S = h->sh;
        S.ready = false;
        S.n = n; S.m = m; S.sym = (dAT_rows == nullptr); S.fill = false; S.csr = false;
        const int64_t lw = ld_for(n);
        const size_t es = h->precision == GOAT_FP32 ? 4 : 8;
        cudaStream_t s = h->stream;
        auto put = [&](DevBuf &dst, const void *src, int64_t rows) {
            dst.ensure((size_t)rows * lw * es);
            GOAT_CUDA(cudaMemsetAsync(dst.p, 0, (size_t)rows * lw * es, s));
            GOAT_CUDA(cudaMemcpy2DAsync(dst.p, lw * es, src, ld * es, n * es, rows, cudaMemcpyDeviceToDevice, s));
        };
        put(S.A, dA_rows, m);
        if (!S.sym) put(S.AT, dAT_rows, m);
        put(S.B, dB, n);
        S.X.ensure((size_t)m * lw * es);
        S.tc = h->precision == GOAT_FP32 && h->gemm != GOAT_GEMM_SIMT;
        if (S.tc) shard_tc_prepare(*h);
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            S.plan = sk_plan<T>((int)n, h->num_sms, (int)m, true);
        });
        h->colpart.ensure(S.plan.colpart_bytes);
        S.bad.ensure((size_t)ld_for(n));
        GOAT_CUDA(cudaStreamSynchronize(s));
        S.ready = true;
    });
}

int goat_shard_setup_csr(goat_handle *h, int64_t n, int64_t m, const goat_csr *dA_rows, const goat_csr *dAT_rows,
                         const goat_csr *dB, const goat_csr *dBT) {
    return guarded([&] {
        require(h && dA_rows && dB && (!dAT_rows) == (!dBT), "NULL argument (A^T rows and B^T go together)");
        check_order(n);
        require(m >= 1 && m <= n, "block rows must be in [1, n]");
        ensure_workspace(*h, n, false);
        auto &S = h->sh;
        S.ready = false;
        S.n = n; S.m = m; S.sym = (dAT_rows == nullptr); S.fill = false; S.csr = true; S.tc = false;
        const size_t es = h->precision == GOAT_FP32 ? 4 : 8;
        cudaStream_t s = h->stream;
        auto put = [&](Handle::Csr &dst, const goat_csr &src, int64_t rows) {
            const int64_t nnz = src.nnz;
            require(nnz >= 0 && src.rowptr && (nnz == 0 || src.colidx), "csr: NULL rowptr/colidx");
            dst.rowptr.ensure((size_t)(rows + 1) * 8);
            dst.col.ensure((size_t)std::max<int64_t>(nnz, 1) * 4);
            dst.nnz = nnz;
            dst.has_val = src.values != nullptr;
            GOAT_CUDA(cudaMemcpyAsync(dst.rowptr.p, src.rowptr, (size_t)(rows + 1) * 8, cudaMemcpyDeviceToDevice, s));
            if (nnz) GOAT_CUDA(cudaMemcpyAsync(dst.col.p, src.colidx, (size_t)nnz * 4, cudaMemcpyDeviceToDevice, s));
            if (dst.has_val) {
                dst.val.ensure((size_t)std::max<int64_t>(nnz, 1) * es);
                if (nnz) GOAT_CUDA(cudaMemcpyAsync(dst.val.p, src.values, (size_t)nnz * es, cudaMemcpyDeviceToDevice, s));
            }
            int *flag = h->ivec.as<int>();
            const int one = 1;
            GOAT_CUDA(cudaMemcpyAsync(flag, &one, sizeof(int), cudaMemcpyHostToDevice, s));
            dispatch(*h, [&](auto *tag) {
                using T = std::remove_pointer_t<decltype(tag)>;
                launch_csr_check<T>(csr_view<T>(dst), (int)rows, (int)n, flag, s);
            });
            int ok = 0;
            GOAT_CUDA(cudaMemcpyAsync(&ok, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
            GOAT_CUDA(cudaStreamSynchronize(s));
            require(ok == 1, "csr: rows must hold strictly increasing column indices in [0, n) and finite values");
        };
        put(h->shB, *dB, n);
        if (!S.sym) put(h->shBT, *dBT, n);
        put(h->shA, *dA_rows, m);  // m rows over n columns
        if (!S.sym) put(h->shAT, *dAT_rows, m);
        const int64_t ldm = ld_for(m);
        S.X.ensure((size_t)2 * n * ldm * es);
        GOAT_CUDA(cudaMemsetAsync(S.X.p, 0, S.X.bytes, s));
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            S.plan = sk_plan<T>((int)n, h->num_sms, (int)m, true);
        });
        h->colpart.ensure(S.plan.colpart_bytes);
        S.bad.ensure((size_t)ld_for(n));
        GOAT_CUDA(cudaStreamSynchronize(s));
        S.ready = true;
    });
}

int goat_shard_gradient(goat_handle *h, const void *dQ_full, void *dOut_rows) {
    return guarded([&] {
        shard_of(h);
        require(dQ_full && dOut_rows, "NULL argument");
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            shard_gradient<T>(*h, static_cast<const T *>(dQ_full), static_cast<T *>(dOut_rows));
        });
        GOAT_CHECK_LAUNCH();
    });
}

int goat_shard_minmax(goat_handle *h, const void *dX_rows, double *out2) {
    return guarded([&] {
        auto &S = shard_of(h);
        require(dX_rows && out2, "NULL argument");
        double *mm = h->scal.as<double>();
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            launch_minmax<T>(static_cast<const T *>(dX_rows), ld_for(S.n), (int)S.n, h->red.as<double>(), mm,
                             h->stream, (int)S.m);
        });
        GOAT_CUDA(cudaMemcpyAsync(h->h_scal, mm, 16, cudaMemcpyDeviceToHost, h->stream));
        GOAT_CUDA(cudaStreamSynchronize(h->stream));
        out2[0] = h->h_scal[0];
        out2[1] = h->h_scal[1];
    });
}

int goat_shard_lot_begin(goat_handle *h, int32_t sense, double lam, double gmin, double gmax, int32_t max_sweeps,
                         double tol) {
    return guarded([&] {
        auto &S = shard_of(h);
        require(sense == GOAT_MINIMIZE || sense == GOAT_MAXIMIZE, "bad objective sense");
        require(lam > 0 && tol > 0 && max_sweeps >= 1, "bad Sinkhorn parameters");
        const double scale = gmax - gmin;  // sinkhorn.py:115-119, global over all ranks
        SkState st0{};
        S.fill = (scale == 0.0);           // sinkhorn.py:121-124: exact barycenter
        if (S.fill) {
            st0.done = 1; st0.sweeps = 0; st0.converged = 1; st0.dev = 0.0;
        } else {
            const bool maximize = (sense == GOAT_MAXIMIZE);
            st0.gmax = maximize ? gmax : gmin;
            st0.coef = maximize ? -lam / scale : lam / scale;
            st0.log_mode = !(std::exp((-lam / scale) * scale) > 0.0);
            st0.k = st0.log_mode ? 1 : 0;
            const bool finish64 = h->precision == GOAT_FP32 && tol < fp32_dev_floor() && fp64_finish_enabled();
            st0.tol = finish64 ? fp32_dev_floor() : tol;
            st0.max_sweeps = max_sweeps;
        }
        S.user_tol = tol;
        S.phase64 = false;
        const int64_t lw = ld_for(S.n);
        GOAT_CUDA(cudaMemsetAsync(h->f[0].p, 0, lw * 8, h->stream));
        GOAT_CUDA(cudaMemsetAsync(h->g[0].p, 0, lw * 8, h->stream));
        *h->h_state = st0;
        GOAT_CUDA(cudaMemcpyAsync(h->state.p, h->h_state, sizeof(SkState), cudaMemcpyHostToDevice, h->stream));
    });
}

int goat_shard_lot_pass(goat_handle *h, const void *dG_rows, double *dSend) {
    return guarded([&] {
        auto &S = shard_of(h);
        require(dG_rows && dSend, "NULL argument");
        if (S.phase64) {
            SkArgs a = shard_sk_args<double>(*h, S.G64.p);
            a.nblk = S.plan64.nblk;
            sk_launch_shard_pass<double>(a, S.plan64, h->bar.as<unsigned>(), dSend, h->stream);
            return;
        }
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            SkArgs a = shard_sk_args<T>(*h, dG_rows);
            sk_launch_shard_pass<T>(a, S.plan, h->bar.as<unsigned>(), dSend, h->stream);
        });
    });
}

int goat_shard_lot_merge(goat_handle *h, const double *dRecv, int32_t world) {
    return guarded([&] {
        auto &S = shard_of(h);
        require(dRecv && world >= 1, "bad argument");
        if (S.phase64) {
            SkArgs a = shard_sk_args<double>(*h, nullptr);
            sk_launch_shard_merge<double>(a, dRecv, world, S.bad.as<unsigned char>(), h->stream);
            return;
        }
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            SkArgs a = shard_sk_args<T>(*h, nullptr);
            sk_launch_shard_merge<T>(a, dRecv, world, h->sh.bad.as<unsigned char>(), h->stream);
        });
    });
}

int goat_shard_lot_repair_pass(goat_handle *h, const void *dG_rows, double *dPairs) {
    return guarded([&] {
        auto &S = shard_of(h);
        require(dG_rows && dPairs, "NULL argument");
        if (S.phase64) {
            SkArgs a = shard_sk_args<double>(*h, S.G64.p);
            sk_launch_shard_repair_pass<double>(a, S.bad.as<unsigned char>(), dPairs, h->stream);
            return;
        }
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            SkArgs a = shard_sk_args<T>(*h, dG_rows);
            sk_launch_shard_repair_pass<T>(a, h->sh.bad.as<unsigned char>(), dPairs, h->stream);
        });
    });
}

int goat_shard_lot_repair_merge(goat_handle *h, const double *dRecvPairs, int32_t world) {
    return guarded([&] {
        shard_of(h);
        require(dRecvPairs && world >= 1, "bad argument");
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            SkArgs a = shard_sk_args<T>(*h, nullptr);
            sk_launch_shard_repair_merge(a, dRecvPairs, world, h->sh.bad.as<unsigned char>(), h->stream);
        });
    });
}

int goat_shard_lot_refine(goat_handle *h, const void *dG_rows, int32_t *started) {
    return guarded([&] {
        auto &S = shard_of(h);
        require(dG_rows && started, "NULL argument");
        *started = 0;
        if (h->precision != GOAT_FP32 || S.fill || S.phase64) return;
        GOAT_CUDA(cudaMemcpyAsync(h->h_state, h->state.p, sizeof(SkState), cudaMemcpyDeviceToHost, h->stream));
        GOAT_CUDA(cudaStreamSynchronize(h->stream));
        SkState st = *h->h_state;
        // the fp32 sweeps stopped at the floor (run_lot: same re-entry rule)
        if (!(st.done && st.converged && S.user_tol < st.tol)) return;
        const int64_t ld = ld_for(S.n);
        S.G64.ensure((size_t)S.m * ld * sizeof(double));
        launch_convert_to_f64<float>(static_cast<const float *>(dG_rows), ld, S.G64.as<double>(), ld, (int)S.n,
                                     h->stream, (int)S.m);
        S.plan64 = sk_plan<double>((int)S.n, h->num_sms, (int)S.m, true);
        h->colpart.ensure(S.plan64.colpart_bytes);
        const int swept = st.sweeps;
        st.done = 0; st.converged = 0; st.pending = 0; st.tol = S.user_tol;
        if (swept > 0) { st.k = swept; st.nostop_k = swept; }
        else {
            st.k = st.log_mode ? 1 : 0;
            GOAT_CUDA(cudaMemsetAsync(h->f[0].p, 0, ld * 8, h->stream));
            GOAT_CUDA(cudaMemsetAsync(h->g[0].p, 0, ld * 8, h->stream));
        }
        *h->h_state = st;
        GOAT_CUDA(cudaMemcpyAsync(h->state.p, h->h_state, sizeof(SkState), cudaMemcpyHostToDevice, h->stream));
        GOAT_CUDA(cudaStreamSynchronize(h->stream));
        S.phase64 = true;
        *started = 1;
    });
}

int goat_shard_lot_status(goat_handle *h, int32_t *done, int32_t *sweeps, int32_t *converged, double *deviation,
                          int32_t *repaired, int32_t *pending) {
    return guarded([&] {
        shard_of(h);
        GOAT_CUDA(cudaMemcpyAsync(h->h_state, h->state.p, sizeof(SkState), cudaMemcpyDeviceToHost, h->stream));
        GOAT_CUDA(cudaStreamSynchronize(h->stream));
        const SkState &st = *h->h_state;
        if (done) *done = st.done;
        if (sweeps) *sweeps = st.sweeps;
        if (converged) *converged = st.converged;
        if (deviation) *deviation = st.dev;
        if (repaired) *repaired = st.repaired;
        if (pending) *pending = st.pending;
    });
}

int goat_shard_lot_emit(goat_handle *h, const void *dG_rows, void *dQ_rows) {
    return guarded([&] {
        auto &S = shard_of(h);
        require(dG_rows && dQ_rows, "NULL argument");
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            if (S.fill) {
                launch_fill<T>(static_cast<T *>(dQ_rows), ld_for(S.n), (int)S.n, 1.0 / (double)S.n, h->stream, (int)S.m);
            } else {
                SkArgs a = shard_sk_args<T>(*h, dG_rows);
                sk_launch_emit<T>(a, static_cast<T *>(dQ_rows), ld_for(S.n), nullptr, 0, nullptr, 0,
                                  h->red.as<double>(), kRedBlocks, h->stream);
            }
        });
    });
}

int goat_shard_dots(goat_handle *h, const void *GP, const void *GQ, const void *P, const void *Q, double *out6) {
    return guarded([&] {
        auto &S = shard_of(h);
        require(GP && GQ && P && Q && out6, "NULL argument");
        double *dots = h->scal.as<double>() + 16;
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            launch_fw_dots<T>(static_cast<const T *>(GP), static_cast<const T *>(GQ), static_cast<const T *>(P),
                              static_cast<const T *>(Q), nullptr, ld_for(S.n), (int)S.n, h->red.as<double>(), dots,
                              h->stream, (int)S.m);
        });
        GOAT_CUDA(cudaMemcpyAsync(h->h_scal + 16, dots, 6 * 8, cudaMemcpyDeviceToHost, h->stream));
        GOAT_CUDA(cudaStreamSynchronize(h->stream));
        for (int q = 0; q < 6; ++q) out6[q] = h->h_scal[16 + q];
    });
}

int goat_shard_axpby(goat_handle *h, double a, const void *dX_rows, double b, void *dY_rows) {
    return guarded([&] {
        auto &S = shard_of(h);
        require(dX_rows && dY_rows, "NULL argument");
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            launch_axpby<T>(a, static_cast<const T *>(dX_rows), b, static_cast<T *>(dY_rows), ld_for(S.n), (int)S.n,
                            h->stream, (int)S.m);
        });
    });
}

int goat_shard_fill(goat_handle *h, double value, void *dX_rows) {
    return guarded([&] {
        auto &S = shard_of(h);
        require(dX_rows, "NULL argument");
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            launch_fill<T>(static_cast<T *>(dX_rows), ld_for(S.n), (int)S.n, value, h->stream, (int)S.m);
        });
    });
}

int goat_lap_device(goat_handle *h, int64_t n, const void *dM, int64_t ldm, int32_t sense, int64_t *assignment,
                    double *objective, int32_t *certified) {
    return guarded([&] {
        require(h && dM && assignment, "NULL argument");
        check_order(n);
        require(ldm >= n, "leading dimension < n");
        require(sense == GOAT_MINIMIZE || sense == GOAT_MAXIMIZE, "sense must be minimize or maximize");
        ensure_workspace(*h, n, false);
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            Ctx c(*h, (int)n);
            const size_t es = sizeof(T);
            h->M.ensure((size_t)n * c.ld * es);
            GOAT_CUDA(cudaMemsetAsync(h->M.p, 0, (size_t)n * c.ld * es, c.s));
            GOAT_CUDA(cudaMemcpy2DAsync(h->M.p, c.ld * es, dM, ldm * es, n * es, n, cudaMemcpyDeviceToDevice, c.s));
            std::vector<int> ph;
            const int cert = run_lap<T>(c, h->M.as<T>(), sense, h->ivec.as<int>(), ph);
            if (certified) *certified = cert;
            for (int64_t r = 0; r < n; ++r) assignment[r] = ph[r];
            if (objective) {
                double *o = h->scal.as<double>() + 56;
                const bool f32 = std::is_same<T, float>::value;
                assign_sum_kernel<<<1, 1024, 0, c.s>>>(f32 ? (const float *)h->M.p : nullptr,
                                                       f32 ? nullptr : (const double *)h->M.p, c.ld,
                                                       h->ivec.as<int>(), (int)n, o);
                note_launch();
                GOAT_CUDA(cudaMemcpyAsync(h->h_scal + 56, o, 8, cudaMemcpyDeviceToHost, c.s));
                sync(c);
                *objective = h->h_scal[56];
            }
        });
    });
}


int goat_fw_core_csr(goat_handle *h, int64_t n, const goat_csr *A, const goat_csr *B, const double *L, int64_t ldl,
                     const double *P0, int64_t ldp, const goat_options *opts, goat_fw_result *res) {
    return guarded([&] {
        require(h && A && B && res && res->assignment && res->hist_obj && res->hist_alpha, "NULL argument");
        check_order(n);
        validate_opts(opts);
        require((!L || ldl >= n) && (!P0 || ldp >= n), "leading dimension < n");
        launch_count() = 0;
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            fw_core_csr<T>(*h, n, *A, *B, false, L, ldl, P0, ldp, opts, res);
        });
        res->gpu_launches = (int32_t)launch_count();
    });
}

int goat_fw_core_csr_device(goat_handle *h, int64_t n, const goat_csr *dA, const goat_csr *dB, const void *dL,
                            int64_t ldl, const void *dP0, int64_t ldp, const goat_options *opts,
                            goat_fw_result *res) {
    return guarded([&] {
        require(h && dA && dB && res && res->assignment && res->hist_obj && res->hist_alpha, "NULL argument");
        check_order(n);
        validate_opts(opts);
        require((!dL || ldl >= n) && (!dP0 || ldp >= n), "leading dimension < n");
        launch_count() = 0;
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            fw_core_csr<T>(*h, n, *dA, *dB, true, dL, ldl, dP0, ldp, opts, res);
        });
        res->gpu_launches = (int32_t)launch_count();
    });
}

int goat_gradient_csr(goat_handle *h, int64_t n, const goat_csr *A, const goat_csr *B, const double *P, int64_t ldp,
                      double *G, int64_t ldg) {
    return guarded([&] {
        require(h && A && B && P && G, "NULL argument");
        check_order(n);
        require(ldp >= n && ldg >= n, "leading dimension < n");
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            csr_setup<T>(*h, (int)n, *A, *B, false);
            h->stage.ensure((size_t)n * ld_for(n) * 8);
            Ctx c(*h, (int)n);
            c.csr = true;
            c.sym = h->csr_sym;
            double *stage = h->stage.as<double>();
            upload<T>(c, P, ldp, h->P.as<T>(), stage);
            gradient<T>(c, (const T *)nullptr, (const T *)nullptr, h->P.as<T>(), h->G.as<T>(), h->T1.as<T>());
            download<T>(c, h->G.as<T>(), G, ldg, stage);
        });
    });
}

int goat_bench_gradient_csr(goat_handle *h, int64_t n, const goat_csr *dA, const goat_csr *dB, const void *dX,
                            int32_t reps, double *ms) {
    return guarded([&] {
        require(h && dA && dB && dX && ms && reps >= 1, "NULL argument");
        check_order(n);
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            csr_setup<T>(*h, (int)n, *dA, *dB, true);
            Ctx c(*h, (int)n);
            c.csr = true;
            c.sym = h->csr_sym;
            const size_t es = sizeof(T);
            GOAT_CUDA(cudaMemcpy2DAsync(h->P.p, c.ld * es, dX, n * es, n * es, n, cudaMemcpyDeviceToDevice, c.s));
            gradient<T>(c, (const T *)nullptr, (const T *)nullptr, h->P.as<T>(), h->G.as<T>(), h->T1.as<T>());
            Timer tm(c.s);
            for (int r = 0; r < reps; ++r)
                gradient<T>(c, (const T *)nullptr, (const T *)nullptr, h->P.as<T>(), h->G.as<T>(), h->T1.as<T>());
            *ms = tm.stop() / reps;
        });
    });
}


int goat_fw_core_seeded(goat_handle *h, int64_t nf, int64_t m, const double *A22, int64_t lda22, const double *B22,
                        int64_t ldb22, const double *A21, int64_t lda21, const double *A12, int64_t lda12,
                        const double *B21, int64_t ldb21, const double *B12, int64_t ldb12, const double *P0,
                        int64_t ldp, const goat_options *opts, goat_fw_result *res) {
    return guarded([&] {
        require(h && A22 && B22 && res && res->assignment && res->hist_obj && res->hist_alpha, "NULL argument");
        require(m >= 1 && A21 && A12 && B21 && B12, "seed blocks must be given (m >= 1)");
        check_order(nf);
        validate_opts(opts);
        require(lda22 >= nf && ldb22 >= nf && lda21 >= m && ldb21 >= m && lda12 >= nf && ldb12 >= nf &&
                    (!P0 || ldp >= nf),
                "leading dimension too small");
        launch_count() = 0;
        dispatch(*h, [&](auto *tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            fw_core_seeded<T>(*h, nf, m, A22, lda22, B22, ldb22, A21, lda21, A12, lda12, B21, ldb21, B12, ldb12,
                              P0, ldp, opts, res);
        });
        res->gpu_launches = (int32_t)launch_count();
    });
}

}  // extern "C"
