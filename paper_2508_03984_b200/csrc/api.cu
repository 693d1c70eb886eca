// C-ABI implementation: context, workspace and the stage pipeline of
// emulate<T> (reference: emulator.cpp:25-78):
//
//   validate (emulator.cpp:12-23)            host checks + device finite flag
//   [FP32 precision on FP64 data: round]     emulator.cpp:84-91
//   K1a scale  (scaling.cpp)                 row/col stats -> exponents
//   K1b truncate + residues (residue.cpp)    int8 K-major planes
//   K2  N residue GEMMs + mod epilogue       tcgen05 kind::i8 -> uint8 U_i
//   K3  accumulate, CRT reduce, unscale      FP64/FP32 C (+ alpha/beta)
//
// The pipeline is organised by column blocks of B and C (nu is
// column-local, mu depends on A — fast mode — or on a max over all columns —
// accurate mode). The device API runs one block; the host API runs several so
// the H2D copy of B block j+1 and the D2H copy of C block j-1 overlap the
// compute of block j on separate streams. Results do not depend on the
// blocking (every stage is column-local apart from the accurate row bound,
// which is an exact max).
//
// Nothing here computes on the CPU: the host validates arguments, sizes the
// workspace and launches kernels. Without a usable CUDA device every compute
// entry point fails with OZK_CUDA_ERROR (no fallback).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include <algorithm>
#include <cstdlib>

#include "ozaki2_b200.h"
#include <nvtx3/nvToolsExt.h>

#include "ozk_internal.h"

namespace ozk {

namespace {
thread_local std::string g_error;

struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
};
}  // namespace

void set_error(const std::string& msg) { g_error = msg; }

unsigned long long* k3_replay_counter(bool create);  // k3_tc.cu

int fast_floor_host(float pp_fast, double ub) {
    // scaling.cpp:50-52, same operations and order (compiled with -ffp-contract=off)
    const double t = std::max(1.0, 0.51 * std::log2(ub));
    return static_cast<int>(std::floor(static_cast<double>(pp_fast) - t));
}

// The step table of fast_floor_host over ub in [1, 2^48] (ub = sum_upper_bound
// of a line's scaled sum of squares: 1 <= ub < 4 (k + 2) for k < 2^31): each
// threshold is the smallest double at which the floor drops, found by
// bisection on the (monotone) bit patterns of positive doubles. Cached per
// pp_fast (the tables of every modulus count share few values).
FastFloorTable fast_floor_table(float pp_fast) {
    static std::mutex mu;
    static std::vector<std::pair<float, FastFloorTable>> cache;
    std::lock_guard<std::mutex> lock(mu);
    for (const auto& e : cache)
        if (std::memcmp(&e.first, &pp_fast, sizeof(float)) == 0) return e.second;
    FastFloorTable T{};
    T.floor0 = fast_floor_host(pp_fast, 1.0);
    auto bits = [](double x) {
        uint64_t u;
        std::memcpy(&u, &x, 8);
        return u;
    };
    auto from = [](uint64_t u) {
        double x;
        std::memcpy(&x, &u, 8);
        return x;
    };
    const uint64_t top = bits(0x1.0p48);
    uint64_t lo = bits(1.0);
    for (int level = T.floor0 - 1; T.n < 24; --level) {
        if (fast_floor_host(pp_fast, from(top)) > level) break;
        uint64_t a = lo, b = top;  // floor(a) > level >= floor(b)
        while (b - a > 1) {
            const uint64_t mid = a + (b - a) / 2;
            if (fast_floor_host(pp_fast, from(mid)) > level)
                a = mid;
            else
                b = mid;
        }
        T.thr[T.n++] = from(b);
        lo = b;
    }
    cache.push_back({pp_fast, T});
    return T;
}

DevConsts to_dev(const ozk_constants& c) {
    DevConsts d{};
    d.n = c.n_moduli;
    d.precision = c.precision;
    for (int i = 0; i < c.n_moduli; ++i) {
        d.p[i] = c.moduli[i];
        d.pinv_mulhi[i] = c.pinv_mulhi[i];
        d.pinv64[i] = c.pinv64[i];
        d.pinv32[i] = c.pinv32[i];
        d.s1[i] = c.s1[i];
        d.s2[i] = c.s2[i];
    }
    d.P1 = c.P1;
    d.P2 = c.P2;
    d.P_inv = c.P_inv;
    d.pp_fast = c.pp_fast;
    d.pp_accu = c.pp_accu;
    for (int i = 0; i < c.n_moduli; ++i) {
        d.s2_m52[i] = -c.s2[i] * 0x1p52;
        d.s1_m52[i] = -c.s1[i] * 0x1p52;
        d.negp[i] = 0u - static_cast<uint32_t>(c.moduli[i]);
        if (i > 0 && c.moduli[i] == 256) d.p256_later = 1;
    }
    d.fast_floor = fast_floor_table(c.pp_fast);
    return d;
}

}  // namespace ozk

using namespace ozk;

namespace {
// One emulated GEMM: constants, operand views and the carved workspace.
struct Job {
    ozk_constants c;
    DevConsts dc;
    int mode;
    int64_t m, n, k, ldu;
    // op(A) / op(B) storage: ta -> A is k x m, tb -> B is n x k (column-major, BLAS 'T').
    // Planes follow the storage, so no transpose is ever materialised:
    //   A: !ta MN-major [N][k][lda_p = ld(m)],  ta K-major [N][m][lda_p = ld(k)]
    //   B: !tb K-major  [N][n][ld = ld(k)],     tb MN-major [N][k][ld = ld(n)]
    bool ta, tb;
    int64_t ld, lda_p, pa_stride, pb_stride;
    const void* a;  // device operands as the kernels read them
    const void* b;
    int64_t lda, ldb;
    int in_f32;
    int32_t *mu, *nu, *ma, *nb, *rowmax, *colmax;
    // accurate mode with k > 2^19: the bound product Abar*Bbar exceeds int32, so it
    // accumulates in int64 (per column block) and its maxima are uint64
    bool wide_bound;
    unsigned long long *rowmax64, *colmax64;
    bool async = false;  // OZK_FLAG_ASYNC: no host sync, deferred non-finite check
    int32_t* flags;  // [0] non-finite input, [4..] K2 lockstep words (1 KB)
    double *amax, *asum, *bmax, *bsum;
    int splits, splits_b;  // k-partials of the row-stat reductions of op(A) (!ta) / op(B) (tb)
    int32_t *cnt_a, *cnt_b;  // last-block counters of the row-stat reductions (A side / B side)
    int8_t *pa, *pb;
    uint8_t* u;
    bool need_products;
};

// a panel plan (make_plan): row panels of op(A)/C, column panels of op(B)/C
struct Plan {
    int64_t mr = 0, nc = 0;
    bool col_outer = true;
    int64_t panels = 1, extra_passes = 0;
    size_t pa = 0, pb = 0, u = 0;
    bool single = true;  // one panel: the whole problem (the two-stream K1 path)
};
}  // namespace

struct ozk_context {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;              // compute stream (user-settable)
    cudaStream_t h2d = nullptr, d2h = nullptr;  // copy streams of ozk_gemm_host
    cudaStream_t side = nullptr;                // B-side K1 chain of ozk_gemm (fork/join events)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int64_t launches = 0;
    Buf planes_a, planes_b, u, stats, ints, flags, f32a, f32b, host_a, host_b, host_c, wide, cbar, counters;
    Buf fused;                  // one-pass K1 row state (k1_fused.cu): A side, then B side; zero between calls
    int64_t fused_m = -1, fused_n = -1;  // the shape the state layout was last cleared for
    int32_t* flags_host = nullptr;  // pinned mirror of the device flag word
    // stage timing (ozk_profile): CUDA events on the compute stream
    bool profiling = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    double stage_ms[OZK_PROFILE_SLOTS] = {};
    int64_t stage_calls[OZK_PROFILE_SLOTS] = {};
    // the column shard between ozk_shard_begin and ozk_shard_end
    bool shard_open = false;
    ozk_config shard_cfg{};
    Job shard{};  // plain pointers into this handle's workspace
    Plan shard_plan{};
    // the row-streamed shard (ozk_shard_stream_*): output and progress
    bool stream_open = false;
    double stream_alpha = 1.0, stream_beta = 0.0;
    void* stream_c = nullptr;
    int64_t stream_ldc = 0, stream_rows = 0;
    int stream_c_f32 = 0;
    int64_t stream_ldu = 0;  // U pitch of the row-streamed shard's per-block products
    // pinned staging of pageable host buffers (ozk_gemm_host), created on first use
    HostStager* stager = nullptr;
    // device workspace limit (0: automatic) and the last call's panel plan
    int64_t ws_limit = 0;
    int64_t last_plan[4] = {0, 0, 0, 0};
};

namespace {

int cuda_fail(const char* what, cudaError_t e) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return OZK_CUDA_ERROR;
}

#define OZK_CUDA(call)                                      \
    do {                                                    \
        const cudaError_t e_ = (call);                      \
        if (e_ != cudaSuccess) return cuda_fail(#call, e_); \
    } while (0)
#define OZK_TRY(call)                  \
    do {                               \
        const int st_ = (call);        \
        if (st_ != OZK_OK) return st_; \
    } while (0)

// entries of Abar*Bbar are <= 64 * 64 * k (an Abar entry is ceil of a value in
// (63, 64] at most): int32 holds them for k < 2^19 (at k = 2^19, 2^31 wraps)
constexpr int64_t kBoundInt32K = int64_t(1) << 19;
inline bool bound_needs_int64(int64_t k) { return k >= kBoundInt32K; }

int ensure(Buf& b, size_t bytes) {
    if (bytes <= b.bytes && b.p) return OZK_OK;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    const size_t want = bytes ? bytes : 16;
    OZK_CUDA(cudaMalloc(&b.p, want));
    b.bytes = want;
    return OZK_OK;
}

// RAII bracket of one stage: an NVTX range on the host timeline (header-only
// NVTX v3: a no-op unless a tool such as nsys / ncu --nvtx is attached) and,
// with ozk_profile on, a start/stop event pair on the compute stream
const char* stage_name(int slot) {
    static const char* names[OZK_PROFILE_SLOTS] = {"ozk K1 scale", "ozk K1 residues", "ozk K2 products",
                                                   "ozk K3 reconstruct", "ozk gemm"};
    return slot >= 0 && slot < OZK_PROFILE_SLOTS ? names[slot] : "ozk";
}
struct StageTimer {
    ozk_context* h;
    int slot;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    StageTimer(ozk_context* hh, int s) : h(hh), slot(s) {
        nvtxRangePushA(stage_name(s));
        if (!h->profiling) return;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, h->stream);
    }
    ~StageTimer() {
        nvtxRangePop();
        if (!h->profiling) return;
        cudaEventRecord(e1, h->stream);
        h->pending.push_back({slot, {e0, e1}});
    }
};

// runs the enclosed stages on the handle's side stream (h->stream swapped)
struct OnSideStream {
    ozk_context* h;
    cudaStream_t saved;
    explicit OnSideStream(ozk_context* hh) : h(hh), saved(hh->stream) { h->stream = h->side; }
    ~OnSideStream() { h->stream = saved; }
};

int check_launch(ozk_context* h, int n_kernels) {
    h->launches += n_kernels;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail("kernel launch", e);
    return OZK_OK;
}

// Resolve the constant table (build_constants is called first, as in
// emulator.cpp:102-108, so an out-of-range N is a ConfigError before any input check).
int resolve(const ozk_config* cfg, ozk_constants& c) {
    if (!cfg) {
        set_error("null config");
        return OZK_CONFIG_ERROR;
    }
    if (cfg->constants) {
        c = *cfg->constants;
        if (c.n_moduli < 2 || c.n_moduli > OZK_MAX_MODULI) {
            set_error("constant table has an invalid modulus count");
            return OZK_CONFIG_ERROR;
        }
        return OZK_OK;
    }
    return ozk_build_constants(cfg->n_moduli, cfg->precision, &c);
}

// validate_inputs (emulator.cpp:12-23) minus the finite scan, which runs on the device
int validate(const ozk_config* cfg, const ozk_constants& c, int64_t m, int64_t n, int64_t k, int64_t lda,
             int64_t ldb) {
    // the configuration's precision (not the table's) decides, as in emulator.cpp:96-99
    if (cfg->precision != OZK_FP32 && cfg->a_type == OZK_R32F) {
        set_error("gemm_emulated: FP32 inputs require cfg.precision == Fp32");
        return OZK_CONFIG_ERROR;
    }
    if (m < 1 || k < 1 || n < 1) {
        set_error("gemm_emulated: empty dimension");
        return OZK_INPUT_ERROR;
    }
    if (cfg->block_k < 1 || cfg->block_k > OZK_ENGINE_MAX_K) {
        set_error("gemm_emulated: block_k must be in [1, 2^17]");
        return OZK_CONFIG_ERROR;
    }
    const bool ta = (cfg->flags & OZK_FLAG_TRANS_A) != 0, tb = (cfg->flags & OZK_FLAG_TRANS_B) != 0;
    if (lda < (ta ? k : m) || ldb < (tb ? n : k)) {
        set_error("gemm_emulated: leading dimension smaller than the matrix");
        return OZK_INPUT_ERROR;
    }
    if (cfg->mode != OZK_FAST && cfg->mode != OZK_ACCURATE) {
        set_error("gemm_emulated: unknown scaling mode");
        return OZK_CONFIG_ERROR;
    }
    if (k > (int64_t(1) << 31) - 1) {
        set_error("k exceeds 2^31");
        return OZK_INPUT_ERROR;
    }
    return OZK_OK;
}


int setup(ozk_context* h, Job& J, const ozk_config* cfg, const ozk_constants& c, int64_t m, int64_t n, int64_t k,
          const void* A, int64_t lda, const void* B, int64_t ldb, bool need_products) {
    J.c = c;
    J.dc = to_dev(c);
    J.dc.fast_fix = (cfg->flags & OZK_FLAG_FAST_EXPONENT_FIX) ? 1 : 0;
    J.mode = cfg->mode;
    J.m = m;
    J.n = n;
    J.k = k;
    J.ta = (cfg->flags & OZK_FLAG_TRANS_A) != 0;
    J.tb = (cfg->flags & OZK_FLAG_TRANS_B) != 0;
    J.lda_p = J.ta ? plane_ld(k) : plane_ld(m);
    J.pa_stride = J.ta ? m * J.lda_p : k * J.lda_p;
    J.ld = J.tb ? plane_ld(n) : plane_ld(k);
    J.pb_stride = J.tb ? k * J.ld : n * J.ld;
    J.ldu = u_ld(m);
    const int N = c.n_moduli;
    J.splits = J.ta ? 1 : row_stats_splits(m, k);
    J.splits_b = J.tb ? row_stats_splits(n, k) : 1;
    OZK_TRY(ensure(h->flags, 2048));
    OZK_TRY(ensure(h->stats, sizeof(double) * (2 * J.splits * m + 2 * J.splits_b * n)));
    OZK_TRY(ensure(h->ints, sizeof(int32_t) * 4 * (m + n)));
    {
        const size_t cbytes = sizeof(int32_t) * (row_stat_groups(m) + row_stat_groups(n) + 2);
        const bool grow = !h->counters.p || cbytes > h->counters.bytes;
        OZK_TRY(ensure(h->counters, cbytes));
        if (grow) OZK_CUDA(cudaMemsetAsync(h->counters.p, 0, h->counters.bytes, h->stream));  // then self-resetting
        J.cnt_a = static_cast<int32_t*>(h->counters.p);
        J.cnt_b = J.cnt_a + row_stat_groups(m) + 1;
    }
    (void)N;
    // the residue planes and U are sized by the caller's panel plan
    // (alloc_plan); without products only the accurate-mode bound operands
    // Abar / Bbar (one plane each, whole problem) are needed here
    if (!need_products && cfg->mode == OZK_ACCURATE) {
        OZK_TRY(ensure(h->planes_a, static_cast<size_t>(J.pa_stride)));
        OZK_TRY(ensure(h->planes_b, static_cast<size_t>(J.pb_stride)));
    }
    J.flags = static_cast<int32_t*>(h->flags.p);
    double* d = static_cast<double*>(h->stats.p);
    J.amax = d;
    J.asum = d + J.splits * m;
    J.bmax = d + 2 * J.splits * m;
    J.bsum = J.bmax + J.splits_b * n;
    int32_t* p = static_cast<int32_t*>(h->ints.p);
    J.mu = p;
    J.nu = J.mu + m;
    J.ma = J.nu + n;
    J.nb = J.ma + m;
    J.rowmax = J.nb + n;
    J.colmax = J.rowmax + m;
    J.wide_bound = cfg->mode == OZK_ACCURATE && bound_needs_int64(k);
    if (J.wide_bound) {
        OZK_TRY(ensure(h->wide, sizeof(unsigned long long) * (m + n)));
        J.rowmax64 = static_cast<unsigned long long*>(h->wide.p);
        J.colmax64 = J.rowmax64 + m;
    }
    J.pa = static_cast<int8_t*>(h->planes_a.p);
    J.pb = static_cast<int8_t*>(h->planes_b.p);
    J.u = static_cast<uint8_t*>(h->u.p);
    J.need_products = need_products;
    J.a = A;
    J.b = B;
    J.lda = lda;
    J.ldb = ldb;
    J.in_f32 = cfg->a_type == OZK_R32F;
    // flag word 0 (non-finite input): cleared per synchronous call; sticky
    // across stream-ordered calls until ozk_sync collects it
    J.async = (cfg->flags & OZK_FLAG_ASYNC) != 0;
    if (!J.async) OZK_CUDA(cudaMemsetAsync(J.flags, 0, sizeof(int32_t), h->stream));
    return OZK_OK;
}

// FP32 precision on FP64 storage (emulator.cpp:84-91): the operands are rounded
// into FP32 staging buffers (A whole, B by column range) before any stage reads them.
// cfg.precision decides, as in the reference; the constant table (which may be
// passed separately, of either precision) only supplies the arithmetic.
bool rounds_inputs(const Job&, const ozk_config* cfg) {
    return cfg->precision == OZK_FP32 && cfg->a_type == OZK_R64F;
}

int round_a(ozk_context* h, Job& J, const ozk_config* cfg) {
    if (!rounds_inputs(J, cfg)) return OZK_OK;
    OZK_TRY(ensure(h->f32a, sizeof(float) * J.m * J.k));
    const int64_t rows = J.ta ? J.k : J.m, cols = J.ta ? J.m : J.k;
    launch_round_to_f32(static_cast<const double*>(J.a), rows, cols, J.lda, static_cast<float*>(h->f32a.p), rows,
                        h->stream);
    J.a = h->f32a.p;
    J.lda = rows;
    J.in_f32 = 1;
    return check_launch(h, 1);
}

// B is rounded block by block into a k x n (tb: n x k) FP32 staging buffer;
// src keeps the caller's FP64 view for the later blocks
int round_b(ozk_context* h, Job& J, const ozk_config* cfg, const void* src, int64_t src_ld, int64_t j0, int64_t nj) {
    if (!rounds_inputs(J, cfg)) return OZK_OK;
    OZK_TRY(ensure(h->f32b, sizeof(float) * J.k * J.n));
    float* dst = static_cast<float*>(h->f32b.p);
    if (J.tb)
        launch_round_to_f32(static_cast<const double*>(src) + j0, nj, J.k, src_ld, dst + j0, J.n, h->stream);
    else
        launch_round_to_f32(static_cast<const double*>(src) + j0 * src_ld, J.k, nj, src_ld, dst + j0 * J.k, J.k,
                            h->stream);
    J.b = h->f32b.p;
    J.ldb = J.tb ? J.n : J.k;
    J.in_f32 = 1;
    return check_launch(h, 1);
}

// first element of op(B)'s column j0 (tb: row j0 of the stored n x k B)
const void* b_block(const Job& J, int64_t j0) {
    const int64_t off = J.tb ? j0 : j0 * J.ldb;
    return J.in_f32 ? static_cast<const void*>(static_cast<const float*>(J.b) + off)
                    : static_cast<const void*>(static_cast<const double*>(J.b) + off);
}

// byte offset of op(B)'s column j0 inside a B plane
int64_t b_plane_off(const Job& J, int64_t j0) { return J.tb ? j0 : j0 * J.ld; }

// what the reductions finalize per line: fast-mode exponents (exp_out), or
// accurate-mode bases (exp_out) with the bound maxima cleared (zero_out);
// element h of line l at base[l*line_step + h*elem_step] for the exact recompute
LineFinal line_final(const Job& J, int32_t* exp_out, int32_t* zero_out, const void* base, int64_t line_step,
                     int64_t elem_step) {
    LineFinal F{};
    F.mode = J.mode;
    F.prec = J.dc.precision;
    F.fix = J.dc.fast_fix;
    F.pp_fast = J.dc.pp_fast;
    F.k = J.k;
    F.exp_out = exp_out;
    F.zero_out = zero_out;
    F.base = base;
    F.is_f32 = J.in_f32;
    F.line_step = line_step;
    F.elem_step = elem_step;
    F.fast_floor = J.dc.fast_floor;
    return F;
}

// op(A)'s rows: row stats over A's rows, or column stats over the stored k x m A^T,
// finalized into mu (fast) or mu' (accurate, rowmax cleared)
void a_line_stats(ozk_context* h, Job& J) {
    const bool fast = J.mode == OZK_FAST;
    const LineFinal F = line_final(J, fast ? J.mu : J.ma, fast ? nullptr : J.rowmax, J.a, J.ta ? J.lda : 1,
                                   J.ta ? 1 : J.lda);
    if (J.ta)
        launch_col_stats(J.a, J.in_f32, J.k, J.m, J.lda, J.amax, J.asum, J.flags, F, h->stream);
    else
        launch_row_stats(J.a, J.in_f32, J.m, J.k, J.lda, J.splits, J.amax, J.asum, J.flags, J.cnt_a, F, h->stream);
}

// residues (kind 0) or the bound plane (kind 1) of op(A), in the layout K2 reads
void a_planes(ozk_context* h, Job& J, const int32_t* mu, int kind, int8_t* pa, int64_t stride) {
    if (J.ta)  // K-major: column i of the stored A^T is row i of op(A), scaled by mu[i]
        launch_b_planes(J.a, J.in_f32, J.k, J.m, J.lda, mu, J.dc, kind, pa, J.lda_p, stride, h->stream);
    else
        launch_a_planes(J.a, J.in_f32, J.m, J.k, J.lda, mu, J.dc, kind, pa, J.lda_p, stride, h->stream);
}

// op(B) columns [j0, j0+nj): planes at b_plane_off(j0)
void b_planes(ozk_context* h, Job& J, int64_t j0, int64_t nj, const int32_t* nu, int kind, int8_t* pb,
              int64_t stride) {
    if (J.tb)  // MN-major: row j of the stored B^T is column j of op(B), scaled by nu[j]
        launch_a_planes(b_block(J, j0), J.in_f32, nj, J.k, J.ldb, nu + j0, J.dc, kind, pb + b_plane_off(J, j0), J.ld,
                        stride, h->stream);
    else
        launch_b_planes(b_block(J, j0), J.in_f32, J.k, nj, J.ldb, nu + j0, J.dc, kind, pb + b_plane_off(J, j0), J.ld,
                        stride, h->stream);
}

// ---- stages ----------------------------------------------------------------------
// rows of A: stats, and fast-mode mu (or accurate-mode mu' + the Abar plane)
int stage_rows(ozk_context* h, Job& J) {
    a_line_stats(h, J);
    OZK_TRY(check_launch(h, 1));
    if (J.mode == OZK_FAST) return OZK_OK;
    a_planes(h, J, J.ma, 1, J.pa, J.pa_stride);
    if (J.wide_bound) OZK_CUDA(cudaMemsetAsync(J.rowmax64, 0, sizeof(unsigned long long) * J.m, h->stream));
    return check_launch(h, 1);
}

// columns [j0, j0+nj) of B: stats and fast-mode nu, or accurate-mode nu', the
// Bbar block and the bound GEMM Abar * Bbar_block (row maxima accumulate)
// part: 0 everything; 1 up to the bound operand (accurate: B-bar planes), which
// needs only B; 2 the bound GEMM alone (needs the A-bar planes too)
int stage_cols(ozk_context* h, Job& J, int64_t j0, int64_t nj, int part = 0) {
    const void* bj = b_block(J, j0);
    // this block's [split][nj] partials
    double* bmax = J.bmax + J.splits_b * j0;
    double* bsum = J.bsum + J.splits_b * j0;
    int8_t* bbar = J.pb + b_plane_off(J, j0);
    if (part == 2) goto bound_gemm;
    {
        const bool fast = J.mode == OZK_FAST;
        const LineFinal F = line_final(J, fast ? J.nu + j0 : J.nb + j0, fast ? nullptr : J.colmax + j0, bj,
                                       J.tb ? 1 : J.ldb, J.tb ? J.ldb : 1);
        if (J.tb)
            launch_row_stats(bj, J.in_f32, nj, J.k, J.ldb, J.splits_b, bmax, bsum, J.flags, J.cnt_b, F, h->stream);
        else
            launch_col_stats(bj, J.in_f32, J.k, nj, J.ldb, bmax, bsum, J.flags, F, h->stream);
    }
    OZK_TRY(check_launch(h, 1));
    if (J.mode == OZK_FAST) return OZK_OK;
    b_planes(h, J, j0, nj, J.nb, 1, J.pb, J.pb_stride);
    if (J.wide_bound) OZK_CUDA(cudaMemsetAsync(J.colmax64 + j0, 0, sizeof(unsigned long long) * nj, h->stream));
    OZK_TRY(check_launch(h, 2));
    if (part == 1) return OZK_OK;
bound_gemm:
    if (J.wide_bound) OZK_TRY(ensure(h->cbar, sizeof(long long) * J.m * nj));
    K2Launch L{};
    L.a_planes = J.pa;
    L.b_planes = bbar;
    L.m = J.m;
    L.n = nj;
    L.k = J.k;
    L.ld = J.ld;
    L.lda = J.lda_p;
    L.a_mn = !J.ta;
    L.b_mn = J.tb;
    L.a_stride = J.pa_stride;
    L.b_stride = J.pb_stride;
    L.n_mod = 1;
    L.kind = K2_MAX;
    L.rowmax = J.rowmax;
    L.colmax = J.colmax + j0;
    L.c = &J.dc;
    L.num_sms = h->num_sms;
    L.sync_counter = reinterpret_cast<unsigned int*>(J.flags + 4);
    if (J.wide_bound) {  // int64 C-bar block, then its maxima (scaling.cpp:118-148 keeps C-bar in int64 too)
        L.kind = K2_ACC64;
        L.out = h->cbar.p;
        L.ldo = J.m;
        OZK_TRY(launch_k2(L, h->stream));
        launch_bound_max64(static_cast<const long long*>(h->cbar.p), J.m, nj, J.m, J.rowmax64, J.colmax64 + j0,
                           h->stream);
        return check_launch(h, (J.k + (1 << 17) - 1) / (1 << 17) + 1);
    }
    OZK_TRY(launch_k2(L, h->stream));
    return check_launch(h, 1);
}

// accurate mode, after every column block: the budgets (scaling.cpp:151-165)
int stage_budget(ozk_context* h, Job& J) {
    if (J.wide_bound)
        launch_accurate_budget64(J.ma, J.rowmax64, J.m, J.mu, J.nb, J.colmax64, J.n, J.nu, J.dc, h->stream);
    else
        launch_accurate_budget(J.ma, J.rowmax, J.m, J.mu, J.nb, J.colmax, J.n, J.nu, J.dc, h->stream);
    return check_launch(h, 1);
}

int stage_row_residues(ozk_context* h, Job& J, const int32_t* mu, int8_t* pa) {
    a_planes(h, J, mu, 0, pa, J.pa_stride);
    return check_launch(h, 1);
}

int stage_col_residues(ozk_context* h, Job& J, int64_t j0, int64_t nj, const int32_t* nu, int8_t* pb,
                       int64_t pb_stride) {
    b_planes(h, J, j0, nj, nu, 0, pb, pb_stride);
    return check_launch(h, 1);
}

// ---- one-pass K1 (k1_fused.cu) ---------------------------------------------------
// The line statistics, the exponents and the planes in one pass over an operand
// (fast mode: the residue planes; accurate mode: the bound plane Abar / Bbar).
// OZK_K1_FUSED is a mask of the one-pass kernels to use: bit 0 the column
// kernel (contiguous lines: B, or a transposed A), bit 1 the row kernel
// (strided lines: A, or a transposed B); 0 selects the two-kernel path (stats
// kernel, then planes kernel) everywhere. Default 1: in the bench step the
// column kernel wins (1.01 vs 0.34 + 0.94 ms at 16384^2) and the row kernel
// loses (1.57 vs 0.39 + 0.94 ms).
int k1_fused_mask() {
    static const int v = [] {
        const char* e = std::getenv("OZK_K1_FUSED");
        return e && *e ? std::atoi(e) : 1;
    }();
    return v;
}
bool k1_fused_enabled() { return k1_fused_mask() != 0; }
bool cols_fused_on() { return (k1_fused_mask() & 1) != 0; }
bool rows_fused_on() { return (k1_fused_mask() & 2) != 0; }

// the row kernel reads two adjacent rows per lane (16 / 8-byte vectors)
// and its planes role stages 64-row column runs with bulk copies (16-byte
// aligned runs of a multiple of 16 bytes): rows and ld multiples of 16 / size
bool rows_fusable(const void* x, int64_t ld, int64_t rows, int in_f32) {
    const int64_t q = in_f32 ? 4 : 2;
    return (reinterpret_cast<uintptr_t>(x) & 15) == 0 && ld % q == 0 && rows % q == 0;
}

// state of the one-pass row kernel: [A side | B side], zeroed when it grows, then self-resetting
int fused_state(ozk_context* h, const Job& J, void** sa, void** sb) {
    const size_t a = (rows_fused_state_bytes(J.m) + 255) / 256 * 256;
    const size_t b = (rows_fused_state_bytes(J.n) + 255) / 256 * 256;
    // the state is all zero between calls, but the regions' layout follows
    // (m, n): cleared whenever the buffer grows or the shape changes (a call
    // that failed mid-way cannot leave stale words at a moved offset)
    const bool grow = !h->fused.p || a + b > h->fused.bytes;
    OZK_TRY(ensure(h->fused, a + b));
    if (grow || h->fused_m != J.m || h->fused_n != J.n) {
        OZK_CUDA(cudaMemsetAsync(h->fused.p, 0, h->fused.bytes, h->stream));
        h->fused_m = J.m;
        h->fused_n = J.n;
    }
    *sa = h->fused.p;
    *sb = static_cast<char*>(h->fused.p) + a;
    return OZK_OK;
}

// op(A)'s rows in one pass: mu and its residue planes (fast), or mu' and Abar (accurate)
bool cols_worth_fusing(int64_t len, int64_t lines);
bool a_fusable(const Job& J) {
    return J.ta ? cols_fused_on() && cols_worth_fusing(J.k, J.m)
                : rows_fused_on() && rows_fusable(J.a, J.lda, J.m, J.in_f32);
}
int stage_rows_fused(ozk_context* h, Job& J, void* state) {
    const bool fast = J.mode == OZK_FAST;
    const LineFinal F = line_final(J, fast ? J.mu : J.ma, fast ? nullptr : J.rowmax, J.a, J.ta ? J.lda : 1,
                                   J.ta ? 1 : J.lda);
    const int kind = fast ? 0 : 1;
    if (J.ta)  // stored k x m: the lines are its columns, the planes K-major
        launch_cols_fused(J.a, J.in_f32, J.k, J.m, J.lda, J.flags, F, J.dc, kind, J.pa, J.lda_p, J.pa_stride,
                          h->num_sms, h->stream);
    else
        launch_rows_fused(J.a, J.in_f32, J.m, J.k, J.lda, state, J.flags, F, J.dc, kind, J.pa,
                          J.lda_p, J.pa_stride, h->num_sms, h->stream);
    if (!fast && J.wide_bound) OZK_CUDA(cudaMemsetAsync(J.rowmax64, 0, sizeof(unsigned long long) * J.m, h->stream));
    return check_launch(h, 1);
}

// columns [j0, j0+nj) of op(B) in one pass: nu and its planes (fast), or nu' and Bbar (accurate)
// the column kernel gives each column a 512-thread block (8 elements per
// thread per pass): below ~4096-element columns most of the block idles and
// its per-column finalize latency shows (1024^3: 0.055 -> 0.062 ms), so short
// or few columns keep the two-kernel path
bool cols_worth_fusing(int64_t len, int64_t lines) {
    static const bool any = std::getenv("OZK_K1_FUSED_ANY") != nullptr;  // tests: every size
    return any || (len >= 4096 && lines >= 1024);
}
bool b_fusable(const Job& J, int64_t j0) {
    return !J.tb ? cols_fused_on() && cols_worth_fusing(J.k, J.n)
                 : rows_fused_on() && rows_fusable(b_block(J, j0), J.ldb, J.n, J.in_f32);
}
int stage_cols_fused(ozk_context* h, Job& J, int64_t j0, int64_t nj, void* state) {
    const bool fast = J.mode == OZK_FAST;
    const void* bj = b_block(J, j0);
    const LineFinal F = line_final(J, fast ? J.nu + j0 : J.nb + j0, fast ? nullptr : J.colmax + j0, bj,
                                   J.tb ? 1 : J.ldb, J.tb ? J.ldb : 1);
    const int kind = fast ? 0 : 1;
    int8_t* dst = J.pb + b_plane_off(J, j0);
    if (J.tb)  // stored n x k: the lines are its rows, the planes MN-major
        launch_rows_fused(bj, J.in_f32, nj, J.k, J.ldb, state, J.flags, F, J.dc, kind, dst, J.ld,
                          J.pb_stride, h->num_sms, h->stream);
    else
        launch_cols_fused(bj, J.in_f32, J.k, nj, J.ldb, J.flags, F, J.dc, kind, dst, J.ld, J.pb_stride, h->num_sms,
                          h->stream);
    if (!fast && J.wide_bound)
        OZK_CUDA(cudaMemsetAsync(J.colmax64 + j0, 0, sizeof(unsigned long long) * nj, h->stream));
    return check_launch(h, 1);
}

int stage_products(ozk_context* h, Job& J, int64_t j0, int64_t nj, const int8_t* pa, int64_t pa_stride,
                   const int8_t* pb, int64_t pb_stride, int kind, void* out, int64_t ldo, int64_t out_stride) {
    K2Launch L{};
    L.a_planes = pa;
    L.b_planes = pb + b_plane_off(J, j0);
    L.m = J.m;
    L.n = nj;
    L.k = J.k;
    L.ld = J.ld;
    L.lda = J.lda_p;
    L.a_mn = !J.ta;
    L.b_mn = J.tb;
    L.a_stride = pa_stride;
    L.b_stride = pb_stride;
    L.n_mod = J.c.n_moduli;
    L.kind = kind == OZK_PRODUCTS_I32 ? K2_I32 : K2_U8;
    const int64_t esz = kind == OZK_PRODUCTS_I32 ? 4 : 1;
    L.out = static_cast<uint8_t*>(out) + j0 * ldo * esz;
    L.ldo = ldo;
    L.out_stride = out_stride;
    L.c = &J.dc;
    L.num_sms = h->num_sms;
    L.sync_counter = reinterpret_cast<unsigned int*>(J.flags + 4);
    OZK_TRY(launch_k2(L, h->stream));
    return check_launch(h, 1);
}

int stage_reconstruct(ozk_context* h, Job& J, int64_t j0, int64_t nj, const uint8_t* u, int64_t ldu,
                      int64_t u_stride, const int32_t* mu, const int32_t* nu, double alpha, double beta, void* C,
                      int64_t ldc, int c_f32) {
    void* cj = c_f32 ? static_cast<void*>(static_cast<float*>(C) + j0 * ldc)
                     : static_cast<void*>(static_cast<double*>(C) + j0 * ldc);
    launch_reconstruct(u + j0 * ldu, ldu, u_stride, J.m, nj, mu, nu + j0, J.dc, alpha, beta, cj, ldc, c_f32,
                       h->stream);
    return check_launch(h, 1);
}

// column block [j0, j0+nj) once mu (and, in accurate mode, every nu) is known:
// B residues -> N GEMMs -> CRT reconstruction
int compute_block(ozk_context* h, Job& J, int64_t j0, int64_t nj, double alpha, double beta, void* C, int64_t ldc,
                  int c_f32) {
    {
        StageTimer t(h, OZK_PROFILE_RESIDUES);
        OZK_TRY(stage_col_residues(h, J, j0, nj, J.nu, J.pb, J.pb_stride));
    }
    {
        StageTimer t(h, OZK_PROFILE_PRODUCTS);
        OZK_TRY(stage_products(h, J, j0, nj, J.pa, J.pa_stride, J.pb, J.pb_stride, OZK_PRODUCTS_U8, J.u, J.ldu,
                               J.n * J.ldu));
    }
    StageTimer t(h, OZK_PROFILE_RECONSTRUCT);
    return stage_reconstruct(h, J, j0, nj, J.u, J.ldu, J.n * J.ldu, J.mu, J.nu, alpha, beta, C, ldc, c_f32);
}

int finish_check(ozk_context* h, Job& J, cudaStream_t s) {
    if (J.async) return OZK_OK;  // deferred to ozk_sync
    OZK_CUDA(cudaMemcpyAsync(h->flags_host, J.flags, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    OZK_CUDA(cudaStreamSynchronize(s));
    if (h->flags_host[0]) {
        set_error("gemm_emulated: non-finite entry in A or B");
        return OZK_INPUT_ERROR;
    }
    return OZK_OK;
}

// scale of the whole problem with device-resident operands (one column block)
int scale_all(ozk_context* h, Job& J, const ozk_config* cfg) {
    const void* b_src = J.b;
    const int64_t b_ld = J.ldb;
    OZK_TRY(round_a(h, J, cfg));
    OZK_TRY(round_b(h, J, cfg, b_src, b_ld, 0, J.n));
    OZK_TRY(stage_rows(h, J));
    OZK_TRY(stage_cols(h, J, 0, J.n));
    if (J.mode == OZK_ACCURATE) OZK_TRY(stage_budget(h, J));
    return OZK_OK;
}

// ---- panel plan (bounded workspace) -------------------------------------------
// The N residue planes of A, of B and the N uint8 product residues U take
// about N bytes per element of A, B and C (60 GB each at 65536^2, N = 14). A
// problem whose workspace exceeds the handle's limit runs in panels: row
// panels of op(A)/C (mr rows) times column panels of op(B)/C (nc columns), the
// planes of one A panel and one B panel and the U of one region live at a
// time. With column panels outside, A's residues are derived once per column
// panel (none extra when one row panel holds all of A), and vice versa; the
// plan takes the shape and order with the fewest extra residue passes that
// fits. Results do not depend on it: after the O(m + n) exponents every stage
// is row/column-local.

// one plane of an op(A) row panel / op(B) column panel, in K2's operand layouts
int64_t a_panel_ld(const Job& J, int64_t mr) { return J.ta ? plane_ld(J.k) : plane_ld(mr); }
int64_t a_panel_plane(const Job& J, int64_t mr) { return J.ta ? mr * a_panel_ld(J, mr) : J.k * a_panel_ld(J, mr); }
int64_t b_panel_ld(const Job& J, int64_t nc) { return J.tb ? plane_ld(nc) : plane_ld(J.k); }
int64_t b_panel_plane(const Job& J, int64_t nc) { return J.tb ? J.k * b_panel_ld(J, nc) : nc * b_panel_ld(J, nc); }

int64_t env_workspace_limit() {
    const char* e = std::getenv("OZK_WORKSPACE_GB");
    return e && *e ? static_cast<int64_t>(std::atof(e) * 1e9) : 0;
}

// bytes the plan may use for planes_a + planes_b + u
int64_t workspace_limit(ozk_context* h) {
    if (h->ws_limit > 0) return h->ws_limit;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
        cudaGetLastError();
        return INT64_MAX;
    }
    const int64_t held = static_cast<int64_t>(h->planes_a.bytes + h->planes_b.bytes + h->u.bytes);
    const int64_t reserve = std::max<int64_t>(int64_t(1) << 30, static_cast<int64_t>(total_b / 10));
    int64_t lim = static_cast<int64_t>(free_b) + held - reserve;
    const int64_t env = env_workspace_limit();
    if (env > 0) lim = env;
    return lim;
}

std::vector<int64_t> panel_candidates(int64_t x) {
    std::vector<int64_t> v{x};
    for (int s = 1; s < 40; ++s) {
        int64_t c = (x + (int64_t(1) << s) - 1) >> s;
        c = (c + 255) / 256 * 256;  // whole 256-wide GEMM tiles
        if (c >= v.back()) continue;
        v.push_back(c);
        if (c <= 256) break;
    }
    return v;
}

Plan make_plan(ozk_context* h, const Job& J, int64_t extra_bytes = 0) {
    const int N = J.c.n_moduli;
    const bool acc = J.mode == OZK_ACCURATE;
    const int64_t es = J.in_f32 ? 4 : 8;
    const int64_t limit = workspace_limit(h) - extra_bytes;
    const double pass_a = double(es + N) * J.m * J.k, pass_b = double(es + N) * J.k * J.n;
    const double region_cost = 256e6;  // ~40 us of HBM per region (launches, partial last waves)
    Plan best;
    double best_cost = 0;
    bool found = false;
    Plan smallest;
    for (int64_t mr : panel_candidates(J.m)) {
        for (int64_t nc : panel_candidates(J.n)) {
            Plan P;
            P.mr = mr;
            P.nc = nc;
            P.pa = static_cast<size_t>(std::max<int64_t>(N * a_panel_plane(J, mr), acc ? J.pa_stride : 0));
            P.pb = static_cast<size_t>(std::max<int64_t>(N * b_panel_plane(J, nc), acc ? J.pb_stride : 0));
            P.u = static_cast<size_t>(N * nc * u_ld(mr));
            const int64_t I = (J.m + mr - 1) / mr, Jn = (J.n + nc - 1) / nc;
            P.panels = I * Jn;
            P.single = I == 1 && Jn == 1;
            const double col = I > 1 ? double(Jn - 1) * pass_a : 0.0;
            const double row = Jn > 1 ? double(I - 1) * pass_b : 0.0;
            P.col_outer = col <= row;
            P.extra_passes = P.col_outer ? (I > 1 ? Jn - 1 : 0) : (Jn > 1 ? I - 1 : 0);
            smallest = P;  // candidates shrink: the last one is the smallest
            if (static_cast<int64_t>(P.pa + P.pb + P.u) > limit) continue;
            const double cost = std::min(col, row) + region_cost * double(P.panels);
            if (!found || cost < best_cost) {
                best = P;
                best_cost = cost;
                found = true;
            }
        }
    }
    return found ? best : smallest;
}

void release(Buf& b) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
}

int alloc_plan(ozk_context* h, Job& J, const Plan& P) {
    // the plan counted what the handle holds as available: if any of the three
    // buffers must grow, all three are released first (growing one while the
    // others keep their old sizes could need more than the limit)
    if (P.pa > h->planes_a.bytes || P.pb > h->planes_b.bytes || P.u > h->u.bytes) {
        release(h->planes_a);
        release(h->planes_b);
        release(h->u);
    }
    OZK_TRY(ensure(h->planes_a, P.pa));
    OZK_TRY(ensure(h->planes_b, P.pb));
    OZK_TRY(ensure(h->u, P.u));
    J.pa = static_cast<int8_t*>(h->planes_a.p);
    J.pb = static_cast<int8_t*>(h->planes_b.p);
    J.u = static_cast<uint8_t*>(h->u.p);
    h->last_plan[0] = P.mr;
    h->last_plan[1] = P.nc;
    h->last_plan[2] = P.panels;
    h->last_plan[3] = P.extra_passes;
    return OZK_OK;
}

// residue planes of op(A)'s rows [r0, r0+mr) at pa (panel layout, offset 0)
int a_panel_residues(ozk_context* h, Job& J, int64_t r0, int64_t mr, int8_t* pa) {
    const int64_t es = J.in_f32 ? 4 : 8;
    const int64_t ld = a_panel_ld(J, mr), stride = a_panel_plane(J, mr);
    if (J.ta)  // K-major: columns r0.. of the stored k x m A^T
        launch_b_planes(static_cast<const char*>(J.a) + es * r0 * J.lda, J.in_f32, J.k, mr, J.lda, J.mu + r0, J.dc, 0,
                        pa, ld, stride, h->stream);
    else
        launch_a_planes(static_cast<const char*>(J.a) + es * r0, J.in_f32, mr, J.k, J.lda, J.mu + r0, J.dc, 0, pa,
                        ld, stride, h->stream);
    return check_launch(h, 1);
}

// residue planes of op(B)'s columns [c0, c0+nc) at pb (panel layout, offset 0)
int b_panel_residues(ozk_context* h, Job& J, int64_t c0, int64_t nc, int8_t* pb) {
    const int64_t ld = b_panel_ld(J, nc), stride = b_panel_plane(J, nc);
    if (J.tb)  // MN-major: rows c0.. of the stored n x k B^T
        launch_a_planes(b_block(J, c0), J.in_f32, nc, J.k, J.ldb, J.nu + c0, J.dc, 0, pb, ld, stride, h->stream);
    else
        launch_b_planes(b_block(J, c0), J.in_f32, J.k, nc, J.ldb, J.nu + c0, J.dc, 0, pb, ld, stride, h->stream);
    return check_launch(h, 1);
}

// C[r0:r0+mr, c0:c0+nc] from an A panel and a B panel: K2 into U, then K3
int panel_region(ozk_context* h, Job& J, int64_t r0, int64_t mr, int64_t c0, int64_t nc, double alpha, double beta,
                 void* C, int64_t ldc, int c_f32) {
    const int64_t ldu = u_ld(mr), ustride = nc * ldu;
    {
        StageTimer t(h, OZK_PROFILE_PRODUCTS);
        K2Launch L{};
        L.a_planes = J.pa;
        L.b_planes = J.pb;
        L.m = mr;
        L.n = nc;
        L.k = J.k;
        L.lda = a_panel_ld(J, mr);
        L.ld = b_panel_ld(J, nc);
        L.a_mn = !J.ta;
        L.b_mn = J.tb;
        L.a_stride = a_panel_plane(J, mr);
        L.b_stride = b_panel_plane(J, nc);
        L.n_mod = J.c.n_moduli;
        L.kind = K2_U8;
        L.out = J.u;
        L.ldo = ldu;
        L.out_stride = ustride;
        L.c = &J.dc;
        L.num_sms = h->num_sms;
        L.sync_counter = reinterpret_cast<unsigned int*>(J.flags + 4);
        OZK_TRY(launch_k2(L, h->stream));
        OZK_TRY(check_launch(h, 1));
    }
    const size_t cs = c_f32 ? 4 : 8;
    StageTimer t(h, OZK_PROFILE_RECONSTRUCT);
    launch_reconstruct(J.u, ldu, ustride, mr, nc, J.mu + r0, J.nu + c0, J.dc, alpha, beta,
                       static_cast<char*>(C) + cs * (c0 * ldc + r0), ldc, c_f32, h->stream);
    return check_launch(h, 1);
}

// every panel once the exponents are known (on the handle's stream)
int run_panels(ozk_context* h, Job& J, const Plan& P, double alpha, double beta, void* C, int64_t ldc, int c_f32) {
    const int64_t I = (J.m + P.mr - 1) / P.mr, Jn = (J.n + P.nc - 1) / P.nc;
    auto a_res = [&](int64_t r0, int64_t mr) {
        StageTimer t(h, OZK_PROFILE_RESIDUES);
        return a_panel_residues(h, J, r0, mr, J.pa);
    };
    auto b_res = [&](int64_t c0, int64_t nc) {
        StageTimer t(h, OZK_PROFILE_RESIDUES);
        return b_panel_residues(h, J, c0, nc, J.pb);
    };
    if (P.col_outer) {
        for (int64_t jb = 0; jb < Jn; ++jb) {
            const int64_t c0 = jb * P.nc, nc = std::min(P.nc, J.n - c0);
            OZK_TRY(b_res(c0, nc));
            for (int64_t ib = 0; ib < I; ++ib) {
                const int64_t r0 = ib * P.mr, mr = std::min(P.mr, J.m - r0);
                if (I > 1 || jb == 0) OZK_TRY(a_res(r0, mr));
                OZK_TRY(panel_region(h, J, r0, mr, c0, nc, alpha, beta, C, ldc, c_f32));
            }
        }
    } else {
        for (int64_t ib = 0; ib < I; ++ib) {
            const int64_t r0 = ib * P.mr, mr = std::min(P.mr, J.m - r0);
            OZK_TRY(a_res(r0, mr));
            for (int64_t jb = 0; jb < Jn; ++jb) {
                const int64_t c0 = jb * P.nc, nc = std::min(P.nc, J.n - c0);
                if (Jn > 1 || ib == 0) OZK_TRY(b_res(c0, nc));
                OZK_TRY(panel_region(h, J, r0, mr, c0, nc, alpha, beta, C, ldc, c_f32));
            }
        }
    }
    return OZK_OK;
}

// accurate mode: the bound GEMM Abar * Bbar (row maxima accumulate across
// column blocks; the int64 product of k >= 2^19 is formed per block of at
// most ~2 GB) and the budgets
int bound_and_budget(ozk_context* h, Job& J) {
    StageTimer t(h, OZK_PROFILE_SCALE);
    int64_t nb = J.n;
    if (J.wide_bound) nb = std::min<int64_t>(J.n, std::max<int64_t>(256, ((int64_t(1) << 31) / (8 * J.m)) / 256 * 256));
    for (int64_t j0 = 0; j0 < J.n; j0 += nb) OZK_TRY(stage_cols(h, J, j0, std::min(nb, J.n - j0), 2));
    return stage_budget(h, J);
}

int single_panel(ozk_context* h, Job& J, double alpha, double beta, void* C, int64_t ldc, int c_f32);

int gemm_device(ozk_context* h, const ozk_config* cfg, const ozk_constants& c, int64_t m, int64_t n, int64_t k,
                double alpha, const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C,
                int64_t ldc) {
    OZK_TRY(validate(cfg, c, m, n, k, lda, ldb));
    if (ldc < m) {
        set_error("gemm_emulated: ldc < m");
        return OZK_INPUT_ERROR;
    }
    OZK_CUDA(cudaSetDevice(h->device));
    Job J{};
    OZK_TRY(setup(h, J, cfg, c, m, n, k, A, lda, B, ldb, true));
    const int64_t f32_bytes = rounds_inputs(J, cfg) ? 4 * (m * k + k * n) : 0;
    const Plan P = make_plan(h, J, f32_bytes);
    OZK_TRY(alloc_plan(h, J, P));
    const int c_f32 = cfg->c_type == OZK_R32F;
    const bool fast = J.mode == OZK_FAST;
    {
        StageTimer total(h, OZK_PROFILE_TOTAL);
        // A's rows on the handle's stream, B's columns on the side stream: the two
        // chains of small K1 kernels overlap (what bounds small problems); they
        // share no buffers (separate partials, exponents and flag words)
        // one pass per operand (k1_fused.cu) where the whole problem is one
        // panel (fast mode writes the residue planes of all of A / B) or in
        // accurate mode (the bound planes always cover the whole problem)
        void *st_a = nullptr, *st_b = nullptr;
        OZK_TRY(fused_state(h, J, &st_a, &st_b));  // before the fork: its first-use memset is on this stream
        OZK_CUDA(cudaEventRecord(h->ev_fork, h->stream));
        OZK_CUDA(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
        const bool whole = P.single || !fast;
        {
            StageTimer t(h, OZK_PROFILE_SCALE);
            OZK_TRY(round_a(h, J, cfg));
        }
        const bool fa = whole && a_fusable(J);
        {
            StageTimer t(h, OZK_PROFILE_SCALE);
            OZK_TRY(fa ? stage_rows_fused(h, J, st_a) : stage_rows(h, J));
        }
        if (fast && P.single && !fa) {
            StageTimer t(h, OZK_PROFILE_RESIDUES);
            OZK_TRY(stage_row_residues(h, J, J.mu, J.pa));
        }
        auto b_chain = [&]() -> int {
            {
                StageTimer t(h, OZK_PROFILE_SCALE);
                OZK_TRY(round_b(h, J, cfg, J.b, J.ldb, 0, n));
            }
            const bool fb = whole && b_fusable(J, 0);
            {
                StageTimer t(h, OZK_PROFILE_SCALE);
                OZK_TRY(fb ? stage_cols_fused(h, J, 0, n, st_b) : stage_cols(h, J, 0, n, fast ? 0 : 1));
            }
            if (fast && P.single && !fb) {
                StageTimer t(h, OZK_PROFILE_RESIDUES);
                OZK_TRY(stage_col_residues(h, J, 0, n, J.nu, J.pb, J.pb_stride));
            }
            return OZK_OK;
        };
        // two one-pass kernels each fill the GPU and keep their lines in L2
        // until the planes pass: after a one-pass A a one-pass B follows on
        // the same stream; otherwise the chains overlap on two streams
        static const bool one_stream = std::getenv("OZK_K1_ONE_STREAM") != nullptr;  // A/B timing knob
        if (one_stream || (fa && (J.tb ? rows_fused_on() : cols_fused_on()))) {
            OZK_TRY(b_chain());
        } else {
            {
                OnSideStream side(h);
                OZK_TRY(b_chain());
                OZK_CUDA(cudaEventRecord(h->ev_join, h->stream));
            }
            OZK_CUDA(cudaStreamWaitEvent(h->stream, h->ev_join, 0));
        }
        // the bound GEMM needs both bound operands, mu and nu need its maxima
        if (!fast) OZK_TRY(bound_and_budget(h, J));
        if (!P.single) {
            OZK_TRY(run_panels(h, J, P, alpha, beta, C, ldc, c_f32));
        } else {
            OZK_TRY(single_panel(h, J, alpha, beta, C, ldc, c_f32));
        }
    }
    return finish_check(h, J, h->stream);
}

// the whole problem as one panel (the residues of fast mode are already issued
// on the two K1 streams): residues (accurate mode), K2, K3
int single_panel(ozk_context* h, Job& J, double alpha, double beta, void* C, int64_t ldc, int c_f32) {
    const int64_t n = J.n;
    {
        if (J.mode != OZK_FAST) {
            // both residue passes at once again (A on this stream, B on the side stream)
            OZK_CUDA(cudaEventRecord(h->ev_fork, h->stream));
            OZK_CUDA(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
            {
                StageTimer t(h, OZK_PROFILE_RESIDUES);
                OZK_TRY(stage_row_residues(h, J, J.mu, J.pa));
            }
            {
                OnSideStream side(h);
                StageTimer t(h, OZK_PROFILE_RESIDUES);
                OZK_TRY(stage_col_residues(h, J, 0, n, J.nu, J.pb, J.pb_stride));
                OZK_CUDA(cudaEventRecord(h->ev_join, h->stream));
            }
            OZK_CUDA(cudaStreamWaitEvent(h->stream, h->ev_join, 0));
        }
        {
            StageTimer t(h, OZK_PROFILE_PRODUCTS);
            OZK_TRY(stage_products(h, J, 0, n, J.pa, J.pa_stride, J.pb, J.pb_stride, OZK_PRODUCTS_U8, J.u, J.ldu,
                                   J.n * J.ldu));
        }
        StageTimer t(h, OZK_PROFILE_RECONSTRUCT);
        OZK_TRY(stage_reconstruct(h, J, 0, n, J.u, J.ldu, J.n * J.ldu, J.mu, J.nu, alpha, beta, C, ldc, c_f32));
    }
    return OZK_OK;
}

int64_t host_block_cols(int64_t n) {
    if (n <= 1024) return n;
    int64_t nb = (n + 7) / 8;     // about 8 blocks
    nb = (nb + 255) / 256 * 256;  // whole 256-column GEMM tiles
    return nb < 512 ? 512 : nb;
}

// ---- streamed host path (fast mode) -------------------------------------------
// Fast-mode mu_i depends on row i of A only and nu_j on column j of B, so C
// block (I, J) can be computed as soon as A's row block I and B's column
// block J are on the device. The copy stream alternates A_0, B_0, A_1, B_1, ...
// (A row blocks are pitched copies); each arrival triggers one rectangular
// region: rows I x all columns that have arrived (after A_I), or all rows that
// have arrived x columns J (after B_J). K2 therefore starts after 2/P of the
// inputs instead of after all of A, and the tail after the last byte arrives
// is one thin region plus its D2H. Results are identical to the unblocked
// call: every stage is row/column-local in fast mode.

int64_t stream_block(int64_t dim);
bool tail_split() {
    static const bool on = std::getenv("OZK_HOST_TAIL") == nullptr || std::atoi(std::getenv("OZK_HOST_TAIL")) != 0;
    return on;
}

// block boundaries along one operand dimension: ~16 blocks of whole 256-wide
// GEMM tiles, the last one split into halving pieces (b/2, b/4, ...) so the
// region computed after the final transfer, and its D2H, are short
std::vector<std::pair<int64_t, int64_t>> stream_blocks(int64_t dim) {
    const int64_t b = stream_block(dim);
    std::vector<std::pair<int64_t, int64_t>> out;
    int64_t r0 = 0;
    while (r0 < dim) {
        int64_t sz = std::min(b, dim - r0);
        const int64_t rest = dim - r0;
        if (rest <= b && rest > 256 && tail_split()) sz = std::max<int64_t>(256, (rest / 2 + 255) / 256 * 256);
        if (sz > rest) sz = rest;
        out.push_back({r0, sz});
        r0 += sz;
    }
    return out;
}

int64_t stream_block(int64_t dim) {
    int64_t b = (dim + 15) / 16;  // ~16 blocks per operand
    b = (b + 255) / 256 * 256;    // whole 256-row/column GEMM tiles
    return b < 512 ? 512 : b;
}

bool use_streamed(const Job& J, const ozk_config* cfg, double beta) {
    return J.mode == OZK_FAST && !J.ta && !J.tb && beta == 0.0 && !rounds_inputs(J, cfg) && J.m >= 2048 &&
           J.n >= 2048 && std::getenv("OZK_HOST_STREAM") == nullptr;
}

// rows [r0, r0+mr) of A, stored as an mr x k column-major block at `a` with
// leading dimension lda: stats, mu, residue planes (fast mode: all row-local)
int row_block_stats(ozk_context* h, Job& J, int64_t r0, int64_t mr, const void* a, int64_t lda) {
    int splits = row_stats_splits(mr, J.k);
    const int64_t cap = J.splits * J.m / mr;  // the [split][rows] partials live in J.amax / J.asum
    if (splits > cap) splits = static_cast<int>(cap < 1 ? 1 : cap);
    launch_row_stats(a, J.in_f32, mr, J.k, lda, splits, J.amax, J.asum, J.flags, J.cnt_a,
                     line_final(J, J.mu + r0, nullptr, a, 1, lda), h->stream);
    return check_launch(h, 1);
}

int rows_block(ozk_context* h, Job& J, int64_t r0, int64_t mr, const void* a, int64_t lda) {
    OZK_TRY(row_block_stats(h, J, r0, mr, a, lda));
    launch_a_planes(a, J.in_f32, mr, J.k, lda, J.mu + r0, J.dc, 0, J.pa + r0, J.lda_p, J.pa_stride, h->stream);
    return check_launch(h, 1);
}

int stream_a_block(ozk_context* h, Job& J, int64_t r0, int64_t mr) {
    const size_t es = J.in_f32 ? 4 : 8;
    return rows_block(h, J, r0, mr, static_cast<const char*>(J.a) + es * r0, J.lda);
}

// C[r0:r0+mr, c0:c0+nc] = alpha (A B)[region] + beta C[region] from the planes:
// K2 over the region's tiles, then K3. C is the full device matrix (ldc).
int region_products(ozk_context* h, Job& J, int64_t r0, int64_t mr, int64_t c0, int64_t nc, double alpha,
                    double beta, void* C, int64_t ldc, int c_f32) {
    {
        StageTimer t(h, OZK_PROFILE_PRODUCTS);
        K2Launch L{};
        L.a_planes = J.pa + r0;  // MN-major: rows are bytes inside a column
        L.b_planes = J.pb + c0 * J.ld;
        L.m = mr;
        L.n = nc;
        L.k = J.k;
        L.ld = J.ld;
        L.lda = J.lda_p;
        L.a_mn = true;
        L.a_stride = J.pa_stride;
        L.b_stride = J.pb_stride;
        L.n_mod = J.c.n_moduli;
        L.kind = K2_U8;
        L.out = J.u + c0 * J.ldu + r0;
        L.ldo = J.ldu;
        L.out_stride = J.n * J.ldu;
        L.c = &J.dc;
        L.num_sms = h->num_sms;
        L.sync_counter = reinterpret_cast<unsigned int*>(J.flags + 4);
        OZK_TRY(launch_k2(L, h->stream));
        OZK_TRY(check_launch(h, 1));
    }
    const size_t cs = c_f32 ? 4 : 8;
    StageTimer t(h, OZK_PROFILE_RECONSTRUCT);
    launch_reconstruct(J.u + c0 * J.ldu + r0, J.ldu, J.n * J.ldu, mr, nc, J.mu + r0, J.nu + c0, J.dc, alpha, beta,
                       static_cast<char*>(C) + cs * (c0 * ldc + r0), ldc, c_f32, h->stream);
    return check_launch(h, 1);
}

// Host <-> device copies of ozk_gemm_host: pinned (or small) caller buffers
// are DMA'd directly on the copy streams; large pageable ones go through the
// handle's pinned staging (host_stage.cpp). up() returns a ticket that
// must be passed to before_wait() before the compute stream waits on the
// copy's event.
struct HostIO {
    ozk_context* h;
    HostStager* st = nullptr;  // non-null: some buffer is staged
    bool stage_a = false, stage_b = false, stage_c = false;
    int64_t up(bool staged, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
               cudaEvent_t done, cudaError_t& err) {
        if (staged) return st->h2d(dst, dpitch, src, spitch, width, height, done);
        err = cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyHostToDevice, h->h2d);
        if (err == cudaSuccess && done) err = cudaEventRecord(done, h->h2d);
        return 0;
    }
    cudaError_t before_wait(int64_t ticket) { return ticket > 0 ? st->wait_issued(ticket) : cudaSuccess; }
    cudaError_t down(bool staged, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                     size_t height, cudaEvent_t ready) {
        if (staged) {
            st->d2h(dst, dpitch, src, spitch, width, height, ready);
            return cudaSuccess;
        }
        cudaError_t e = cudaStreamWaitEvent(h->d2h, ready, 0);
        if (e == cudaSuccess) e = cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDeviceToHost, h->d2h);
        return e;
    }
};
// every exit of ozk_gemm_host waits for the staging threads (they hold the
// caller's pointers)
struct StagerFinish {
    HostStager* st;
    ~StagerFinish() {
        if (st) st->finish();
    }
};

// C[r0:r0+mr, c0:c0+nc] from the planes (K2 + K3), then its D2H on the copy stream
// (the device staging C is m x n with pitch m; the caller's C has pitch ldc)
int stream_region(ozk_context* h, HostIO& io, Job& J, int64_t r0, int64_t mr, int64_t c0, int64_t nc, double alpha,
                  int c_f32, void* C_host, int64_t ldc, cudaEvent_t done) {
    const int64_t ldd = J.m;
    OZK_TRY(region_products(h, J, r0, mr, c0, nc, alpha, 0.0, h->host_c.p, ldd, c_f32));
    const size_t cs = c_f32 ? 4 : 8;
    const char* cdev = static_cast<const char*>(h->host_c.p) + cs * (c0 * ldd + r0);
    OZK_CUDA(cudaEventRecord(done, h->stream));
    OZK_CUDA(io.down(io.stage_c, static_cast<char*>(C_host) + cs * (c0 * ldc + r0), cs * ldc, cdev, cs * ldd, cs * mr,
                     nc, done));
    return OZK_OK;
}

int gemm_host_streamed(ozk_context* h, HostIO& io, Job& J, double alpha, const void* A, int64_t lda, const void* B,
                       int64_t ldb, void* C, int64_t ldc, int c_f32) {
    const size_t es = J.in_f32 ? 4 : 8;
    const int64_t m = J.m, n = J.n, k = J.k;
    const auto blocks_a = stream_blocks(m), blocks_b = stream_blocks(n);
    const int na = static_cast<int>(blocks_a.size()), nb = static_cast<int>(blocks_b.size());
    std::vector<cudaEvent_t> ev(na + nb + na + nb + 1);
    for (auto& e : ev) OZK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    struct EventGuard {  // the staging threads use these events: they finish first
        std::vector<cudaEvent_t>& v;
        HostStager* st;
        ~EventGuard() {
            if (st) st->finish();
            for (auto& e : v) cudaEventDestroy(e);
        }
    } guard{ev, io.st};
    cudaEvent_t evStart = ev.back();
    auto ev_a = [&](int i) { return ev[i]; };
    auto ev_b = [&](int j) { return ev[na + j]; };
    auto ev_ra = [&](int i) { return ev[na + nb + i]; };
    auto ev_rb = [&](int j) { return ev[na + nb + na + j]; };
    OZK_CUDA(cudaEventRecord(evStart, h->stream));
    OZK_CUDA(cudaStreamWaitEvent(h->h2d, evStart, 0));
    OZK_CUDA(cudaStreamWaitEvent(h->d2h, evStart, 0));
    // the copy stream: A_0, B_0, A_1, B_1, ...
    std::vector<int64_t> tk_a(na, 0), tk_b(nb, 0);
    cudaError_t ce = cudaSuccess;
    for (int s = 0; s < na || s < nb; ++s) {
        if (s < na) {
            const int64_t r0 = blocks_a[s].first, mr = blocks_a[s].second;
            tk_a[s] = io.up(io.stage_a, static_cast<char*>(h->host_a.p) + es * r0, es * m,
                            static_cast<const char*>(A) + es * r0, es * lda, es * mr, k, ev_a(s), ce);
            OZK_CUDA(ce);
        }
        if (s < nb) {
            const int64_t c0 = blocks_b[s].first, nc = blocks_b[s].second;
            tk_b[s] = io.up(io.stage_b, static_cast<char*>(h->host_b.p) + es * k * c0, es * k,
                            static_cast<const char*>(B) + es * ldb * c0, es * ldb, es * k, nc, ev_b(s), ce);
            OZK_CUDA(ce);
        }
    }
    StageTimer total(h, OZK_PROFILE_TOTAL);
    int64_t rows_in = 0, cols_in = 0;  // prefix of A rows / B columns already on the device
    for (int s = 0; s < na || s < nb; ++s) {
        if (s < na) {
            const int64_t r0 = blocks_a[s].first, mr = blocks_a[s].second;
            OZK_CUDA(io.before_wait(tk_a[s]));
            OZK_CUDA(cudaStreamWaitEvent(h->stream, ev_a(s), 0));
            {
                StageTimer t(h, OZK_PROFILE_SCALE);
                OZK_TRY(stream_a_block(h, J, r0, mr));
            }
            rows_in = r0 + mr;
            if (cols_in > 0) OZK_TRY(stream_region(h, io, J, r0, mr, 0, cols_in, alpha, c_f32, C, ldc, ev_ra(s)));
        }
        if (s < nb) {
            const int64_t c0 = blocks_b[s].first, nc = blocks_b[s].second;
            OZK_CUDA(io.before_wait(tk_b[s]));
            OZK_CUDA(cudaStreamWaitEvent(h->stream, ev_b(s), 0));
            {
                StageTimer t(h, OZK_PROFILE_SCALE);
                OZK_TRY(stage_cols(h, J, c0, nc));
            }
            {
                StageTimer t(h, OZK_PROFILE_RESIDUES);
                OZK_TRY(stage_col_residues(h, J, c0, nc, J.nu, J.pb, J.pb_stride));
            }
            cols_in = c0 + nc;
            if (rows_in > 0) OZK_TRY(stream_region(h, io, J, 0, rows_in, c0, nc, alpha, c_f32, C, ldc, ev_rb(s)));
        }
    }
    return OZK_OK;
}

// Host operands: H2D of A, then of B column blocks, on one copy stream; the
// compute of block j waits for its B block; C block j leaves on a second copy
// stream while block j+1 computes.
int gemm_host(ozk_context* h, const ozk_config* cfg, const ozk_constants& c, int64_t m, int64_t n, int64_t k,
              double alpha, const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C,
              int64_t ldc) {
    ozk_config hc = *cfg;  // host buffers: the call always completes (no OZK_FLAG_ASYNC)
    hc.flags &= ~OZK_FLAG_ASYNC;
    cfg = &hc;
    OZK_TRY(validate(cfg, c, m, n, k, lda, ldb));
    if (ldc < m) {
        set_error("gemm_emulated: ldc < m");
        return OZK_INPUT_ERROR;
    }
    OZK_CUDA(cudaSetDevice(h->device));
    if (!h->h2d) OZK_CUDA(cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking));
    if (!h->d2h) OZK_CUDA(cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking));
    const size_t es = cfg->a_type == OZK_R32F ? 4 : 8, cs = cfg->c_type == OZK_R32F ? 4 : 8;
    const bool ta = (cfg->flags & OZK_FLAG_TRANS_A) != 0, tb = (cfg->flags & OZK_FLAG_TRANS_B) != 0;
    // device staging is dense (pitch = stored rows); every transfer is a pitched
    // copy of the stored rows only, so a caller's ld > rows (a submatrix view)
    // is neither over-read nor, for C, written outside its rows
    const int64_t rows_a = ta ? k : m, cols_a = ta ? m : k, rows_b = tb ? n : k;
    OZK_TRY(ensure(h->host_a, es * rows_a * cols_a));
    OZK_TRY(ensure(h->host_b, es * rows_b * (tb ? k : n)));
    OZK_TRY(ensure(h->host_c, cs * m * n));
    Job J{};
    OZK_TRY(setup(h, J, cfg, c, m, n, k, h->host_a.p, rows_a, h->host_b.p, rows_b, true));
    const Plan P = make_plan(h, J, rounds_inputs(J, cfg) ? 4 * (m * k + k * n) : 0);
    if (!P.single) {
        // too large for one panel: the operands go to the device whole, the
        // panelled device call runs, C comes back (no copy/compute overlap)
        const int64_t cols_b = tb ? k : n;
        OZK_CUDA(cudaMemcpy2DAsync(h->host_a.p, es * rows_a, A, es * lda, es * rows_a, cols_a, cudaMemcpyHostToDevice,
                                   h->stream));
        OZK_CUDA(cudaMemcpy2DAsync(h->host_b.p, es * rows_b, B, es * ldb, es * rows_b, cols_b, cudaMemcpyHostToDevice,
                                   h->stream));
        if (beta != 0.0)
            OZK_CUDA(cudaMemcpy2DAsync(h->host_c.p, cs * m, C, cs * ldc, cs * m, n, cudaMemcpyHostToDevice, h->stream));
        OZK_TRY(gemm_device(h, cfg, c, m, n, k, alpha, h->host_a.p, rows_a, h->host_b.p, rows_b, beta, h->host_c.p,
                            m));
        OZK_CUDA(cudaMemcpy2DAsync(C, cs * ldc, h->host_c.p, cs * m, cs * m, n, cudaMemcpyDeviceToHost, h->stream));
        OZK_CUDA(cudaStreamSynchronize(h->stream));
        return OZK_OK;
    }
    OZK_TRY(alloc_plan(h, J, P));
    const void* b_src = h->host_b.p;
    const int c_f32 = cfg->c_type == OZK_R32F;
    // large pageable operands go through the pinned staging ring (OZK_HOST_STAGE=0: plain copies)
    HostIO io{h};
    {
        static const bool stage_on = std::getenv("OZK_HOST_STAGE") == nullptr || std::atoi(std::getenv("OZK_HOST_STAGE")) != 0;
        const size_t big = size_t(4) << 20;
        io.stage_a = stage_on && es * rows_a * cols_a >= big && host_is_pageable(A);
        io.stage_b = stage_on && es * rows_b * (tb ? k : n) >= big && host_is_pageable(B);
        io.stage_c = stage_on && cs * m * n >= big && host_is_pageable(C);
        if (io.stage_a || io.stage_b || io.stage_c) {
            if (!h->stager) h->stager = new HostStager(h->device);
            OZK_CUDA(h->stager->begin(h->h2d, h->d2h));
            io.st = h->stager;
        }
    }
    StagerFinish stager_finish{io.st};
    auto staged_done = [&]() -> int {
        if (io.st) OZK_CUDA(io.st->finish());
        return OZK_OK;
    };
    if (use_streamed(J, cfg, beta)) {
        OZK_CUDA(cudaSetDevice(h->device));
        OZK_TRY(gemm_host_streamed(h, io, J, alpha, A, lda, B, ldb, C, ldc, c_f32));
        OZK_TRY(staged_done());
        OZK_CUDA(cudaStreamSynchronize(h->d2h));
        return finish_check(h, J, h->stream);
    }
    const int64_t nb = host_block_cols(n);
    const int nblk = static_cast<int>((n + nb - 1) / nb);
    std::vector<cudaEvent_t> ev(2 * nblk + 2);
    for (auto& e : ev) OZK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    struct EventGuard {  // the staging threads use these events: they finish first
        std::vector<cudaEvent_t>& v;
        HostStager* st;
        ~EventGuard() {
            if (st) st->finish();
            for (auto& e : v) cudaEventDestroy(e);
        }
    } guard{ev, io.st};
    cudaEvent_t evA = ev[0], evStart = ev[1];
    auto ev_b = [&](int b) { return ev[2 + b]; };
    auto ev_c = [&](int b) { return ev[2 + nblk + b]; };
    auto block = [&](int b, int64_t& j0, int64_t& nj) {
        j0 = b * nb;
        nj = (n - j0 < nb) ? n - j0 : nb;
    };
    // the copy stream starts after the compute stream's earlier work (workspace reuse)
    OZK_CUDA(cudaEventRecord(evStart, h->stream));
    OZK_CUDA(cudaStreamWaitEvent(h->h2d, evStart, 0));
    OZK_CUDA(cudaStreamWaitEvent(h->d2h, evStart, 0));
    cudaError_t ce = cudaSuccess;
    const int64_t tk_a = io.up(io.stage_a, h->host_a.p, es * rows_a, A, es * lda, es * rows_a, cols_a, evA, ce);
    OZK_CUDA(ce);
    std::vector<int64_t> tk_b(nblk, 0);
    for (int b = 0; b < nblk; ++b) {
        int64_t j0, nj;
        block(b, j0, nj);
        cudaEvent_t after_b = beta != 0.0 ? nullptr : ev_b(b);
        if (tb)  // op(B) columns = rows j0.. of the stored n x k B
            tk_b[b] = io.up(io.stage_b, static_cast<char*>(h->host_b.p) + es * j0, es * rows_b,
                            static_cast<const char*>(B) + es * j0, es * ldb, es * nj, k, after_b, ce);
        else
            tk_b[b] = io.up(io.stage_b, static_cast<char*>(h->host_b.p) + es * rows_b * j0, es * rows_b,
                            static_cast<const char*>(B) + es * ldb * j0, es * ldb, es * rows_b, nj, after_b, ce);
        OZK_CUDA(ce);
        if (beta != 0.0) {
            // the block's event after both copies: a direct copy after a staged
            // one would not be ordered behind it, so C follows B's route
            const int64_t t = io.up(io.stage_b || io.stage_c, static_cast<char*>(h->host_c.p) + cs * m * j0, cs * m,
                                    static_cast<const char*>(C) + cs * ldc * j0, cs * ldc, cs * m, nj, ev_b(b), ce);
            OZK_CUDA(ce);
            tk_b[b] = std::max(tk_b[b], t);
        }
    }
    {
        StageTimer total(h, OZK_PROFILE_TOTAL);
        OZK_CUDA(io.before_wait(tk_a));
        OZK_CUDA(cudaStreamWaitEvent(h->stream, evA, 0));
        OZK_TRY(round_a(h, J, cfg));
        {
            StageTimer t(h, OZK_PROFILE_SCALE);
            OZK_TRY(stage_rows(h, J));
        }
        if (J.mode == OZK_ACCURATE) {
            for (int b = 0; b < nblk; ++b) {  // bound GEMM per arriving block
                int64_t j0, nj;
                block(b, j0, nj);
                OZK_CUDA(io.before_wait(tk_b[b]));
                OZK_CUDA(cudaStreamWaitEvent(h->stream, ev_b(b), 0));
                OZK_TRY(round_b(h, J, cfg, b_src, rows_b, j0, nj));
                StageTimer t(h, OZK_PROFILE_SCALE);
                OZK_TRY(stage_cols(h, J, j0, nj));
            }
            StageTimer t(h, OZK_PROFILE_SCALE);
            OZK_TRY(stage_budget(h, J));
        }
        {
            StageTimer t(h, OZK_PROFILE_RESIDUES);
            OZK_TRY(stage_row_residues(h, J, J.mu, J.pa));
        }
        for (int b = 0; b < nblk; ++b) {
            int64_t j0, nj;
            block(b, j0, nj);
            if (J.mode == OZK_FAST) {
                OZK_CUDA(io.before_wait(tk_b[b]));
                OZK_CUDA(cudaStreamWaitEvent(h->stream, ev_b(b), 0));
                OZK_TRY(round_b(h, J, cfg, b_src, rows_b, j0, nj));
                StageTimer t(h, OZK_PROFILE_SCALE);
                OZK_TRY(stage_cols(h, J, j0, nj));
            }
            OZK_TRY(compute_block(h, J, j0, nj, alpha, beta, h->host_c.p, m, c_f32));
            OZK_CUDA(cudaEventRecord(ev_c(b), h->stream));
            OZK_CUDA(io.down(io.stage_c, static_cast<char*>(C) + cs * ldc * j0, cs * ldc,
                             static_cast<const char*>(h->host_c.p) + cs * m * j0, cs * m, cs * m, nj, ev_c(b)));
        }
    }
    OZK_TRY(staged_done());
    OZK_CUDA(cudaStreamSynchronize(h->d2h));
    return finish_check(h, J, h->stream);
}

}  // namespace

extern "C" {

const char* ozk_last_error(void) { return g_error.c_str(); }
int ozk_version(void) { return 2; }

ozk_config ozk_default_config(int n_moduli, int mode, int precision) {
    ozk_config c{};
    c.n_moduli = n_moduli;
    c.mode = mode;
    c.precision = precision;
    c.a_type = precision == OZK_FP32 ? OZK_R32F : OZK_R64F;
    c.c_type = OZK_R64F;
    c.block_k = OZK_ENGINE_MAX_K;
    c.constants = nullptr;
    return c;
}

int ozk_create(ozk_handle* handle, int device) {
    if (!handle) return OZK_INPUT_ERROR;
    *handle = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        set_error("no CUDA device available (this library has no CPU fallback)");
        return OZK_CUDA_ERROR;
    }
    if (device < 0 || device >= count) {
        set_error("device ordinal out of range");
        return OZK_INPUT_ERROR;
    }
    cudaDeviceProp prop{};
    OZK_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        set_error(std::string("needs an sm_100 (B200) device, found ") + prop.name);
        return OZK_CUDA_ERROR;
    }
    OZK_CUDA(cudaSetDevice(device));
    auto* h = new ozk_context();
    h->device = device;
    h->num_sms = prop.multiProcessorCount;
    e = cudaMallocHost(reinterpret_cast<void**>(&h->flags_host), 64);
    if (e != cudaSuccess) {
        delete h;
        return cuda_fail("cudaMallocHost", e);
    }
    if (cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess) {
        ozk_destroy(h);
        set_error("side stream / events");
        return OZK_CUDA_ERROR;
    }
    // the device flag words (non-finite, flagged lines, K2 lockstep counters):
    // allocated and cleared once, so the sticky OZK_FLAG_ASYNC word starts at 0
    if (ensure(h->flags, 2048) != OZK_OK || cudaMemset(h->flags.p, 0, 2048) != cudaSuccess) {
        const std::string err = ozk_last_error();
        ozk_destroy(h);
        set_error("flag buffer: " + err);
        return OZK_CUDA_ERROR;
    }
    *handle = h;
    return OZK_OK;
}

int ozk_destroy(ozk_handle h) {
    if (!h) return OZK_OK;
    cudaSetDevice(h->device);
    for (Buf* b : {&h->wide, &h->cbar, &h->counters, &h->fused, &h->planes_a, &h->planes_b, &h->u, &h->stats, &h->ints,
                   &h->flags, &h->f32a, &h->f32b, &h->host_a,
                   &h->host_b, &h->host_c})
        if (b->p) cudaFree(b->p);
    if (h->flags_host) cudaFreeHost(h->flags_host);
    delete h->stager;
    if (h->side) cudaStreamDestroy(h->side);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    if (h->h2d) cudaStreamDestroy(h->h2d);
    if (h->d2h) cudaStreamDestroy(h->d2h);
    for (auto& p : h->pending) {
        cudaEventDestroy(p.second.first);
        cudaEventDestroy(p.second.second);
    }
    delete h;
    return OZK_OK;
}

int ozk_set_stream(ozk_handle h, void* stream) {
    if (!h) return OZK_INPUT_ERROR;
    h->stream = static_cast<cudaStream_t>(stream);
    return OZK_OK;
}

int64_t ozk_kernel_launches(ozk_handle h) { return h ? h->launches : 0; }

int ozk_profile(ozk_handle h, int enable) {
    if (!h) return OZK_INPUT_ERROR;
    h->profiling = enable != 0;
    return OZK_OK;
}

int ozk_profile_read(ozk_handle h, double* ms, int64_t* calls, int reset) {
    if (!h) return OZK_INPUT_ERROR;
    OZK_CUDA(cudaSetDevice(h->device));
    for (auto& p : h->pending) {
        float t = 0.f;
        OZK_CUDA(cudaEventSynchronize(p.second.second));
        OZK_CUDA(cudaEventElapsedTime(&t, p.second.first, p.second.second));
        h->stage_ms[p.first] += t;
        h->stage_calls[p.first] += 1;
        cudaEventDestroy(p.second.first);
        cudaEventDestroy(p.second.second);
    }
    h->pending.clear();
    for (int i = 0; i < OZK_PROFILE_SLOTS; ++i) {
        if (ms) ms[i] = h->stage_ms[i];
        if (calls) calls[i] = h->stage_calls[i];
        if (reset) {
            h->stage_ms[i] = 0.0;
            h->stage_calls[i] = 0;
        }
    }
    return OZK_OK;
}

int ozk_k3_replays(ozk_handle h, unsigned long long* count, int reset) {
    if (!h) return OZK_INPUT_ERROR;
    OZK_CUDA(cudaSetDevice(h->device));
    unsigned long long* d = k3_replay_counter(true);
    if (!d) return cuda_fail("k3 replay counter", cudaErrorMemoryAllocation);
    OZK_CUDA(cudaDeviceSynchronize());
    unsigned long long v = 0;
    OZK_CUDA(cudaMemcpy(&v, d, sizeof(v), cudaMemcpyDeviceToHost));
    if (count) *count = v;
    if (reset) OZK_CUDA(cudaMemset(d, 0, sizeof(v)));
    return OZK_OK;
}

int64_t ozk_plane_ld(int64_t k) { return plane_ld(k); }

int ozk_fast_floor(float pp_fast, double ub, int from_table) {
    if (!from_table) return fast_floor_host(pp_fast, ub);
    const FastFloorTable T = fast_floor_table(pp_fast);
    int f = T.floor0;
    for (int i = 0; i < T.n; ++i) f -= ub >= T.thr[i] ? 1 : 0;
    return f;
}

int ozk_set_workspace_limit(ozk_handle h, int64_t bytes) {
    if (!h || bytes < 0) return OZK_INPUT_ERROR;
    h->ws_limit = bytes;
    return OZK_OK;
}

int64_t ozk_workspace_bytes(ozk_handle h) {
    if (!h) return 0;
    int64_t total = 0;
    for (const Buf* b : {&h->wide, &h->cbar, &h->counters, &h->fused, &h->planes_a, &h->planes_b, &h->u, &h->stats,
                         &h->ints, &h->flags, &h->f32a, &h->f32b, &h->host_a, &h->host_b, &h->host_c})
        total += static_cast<int64_t>(b->bytes);
    return total;
}

int ozk_release_workspace(ozk_handle h) {
    if (!h) return OZK_INPUT_ERROR;
    if (h->shard_open || h->stream_open) {
        set_error("ozk_release_workspace: a shard is open on this handle");
        return OZK_INPUT_ERROR;
    }
    OZK_CUDA(cudaSetDevice(h->device));
    OZK_CUDA(cudaDeviceSynchronize());
    for (Buf* b : {&h->wide, &h->cbar, &h->planes_a, &h->planes_b, &h->u, &h->f32a, &h->f32b, &h->host_a, &h->host_b,
                   &h->host_c})
        release(*b);
    return OZK_OK;
}

int ozk_last_plan(ozk_handle h, int64_t out[4]) {
    if (!h || !out) return OZK_INPUT_ERROR;
    for (int i = 0; i < 4; ++i) out[i] = h->last_plan[i];
    return OZK_OK;
}

int ozk_sync(ozk_handle h) {
    if (!h) return OZK_INPUT_ERROR;
    OZK_CUDA(cudaSetDevice(h->device));
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    if (!h->flags.p) return OZK_OK;
    OZK_CUDA(cudaMemcpy(h->flags_host, h->flags.p, sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (h->flags_host[0]) {
        OZK_CUDA(cudaMemset(h->flags.p, 0, sizeof(int32_t)));
        set_error("gemm_emulated: non-finite entry in A or B");
        return OZK_INPUT_ERROR;
    }
    return OZK_OK;
}

int ozk_gemm(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, double alpha, const void* A,
             int64_t lda, const void* B, int64_t ldb, double beta, void* C, int64_t ldc) {
    if (!h) return OZK_INPUT_ERROR;
    ozk_constants c;
    OZK_TRY(resolve(cfg, c));
    return gemm_device(h, cfg, c, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
}

int ozk_gemm_host(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, double alpha,
                  const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C, int64_t ldc) {
    if (!h) return OZK_INPUT_ERROR;
    ozk_constants c;
    OZK_TRY(resolve(cfg, c));
    return gemm_host(h, cfg, c, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
}

int ozk_dgemm(ozk_handle h, int n_moduli, int mode, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
              int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
    const ozk_config cfg = ozk_default_config(n_moduli, mode, OZK_FP64);
    return ozk_gemm(h, &cfg, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
}

int ozk_sgemm(ozk_handle h, int n_moduli, int mode, int64_t m, int64_t n, int64_t k, float alpha, const float* A,
              int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc) {
    ozk_config cfg = ozk_default_config(n_moduli, mode, OZK_FP32);
    cfg.c_type = OZK_R32F;
    return ozk_gemm(h, &cfg, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
}

int ozk_dgemm_ex(ozk_handle h, int n_moduli, int mode, char transa, char transb, int64_t m, int64_t n, int64_t k,
                 double alpha, const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
                 int64_t ldc) {
    auto flag = [](char t, int bit, int32_t& f) {
        if (t == 'N' || t == 'n') return true;
        if (t == 'T' || t == 't' || t == 'C' || t == 'c') {
            f |= bit;
            return true;
        }
        return false;
    };
    ozk_config cfg = ozk_default_config(n_moduli, mode, OZK_FP64);
    if (!flag(transa, OZK_FLAG_TRANS_A, cfg.flags) || !flag(transb, OZK_FLAG_TRANS_B, cfg.flags)) {
        set_error("ozk_dgemm_ex: trans must be 'N' or 'T'");
        return OZK_CONFIG_ERROR;
    }
    return ozk_gemm(h, &cfg, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
}

int ozk_gemm_strided_batched(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, double alpha,
                             const void* A, int64_t lda, int64_t stride_a, const void* B, int64_t ldb,
                             int64_t stride_b, double beta, void* C, int64_t ldc, int64_t stride_c, int64_t batch) {
    if (!h) return OZK_INPUT_ERROR;
    if (batch < 0) {
        set_error("ozk_gemm_strided_batched: negative batch");
        return OZK_INPUT_ERROR;
    }
    ozk_constants c;
    OZK_TRY(resolve(cfg, c));  // the table is built once for the batch
    const size_t ea = cfg->a_type == OZK_R32F ? 4 : 8, ec = cfg->c_type == OZK_R32F ? 4 : 8;
    for (int64_t b = 0; b < batch; ++b)
        OZK_TRY(gemm_device(h, cfg, c, m, n, k, alpha, static_cast<const char*>(A) + ea * stride_a * b, lda,
                            static_cast<const char*>(B) + ea * stride_b * b, ldb, beta,
                            static_cast<char*>(C) + ec * stride_c * b, ldc));
    return OZK_OK;
}

int ozk_shard_begin(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, const void* A,
                    int64_t lda, const void* B, int64_t ldb) {
    if (!h) return OZK_INPUT_ERROR;
    ozk_constants c;
    OZK_TRY(resolve(cfg, c));
    OZK_TRY(validate(cfg, c, m, n, k, lda, ldb));
    if (cfg->mode == OZK_ACCURATE && bound_needs_int64(k)) {
        // ozk_shard_rowmax exchanges int32 maxima
        set_error("column-shard accurate mode supports k < 2^19");
        return OZK_INPUT_ERROR;
    }
    OZK_CUDA(cudaSetDevice(h->device));
    Job& J = h->shard;
    J = Job{};
    OZK_TRY(setup(h, J, cfg, c, m, n, k, A, lda, B, ldb, true));
    h->shard_plan = make_plan(h, J, rounds_inputs(J, cfg) ? 4 * (m * k + k * n) : 0);
    OZK_TRY(alloc_plan(h, J, h->shard_plan));
    h->shard_cfg = *cfg;
    h->shard_cfg.constants = nullptr;  // resolved into J.c
    {
        StageTimer t(h, OZK_PROFILE_SCALE);
        const void* b_src = J.b;
        OZK_TRY(round_a(h, J, cfg));
        OZK_TRY(round_b(h, J, cfg, b_src, ldb, 0, n));
        OZK_TRY(stage_rows(h, J));
        OZK_TRY(stage_cols(h, J, 0, n));  // accurate: partial row maxima over this shard's columns
    }
    h->shard_open = true;
    return OZK_OK;
}

int32_t* ozk_shard_rowmax(ozk_handle h) {
    if (!h || !h->shard_open) return nullptr;
    return h->shard.rowmax;
}

int ozk_shard_end(ozk_handle h, double alpha, double beta, void* C, int64_t ldc) {
    if (!h || !h->shard_open) {
        set_error("ozk_shard_end without ozk_shard_begin");
        return OZK_INPUT_ERROR;
    }
    h->shard_open = false;
    Job& J = h->shard;
    if (ldc < J.m) {
        set_error("gemm_emulated: ldc < m");
        return OZK_INPUT_ERROR;
    }
    OZK_CUDA(cudaSetDevice(h->device));
    if (J.mode == OZK_ACCURATE) {
        StageTimer t(h, OZK_PROFILE_SCALE);
        OZK_TRY(stage_budget(h, J));
    }
    const int c_f32 = h->shard_cfg.c_type == OZK_R32F;
    if (!h->shard_plan.single) {
        OZK_TRY(run_panels(h, J, h->shard_plan, alpha, beta, C, ldc, c_f32));
        return finish_check(h, J, h->stream);
    }
    {
        StageTimer t(h, OZK_PROFILE_RESIDUES);
        OZK_TRY(stage_row_residues(h, J, J.mu, J.pa));
    }
    OZK_TRY(compute_block(h, J, 0, J.n, alpha, beta, C, ldc, c_f32));
    return finish_check(h, J, h->stream);
}

int ozk_shard_stream_begin(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, const void* B,
                           int64_t ldb, double alpha, double beta, void* C, int64_t ldc) {
    if (!h) return OZK_INPUT_ERROR;
    ozk_constants c;
    OZK_TRY(resolve(cfg, c));
    OZK_TRY(validate(cfg, c, m, n, k, m, ldb));
    if (cfg->mode != OZK_FAST || (cfg->flags & (OZK_FLAG_TRANS_A | OZK_FLAG_TRANS_B)) ||
        (cfg->precision == OZK_FP32 && cfg->a_type == OZK_R64F)) {
        // accurate-mode mu needs every column's bound first; rounding / transposed
        // operands keep the whole-A path (ozk_shard_begin)
        set_error("row-streamed shard: fast mode, untransposed operands stored in the compute precision only");
        return OZK_CONFIG_ERROR;
    }
    if (ldc < m) {
        set_error("gemm_emulated: ldc < m");
        return OZK_INPUT_ERROR;
    }
    OZK_CUDA(cudaSetDevice(h->device));
    Job& J = h->shard;
    J = Job{};
    OZK_TRY(setup(h, J, cfg, c, m, n, k, nullptr, m, B, ldb, true));
    // the shard's B planes live for the whole call; A's planes and U are per
    // row block (sized, and reused, in ozk_shard_stream_rows)
    OZK_TRY(ensure(h->planes_b, static_cast<size_t>(c.n_moduli * J.pb_stride)));
    J.pb = static_cast<int8_t*>(h->planes_b.p);
    h->shard_cfg = *cfg;
    h->shard_cfg.constants = nullptr;
    h->stream_alpha = alpha;
    h->stream_beta = beta;
    h->stream_c = C;
    h->stream_ldc = ldc;
    h->stream_c_f32 = cfg->c_type == OZK_R32F;
    h->stream_rows = 0;
    {
        StageTimer t(h, OZK_PROFILE_SCALE);
        OZK_TRY(stage_cols(h, J, 0, n));
    }
    {
        StageTimer t(h, OZK_PROFILE_RESIDUES);
        OZK_TRY(stage_col_residues(h, J, 0, n, J.nu, J.pb, J.pb_stride));
    }
    h->stream_open = true;
    return OZK_OK;
}

int ozk_shard_stream_rows(ozk_handle h, int64_t r0, int64_t mr, const void* A_rows, int64_t lda_rows) {
    if (!h || !h->stream_open) {
        set_error("ozk_shard_stream_rows without ozk_shard_stream_begin");
        return OZK_INPUT_ERROR;
    }
    Job& J = h->shard;
    if (r0 < 0 || mr < 1 || r0 + mr > J.m || lda_rows < mr || !A_rows || r0 % 16 != 0) {
        set_error("ozk_shard_stream_rows: row block outside [0, m), lda < rows, or r0 not a multiple of 16");
        return OZK_INPUT_ERROR;
    }
    OZK_CUDA(cudaSetDevice(h->device));
    // this block's planes and U at offset 0 of buffers sized for the block: the
    // blocks run in stream order, so one buffer of each serves them all
    const int N = J.c.n_moduli;
    OZK_TRY(ensure(h->planes_a, static_cast<size_t>(N * a_panel_plane(J, mr))));
    OZK_TRY(ensure(h->u, static_cast<size_t>(N * J.n * u_ld(mr))));
    J.pa = static_cast<int8_t*>(h->planes_a.p);
    J.u = static_cast<uint8_t*>(h->u.p);
    {
        StageTimer t(h, OZK_PROFILE_SCALE);
        OZK_TRY(row_block_stats(h, J, r0, mr, A_rows, lda_rows));
    }
    {
        StageTimer t(h, OZK_PROFILE_RESIDUES);
        launch_a_planes(A_rows, J.in_f32, mr, J.k, lda_rows, J.mu + r0, J.dc, 0, J.pa, a_panel_ld(J, mr),
                        a_panel_plane(J, mr), h->stream);
        OZK_TRY(check_launch(h, 1));
    }
    h->stream_rows += mr;
    return panel_region(h, J, r0, mr, 0, J.n, h->stream_alpha, h->stream_beta, h->stream_c, h->stream_ldc,
                        h->stream_c_f32);
}

int ozk_shard_stream_end(ozk_handle h) {
    if (!h || !h->stream_open) {
        set_error("ozk_shard_stream_end without ozk_shard_stream_begin");
        return OZK_INPUT_ERROR;
    }
    h->stream_open = false;
    Job& J = h->shard;
    if (h->stream_rows != J.m) {
        set_error("ozk_shard_stream_end: the row blocks do not cover the m rows of A");
        return OZK_INPUT_ERROR;
    }
    OZK_CUDA(cudaSetDevice(h->device));
    return finish_check(h, J, h->stream);
}

int ozk_stage_scale(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                    const void* B, int64_t ldb, int32_t* mu_exp, int32_t* nu_exp) {
    if (!h) return OZK_INPUT_ERROR;
    ozk_constants c;
    OZK_TRY(resolve(cfg, c));
    OZK_TRY(validate(cfg, c, m, n, k, lda, ldb));
    OZK_CUDA(cudaSetDevice(h->device));
    Job J{};
    OZK_TRY(setup(h, J, cfg, c, m, n, k, A, lda, B, ldb, false));
    OZK_TRY(scale_all(h, J, cfg));
    OZK_CUDA(cudaMemcpyAsync(mu_exp, J.mu, sizeof(int32_t) * m, cudaMemcpyDeviceToDevice, h->stream));
    OZK_CUDA(cudaMemcpyAsync(nu_exp, J.nu, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, h->stream));
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
}

int ozk_stage_residues(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, const void* A,
                       int64_t lda, const void* B, int64_t ldb, const int32_t* mu_exp, const int32_t* nu_exp,
                       int8_t* a_planes, int8_t* b_planes) {
    if (!h) return OZK_INPUT_ERROR;
    ozk_constants c;
    OZK_TRY(resolve(cfg, c));
    OZK_TRY(validate(cfg, c, m, n, k, lda, ldb));
    OZK_CUDA(cudaSetDevice(h->device));
    if (cfg->flags & (OZK_FLAG_TRANS_A | OZK_FLAG_TRANS_B)) {
        set_error("ozk_stage_residues: the stage API takes untransposed operands");
        return OZK_CONFIG_ERROR;
    }
    Job J{};
    OZK_TRY(setup(h, J, cfg, c, m, n, k, A, lda, B, ldb, false));
    const void* b_src = J.b;
    OZK_TRY(round_a(h, J, cfg));
    OZK_TRY(round_b(h, J, cfg, b_src, ldb, 0, n));
    OZK_TRY(stage_row_residues(h, J, mu_exp, a_planes));
    OZK_TRY(stage_col_residues(h, J, 0, n, nu_exp, b_planes, J.pb_stride));
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
}

int ozk_stage_products(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, const int8_t* a_planes,
                       const int8_t* b_planes, int kind, void* out, int64_t ldo) {
    if (!h) return OZK_INPUT_ERROR;
    ozk_constants c;
    OZK_TRY(resolve(cfg, c));
    if (m < 1 || n < 1 || k < 1 || ldo < m) {
        set_error("ozk_stage_products: bad dimensions");
        return OZK_INPUT_ERROR;
    }
    if (k > OZK_ENGINE_MAX_K && kind == OZK_PRODUCTS_I32) {  // int8_engine.cpp:44 (U8 runs blocked)
        set_error("int8_gemm: k exceeds 2^17, use blocked_int8_gemm");
        return OZK_INPUT_ERROR;
    }
    OZK_CUDA(cudaSetDevice(h->device));
    OZK_TRY(ensure(h->flags, 2048));
    Job J{};
    J.flags = static_cast<int32_t*>(h->flags.p);
    J.c = c;
    J.dc = to_dev(c);
    J.m = m;
    J.n = n;
    J.k = k;
    J.ld = plane_ld(k);
    J.lda_p = plane_ld(m);
    OZK_TRY(stage_products(h, J, 0, n, a_planes, k * J.lda_p, b_planes, n * J.ld, kind, out, ldo, ldo * n));
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
}

int ozk_stage_reconstruct(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, const uint8_t* U, int64_t ldu,
                          const int32_t* mu_exp, const int32_t* nu_exp, double alpha, double beta, void* C,
                          int64_t ldc) {
    if (!h) return OZK_INPUT_ERROR;
    ozk_constants c;
    OZK_TRY(resolve(cfg, c));
    if (m < 1 || n < 1 || ldu < m || ldc < m || (ldu % 8) != 0) {
        set_error("ozk_stage_reconstruct: bad dimensions (ldu must be a multiple of 8)");
        return OZK_INPUT_ERROR;
    }
    OZK_CUDA(cudaSetDevice(h->device));
    Job J{};
    J.c = c;
    J.dc = to_dev(c);
    J.m = m;
    J.n = n;
    OZK_TRY(stage_reconstruct(h, J, 0, n, U, ldu, ldu * n, mu_exp, nu_exp, alpha, beta, C, ldc,
                              cfg->c_type == OZK_R32F));
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
}

int ozk_int8_gemm(ozk_handle h, int64_t m, int64_t n, int64_t k, const int8_t* A, int64_t lda, const int8_t* B,
                  int64_t ldb, int32_t* C, int64_t ldc) {
    if (!h) return OZK_INPUT_ERROR;
    if (m < 0 || n < 0 || k < 0 || lda < m || ldb < k || ldc < m || (lda % 16) || (ldb % 16)) {
        set_error("int8_gemm: bad dimensions (lda, ldb must be multiples of 16)");
        return OZK_INPUT_ERROR;
    }
    if (k > OZK_ENGINE_MAX_K) {
        set_error("int8_gemm: k exceeds 2^17, use blocked_int8_gemm");
        return OZK_INPUT_ERROR;
    }
    OZK_CUDA(cudaSetDevice(h->device));
    if (m == 0 || n == 0) return OZK_OK;
    if (k == 0) {
        for (int64_t j = 0; j < n; ++j) OZK_CUDA(cudaMemsetAsync(C + j * ldc, 0, sizeof(int32_t) * m, h->stream));
        OZK_CUDA(cudaStreamSynchronize(h->stream));
        return OZK_OK;
    }
    OZK_TRY(ensure(h->flags, 2048));
    Job J{};
    J.flags = static_cast<int32_t*>(h->flags.p);
    J.c.n_moduli = 1;  // one plane, raw int32 output: no modulus involved
    J.dc.n = 1;
    J.m = m;
    J.n = n;
    J.k = k;
    J.ld = ldb;
    J.lda_p = lda;
    OZK_TRY(stage_products(h, J, 0, n, A, k * lda, B, n * ldb, OZK_PRODUCTS_I32, C, ldc, ldc * n));
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
}

int ozk_int8_gemm_reference(ozk_handle h, int64_t m, int64_t n, int64_t k, const int8_t* A, int64_t lda,
                            const int8_t* B, int64_t ldb, int32_t* C, int64_t ldc) {
    if (!h) return OZK_INPUT_ERROR;
    if (m < 0 || n < 0 || k < 0 || lda < m || ldb < k || ldc < m) {
        set_error("int8_gemm_reference: bad dimensions");
        return OZK_INPUT_ERROR;
    }
    if (k > OZK_ENGINE_MAX_K) {
        set_error("int8_gemm_reference: k exceeds 2^17");
        return OZK_INPUT_ERROR;
    }
    OZK_CUDA(cudaSetDevice(h->device));
    if (m == 0 || n == 0) return OZK_OK;
    launch_int8_gemm_simple(A, B, m, n, k, lda, ldb, C, ldc, h->stream);
    OZK_TRY(check_launch(h, 1));
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
}

int ozk_truncate_scale(ozk_handle h, int type, int64_t rows, int64_t cols, const void* x, int64_t ldx,
                       const int32_t* scale_exp, int side, void* out, int64_t ldo) {
    if (!h || rows < 0 || cols < 0 || ldx < rows || ldo < rows) return OZK_INPUT_ERROR;
    OZK_CUDA(cudaSetDevice(h->device));
    if (rows * cols == 0) return OZK_OK;
    launch_truncate(type == OZK_R32F, x, rows, cols, ldx, scale_exp, side, out, ldo, h->stream);
    OZK_TRY(check_launch(h, 1));
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
}

int ozk_residues(ozk_handle h, const ozk_config* cfg, int64_t rows, int64_t cols, const void* x, int64_t ldx,
                 int8_t* planes, int64_t ldp) {
    if (!h) return OZK_INPUT_ERROR;
    ozk_constants c;
    OZK_TRY(resolve(cfg, c));
    if (rows < 0 || cols < 0 || ldx < rows || ldp < rows) return OZK_INPUT_ERROR;
    OZK_CUDA(cudaSetDevice(h->device));
    if (rows * cols == 0) return OZK_OK;
    launch_residues_literal(cfg->a_type == OZK_R32F, x, rows, cols, ldx, to_dev(c), planes, ldp, h->stream);
    OZK_TRY(check_launch(h, 1));
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
}

int ozk_mod_u8_array(ozk_handle h, int64_t count, const int32_t* x, int32_t p, int32_t pinv_mulhi, uint8_t* out) {
    if (!h || count < 0) return OZK_INPUT_ERROR;
    OZK_CUDA(cudaSetDevice(h->device));
    if (!count) return OZK_OK;
    launch_mod_u8(x, count, p, pinv_mulhi, out, h->stream);
    OZK_TRY(check_launch(h, 1));
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
}

int ozk_accumulate(ozk_handle h, const ozk_config* cfg, int64_t count, const uint8_t* u, double* c1, double* c2) {
    if (!h || count < 0) return OZK_INPUT_ERROR;
    ozk_constants c;
    OZK_TRY(resolve(cfg, c));
    OZK_CUDA(cudaSetDevice(h->device));
    if (!count) return OZK_OK;
    launch_accumulate(u, count, to_dev(c), c1, c2, h->stream);
    OZK_TRY(check_launch(h, 1));
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
}

int ozk_crt_reduce(ozk_handle h, const ozk_config* cfg, int64_t count, const double* c1, const double* c2,
                   double* out) {
    if (!h || count < 0) return OZK_INPUT_ERROR;
    ozk_constants c;
    OZK_TRY(resolve(cfg, c));
    OZK_CUDA(cudaSetDevice(h->device));
    if (!count) return OZK_OK;
    launch_crt_reduce(c1, c2, count, to_dev(c), out, h->stream);
    OZK_TRY(check_launch(h, 1));
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
}

int ozk_unscale(ozk_handle h, int64_t m, int64_t n, const double* cpp, int64_t ldc, const int32_t* mu_exp,
                const int32_t* nu_exp, double* out, int64_t ldo) {
    if (!h || m < 0 || n < 0 || ldc < m || ldo < m) return OZK_INPUT_ERROR;
    OZK_CUDA(cudaSetDevice(h->device));
    if (m * n == 0) return OZK_OK;
    launch_unscale(cpp, m, n, ldc, mu_exp, nu_exp, out, ldo, h->stream);
    OZK_TRY(check_launch(h, 1));
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
}

}  // extern "C"
