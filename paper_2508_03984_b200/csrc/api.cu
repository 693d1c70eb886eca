// C-ABI implementation: context, workspace and the stage pipeline of
// emulate<T> (reference: emulator.cpp:25-78), all on one CUDA stream:
//
//   validate (emulator.cpp:12-23)            host checks + device finite flag
//   [FP32 precision on FP64 data: round]     emulator.cpp:84-91
//   K1a scale  (scaling.cpp)                 row/col stats -> exponents
//   K1b truncate + residues (residue.cpp)    int8 K-major planes
//   K2  N residue GEMMs + mod epilogue       tcgen05 kind::i8 -> uint8 U_i
//   K3  accumulate, CRT reduce, unscale      FP64/FP32 C (+ alpha/beta)
//
// Nothing here computes on the CPU: the host only validates arguments, sizes
// the workspace and launches kernels. Without a usable CUDA device every
// compute entry point fails with OZK_CUDA_ERROR (no fallback).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "ozaki2_b200.h"
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
    return d;
}

}  // namespace ozk

using namespace ozk;

struct ozk_context {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    int64_t launches = 0;
    Buf planes_a, planes_b, u, stats, ints, flags, f32a, f32b, host_a, host_b, host_c;
    int32_t* flags_host = nullptr;  // pinned mirror of the device flag word
    // stage timing (ozk_profile): CUDA events on the launching stream
    bool profiling = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    double stage_ms[OZK_PROFILE_SLOTS] = {};
    int64_t stage_calls[OZK_PROFILE_SLOTS] = {};
};

namespace {

int cuda_fail(const char* what, cudaError_t e) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return OZK_CUDA_ERROR;
}

#define OZK_CUDA(call)                                         \
    do {                                                       \
        const cudaError_t e_ = (call);                         \
        if (e_ != cudaSuccess) return cuda_fail(#call, e_);    \
    } while (0)

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

// RAII bracket recording a start/stop event pair for one stage slot
struct StageTimer {
    ozk_context* h;
    int slot;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    StageTimer(ozk_context* hh, int s) : h(hh), slot(s) {
        if (!h->profiling) return;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, h->stream);
    }
    ~StageTimer() {
        if (!h->profiling) return;
        cudaEventRecord(e1, h->stream);
        h->pending.push_back({slot, {e0, e1}});
    }
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
    if (c.precision == OZK_FP64 && cfg->a_type == OZK_R32F) {
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
    if (lda < m || ldb < k) {
        set_error("gemm_emulated: leading dimension smaller than the matrix");
        return OZK_INPUT_ERROR;
    }
    if (cfg->mode != OZK_FAST && cfg->mode != OZK_ACCURATE) {
        set_error("gemm_emulated: unknown scaling mode");
        return OZK_CONFIG_ERROR;
    }
    if (k > OZK_ENGINE_MAX_K) {
        // TODO(next round): chunked k > 2^17 (emulator.cpp:57-73); the per-modulus
        // U_i do not depend on the blocking, so this is a K2 chunk loop.
        set_error("k > 2^17 is not supported yet");
        return OZK_INPUT_ERROR;
    }
    return OZK_OK;
}

struct Inputs {
    const void* a;
    const void* b;
    int64_t lda, ldb;
    int is_f32;
};

// FP32 precision with FP64 storage: round both operands first (emulator.cpp:84-91)
int prepare_inputs(ozk_context* h, const ozk_config* cfg, const ozk_constants& c, int64_t m, int64_t n, int64_t k,
                   const void* A, int64_t lda, const void* B, int64_t ldb, Inputs& in) {
    in = {A, B, lda, ldb, cfg->a_type == OZK_R32F};
    if (c.precision == OZK_FP32 && cfg->a_type == OZK_R64F) {
        int st;
        if ((st = ensure(h->f32a, sizeof(float) * m * k))) return st;
        if ((st = ensure(h->f32b, sizeof(float) * k * n))) return st;
        launch_round_to_f32(static_cast<const double*>(A), m, k, lda, static_cast<float*>(h->f32a.p), h->stream);
        launch_round_to_f32(static_cast<const double*>(B), k, n, ldb, static_cast<float*>(h->f32b.p), h->stream);
        if ((st = check_launch(h, 2))) return st;
        in = {h->f32a.p, h->f32b.p, m, k, 1};
    }
    return OZK_OK;
}


// int32 scratch layout inside h->ints
struct IntScratch {
    int32_t *mu, *nu, *ma, *nb, *rowmax, *colmax, *flag_rows, *flag_cols;
};
IntScratch carve_ints(ozk_context* h, int64_t m, int64_t n) {
    int32_t* p = static_cast<int32_t*>(h->ints.p);
    IntScratch s;
    s.mu = p;
    s.nu = s.mu + m;
    s.ma = s.nu + n;
    s.nb = s.ma + m;
    s.rowmax = s.nb + n;
    s.colmax = s.rowmax + m;
    s.flag_rows = s.colmax + n;
    s.flag_cols = s.flag_rows + m;
    return s;
}

// K1a. mu/nu exponents into (mu, nu); may use planes_a/planes_b as scratch (accurate).
int run_scale(ozk_context* h, const ozk_constants& c, int mode, int64_t m, int64_t n, int64_t k, const Inputs& in,
              int32_t* mu, int32_t* nu, int32_t* flags_dev) {
    int st;
    const DevConsts dc = to_dev(c);
    LineStats ls{};
    ls.splits = row_stats_splits(m, k);
    if ((st = ensure(h->stats, sizeof(double) * (2 * ls.splits * m + 2 * n)))) return st;
    double* d = static_cast<double*>(h->stats.p);
    ls.amax = d;
    ls.asum = d + ls.splits * m;
    ls.bmax = d + 2 * ls.splits * m;
    ls.bsum = ls.bmax + n;
    ls.nonfinite = flags_dev;
    if ((st = ensure(h->ints, sizeof(int32_t) * 5 * (m + n)))) return st;
    IntScratch is = carve_ints(h, m, n);

    launch_row_stats(in.a, in.is_f32, m, k, in.lda, ls, h->stream);
    launch_col_stats(in.b, in.is_f32, k, n, in.ldb, ls, h->stream);
    if ((st = check_launch(h, 2))) return st;
    if (mode == OZK_FAST) {
        launch_fast_finalize(ls, m, n, k, dc, mu, nu, flags_dev + 1, is.flag_rows, is.flag_cols, h->stream);
        launch_fast_exact(in.a, in.b, in.is_f32, m, n, k, in.lda, in.ldb, dc, flags_dev + 1, is.flag_rows,
                          is.flag_cols, mu, nu, h->stream);
        return check_launch(h, 2);
    }
    // accurate: mu' exponents, Abar/Bbar planes, bound GEMM with max epilogue, budget
    launch_accurate_base(ls, m, n, is.ma, is.nb, h->stream);
    const int64_t ld = plane_ld(k);
    if ((st = ensure(h->planes_a, static_cast<size_t>(m * ld * (c.n_moduli > 1 ? c.n_moduli : 1))))) return st;
    if ((st = ensure(h->planes_b, static_cast<size_t>(n * ld * (c.n_moduli > 1 ? c.n_moduli : 1))))) return st;
    int8_t* abar = static_cast<int8_t*>(h->planes_a.p);
    int8_t* bbar = static_cast<int8_t*>(h->planes_b.p);
    launch_a_planes(in.a, in.is_f32, m, k, in.lda, is.ma, dc, 1, abar, ld, h->stream);
    launch_b_planes(in.b, in.is_f32, k, n, in.ldb, is.nb, dc, 1, bbar, ld, h->stream);
    OZK_CUDA(cudaMemsetAsync(is.rowmax, 0, sizeof(int32_t) * (m + n), h->stream));
    if ((st = check_launch(h, 3))) return st;
    K2Launch L{};
    L.a_planes = abar;
    L.b_planes = bbar;
    L.m = m;
    L.n = n;
    L.k = k;
    L.ld = ld;
    L.n_mod = 1;
    L.kind = K2_MAX;
    L.rowmax = is.rowmax;
    L.colmax = is.colmax;
    L.c = &dc;
    L.num_sms = h->num_sms;
    if ((st = launch_k2(L, h->stream))) return st;
    launch_accurate_budget(is.ma, is.nb, is.rowmax, is.colmax, m, n, dc, mu, nu, h->stream);
    return check_launch(h, 2);
}

int run_residues(ozk_context* h, const ozk_constants& c, int64_t m, int64_t n, int64_t k, const Inputs& in,
                 const int32_t* mu, const int32_t* nu, int8_t* pa, int8_t* pb) {
    const DevConsts dc = to_dev(c);
    const int64_t ld = plane_ld(k);
    launch_a_planes(in.a, in.is_f32, m, k, in.lda, mu, dc, 0, pa, ld, h->stream);
    launch_b_planes(in.b, in.is_f32, k, n, in.ldb, nu, dc, 0, pb, ld, h->stream);
    return check_launch(h, 2);
}

int run_products(ozk_context* h, const ozk_constants& c, int64_t m, int64_t n, int64_t k, const int8_t* pa,
                 const int8_t* pb, int kind, void* out, int64_t ldo) {
    const DevConsts dc = to_dev(c);
    K2Launch L{};
    L.a_planes = pa;
    L.b_planes = pb;
    L.m = m;
    L.n = n;
    L.k = k;
    L.ld = plane_ld(k);
    L.n_mod = c.n_moduli;
    L.kind = kind == OZK_PRODUCTS_I32 ? K2_I32 : K2_U8;
    L.out = out;
    L.ldo = ldo;
    L.c = &dc;
    L.num_sms = h->num_sms;
    const int st = launch_k2(L, h->stream);
    if (st) return st;
    return check_launch(h, 1);
}

int finish_check(ozk_context* h, int32_t* flags_dev) {
    OZK_CUDA(cudaMemcpyAsync(h->flags_host, flags_dev, sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    if (h->flags_host[0]) {
        set_error("gemm_emulated: non-finite entry in A or B");
        return OZK_INPUT_ERROR;
    }
    return OZK_OK;
}

int gemm_device(ozk_context* h, const ozk_config* cfg, const ozk_constants& c, int64_t m, int64_t n, int64_t k,
                double alpha, const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C,
                int64_t ldc, bool sync_check) {
    int st;
    if ((st = validate(cfg, c, m, n, k, lda, ldb))) return st;
    if (ldc < m) {
        set_error("gemm_emulated: ldc < m");
        return OZK_INPUT_ERROR;
    }
    OZK_CUDA(cudaSetDevice(h->device));
    if ((st = ensure(h->flags, 64))) return st;
    int32_t* flags_dev = static_cast<int32_t*>(h->flags.p);
    OZK_CUDA(cudaMemsetAsync(flags_dev, 0, 64, h->stream));

    Inputs in;
    if ((st = prepare_inputs(h, cfg, c, m, n, k, A, lda, B, ldb, in))) return st;

    const int64_t ld = plane_ld(k), ldu = u_ld(m);
    const int N = c.n_moduli;
    if ((st = ensure(h->planes_a, static_cast<size_t>(N * m * ld)))) return st;
    if ((st = ensure(h->planes_b, static_cast<size_t>(N * n * ld)))) return st;
    if ((st = ensure(h->u, static_cast<size_t>(N * n * ldu)))) return st;
    if ((st = ensure(h->ints, sizeof(int32_t) * 5 * (m + n)))) return st;
    IntScratch is = carve_ints(h, m, n);

    {
        StageTimer total(h, OZK_PROFILE_TOTAL);
        {
            StageTimer t(h, OZK_PROFILE_SCALE);
            if ((st = run_scale(h, c, cfg->mode, m, n, k, in, is.mu, is.nu, flags_dev))) return st;
        }
        is = carve_ints(h, m, n);  // ints may have been re-allocated
        int8_t* pa = static_cast<int8_t*>(h->planes_a.p);
        int8_t* pb = static_cast<int8_t*>(h->planes_b.p);
        {
            StageTimer t(h, OZK_PROFILE_RESIDUES);
            if ((st = run_residues(h, c, m, n, k, in, is.mu, is.nu, pa, pb))) return st;
        }
        {
            StageTimer t(h, OZK_PROFILE_PRODUCTS);
            if ((st = run_products(h, c, m, n, k, pa, pb, OZK_PRODUCTS_U8, h->u.p, ldu))) return st;
        }
        {
            StageTimer t(h, OZK_PROFILE_RECONSTRUCT);
            launch_reconstruct(static_cast<const uint8_t*>(h->u.p), ldu, m, n, is.mu, is.nu, to_dev(c), alpha, beta, C,
                               ldc, cfg->c_type == OZK_R32F, h->stream);
            if ((st = check_launch(h, 1))) return st;
        }
    }
    return sync_check ? finish_check(h, flags_dev) : OZK_OK;
}

}  // namespace

extern "C" {

const char* ozk_last_error(void) { return g_error.c_str(); }
int ozk_version(void) { return 1; }

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
    *handle = h;
    return OZK_OK;
}

int ozk_destroy(ozk_handle h) {
    if (!h) return OZK_OK;
    cudaSetDevice(h->device);
    for (Buf* b : {&h->planes_a, &h->planes_b, &h->u, &h->stats, &h->ints, &h->flags, &h->f32a, &h->f32b, &h->host_a,
                   &h->host_b, &h->host_c})
        if (b->p) cudaFree(b->p);
    if (h->flags_host) cudaFreeHost(h->flags_host);
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

int64_t ozk_plane_ld(int64_t k) { return plane_ld(k); }

int ozk_gemm(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, double alpha, const void* A,
             int64_t lda, const void* B, int64_t ldb, double beta, void* C, int64_t ldc) {
    if (!h) return OZK_INPUT_ERROR;
    ozk_constants c;
    int st = resolve(cfg, c);
    if (st) return st;
    return gemm_device(h, cfg, c, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, true);
}

int ozk_gemm_host(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, double alpha,
                  const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C, int64_t ldc) {
    if (!h) return OZK_INPUT_ERROR;
    ozk_constants c;
    int st = resolve(cfg, c);
    if (st) return st;
    if ((st = validate(cfg, c, m, n, k, lda, ldb))) return st;
    if (ldc < m) {
        set_error("gemm_emulated: ldc < m");
        return OZK_INPUT_ERROR;
    }
    OZK_CUDA(cudaSetDevice(h->device));
    const size_t es = cfg->a_type == OZK_R32F ? 4 : 8, cs = cfg->c_type == OZK_R32F ? 4 : 8;
    if ((st = ensure(h->host_a, es * lda * k))) return st;
    if ((st = ensure(h->host_b, es * ldb * n))) return st;
    if ((st = ensure(h->host_c, cs * ldc * n))) return st;
    OZK_CUDA(cudaMemcpyAsync(h->host_a.p, A, es * lda * k, cudaMemcpyHostToDevice, h->stream));
    OZK_CUDA(cudaMemcpyAsync(h->host_b.p, B, es * ldb * n, cudaMemcpyHostToDevice, h->stream));
    if (beta != 0.0) OZK_CUDA(cudaMemcpyAsync(h->host_c.p, C, cs * ldc * n, cudaMemcpyHostToDevice, h->stream));
    if ((st = gemm_device(h, cfg, c, m, n, k, alpha, h->host_a.p, lda, h->host_b.p, ldb, beta, h->host_c.p, ldc,
                          true)))
        return st;
    OZK_CUDA(cudaMemcpyAsync(C, h->host_c.p, cs * ldc * n, cudaMemcpyDeviceToHost, h->stream));
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
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

int ozk_stage_scale(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                    const void* B, int64_t ldb, int32_t* mu_exp, int32_t* nu_exp) {
    if (!h) return OZK_INPUT_ERROR;
    ozk_constants c;
    int st = resolve(cfg, c);
    if (st) return st;
    if ((st = validate(cfg, c, m, n, k, lda, ldb))) return st;
    OZK_CUDA(cudaSetDevice(h->device));
    if ((st = ensure(h->flags, 64))) return st;
    int32_t* flags_dev = static_cast<int32_t*>(h->flags.p);
    OZK_CUDA(cudaMemsetAsync(flags_dev, 0, 64, h->stream));
    Inputs in;
    if ((st = prepare_inputs(h, cfg, c, m, n, k, A, lda, B, ldb, in))) return st;
    if ((st = run_scale(h, c, cfg->mode, m, n, k, in, mu_exp, nu_exp, flags_dev))) return st;
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
}

int ozk_stage_residues(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, const void* A,
                       int64_t lda, const void* B, int64_t ldb, const int32_t* mu_exp, const int32_t* nu_exp,
                       int8_t* a_planes, int8_t* b_planes) {
    if (!h) return OZK_INPUT_ERROR;
    ozk_constants c;
    int st = resolve(cfg, c);
    if (st) return st;
    if ((st = validate(cfg, c, m, n, k, lda, ldb))) return st;
    OZK_CUDA(cudaSetDevice(h->device));
    Inputs in;
    if ((st = prepare_inputs(h, cfg, c, m, n, k, A, lda, B, ldb, in))) return st;
    if ((st = run_residues(h, c, m, n, k, in, mu_exp, nu_exp, a_planes, b_planes))) return st;
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
}

int ozk_stage_products(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, const int8_t* a_planes,
                       const int8_t* b_planes, int kind, void* out, int64_t ldo) {
    if (!h) return OZK_INPUT_ERROR;
    ozk_constants c;
    int st = resolve(cfg, c);
    if (st) return st;
    if (m < 1 || n < 1 || k < 1 || ldo < m) {
        set_error("ozk_stage_products: bad dimensions");
        return OZK_INPUT_ERROR;
    }
    if (k > OZK_ENGINE_MAX_K) {
        set_error("int8_gemm: k exceeds 2^17, use blocked_int8_gemm");
        return OZK_INPUT_ERROR;
    }
    OZK_CUDA(cudaSetDevice(h->device));
    if ((st = run_products(h, c, m, n, k, a_planes, b_planes, kind, out, ldo))) return st;
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
}

int ozk_stage_reconstruct(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, const uint8_t* U, int64_t ldu,
                          const int32_t* mu_exp, const int32_t* nu_exp, double alpha, double beta, void* C,
                          int64_t ldc) {
    if (!h) return OZK_INPUT_ERROR;
    ozk_constants c;
    int st = resolve(cfg, c);
    if (st) return st;
    if (m < 1 || n < 1 || ldu < m || ldc < m || (ldu % 4) != 0) {
        set_error("ozk_stage_reconstruct: bad dimensions (ldu must be a multiple of 4)");
        return OZK_INPUT_ERROR;
    }
    OZK_CUDA(cudaSetDevice(h->device));
    launch_reconstruct(U, ldu, m, n, mu_exp, nu_exp, to_dev(c), alpha, beta, C, ldc, cfg->c_type == OZK_R32F,
                       h->stream);
    if ((st = check_launch(h, 1))) return st;
    OZK_CUDA(cudaStreamSynchronize(h->stream));
    return OZK_OK;
}

}  // extern "C"
