// The reference's C++ API (include/crtgemm/*.hpp) on top of the C ABI.
//
// gemm_emulated keeps the reference signatures (emulator.hpp:20-35) and value
// semantics: host Matrix<T> in, EmulationResult out. Every call goes to the
// B200 through ozk_gemm_host (H2D, K1 -> K2 -> K3, D2H); status codes become
// the reference exceptions. A process-wide context (device OZK_DEVICE, default
// 0) is shared under a mutex, which keeps the API reentrant like the
// reference (crt_tables.cpp:190-196 is its only shared state).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <sys/mman.h>

#include <cuda_runtime.h>

#include "crtgemm/emulator.hpp"
#include "crtgemm/errors.hpp"
#include "crtgemm/int8_engine.hpp"
#include "crtgemm/reconstruct.hpp"
#include "crtgemm/residue.hpp"
#include "crtgemm/scaling.hpp"
#include "ozaki2_b200.h"

namespace crtgemm {
namespace {

[[noreturn]] void raise(int status) {
    const std::string msg = ozk_last_error();
    switch (status) {
        case OZK_CONFIG_ERROR:
            throw ConfigError(msg);
        case OZK_INPUT_ERROR:
            throw InputError(msg);
        case OZK_DOMAIN_ERROR:
            throw std::domain_error(msg);
        default:
            throw std::runtime_error("ozaki2_b200: " + msg);
    }
}

void check(int status) {
    if (status != OZK_OK) raise(status);
}

std::mutex g_mtx;
ozk_handle g_handle = nullptr;

ozk_handle handle_locked() {
    if (!g_handle) {
        const char* env = std::getenv("OZK_DEVICE");
        check(ozk_create(&g_handle, env ? std::atoi(env) : 0));
    }
    return g_handle;
}

// The result matrix of a large call: Matrix<double>(m, n) value-initialises
// fresh pages, and at 16384^2 (2 GB) the first-touch page faults of that
// memset cost ~0.8 s on one thread — far more than the emulated GEMM. The
// storage is reserved first, the kernel asked for transparent huge pages,
// the pages are populated by several threads at once (MADV_POPULATE_WRITE,
// Linux >= 5.14; silently skipped where unsupported), and only then is the
// vector resized (value-initialised) over memory that is already mapped.
// Same type, same contents (zeros) as the reference's Matrix ctor.
Matrix<double> result_matrix(std::int64_t rows, std::int64_t cols) {
    constexpr std::size_t kBig = std::size_t(64) << 20;
    const std::size_t n = static_cast<std::size_t>(rows * cols), bytes = n * sizeof(double);
    if (bytes < kBig) return Matrix<double>(rows, cols);
    Matrix<double> c;
    c.data.reserve(n);
    const std::size_t page = 4096;
    const std::uintptr_t lo = (reinterpret_cast<std::uintptr_t>(c.data.data()) + page - 1) / page * page;
    const std::uintptr_t hi = (reinterpret_cast<std::uintptr_t>(c.data.data()) + bytes) / page * page;
    if (hi > lo) {
#ifdef MADV_HUGEPAGE
        madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
#endif
#ifndef MADV_POPULATE_WRITE
#define MADV_POPULATE_WRITE 23
#endif
        const unsigned hw = std::thread::hardware_concurrency();
        const std::size_t nt = std::min<std::size_t>(hw ? hw : 4, 16);
        const std::size_t chunk = ((hi - lo) / nt + (std::size_t(2) << 20) - 1) / (std::size_t(2) << 20) * (std::size_t(2) << 20);
        std::vector<std::thread> ts;
        for (std::uintptr_t p = lo; p < hi; p += chunk) {
            const std::size_t len = std::min<std::size_t>(chunk, hi - p);
            ts.emplace_back([p, len] { madvise(reinterpret_cast<void*>(p), len, MADV_POPULATE_WRITE); });
        }
        for (auto& t : ts) t.join();
    }
    c.data.resize(n);
    c.rows = rows;
    c.cols = cols;
    return c;
}

int prec_code(Precision p) { return p == Precision::Fp64 ? OZK_FP64 : OZK_FP32; }
int mode_code(ScaleMode m) { return m == ScaleMode::Fast ? OZK_FAST : OZK_ACCURATE; }

ozk_constants to_c(const CrtConstants& c) {
    ozk_constants o{};
    o.n_moduli = c.n();
    o.precision = prec_code(c.precision);
    for (int i = 0; i < c.n() && i < OZK_MAX_MODULI; ++i) {
        const auto ii = static_cast<std::size_t>(i);
        o.moduli[i] = c.modulus_set.moduli[ii];
        o.q[i] = c.q[ii];
        o.beta[i] = c.beta[ii];
        o.s1[i] = c.s1[ii];
        o.s2[i] = c.s2[ii];
        o.pinv64[i] = c.pinv64[ii];
        o.pinv32[i] = c.pinv32[ii];
        o.pinv_mulhi[i] = c.pinv_mulhi[ii];
    }
    o.P1 = c.P1;
    o.P2 = c.P2;
    o.P_inv = c.P_inv;
    o.pp_fast = c.pp_fast;
    o.pp_accu = c.pp_accu;
    for (std::size_t i = 0; i < c.big_P.limbs.size() && i < 6; ++i) o.P_limbs[i] = c.big_P.limbs[i];
    o.P_bits = c.big_P.bits();
    return o;
}

CrtConstants from_c(const ozk_constants& o) {
    CrtConstants c;
    c.modulus_set.n_moduli = o.n_moduli;
    c.precision = o.precision == OZK_FP64 ? Precision::Fp64 : Precision::Fp32;
    for (int i = 0; i < o.n_moduli; ++i) {
        c.modulus_set.moduli.push_back(o.moduli[i]);
        c.q.push_back(static_cast<long>(o.q[i]));
        c.beta.push_back(o.beta[i]);
        c.s1.push_back(o.s1[i]);
        c.s2.push_back(o.s2[i]);
        c.pinv64.push_back(o.pinv64[i]);
        c.pinv32.push_back(o.pinv32[i]);
        c.pinv_mulhi.push_back(o.pinv_mulhi[i]);
    }
    c.P1 = o.P1;
    c.P2 = o.P2;
    c.P_inv = o.P_inv;
    c.pp_fast = o.pp_fast;
    c.pp_accu = o.pp_accu;
    c.big_P.limbs.assign(o.P_limbs, o.P_limbs + 6);
    return c;
}

// validate_inputs order of emulator.cpp:12-23 for the host-visible checks
template <typename T>
void validate_host(const Matrix<T>& a, const Matrix<T>& b, const EmuConfig& cfg) {
    if (a.cols != b.rows) throw InputError("gemm_emulated: inner dimensions disagree");
    if (a.rows < 1 || a.cols < 1 || b.cols < 1) throw InputError("gemm_emulated: empty dimension");
    if (cfg.block_k < 1 || cfg.block_k > kEngineMaxK) throw ConfigError("gemm_emulated: block_k must be in [1, 2^17]");
    if (cfg.threads < 1) throw ConfigError("gemm_emulated: threads must be >= 1");
}

template <typename T>
EmulationResult run(const Matrix<T>& a, const Matrix<T>& b, const EmuConfig& cfg, const CrtConstants& consts) {
    validate_host(a, b, cfg);
    ozk_constants oc = to_c(consts);
    // cfg.precision decides the FP32 rounding and the FP32-input check
    // (emulator.cpp:84-99); the table supplies the arithmetic
    ozk_config c = ozk_default_config(consts.n(), mode_code(cfg.mode), prec_code(cfg.precision));
    c.a_type = sizeof(T) == 4 ? OZK_R32F : OZK_R64F;
    c.c_type = OZK_R64F;
    c.block_k = cfg.block_k;
    c.constants = &oc;
    EmulationResult r;
    r.n_moduli = consts.n();
    r.mode = cfg.mode;
    r.precision = consts.precision;
    r.c = result_matrix(a.rows, b.cols);
    std::lock_guard<std::mutex> lock(g_mtx);
    check(ozk_gemm_host(handle_locked(), &c, a.rows, b.cols, a.cols, 1.0, a.data.data(), a.rows, b.data.data(),
                        b.rows, 0.0, r.c.data.data(), a.rows));
    return r;
}

// device scratch for the stage helpers (RAII)
struct Dev {
    void* p = nullptr;
    explicit Dev(size_t bytes) {
        if (bytes && cudaMalloc(&p, bytes) != cudaSuccess) throw std::runtime_error("ozaki2_b200: cudaMalloc failed");
    }
    ~Dev() {
        if (p) cudaFree(p);
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

void up(void* dst, const void* src, size_t bytes) {
    if (bytes && cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("ozaki2_b200: H2D copy failed");
}
void down(void* dst, const void* src, size_t bytes) {
    if (bytes && cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
        throw std::runtime_error("ozaki2_b200: D2H copy failed");
}

std::vector<std::int32_t> exps_of(const std::vector<double>& scale) {
    std::vector<std::int32_t> e(scale.size());
    for (std::size_t i = 0; i < scale.size(); ++i) e[i] = std::ilogb(scale[i]);
    return e;
}

template <typename T>
ScalePair scale_impl(const Matrix<T>& a, const Matrix<T>& b, const CrtConstants& c, ScaleMode mode) {
    ozk_constants oc = to_c(c);
    ozk_config cfg = ozk_default_config(c.n(), mode_code(mode), prec_code(c.precision));
    cfg.a_type = sizeof(T) == 4 ? OZK_R32F : OZK_R64F;
    cfg.constants = &oc;
    const std::int64_t m = a.rows, k = a.cols, n = b.cols;
    Dev da(sizeof(T) * a.data.size()), db(sizeof(T) * b.data.size()), dmu(4 * m + 4), dnu(4 * n + 4);
    up(da.p, a.data.data(), sizeof(T) * a.data.size());
    up(db.p, b.data.data(), sizeof(T) * b.data.size());
    std::lock_guard<std::mutex> lock(g_mtx);
    check(ozk_stage_scale(handle_locked(), &cfg, m, n, k, da.p, m, db.p, k, dmu.as<std::int32_t>(),
                          dnu.as<std::int32_t>()));
    std::vector<std::int32_t> mu(m), nu(n);
    down(mu.data(), dmu.p, 4 * m);
    down(nu.data(), dnu.p, 4 * n);
    ScalePair s;
    s.mode = mode;
    for (auto e : mu) s.mu.push_back(std::ldexp(1.0, e));
    for (auto e : nu) s.nu.push_back(std::ldexp(1.0, e));
    return s;
}

template <typename T>
Matrix<T> truncate_impl(const Matrix<T>& m, const std::vector<double>& scale, Side side) {
    const auto e = exps_of(scale);
    Matrix<T> out(m.rows, m.cols);
    Dev dx(sizeof(T) * m.data.size()), dout(sizeof(T) * m.data.size()), de(4 * e.size() + 4);
    up(dx.p, m.data.data(), sizeof(T) * m.data.size());
    up(de.p, e.data(), 4 * e.size());
    std::lock_guard<std::mutex> lock(g_mtx);
    check(ozk_truncate_scale(handle_locked(), sizeof(T) == 4 ? OZK_R32F : OZK_R64F, m.rows, m.cols, dx.p, m.rows,
                             de.as<std::int32_t>(), side == Side::Row ? 0 : 1, dout.p, m.rows));
    down(out.data.data(), dout.p, sizeof(T) * m.data.size());
    return out;
}

template <typename T>
ResidueSlices residues_impl(const Matrix<T>& m, const CrtConstants& c) {
    ozk_constants oc = to_c(c);
    ozk_config cfg = ozk_default_config(c.n(), OZK_FAST, prec_code(c.precision));
    cfg.a_type = sizeof(T) == 4 ? OZK_R32F : OZK_R64F;
    cfg.constants = &oc;
    const std::int64_t cnt = m.size();
    Dev dx(sizeof(T) * cnt + 8), dp(static_cast<size_t>(c.n() * cnt) + 8);
    up(dx.p, m.data.data(), sizeof(T) * cnt);
    {
        std::lock_guard<std::mutex> lock(g_mtx);
        check(ozk_residues(handle_locked(), &cfg, m.rows, m.cols, dx.p, m.rows, dp.as<std::int8_t>(), m.rows));
    }
    ResidueSlices rs;
    rs.n_moduli = c.n();
    rs.rows = m.rows;
    rs.cols = m.cols;
    for (int i = 0; i < c.n(); ++i) {
        Matrix<std::int8_t> sl(m.rows, m.cols);
        down(sl.data.data(), dp.as<std::int8_t>() + i * cnt, static_cast<size_t>(cnt));
        rs.slices.push_back(std::move(sl));
    }
    return rs;
}

}  // namespace

// ---- BigInt -------------------------------------------------------------------
int BigInt::bits() const {
    for (std::size_t i = limbs.size(); i-- > 0;)
        if (limbs[i]) return static_cast<int>(32 * i) + 32 - __builtin_clz(limbs[i]);
    return 0;
}

double BigInt::to_double() const {
    // nearest double, ties to even, from the top 64 bits plus a sticky bit
    const int nb = bits();
    if (nb == 0) return 0.0;
    auto bit = [&](int b) { return (limbs[static_cast<std::size_t>(b / 32)] >> (b % 32)) & 1u; };
    std::uint64_t head = 0;
    const int lo = nb > 64 ? nb - 64 : 0;
    for (int b = nb - 1; b >= lo; --b) head = (head << 1) | bit(b);
    bool sticky = false;
    for (int b = 0; b < lo && !sticky; ++b) sticky = bit(b);
    const int hb = nb - lo;  // bits in head
    if (hb <= 53) return std::ldexp(static_cast<double>(head), lo);
    const int drop = hb - 53;
    const std::uint64_t rest = head & ((std::uint64_t(1) << drop) - 1);
    std::uint64_t top = head >> drop;
    const std::uint64_t half = std::uint64_t(1) << (drop - 1);
    if (rest > half || (rest == half && (sticky || (top & 1u)))) ++top;
    else if (rest == half && !sticky && !(top & 1u)) {}
    return std::ldexp(static_cast<double>(top), lo + drop);
}

// ---- crt_tables ------------------------------------------------------------------
ModulusSet select_moduli(int n_moduli) {
    ModulusSet s;
    std::int32_t buf[OZK_MAX_MODULI];
    check(ozk_select_moduli(n_moduli, buf));
    s.n_moduli = n_moduli;
    s.moduli.assign(buf, buf + n_moduli);
    return s;
}

long mod_inverse(long a, long m) {
    int st = 0;
    const auto r = ozk_mod_inverse(a, m, &st);
    check(st);
    return static_cast<long>(r);
}

const CrtConstants& build_constants(int n_moduli, Precision precision) {
    static std::mutex mtx;
    static std::map<std::pair<int, int>, std::unique_ptr<CrtConstants>> cache;
    ozk_constants o;
    check(ozk_build_constants(n_moduli, prec_code(precision), &o));
    std::lock_guard<std::mutex> lock(mtx);
    auto& slot = cache[{n_moduli, prec_code(precision)}];
    if (!slot) slot = std::make_unique<CrtConstants>(from_c(o));
    return *slot;
}

std::string dump_tables_csv(const CrtConstants& c) {
    const ozk_constants o = to_c(c);
    std::string buf(static_cast<std::size_t>(64 + 160 * c.n()), '\0');
    check(ozk_dump_tables_csv(&o, buf.data(), static_cast<std::int64_t>(buf.size())));
    buf.resize(std::strlen(buf.c_str()));
    return buf;
}

// ---- emulator ------------------------------------------------------------------
EmulationResult gemm_emulated(const Matrix<double>& a, const Matrix<double>& b, const EmuConfig& cfg,
                              const CrtConstants& consts) {
    return run(a, b, cfg, consts);
}

EmulationResult gemm_emulated(const Matrix<float>& a, const Matrix<float>& b, const EmuConfig& cfg,
                              const CrtConstants& consts) {
    if (cfg.precision != Precision::Fp32) throw ConfigError("gemm_emulated: FP32 inputs require cfg.precision == Fp32");
    return run(a, b, cfg, consts);
}

EmulationResult gemm_emulated(const Matrix<double>& a, const Matrix<double>& b, const EmuConfig& cfg) {
    return gemm_emulated(a, b, cfg, build_constants(cfg.n_moduli, cfg.precision));
}

EmulationResult gemm_emulated(const Matrix<float>& a, const Matrix<float>& b, const EmuConfig& cfg) {
    return gemm_emulated(a, b, cfg, build_constants(cfg.n_moduli, cfg.precision));
}

// ---- stage functions (the reference's public stage API, on the GPU) ------------
ScalePair scale_fast(const Matrix<double>& a, const Matrix<double>& b, const CrtConstants& c) {
    return scale_impl(a, b, c, ScaleMode::Fast);
}
ScalePair scale_fast(const Matrix<float>& a, const Matrix<float>& b, const CrtConstants& c) {
    return scale_impl(a, b, c, ScaleMode::Fast);
}
ScalePair scale_accurate(const Matrix<double>& a, const Matrix<double>& b, const CrtConstants& c,
                         std::int64_t block_k, int /*n_threads*/) {
    if (block_k < 1) throw InputError("blocked_int8_gemm: invalid block_k");  // int8_engine.cpp:86
    return scale_impl(a, b, c, ScaleMode::Accurate);
}
ScalePair scale_accurate(const Matrix<float>& a, const Matrix<float>& b, const CrtConstants& c,
                         std::int64_t block_k, int /*n_threads*/) {
    if (block_k < 1) throw InputError("blocked_int8_gemm: invalid block_k");
    return scale_impl(a, b, c, ScaleMode::Accurate);
}

Matrix<double> truncate_scale(const Matrix<double>& m, const std::vector<double>& scale, Side side) {
    return truncate_impl(m, scale, side);
}
Matrix<float> truncate_scale(const Matrix<float>& m, const std::vector<double>& scale, Side side) {
    return truncate_impl(m, scale, side);
}
ResidueSlices to_residue_slices(const Matrix<double>& m, const CrtConstants& c) { return residues_impl(m, c); }
ResidueSlices to_residue_slices(const Matrix<float>& m, const CrtConstants& c) { return residues_impl(m, c); }

Int32ProductMatrix int8_gemm(const Matrix<std::int8_t>& a, const Matrix<std::int8_t>& b, int /*n_threads*/) {
    if (a.cols != b.rows) throw InputError("int8_gemm: inner dimensions disagree");
    if (a.cols > kEngineMaxK) throw InputError("int8_gemm: k exceeds 2^17, use blocked_int8_gemm");
    const std::int64_t m = a.rows, k = a.cols, n = b.cols;
    const std::int64_t lda = (m + 15) / 16 * 16, ldb = (k + 15) / 16 * 16;
    Int32ProductMatrix out;
    out.k_used = k;
    out.data = Matrix<std::int32_t>(m, n);
    Dev da(static_cast<size_t>(lda * k) + 16), db(static_cast<size_t>(ldb * n) + 16), dc(4 * m * n + 16);
    if (k && m && cudaMemcpy2D(da.p, lda, a.data.data(), m, m, k, cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("ozaki2_b200: H2D copy failed");
    if (k && n && cudaMemcpy2D(db.p, ldb, b.data.data(), k, k, n, cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("ozaki2_b200: H2D copy failed");
    {
        std::lock_guard<std::mutex> lock(g_mtx);
        check(ozk_int8_gemm(handle_locked(), m, n, k, da.as<std::int8_t>(), lda, db.as<std::int8_t>(), ldb,
                            dc.as<std::int32_t>(), m));
    }
    down(out.data.data.data(), dc.p, 4 * static_cast<size_t>(m * n));
    return out;
}

// The reference keeps a triple loop here as an in-tree cross-check of its
// tiled kernel (int8_engine.cpp:66-80); here it is a plain CUDA-core kernel
// (ozk_int8_gemm_reference), independent of the tensor-core engine, so the
// cross-check still compares two implementations.
Int32ProductMatrix int8_gemm_reference(const Matrix<std::int8_t>& a, const Matrix<std::int8_t>& b) {
    if (a.cols != b.rows) throw InputError("int8_gemm_reference: inner dimensions disagree");
    if (a.cols > kEngineMaxK) throw InputError("int8_gemm_reference: k exceeds 2^17");
    const std::int64_t m = a.rows, k = a.cols, n = b.cols;
    Int32ProductMatrix out;
    out.k_used = k;
    out.data = Matrix<std::int32_t>(m, n);
    Dev da(static_cast<size_t>(m * k) + 16), db(static_cast<size_t>(k * n) + 16), dc(4 * m * n + 16);
    up(da.p, a.data.data(), static_cast<size_t>(m * k));
    up(db.p, b.data.data(), static_cast<size_t>(k * n));
    {
        std::lock_guard<std::mutex> lock(g_mtx);
        check(ozk_int8_gemm_reference(handle_locked(), m, n, k, da.as<std::int8_t>(), m > 0 ? m : 1,
                                      db.as<std::int8_t>(), k > 0 ? k : 1, dc.as<std::int32_t>(), m > 0 ? m : 1));
    }
    down(out.data.data.data(), dc.p, 4 * static_cast<size_t>(m * n));
    return out;
}

std::vector<Int32ProductMatrix> blocked_int8_gemm(const Matrix<std::int8_t>& a, const Matrix<std::int8_t>& b,
                                                  std::int64_t block_k, int n_threads) {
    if (a.cols != b.rows) throw InputError("blocked_int8_gemm: inner dimensions disagree");
    if (block_k < 1 || block_k > kEngineMaxK) throw InputError("blocked_int8_gemm: invalid block_k");
    std::vector<Int32ProductMatrix> out;
    for (std::int64_t h0 = 0; h0 < a.cols; h0 += block_k) {
        const std::int64_t len = std::min(block_k, a.cols - h0);
        out.push_back(int8_gemm(column_block(a, h0, len), row_block(b, h0, len), n_threads));
    }
    if (out.empty()) {
        Int32ProductMatrix zero;
        zero.data = Matrix<std::int32_t>(a.rows, b.cols);
        out.push_back(std::move(zero));
    }
    return out;
}

ResidueProducts reduce_products_u8(const std::vector<Int32ProductMatrix>& prods, const CrtConstants& c) {
    if (static_cast<int>(prods.size()) != c.n())
        throw InputError("reduce_products_u8: product count does not match modulus count");
    ResidueProducts out;
    for (int i = 0; i < c.n(); ++i) {
        const auto& src = prods[static_cast<std::size_t>(i)].data;
        const std::int64_t cnt = src.size();
        Dev dx(4 * static_cast<size_t>(cnt) + 4), du(static_cast<size_t>(cnt) + 4);
        up(dx.p, src.data.data(), 4 * static_cast<size_t>(cnt));
        {
            std::lock_guard<std::mutex> lock(g_mtx);
            check(ozk_mod_u8_array(handle_locked(), cnt, dx.as<std::int32_t>(),
                                   c.modulus_set.moduli[static_cast<std::size_t>(i)],
                                   c.pinv_mulhi[static_cast<std::size_t>(i)], du.as<std::uint8_t>()));
        }
        Matrix<std::uint8_t> u(src.rows, src.cols);
        down(u.data.data(), du.p, static_cast<size_t>(cnt));
        out.u.push_back(std::move(u));
    }
    return out;
}

std::pair<Matrix<double>, Matrix<double>> accumulate(const ResidueProducts& u, const CrtConstants& c) {
    if (static_cast<int>(u.u.size()) != c.n()) throw InputError("accumulate: residue count does not match modulus count");
    const std::int64_t rows = u.u.front().rows, cols = u.u.front().cols, cnt = rows * cols;
    ozk_constants oc = to_c(c);
    ozk_config cfg = ozk_default_config(c.n(), OZK_FAST, prec_code(c.precision));
    cfg.constants = &oc;
    Dev du(static_cast<size_t>(c.n() * cnt) + 4), d1(8 * static_cast<size_t>(cnt) + 8), d2(8 * static_cast<size_t>(cnt) + 8);
    for (int i = 0; i < c.n(); ++i) up(du.as<std::uint8_t>() + i * cnt, u.u[static_cast<std::size_t>(i)].data.data(), cnt);
    {
        std::lock_guard<std::mutex> lock(g_mtx);
        check(ozk_accumulate(handle_locked(), &cfg, cnt, du.as<std::uint8_t>(), d1.as<double>(), d2.as<double>()));
    }
    Matrix<double> c1(rows, cols), c2(rows, cols);
    down(c1.data.data(), d1.p, 8 * static_cast<size_t>(cnt));
    down(c2.data.data(), d2.p, 8 * static_cast<size_t>(cnt));
    return {std::move(c1), std::move(c2)};
}

Matrix<double> crt_reduce(const Matrix<double>& c1, const Matrix<double>& c2, const CrtConstants& c) {
    if (c1.rows != c2.rows || c1.cols != c2.cols) throw InputError("crt_reduce: shape mismatch");
    const std::int64_t cnt = c1.size();
    ozk_constants oc = to_c(c);
    ozk_config cfg = ozk_default_config(c.n(), OZK_FAST, prec_code(c.precision));
    cfg.constants = &oc;
    Dev d1(8 * static_cast<size_t>(cnt) + 8), d2(8 * static_cast<size_t>(cnt) + 8), dout(8 * static_cast<size_t>(cnt) + 8);
    up(d1.p, c1.data.data(), 8 * static_cast<size_t>(cnt));
    up(d2.p, c2.data.data(), 8 * static_cast<size_t>(cnt));
    {
        std::lock_guard<std::mutex> lock(g_mtx);
        check(ozk_crt_reduce(handle_locked(), &cfg, cnt, d1.as<double>(), d2.as<double>(), dout.as<double>()));
    }
    Matrix<double> out(c1.rows, c1.cols);
    down(out.data.data(), dout.p, 8 * static_cast<size_t>(cnt));
    return out;
}

EmulationResult unscale(const Matrix<double>& cpp, const ScalePair& scales, const CrtConstants& c) {
    const std::int64_t m = cpp.rows, n = cpp.cols;
    if (static_cast<std::int64_t>(scales.mu.size()) != m || static_cast<std::int64_t>(scales.nu.size()) != n)
        throw InputError("unscale: scale vector length mismatch");
    const auto mu = exps_of(scales.mu), nu = exps_of(scales.nu);
    Dev dc(8 * static_cast<size_t>(m * n) + 8), dout(8 * static_cast<size_t>(m * n) + 8), dmu(4 * m + 4), dnu(4 * n + 4);
    up(dc.p, cpp.data.data(), 8 * static_cast<size_t>(m * n));
    up(dmu.p, mu.data(), 4 * m);
    up(dnu.p, nu.data(), 4 * n);
    {
        std::lock_guard<std::mutex> lock(g_mtx);
        check(ozk_unscale(handle_locked(), m, n, dc.as<double>(), m, dmu.as<std::int32_t>(), dnu.as<std::int32_t>(),
                          dout.as<double>(), m));
    }
    EmulationResult r;
    r.n_moduli = c.n();
    r.mode = scales.mode;
    r.precision = c.precision;
    r.c = Matrix<double>(m, n);
    down(r.c.data.data(), dout.p, 8 * static_cast<size_t>(m * n));
    return r;
}

Matrix<float> to_fp32(const Matrix<double>& m) {
    Matrix<float> out(m.rows, m.cols);
    for (std::size_t e = 0; e < m.data.size(); ++e) out.data[e] = static_cast<float>(m.data[e]);
    return out;
}

}  // namespace crtgemm
