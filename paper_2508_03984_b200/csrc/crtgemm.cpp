// The reference's C++ API (include/crtgemm/*.hpp) on top of the C ABI.
//
// gemm_emulated keeps the reference signatures (emulator.hpp:20-35) and value
// semantics: host Matrix<T> in, EmulationResult out. Every call goes to the
// B200 through ozk_gemm_host (H2D, K1 -> K2 -> K3, D2H); status codes become
// the reference exceptions. A process-wide context (device OZK_DEVICE, default
// 0) is shared under a mutex, which keeps the API reentrant like the
// reference (crt_tables.cpp:190-196 is its only shared state).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>

#include "crtgemm/emulator.hpp"
#include "crtgemm/errors.hpp"
#include "crtgemm/residue.hpp"
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
    ozk_config c = ozk_default_config(consts.n(), mode_code(cfg.mode), prec_code(consts.precision));
    c.a_type = sizeof(T) == 4 ? OZK_R32F : OZK_R64F;
    c.c_type = OZK_R64F;
    c.block_k = cfg.block_k;
    c.constants = &oc;
    EmulationResult r;
    r.n_moduli = consts.n();
    r.mode = cfg.mode;
    r.precision = consts.precision;
    r.c = Matrix<double>(a.rows, b.cols);
    std::lock_guard<std::mutex> lock(g_mtx);
    check(ozk_gemm_host(handle_locked(), &c, a.rows, b.cols, a.cols, 1.0, a.data.data(), a.rows, b.data.data(),
                        b.rows, 0.0, r.c.data.data(), a.rows));
    return r;
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

Matrix<float> to_fp32(const Matrix<double>& m) {
    Matrix<float> out(m.rows, m.cols);
    for (std::size_t e = 0; e < m.data.size(); ++e) out.data[e] = static_cast<float>(m.data[e]);
    return out;
}

}  // namespace crtgemm
