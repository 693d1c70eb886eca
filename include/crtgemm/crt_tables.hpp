// Drop-in for crt_tables.hpp:11-79. Same names, fields and semantics; the
// only difference is that P is held in a small fixed-width integer (BigInt)
// instead of GMP's mpz_class, so callers need no GMP.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace crtgemm {

enum class Precision { Fp64, Fp32 };
inline const char* to_string(Precision p) { return p == Precision::Fp64 ? "fp64" : "fp32"; }

inline constexpr int kMinModuli = 2;
inline constexpr int kMaxModuliF64 = 20;
inline constexpr int kMaxModuliF32 = 18;
inline int max_moduli(Precision p) { return p == Precision::Fp64 ? kMaxModuliF64 : kMaxModuliF32; }

struct ModulusSet {
    int n_moduli = 0;
    std::vector<int> moduli;
};

// P = prod p_i < 2^157 as little-endian 32-bit limbs
struct BigInt {
    std::vector<std::uint32_t> limbs;
    int bits() const;
    double to_double() const;  // nearest
};

struct CrtConstants {
    ModulusSet modulus_set;
    Precision precision = Precision::Fp64;
    BigInt big_P;
    std::vector<long> q;
    std::vector<int> beta;
    double P1 = 0.0;
    double P2 = 0.0;
    double P_inv = 0.0;
    float pp_fast = 0.0f;
    float pp_accu = 0.0f;
    std::vector<double> s1;
    std::vector<double> s2;
    std::vector<double> pinv64;
    std::vector<float> pinv32;
    std::vector<std::int32_t> pinv_mulhi;
    int n() const { return modulus_set.n_moduli; }
};

ModulusSet select_moduli(int n_moduli);                                // throws ConfigError
long mod_inverse(long a, long m);                                      // throws std::domain_error
const CrtConstants& build_constants(int n_moduli, Precision precision);  // cached, throws ConfigError
std::string dump_tables_csv(const CrtConstants& c);

}  // namespace crtgemm
