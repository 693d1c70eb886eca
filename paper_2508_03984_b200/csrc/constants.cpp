// Host-side CRT constant tables (reference: crt_tables.cpp:15-209).
//
// The reference builds these with GMP. Every quantity here fits in 192 bits
// (P < 2^157, W_i = (P/p_i) q_i < 2^165 for N <= 20), so a fixed three-limb
// integer with exact arithmetic reproduces the tables bit-for-bit without the
// GMP dependency. Tables are immutable and cached per (N, precision) under a
// mutex like build_constants (crt_tables.cpp:186-197).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "ozaki2_b200.h"
#include "ozk_internal.h"

namespace ozk {
namespace {

using u64 = std::uint64_t;
using u128 = unsigned __int128;

// Unsigned 192-bit integer, little-endian 64-bit limbs.
struct U192 {
    u64 w[3] = {0, 0, 0};

    static U192 from(u64 v) {
        U192 r;
        r.w[0] = v;
        return r;
    }
    bool zero() const { return !(w[0] | w[1] | w[2]); }
    int bits() const {
        for (int i = 2; i >= 0; --i)
            if (w[i]) return 64 * i + 64 - __builtin_clzll(w[i]);
        return 0;
    }
    bool bit(int b) const { return b >= 0 && b < 192 && ((w[b >> 6] >> (b & 63)) & 1u); }
    bool any_below(int b) const {  // any of bits [0, b)
        for (int i = 0; i < 3 && b > 0; ++i, b -= 64) {
            const u64 mask = b >= 64 ? ~u64(0) : ((u64(1) << b) - 1);
            if (w[i] & mask) return true;
        }
        return false;
    }
    U192 shr(int s) const {
        U192 r;
        if (s >= 192) return r;
        const int q = s >> 6, b = s & 63;
        for (int i = 0; i + q < 3; ++i) {
            u64 v = w[i + q] >> b;
            if (b && i + q + 1 < 3) v |= w[i + q + 1] << (64 - b);
            r.w[i] = v;
        }
        return r;
    }
    U192 shl(int s) const {
        U192 r;
        if (s >= 192) return r;
        const int q = s >> 6, b = s & 63;
        for (int i = 2; i >= q; --i) {
            u64 v = w[i - q] << b;
            if (b && i - q - 1 >= 0) v |= w[i - q - 1] >> (64 - b);
            r.w[i] = v;
        }
        return r;
    }
    void mul_small(u64 s) {
        u128 carry = 0;
        for (auto& x : w) {
            const u128 t = static_cast<u128>(x) * s + carry;
            x = static_cast<u64>(t);
            carry = t >> 64;
        }
    }
    u64 div_small(u64 d) {
        u128 rem = 0;
        for (int i = 2; i >= 0; --i) {
            const u128 cur = (rem << 64) | w[i];
            w[i] = static_cast<u64>(cur / d);
            rem = cur % d;
        }
        return static_cast<u64>(rem);
    }
    void add_small(u64 s) {
        for (auto& x : w) {
            const u64 old = x;
            x += s;
            if (x >= old) return;
            s = 1;
        }
    }
    friend int cmp(const U192& a, const U192& b) {
        for (int i = 2; i >= 0; --i)
            if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
        return 0;
    }
    friend U192 sub(const U192& a, const U192& b) {  // a >= b
        U192 r;
        u64 borrow = 0;
        for (int i = 0; i < 3; ++i) {
            const u64 t = a.w[i] - b.w[i];
            const u64 t2 = t - borrow;
            borrow = (a.w[i] < b.w[i]) || (t < borrow);
            r.w[i] = t2;
        }
        return r;
    }
    double exact_small() const { return static_cast<double>(w[0]); }  // callers keep <= 54 bits
};

// nearest double, ties to even (to_double_nearest, crt_tables.cpp:50-67)
double nearest(const U192& z, bool negative = false) {
    if (z.zero()) return 0.0;
    const int nb = z.bits();
    double mag;
    if (nb <= 53) {
        mag = z.exact_small();
    } else {
        const int drop = nb - 53;
        U192 head = z.shr(drop);
        if (z.bit(drop - 1) && (z.any_below(drop - 1) || (head.w[0] & 1u))) head.add_small(1);
        mag = std::ldexp(head.exact_small(), drop);
    }
    return negative ? -mag : mag;
}

// nearest double of 1/P (ratio_to_double_nearest(1, P), crt_tables.cpp:69-95):
// the quotient 2^s / P with s = 54 + bits(P) carries 54..56 bits, then the
// same half-to-even rounding with the division remainder as sticky.
double reciprocal_nearest(const U192& P) {
    const int s = 54 + P.bits();
    // long division of 2^s by P; P < 2^157 so rem < 2^158 never overflows 192 bits
    U192 rem, quot;
    for (int b = s; b >= 0; --b) {
        rem = rem.shl(1);
        if (b == s) rem.add_small(1);
        quot = quot.shl(1);
        if (cmp(rem, P) >= 0) {
            rem = sub(rem, P);
            quot.add_small(1);
        }
    }
    const int drop = quot.bits() - 53;
    bool sticky = !rem.zero();
    if (drop > 0) {
        const bool round = quot.bit(drop - 1);
        sticky = sticky || quot.any_below(drop - 1);
        quot = quot.shr(drop);
        if (round && (sticky || (quot.w[0] & 1u))) quot.add_small(1);
    }
    return std::ldexp(quot.exact_small(), (drop > 0 ? drop : 0) - s);
}

// log2_mpz (crt_tables.cpp:97-105): the top 64 bits converted the way
// mpz_get_d does it (truncation to 53 bits), then libm log2 + shift.
double log2_big(const U192& z) {
    const int nb = z.bits();
    const int shift = nb > 64 ? nb - 64 : 0;
    u64 head = z.shr(shift).w[0];
    const int hb = nb - shift;
    if (hb > 53) head &= ~((u64(1) << (hb - 53)) - 1);
    return std::log2(static_cast<double>(head)) + static_cast<double>(shift);
}

int gcd_i(int a, int b) {
    while (b) {
        const int t = a % b;
        a = b;
        b = t;
    }
    return a;
}

int make_table(int n, int precision, ozk_constants* c) {
    std::memset(c, 0, sizeof *c);
    c->n_moduli = n;
    c->precision = precision;
    ozk_select_moduli(n, c->moduli);
    const int32_t* p = c->moduli;

    U192 P = U192::from(1);
    for (int i = 0; i < n; ++i) P.mul_small(static_cast<u64>(p[i]));
    c->P_bits = P.bits();
    for (int i = 0; i < 6; ++i) c->P_limbs[i] = static_cast<uint32_t>(P.w[i / 2] >> (32 * (i % 2)));

    // q_i = ((P/p_i) mod p_i)^-1 mod p_i  (crt_tables.cpp:124-131)
    for (int i = 0; i < n; ++i) {
        int64_t r = 1;
        for (int j = 0; j < n; ++j)
            if (j != i) r = (r * (p[j] % p[i])) % p[i];
        int st = 0;
        c->q[i] = ozk_mod_inverse(r, p[i], &st);
    }

    // P1 = nearest(P), P2 = nearest(P - P1) for fp64 (crt_tables.cpp:133-136)
    c->P1 = nearest(P);
    if (precision == OZK_FP64) {
        int ex = 0;
        const double fr = std::frexp(c->P1, &ex);
        U192 p1 = U192::from(static_cast<u64>(std::ldexp(fr, 53)));
        p1 = ex >= 53 ? p1.shl(ex - 53) : p1.shr(53 - ex);
        c->P2 = cmp(P, p1) >= 0 ? nearest(sub(P, p1)) : nearest(sub(p1, P), true);
    }
    c->P_inv = reciprocal_nearest(P);

    // per-side scale budgets (crt_tables.cpp:138-140)
    const double half_log = 0.5 * log2_big(sub(P, U192::from(1)));
    c->pp_fast = static_cast<float>(half_log - 1.5);
    c->pp_accu = static_cast<float>(half_log - 0.5);

    // W_i = (P/p_i) q_i with the common-grid head/tail split (crt_tables.cpp:142-171)
    U192 w[OZK_MAX_MODULI];
    int wbits[OZK_MAX_MODULI];
    int wmax = 0;
    for (int i = 0; i < n; ++i) {
        w[i] = P;
        w[i].div_small(static_cast<u64>(p[i]));
        w[i].mul_small(static_cast<u64>(c->q[i]));
        wbits[i] = w[i].bits();
        wmax = wbits[i] > wmax ? wbits[i] : wmax;
    }
    int cl2n = 0;
    while ((1 << cl2n) < n) ++cl2n;
    const int lmax = wmax - 1;
    const int cut = lmax + cl2n - 44 > 0 ? lmax + cl2n - 44 : 0;
    for (int i = 0; i < n; ++i) {
        c->beta[i] = 53 - 8 - cl2n + (wbits[i] - 1 - lmax);
        if (precision == OZK_FP32) {
            c->s1[i] = nearest(w[i]);
            c->s2[i] = 0.0;
        } else {
            const U192 head = w[i].shr(cut).shl(cut);
            c->s1[i] = nearest(head);
            c->s2[i] = nearest(sub(w[i], head));
        }
    }
    for (int i = 0; i < n; ++i) {  // crt_tables.cpp:173-180
        c->pinv64[i] = 1.0 / static_cast<double>(p[i]);
        c->pinv32[i] = 1.0f / static_cast<float>(p[i]);
        c->pinv_mulhi[i] = static_cast<int32_t>((u64(1) << 32) / static_cast<u64>(p[i]) - 1);
    }
    return OZK_OK;
}

}  // namespace

const ozk_constants* cached_constants(int n, int precision) {
    static std::mutex mtx;
    static std::map<std::pair<int, int>, ozk_constants> cache;
    std::lock_guard<std::mutex> lock(mtx);
    auto key = std::make_pair(n, precision);
    auto it = cache.find(key);
    if (it == cache.end()) {
        ozk_constants c;
        make_table(n, precision, &c);
        it = cache.emplace(key, c).first;
    }
    return &it->second;
}

}  // namespace ozk

extern "C" {

int ozk_select_moduli(int n, int32_t* out) {
    if (n < 2 || n > OZK_MAX_MODULI) {
        ozk::set_error("modulus count must be in [2, 20], got " + std::to_string(n));
        return OZK_CONFIG_ERROR;
    }
    int kept = 0;
    for (int cand = 256; cand >= 2 && kept < n; --cand) {
        bool coprime = true;
        for (int j = 0; j < kept && coprime; ++j) coprime = ozk::gcd_i(out[j], cand) == 1;
        if (coprime) out[kept++] = cand;
    }
    return OZK_OK;
}

int64_t ozk_mod_inverse(int64_t a, int64_t m, int* status) {
    *status = OZK_OK;
    if (m < 2) {
        *status = OZK_DOMAIN_ERROR;
        ozk::set_error("modulus must be >= 2");
        return 0;
    }
    int64_t r0 = m, r1 = ((a % m) + m) % m, t0 = 0, t1 = 1;
    while (r1) {
        const int64_t qt = r0 / r1;
        const int64_t r2 = r0 - qt * r1, t2 = t0 - qt * t1;
        r0 = r1;
        r1 = r2;
        t0 = t1;
        t1 = t2;
    }
    if (r0 != 1) {
        *status = OZK_DOMAIN_ERROR;
        ozk::set_error("arguments are not coprime");
        return 0;
    }
    return ((t0 % m) + m) % m;
}

int ozk_build_constants(int n, int precision, ozk_constants* out) {
    const int maxn = precision == OZK_FP64 ? 20 : 18;  // crt_tables.hpp:17-21
    if ((precision != OZK_FP64 && precision != OZK_FP32) || n < 2 || n > maxn) {
        ozk::set_error("modulus count " + std::to_string(n) + " out of range [2, " + std::to_string(maxn) +
                       "] for " + (precision == OZK_FP64 ? "fp64" : "fp32"));
        return OZK_CONFIG_ERROR;
    }
    *out = *ozk::cached_constants(n, precision);
    return OZK_OK;
}

int ozk_dump_tables_csv(const ozk_constants* c, char* buf, int64_t buflen) {
    std::string s = "p,q,beta,s1,s2\n";
    char line[160];
    for (int i = 0; i < c->n_moduli; ++i) {
        std::snprintf(line, sizeof line, "%d,%ld,%d,%a,%a\n", c->moduli[i], static_cast<long>(c->q[i]), c->beta[i],
                      c->s1[i], c->s2[i]);
        s += line;
    }
    if (buflen <= 0) return OZK_INPUT_ERROR;
    std::strncpy(buf, s.c_str(), static_cast<size_t>(buflen - 1));
    buf[buflen - 1] = 0;
    return static_cast<int64_t>(s.size()) < buflen ? OZK_OK : OZK_INPUT_ERROR;
}

}  // extern "C"
