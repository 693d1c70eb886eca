// Eager mpz_class over the GMP C runtime, covering exactly the operations the
// reference sources use (crt_tables.cpp, oracle.cpp). TEST INFRASTRUCTURE ONLY:
// it exists so oracle/_ref can be compiled from the untouched reference
// sources; the product never includes it.
#pragma once

#include <type_traits>
#include <utility>

#include "gmp.h"

class mpz_class {
public:
    mpz_class() { __gmpz_init(v_); }
    mpz_class(const mpz_class& o) { __gmpz_init_set(v_, o.v_); }
    mpz_class(mpz_class&& o) noexcept {
        __gmpz_init(v_);
        std::swap(v_[0], o.v_[0]);
    }
    template <typename I, typename std::enable_if<std::is_integral<I>::value, int>::type = 0>
    mpz_class(I x) {  // NOLINT(google-explicit-constructor): mirrors gmpxx
        if (std::is_signed<I>::value)
            __gmpz_init_set_si(v_, static_cast<long>(x));
        else
            __gmpz_init_set_ui(v_, static_cast<unsigned long>(x));
    }
    explicit mpz_class(double d) { __gmpz_init_set_d(v_, d); }
    ~mpz_class() { __gmpz_clear(v_); }

    mpz_class& operator=(const mpz_class& o) {
        if (this != &o) __gmpz_set(v_, o.v_);
        return *this;
    }
    mpz_class& operator=(mpz_class&& o) noexcept {
        std::swap(v_[0], o.v_[0]);
        return *this;
    }
    template <typename I, typename std::enable_if<std::is_integral<I>::value, int>::type = 0>
    mpz_class& operator=(I x) {
        if (std::is_signed<I>::value)
            __gmpz_set_si(v_, static_cast<long>(x));
        else
            __gmpz_set_ui(v_, static_cast<unsigned long>(x));
        return *this;
    }

    double get_d() const { return __gmpz_get_d(v_); }
    __mpz_struct* get_mpz_t() { return v_; }
    const __mpz_struct* get_mpz_t() const { return v_; }

    friend mpz_class operator+(const mpz_class& a, const mpz_class& b) {
        mpz_class r;
        __gmpz_add(r.v_, a.v_, b.v_);
        return r;
    }
    friend mpz_class operator-(const mpz_class& a, const mpz_class& b) {
        mpz_class r;
        __gmpz_sub(r.v_, a.v_, b.v_);
        return r;
    }
    friend mpz_class operator*(const mpz_class& a, const mpz_class& b) {
        mpz_class r;
        __gmpz_mul(r.v_, a.v_, b.v_);
        return r;
    }
    friend mpz_class operator/(const mpz_class& a, const mpz_class& b) {
        mpz_class r;
        __gmpz_tdiv_q(r.v_, a.v_, b.v_);
        return r;
    }
    friend mpz_class operator&(const mpz_class& a, const mpz_class& b) {
        mpz_class r;
        __gmpz_and(r.v_, a.v_, b.v_);
        return r;
    }
    template <typename I, typename std::enable_if<std::is_integral<I>::value, int>::type = 0>
    friend mpz_class operator<<(const mpz_class& a, I s) {
        mpz_class r;
        __gmpz_mul_2exp(r.v_, a.v_, static_cast<mp_bitcnt_t>(s));
        return r;
    }
    template <typename I, typename std::enable_if<std::is_integral<I>::value, int>::type = 0>
    friend mpz_class operator>>(const mpz_class& a, I s) {
        mpz_class r;
        __gmpz_fdiv_q_2exp(r.v_, a.v_, static_cast<mp_bitcnt_t>(s));
        return r;
    }
    mpz_class& operator+=(const mpz_class& b) {
        __gmpz_add(v_, v_, b.v_);
        return *this;
    }
    mpz_class& operator-=(const mpz_class& b) {
        __gmpz_sub(v_, v_, b.v_);
        return *this;
    }
    mpz_class& operator*=(const mpz_class& b) {
        __gmpz_mul(v_, v_, b.v_);
        return *this;
    }
    template <typename I, typename std::enable_if<std::is_integral<I>::value, int>::type = 0>
    mpz_class& operator<<=(I s) {
        __gmpz_mul_2exp(v_, v_, static_cast<mp_bitcnt_t>(s));
        return *this;
    }
    template <typename I, typename std::enable_if<std::is_integral<I>::value, int>::type = 0>
    mpz_class& operator>>=(I s) {
        __gmpz_fdiv_q_2exp(v_, v_, static_cast<mp_bitcnt_t>(s));
        return *this;
    }

    friend int cmp(const mpz_class& a, const mpz_class& b) { return __gmpz_cmp(a.v_, b.v_); }
    friend bool operator==(const mpz_class& a, const mpz_class& b) { return cmp(a, b) == 0; }
    friend bool operator!=(const mpz_class& a, const mpz_class& b) { return cmp(a, b) != 0; }
    friend bool operator<(const mpz_class& a, const mpz_class& b) { return cmp(a, b) < 0; }
    friend bool operator<=(const mpz_class& a, const mpz_class& b) { return cmp(a, b) <= 0; }
    friend bool operator>(const mpz_class& a, const mpz_class& b) { return cmp(a, b) > 0; }
    friend bool operator>=(const mpz_class& a, const mpz_class& b) { return cmp(a, b) >= 0; }

    friend mpz_class abs(const mpz_class& a) {
        mpz_class r;
        __gmpz_abs(r.v_, a.v_);
        return r;
    }

private:
    mpz_t v_;
};
