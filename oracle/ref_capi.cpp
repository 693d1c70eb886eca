// C entry points over the UNMODIFIED reference library (/root/reference/proj),
// compiled into oracle/_ref/libcrtgemm_ref.so by oracle/Makefile.
//
// TEST INFRASTRUCTURE ONLY. This file is the checker's window into the real
// reference: the parity tests and bench.py's cpu_baseline / --impl reference
// leg call it through ctypes. The product never links it.
//
// Every function maps 1:1 onto a public reference symbol:
//   build_constants        crt_tables.cpp:186     scale_fast/scale_accurate scaling.cpp:171-184
//   truncate_scale         residue.cpp:46-51      to_residue_slices         residue.cpp:52-57
//   rmod_fast              residue.hpp:39-53      int8_gemm(_reference)     int8_engine.cpp:42-80
//   mod_u8                 reconstruct.hpp:31     accumulate/crt_reduce     reconstruct.cpp:22-47
//   unscale                reconstruct.cpp:49     gemm_emulated             emulator.cpp:82-108
//   exact_gemm + compare   oracle.cpp:39-157      plain_gemm                oracle.cpp:159-173
// Exceptions map to the status codes of include/ozaki2_b200.h
// (1 ConfigError, 2 InputError, 4 std::domain_error, 5 anything else).
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "crtgemm/crt_tables.hpp"
#include "crtgemm/emulator.hpp"
#include "crtgemm/errors.hpp"
#include "crtgemm/int8_engine.hpp"
#include "crtgemm/oracle.hpp"
#include "crtgemm/reconstruct.hpp"
#include "crtgemm/residue.hpp"
#include "crtgemm/scaling.hpp"

using namespace crtgemm;

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_last_error = e.what();
        return 1;
    } catch (const InputError& e) {
        g_last_error = e.what();
        return 2;
    } catch (const std::domain_error& e) {
        g_last_error = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return 5;
    }
}

Precision prec_of(int p) { return p == 0 ? Precision::Fp64 : Precision::Fp32; }
ScaleMode mode_of(int m) { return m == 0 ? ScaleMode::Fast : ScaleMode::Accurate; }

template <typename T>
Matrix<T> wrap(const T* p, int64_t rows, int64_t cols) {
    Matrix<T> m(rows, cols);
    if (rows * cols) std::memcpy(m.data.data(), p, sizeof(T) * static_cast<size_t>(rows * cols));
    return m;
}

template <typename T>
void unwrap(const Matrix<T>& m, T* out) {
    if (m.size()) std::memcpy(out, m.data.data(), sizeof(T) * static_cast<size_t>(m.size()));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

int ref_select_moduli(int n, int* out) {
    return guarded([&] {
        auto s = select_moduli(n);
        for (int i = 0; i < n; ++i) out[i] = s.moduli[static_cast<size_t>(i)];
    });
}

long ref_mod_inverse(long a, long m, int* status) {
    long r = 0;
    *status = guarded([&] { r = mod_inverse(a, m); });
    return r;
}

int ref_constants(int n, int prec, int* moduli, long* q, int* beta, double* p1p2pinv, float* pp,
                  double* s1, double* s2, double* pinv64, float* pinv32, int32_t* pinv_mulhi, int* p_bits) {
    return guarded([&] {
        const CrtConstants& c = build_constants(n, prec_of(prec));
        for (int i = 0; i < n; ++i) {
            const auto ii = static_cast<size_t>(i);
            moduli[i] = c.modulus_set.moduli[ii];
            q[i] = c.q[ii];
            beta[i] = c.beta[ii];
            s1[i] = c.s1[ii];
            s2[i] = c.s2[ii];
            pinv64[i] = c.pinv64[ii];
            pinv32[i] = c.pinv32[ii];
            pinv_mulhi[i] = c.pinv_mulhi[ii];
        }
        p1p2pinv[0] = c.P1;
        p1p2pinv[1] = c.P2;
        p1p2pinv[2] = c.P_inv;
        pp[0] = c.pp_fast;
        pp[1] = c.pp_accu;
        *p_bits = static_cast<int>(mpz_sizeinbase(c.big_P.get_mpz_t(), 2));
    });
}

int ref_dump_tables_csv(int n, int prec, char* buf, int buflen) {
    return guarded([&] {
        const std::string s = dump_tables_csv(build_constants(n, prec_of(prec)));
        std::strncpy(buf, s.c_str(), static_cast<size_t>(buflen - 1));
        buf[buflen - 1] = 0;
    });
}

#define REF_GEMM(NAME, T)                                                                                \
    int NAME(int64_t m, int64_t n, int64_t k, const T* a, const T* b, int n_moduli, int mode, int prec,    \
             int64_t block_k, int threads, double* c) {                                                   \
        return guarded([&] {                                                                             \
            EmuConfig cfg;                                                                               \
            cfg.n_moduli = n_moduli;                                                                     \
            cfg.mode = mode_of(mode);                                                                    \
            cfg.precision = prec_of(prec);                                                               \
            cfg.block_k = block_k;                                                                       \
            cfg.threads = threads;                                                                       \
            EmulationResult r = gemm_emulated(wrap(a, m, k), wrap(b, k, n), cfg);                        \
            unwrap(r.c, c);                                                                              \
        });                                                                                              \
    }
REF_GEMM(ref_gemm_f64, double)
REF_GEMM(ref_gemm_f32, float)

// the explicit-constants overloads (emulator.hpp:29-32): cfg.precision and the
// table's precision chosen independently
#define REF_GEMM_TBL(NAME, T)                                                                            \
    int NAME(int64_t m, int64_t n, int64_t k, const T* a, const T* b, int n_moduli, int mode, int prec,    \
             int table_prec, int64_t block_k, int threads, double* c) {                                   \
        return guarded([&] {                                                                             \
            EmuConfig cfg;                                                                               \
            cfg.n_moduli = n_moduli;                                                                     \
            cfg.mode = mode_of(mode);                                                                    \
            cfg.precision = prec_of(prec);                                                               \
            cfg.block_k = block_k;                                                                       \
            cfg.threads = threads;                                                                       \
            const CrtConstants& cs = build_constants(n_moduli, prec_of(table_prec));                     \
            EmulationResult r = gemm_emulated(wrap(a, m, k), wrap(b, k, n), cfg, cs);                    \
            unwrap(r.c, c);                                                                              \
        });                                                                                              \
    }
REF_GEMM_TBL(ref_gemm_tbl_f64, double)
REF_GEMM_TBL(ref_gemm_tbl_f32, float)

#define REF_SCALE(NAME, T)                                                                               \
    int NAME(int64_t m, int64_t n, int64_t k, const T* a, const T* b, int n_moduli, int mode, int prec,    \
             int64_t block_k, int threads, double* mu, double* nu) {                                      \
        return guarded([&] {                                                                             \
            const CrtConstants& c = build_constants(n_moduli, prec_of(prec));                            \
            const auto A = wrap(a, m, k);                                                                \
            const auto B = wrap(b, k, n);                                                                \
            ScalePair s = mode == 0 ? scale_fast(A, B, c) : scale_accurate(A, B, c, block_k, threads);   \
            std::memcpy(mu, s.mu.data(), sizeof(double) * static_cast<size_t>(m));                      \
            std::memcpy(nu, s.nu.data(), sizeof(double) * static_cast<size_t>(n));                      \
        });                                                                                              \
    }
REF_SCALE(ref_scale_f64, double)
REF_SCALE(ref_scale_f32, float)

// side: 0 = Row (scale indexed by row), 1 = Col. planes: n_moduli consecutive
// column-major rows x cols int8 slices.
#define REF_RESIDUES(NAME, T)                                                                            \
    int NAME(int64_t rows, int64_t cols, const T* mat, const double* scale, int side, int n_moduli,       \
             int prec, T* truncated, int8_t* planes) {                                                    \
        return guarded([&] {                                                                             \
            const CrtConstants& c = build_constants(n_moduli, prec_of(prec));                            \
            const int64_t len = side == 0 ? rows : cols;                                                 \
            std::vector<double> sc(scale, scale + len);                                                  \
            Matrix<T> tr = truncate_scale(wrap(mat, rows, cols), sc, side == 0 ? Side::Row : Side::Col); \
            unwrap(tr, truncated);                                                                       \
            ResidueSlices rs = to_residue_slices(tr, c);                                                 \
            for (int i = 0; i < n_moduli; ++i) unwrap(rs.slices[static_cast<size_t>(i)], planes + i * rows * cols); \
        });                                                                                              \
    }
REF_RESIDUES(ref_residues_f64, double)
REF_RESIDUES(ref_residues_f32, float)

int ref_rmod_fast_f64(const double* x, int64_t count, int modulus_index, int n_moduli, int8_t* out) {
    return guarded([&] {
        const CrtConstants& c = build_constants(n_moduli, Precision::Fp64);
        for (int64_t e = 0; e < count; ++e) out[e] = rmod_fast(x[e], modulus_index, c);
    });
}

int ref_rmod_fast_f32(const float* x, int64_t count, int modulus_index, int n_moduli, int8_t* out) {
    return guarded([&] {
        const CrtConstants& c = build_constants(n_moduli, Precision::Fp32);
        for (int64_t e = 0; e < count; ++e) out[e] = rmod_fast(x[e], modulus_index, c);
    });
}

int ref_mod_u8(const int32_t* x, int64_t count, int32_t p, int32_t pinv_mulhi, uint8_t* out) {
    for (int64_t e = 0; e < count; ++e) out[e] = mod_u8(x[e], p, pinv_mulhi);
    return 0;
}

int ref_int8_gemm(int64_t m, int64_t n, int64_t k, const int8_t* a, const int8_t* b, int threads, int use_reference,
                  int32_t* c) {
    return guarded([&] {
        const auto A = wrap(a, m, k);
        const auto B = wrap(b, k, n);
        Int32ProductMatrix p = use_reference ? int8_gemm_reference(A, B) : int8_gemm(A, B, threads);
        unwrap(p.data, c);
    });
}

// u: n_moduli consecutive rows x cols uint8 matrices (column-major)
int ref_accumulate(int n_moduli, int prec, int64_t rows, int64_t cols, const uint8_t* u, double* c1, double* c2) {
    return guarded([&] {
        const CrtConstants& c = build_constants(n_moduli, prec_of(prec));
        ResidueProducts rp;
        for (int i = 0; i < n_moduli; ++i) rp.u.push_back(wrap(u + i * rows * cols, rows, cols));
        auto pr = accumulate(rp, c);
        unwrap(pr.first, c1);
        unwrap(pr.second, c2);
    });
}

int ref_crt_reduce(int n_moduli, int prec, int64_t count, const double* c1, const double* c2, double* out) {
    return guarded([&] {
        const CrtConstants& c = build_constants(n_moduli, prec_of(prec));
        Matrix<double> r = crt_reduce(wrap(c1, count, 1), wrap(c2, count, 1), c);
        unwrap(r, out);
    });
}

int ref_unscale(int n_moduli, int prec, int64_t m, int64_t n, const double* cpp, const double* mu, const double* nu,
                double* out) {
    return guarded([&] {
        const CrtConstants& c = build_constants(n_moduli, prec_of(prec));
        ScalePair s;
        s.mu.assign(mu, mu + m);
        s.nu.assign(nu, nu + n);
        EmulationResult r = unscale(wrap(cpp, m, n), s, c);
        unwrap(r.c, out);
    });
}

// exact oracle: report[0]=max_rel_err, report[1]=median_rel_err, report[2]=exact_match
#define REF_COMPARE(NAME, T)                                                                              \
    int NAME(int64_t m, int64_t n, int64_t k, const T* a, const T* b, const double* c, double* report) {   \
        return guarded([&] {                                                                              \
            ExactMatrix ex = exact_gemm(wrap(a, m, k), wrap(b, k, n));                                     \
            ErrorReport r = compare(wrap(c, m, n), ex);                                                   \
            report[0] = r.max_rel_err;                                                                    \
            report[1] = r.median_rel_err;                                                                 \
            report[2] = r.exact_match ? 1.0 : 0.0;                                                        \
        });                                                                                               \
    }
REF_COMPARE(ref_exact_compare_f64, double)
REF_COMPARE(ref_exact_compare_f32, float)

// the exact product (oracle.cpp exact_gemm) rounded to the nearest FP64 per
// entry (ExactMatrix::value_rounded): compare()'s denominator, so one exact
// GEMM serves the error of many candidate results
#define REF_EXACT_ROUNDED(NAME, T)                                                                       \
    int NAME(int64_t m, int64_t n, int64_t k, const T* a, const T* b, double* out) {                     \
        return guarded([&] {                                                                             \
            const ExactMatrix ex = exact_gemm(wrap(a, m, k), wrap(b, k, n));                             \
            for (int64_t j = 0; j < n; ++j)                                                              \
                for (int64_t i = 0; i < m; ++i) out[i + j * m] = ex.value_rounded(i, j);                 \
        });                                                                                              \
    }
REF_EXACT_ROUNDED(ref_exact_rounded_f64, double)
REF_EXACT_ROUNDED(ref_exact_rounded_f32, float)

int ref_plain_gemm_f64(int64_t m, int64_t n, int64_t k, const double* a, const double* b, double* c) {
    return guarded([&] { unwrap(plain_gemm(wrap(a, m, k), wrap(b, k, n)), c); });
}

int ref_plain_gemm_f32(int64_t m, int64_t n, int64_t k, const float* a, const float* b, float* c) {
    return guarded([&] { unwrap(plain_gemm(wrap(a, m, k), wrap(b, k, n)), c); });
}

}  // extern "C"
