/* ozk_oracle — plain-C CPU restatement of the reference Ozaki-II emulation
 * (/root/reference/proj, crtgemm), used ONLY as the checker.
 *
 * TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library. The product path
 * (paper_2508_03984_b200/) never links or calls it.
 *
 * Parity pins: tests/test_oracle.py checks every function here against
 *   (1) the SPEC.md known-answer examples and SURVEY Appendix A golden tables,
 *   (2) tests/golden/ fixtures produced by the real reference (oracle/_ref),
 *   (3) oracle/_ref itself on random inputs when that library is present.
 *
 * Layout conventions follow the reference: column-major, ld == rows
 * (matrix.hpp:9-32). Residue planes are N consecutive column-major slices.
 * precision: 0 = fp64, 1 = fp32. mode: 0 = fast, 1 = accurate.
 * Status: 0 ok, 1 ConfigError, 2 InputError (errors.hpp:8-16).
 */
#ifndef OZK_ORACLE_H
#define OZK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OZO_MAX_MODULI 20

typedef struct {
    int n_moduli;
    int precision;
    int moduli[OZO_MAX_MODULI];
    long q[OZO_MAX_MODULI];
    int beta[OZO_MAX_MODULI];
    double P1, P2, P_inv;
    float pp_fast, pp_accu;
    double s1[OZO_MAX_MODULI], s2[OZO_MAX_MODULI];
    double pinv64[OZO_MAX_MODULI];
    float pinv32[OZO_MAX_MODULI];
    int32_t pinv_mulhi[OZO_MAX_MODULI];
    int P_bits;
} ozo_constants;

int ozo_select_moduli(int n, int* out);
long ozo_mod_inverse(long a, long m, int* status);
int ozo_build_constants(int n_moduli, int precision, ozo_constants* out);

/* stage 1a: scale exponents (mu = 2^mu_exp, nu = 2^nu_exp). */
int ozo_scale_f64(const double* a, const double* b, int64_t m, int64_t n, int64_t k, const ozo_constants* c,
                  int mode, int64_t block_k, int32_t* mu_exp, int32_t* nu_exp);
int ozo_scale_f32(const float* a, const float* b, int64_t m, int64_t n, int64_t k, const ozo_constants* c, int mode,
                  int64_t block_k, int32_t* mu_exp, int32_t* nu_exp);

/* stage 1b: truncate_scale + to_residue_slices. side 0 = row scale, 1 = column scale. */
void ozo_truncate_f64(const double* x, int64_t rows, int64_t cols, const int32_t* scale_exp, int side, double* out);
void ozo_truncate_f32(const float* x, int64_t rows, int64_t cols, const int32_t* scale_exp, int side, float* out);
int8_t ozo_rmod_fast_f64(double x, int p, double pinv64, float pinv32, int n_moduli);
int8_t ozo_rmod_fast_f32(float x, int p, float pinv32, int n_moduli);
void ozo_residues_f64(const double* xp, int64_t count, const ozo_constants* c, int8_t* planes);
void ozo_residues_f32(const float* xp, int64_t count, const ozo_constants* c, int8_t* planes);

/* stage 2: wrapping int8 x int8 -> int32 product, column-major */
void ozo_int8_gemm(const int8_t* a, const int8_t* b, int64_t m, int64_t n, int64_t k, int32_t* c);
uint8_t ozo_mod_u8(int32_t x, int32_t p, int32_t pinv_mulhi);

/* stage 3 */
void ozo_accumulate(const uint8_t* u, int64_t count, const ozo_constants* c, double* c1, double* c2);
double ozo_crt_reduce_element(double c1, double c2, const ozo_constants* c);
void ozo_unscale(const double* cpp, int64_t m, int64_t n, const int32_t* mu_exp, const int32_t* nu_exp, double* out);

/* full pipeline (emulator.cpp:25-78). c is m x n FP64, column-major. */
int ozo_gemm_f64(const double* a, const double* b, int64_t m, int64_t n, int64_t k, int n_moduli, int mode,
                 int64_t block_k, double* c);
int ozo_gemm_f32(const float* a, const float* b, int64_t m, int64_t n, int64_t k, int n_moduli, int mode,
                 int64_t block_k, double* c);
/* full pipeline with explicit constants (emulator.hpp:29-32; fault injection) */
int ozo_gemm_f64_consts(const double* a, const double* b, int64_t m, int64_t n, int64_t k, const ozo_constants* c,
                        int mode, int64_t block_k, double* out);

/* pipeline with caller-given exponents (sharding checks) and the accurate budget */
int ozo_gemm_f64_scaled(const double* a, const double* b, int64_t m, int64_t n, int64_t k, const ozo_constants* c,
                        const int32_t* mu, const int32_t* nu, int64_t block_k, double* out);
int ozo_gemm_f32_scaled(const float* a, const float* b, int64_t m, int64_t n, int64_t k, const ozo_constants* c,
                        const int32_t* mu, const int32_t* nu, int64_t block_k, double* out);
int ozo_accurate_exponent(int64_t cmax, int base, const ozo_constants* c);

/* debug: the uint8 residue products U_i of the pipeline (N consecutive m x n slices) */
int ozo_products_u8_f64(const double* a, const double* b, int64_t m, int64_t n, int64_t k, int n_moduli, int mode,
                        int64_t block_k, uint8_t* u);

#ifdef __cplusplus
}
#endif

#endif
