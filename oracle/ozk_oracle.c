/* ozk_oracle.c — plain-C restatement of the reference Ozaki-II emulation.
 *
 * TEST INFRASTRUCTURE ONLY (see ozk_oracle.h): the checker for the CUDA path,
 * never the thing measured or shipped. Compiled with -ffp-contract=off so every
 * `a + b*c` below rounds twice exactly like the reference build.
 *
 * Each function cites the reference line(s) it restates; paths are relative to
 * /root/reference/proj. Big-integer table construction (reference: GMP, in
 * crt_tables.cpp) is restated with a fixed 256-bit unsigned integer, which is
 * ample: P < 2^157 and W_i = (P/p_i) q_i < 2^165 for N <= 20.
 */
#include "ozk_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------------
 * 256-bit unsigned integer (little-endian 32-bit limbs)
 * ------------------------------------------------------------------------- */
#define BN_LIMBS 8
typedef struct {
    uint32_t w[BN_LIMBS];
} bn;

static void bn_zero(bn* a) { memset(a, 0, sizeof *a); }
static void bn_set_u64(bn* a, uint64_t v) {
    bn_zero(a);
    a->w[0] = (uint32_t)v;
    a->w[1] = (uint32_t)(v >> 32);
}
static int bn_is_zero(const bn* a) {
    for (int i = 0; i < BN_LIMBS; ++i)
        if (a->w[i]) return 0;
    return 1;
}
static int bn_cmp(const bn* a, const bn* b) {
    for (int i = BN_LIMBS - 1; i >= 0; --i)
        if (a->w[i] != b->w[i]) return a->w[i] < b->w[i] ? -1 : 1;
    return 0;
}
static void bn_mul_small(bn* a, uint32_t s) {
    uint64_t carry = 0;
    for (int i = 0; i < BN_LIMBS; ++i) {
        uint64_t t = (uint64_t)a->w[i] * s + carry;
        a->w[i] = (uint32_t)t;
        carry = t >> 32;
    }
}
static uint32_t bn_div_small(bn* a, uint32_t d) { /* a /= d, returns remainder */
    uint64_t rem = 0;
    for (int i = BN_LIMBS - 1; i >= 0; --i) {
        uint64_t cur = (rem << 32) | a->w[i];
        a->w[i] = (uint32_t)(cur / d);
        rem = cur % d;
    }
    return (uint32_t)rem;
}
static void bn_sub(bn* r, const bn* a, const bn* b) { /* r = a - b, a >= b */
    int64_t borrow = 0;
    for (int i = 0; i < BN_LIMBS; ++i) {
        int64_t t = (int64_t)a->w[i] - b->w[i] - borrow;
        borrow = t < 0;
        r->w[i] = (uint32_t)(t + (borrow ? ((int64_t)1 << 32) : 0));
    }
}
static void bn_add_small(bn* a, uint32_t s) {
    uint64_t carry = s;
    for (int i = 0; i < BN_LIMBS && carry; ++i) {
        uint64_t t = (uint64_t)a->w[i] + carry;
        a->w[i] = (uint32_t)t;
        carry = t >> 32;
    }
}
static int bn_bits(const bn* a) { /* mpz_sizeinbase(., 2) for a > 0 */
    for (int i = BN_LIMBS - 1; i >= 0; --i)
        if (a->w[i]) {
            int b = 32;
            while (!(a->w[i] >> (b - 1))) --b;
            return i * 32 + b;
        }
    return 0;
}
static int bn_tstbit(const bn* a, int bit) { return (a->w[bit / 32] >> (bit % 32)) & 1u; }
static void bn_shr(bn* r, const bn* a, int s) {
    bn t;
    bn_zero(&t);
    for (int i = 0; i < BN_LIMBS * 32; ++i)
        if (i + s < BN_LIMBS * 32 && bn_tstbit(a, i + s)) t.w[i / 32] |= 1u << (i % 32);
    *r = t;
}
static void bn_shl(bn* r, const bn* a, int s) {
    bn t;
    bn_zero(&t);
    for (int i = 0; i + s < BN_LIMBS * 32; ++i)
        if (bn_tstbit(a, i)) t.w[(i + s) / 32] |= 1u << ((i + s) % 32);
    *r = t;
}
static int bn_low_nonzero(const bn* a, int nbits) { /* any of bits [0, nbits) set */
    for (int i = 0; i < nbits; ++i)
        if (bn_tstbit(a, i)) return 1;
    return 0;
}
/* exact value of an integer below 2^64 (all callers ensure <= 54 bits) */
static double bn_get_d_small(const bn* a) { return (double)a->w[1] * 4294967296.0 + (double)a->w[0]; }

/* to_double_nearest, crt_tables.cpp:50-67 (round half to even on the 53-bit head) */
static double bn_to_double_nearest(const bn* z, int negative) {
    if (bn_is_zero(z)) return 0.0;
    const int bits = bn_bits(z);
    double mag;
    if (bits <= 53) {
        mag = bn_get_d_small(z);
    } else {
        const int drop = bits - 53;
        const int roundbit = bn_tstbit(z, drop - 1);
        const int sticky = bn_low_nonzero(z, drop - 1);
        bn head;
        bn_shr(&head, z, drop);
        if (roundbit && (sticky || bn_tstbit(&head, 0))) bn_add_small(&head, 1);
        mag = ldexp(bn_get_d_small(&head), drop);
    }
    return negative ? -mag : mag;
}

/* ratio_to_double_nearest(1, P), crt_tables.cpp:69-95, restated for num = 1:
 * e = 1 - bits(P); s = 55 - e; quot, rem = floor division of 2^s by P. */
static double bn_recip_nearest(const bn* P) {
    const int e = 1 - bn_bits(P);
    const int s = 55 - e; /* > 0 always */
    /* long division of 2^s by P, bit by bit */
    bn rem, quot, one;
    bn_zero(&rem);
    bn_zero(&quot);
    bn_set_u64(&one, 1);
    for (int bit = s; bit >= 0; --bit) {
        bn_shl(&rem, &rem, 1);
        if (bit == s) bn_add_small(&rem, 1);
        bn_shl(&quot, &quot, 1);
        if (bn_cmp(&rem, P) >= 0) {
            bn_sub(&rem, &rem, P);
            bn_add_small(&quot, 1);
        }
    }
    const int qbits = bn_bits(&quot);
    const int drop = qbits - 53;
    int sticky = !bn_is_zero(&rem);
    if (drop > 0) {
        const int roundbit = bn_tstbit(&quot, drop - 1);
        sticky = sticky || bn_low_nonzero(&quot, drop - 1);
        bn_shr(&quot, &quot, drop);
        if (roundbit && (sticky || bn_tstbit(&quot, 0))) bn_add_small(&quot, 1);
    }
    (void)one;
    return ldexp(bn_get_d_small(&quot), (drop > 0 ? drop : 0) - s);
}

/* log2_mpz, crt_tables.cpp:97-105. mpz_get_d truncates toward zero, so the
 * 64-bit head is truncated to 53 significant bits before the conversion. */
static double bn_log2(const bn* z) {
    const int bits = bn_bits(z);
    const int shift = bits - 64 > 0 ? bits - 64 : 0;
    bn head;
    bn_shr(&head, z, shift);
    uint64_t h = ((uint64_t)head.w[1] << 32) | head.w[0];
    const int hb = bits - shift;
    if (hb > 53) h &= ~((((uint64_t)1) << (hb - 53)) - 1);
    return log2((double)h) + (double)shift;
}

/* ---------------------------------------------------------------------------
 * constants (crt_tables.cpp)
 * ------------------------------------------------------------------------- */
static int gcd_int(int a, int b) {
    while (b) {
        int t = a % b;
        a = b;
        b = t;
    }
    return a;
}

/* select_moduli, crt_tables.cpp:15-30 */
int ozo_select_moduli(int n, int* out) {
    if (n < 2 || n > 20) return 1;
    int cnt = 0;
    for (int cand = 256; cand >= 2 && cnt < n; --cand) {
        int ok = 1;
        for (int j = 0; j < cnt; ++j)
            if (gcd_int(out[j], cand) != 1) {
                ok = 0;
                break;
            }
        if (ok) out[cnt++] = cand;
    }
    return 0;
}

/* mod_inverse, crt_tables.cpp:32-48 (status 4 = std::domain_error) */
long ozo_mod_inverse(long a, long m, int* status) {
    *status = 0;
    if (m < 2) {
        *status = 4;
        return 0;
    }
    long r0 = m, r1 = ((a % m) + m) % m, t0 = 0, t1 = 1;
    while (r1 != 0) {
        long quot = r0 / r1;
        long r2 = r0 - quot * r1, t2 = t0 - quot * t1;
        r0 = r1;
        r1 = r2;
        t0 = t1;
        t1 = t2;
    }
    if (r0 != 1) {
        *status = 4;
        return 0;
    }
    return ((t0 % m) + m) % m;
}

/* build_constants / make_constants, crt_tables.cpp:115-197 (no cache needed) */
int ozo_build_constants(int n, int precision, ozo_constants* c) {
    const int maxn = precision == 0 ? 20 : 18; /* crt_tables.hpp:17-21 */
    if (n < 2 || n > maxn) return 1;
    memset(c, 0, sizeof *c);
    c->n_moduli = n;
    c->precision = precision;
    ozo_select_moduli(n, c->moduli);
    const int* p = c->moduli;

    bn P; /* :121-122 */
    bn_set_u64(&P, 1);
    for (int i = 0; i < n; ++i) bn_mul_small(&P, (uint32_t)p[i]);
    c->P_bits = bn_bits(&P);

    for (int i = 0; i < n; ++i) { /* :125-131 */
        long r = 1;
        for (int j = 0; j < n; ++j)
            if (j != i) r = (r * (p[j] % p[i])) % p[i];
        int st;
        c->q[i] = ozo_mod_inverse(r, p[i], &st);
    }

    /* :133-136 */
    c->P1 = bn_to_double_nearest(&P, 0);
    if (precision == 0) {
        /* P - P1 (P1 is an integer < 2^160: rebuild it exactly from its bits) */
        int ex;
        const double fr = frexp(c->P1, &ex);
        bn p1z;
        if (ex <= 53) {
            bn_set_u64(&p1z, (uint64_t)c->P1);
        } else {
            bn_set_u64(&p1z, (uint64_t)ldexp(fr, 53));
            bn_shl(&p1z, &p1z, ex - 53);
        }
        bn diff;
        if (bn_cmp(&P, &p1z) >= 0) {
            bn_sub(&diff, &P, &p1z);
            c->P2 = bn_to_double_nearest(&diff, 0);
        } else {
            bn_sub(&diff, &p1z, &P);
            c->P2 = bn_to_double_nearest(&diff, 1);
        }
    } else {
        c->P2 = 0.0;
    }
    c->P_inv = bn_recip_nearest(&P);

    /* :138-140 */
    bn Pm1 = P;
    bn one;
    bn_set_u64(&one, 1);
    bn_sub(&Pm1, &P, &one);
    const double half_log = 0.5 * bn_log2(&Pm1);
    c->pp_fast = (float)(half_log - 1.5);
    c->pp_accu = (float)(half_log - 0.5);

    /* :143-171 */
    bn w[OZO_MAX_MODULI];
    int wbits[OZO_MAX_MODULI];
    int wbits_max = 0;
    for (int i = 0; i < n; ++i) {
        w[i] = P;
        bn_div_small(&w[i], (uint32_t)p[i]);
        bn_mul_small(&w[i], (uint32_t)c->q[i]);
        wbits[i] = bn_bits(&w[i]);
        if (wbits[i] > wbits_max) wbits_max = wbits[i];
    }
    int cl2n = 0; /* ceil_log2_int, :109-113 */
    while ((1 << cl2n) < n) ++cl2n;
    const int lmax = wbits_max - 1;
    for (int i = 0; i < n; ++i) {
        const int li = wbits[i] - 1;
        c->beta[i] = 53 - 8 - cl2n + (li - lmax);
        if (precision == 1) {
            c->s1[i] = bn_to_double_nearest(&w[i], 0);
            c->s2[i] = 0.0;
            continue;
        }
        const int cut = lmax + cl2n - 44 > 0 ? lmax + cl2n - 44 : 0;
        bn head, tail;
        bn_shr(&head, &w[i], cut);
        bn_shl(&head, &head, cut);
        bn_sub(&tail, &w[i], &head);
        c->s1[i] = bn_to_double_nearest(&head, 0);
        c->s2[i] = bn_to_double_nearest(&tail, 0);
    }

    for (int i = 0; i < n; ++i) { /* :173-180 */
        c->pinv64[i] = 1.0 / (double)p[i];
        c->pinv32[i] = 1.0f / (float)p[i];
        c->pinv_mulhi[i] = (int32_t)((((uint64_t)1) << 32) / (uint64_t)p[i] - 1);
    }
    return 0;
}

/* ---------------------------------------------------------------------------
 * stage 1a: scaling (scaling.cpp)
 * ------------------------------------------------------------------------- */
static int magnitude_cap(int prec) { return prec == 0 ? 72 : 44; }    /* :15 */
static int exponent_clamp(int prec) { return prec == 0 ? 1021 : 125; } /* :18 */
static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* sum_upper_bound, :45-47 */
static double sum_upper_bound(double s, int64_t terms) {
    return s * (1.0 + 2.0 * (double)(terms + 2) * 0x1.0p-53);
}

/* fast_exponent, :50-56 (reference defect kept: no "- max_exp" term) */
static int fast_exponent(double norm_sq_ub, int max_exp, const ozo_constants* c) {
    const double l = 0.51 * log2(norm_sq_ub);
    const double t = l > 1.0 ? l : 1.0;
    int e = (int)floor((double)c->pp_fast - t);
    const int cap = magnitude_cap(c->precision) - 1 - max_exp;
    if (e > cap) e = cap;
    const int cl = exponent_clamp(c->precision);
    return clampi(e, -cl, cl);
}

/* value accessor so one body serves both input precisions (scaling.cpp
 * templates on T and widens with static_cast<double>) */
#define SCALE_BODY(T)                                                                                        \
    const int prec = c->precision;                                                                             \
    double* amax = (double*)calloc((size_t)m, sizeof(double));                                                 \
    for (int64_t j = 0; j < k; ++j) /* row_abs_max :20-31 */                                                   \
        for (int64_t i = 0; i < m; ++i) {                                                                      \
            const double v = fabs((double)a[i + j * m]);                                                       \
            if (v > amax[i]) amax[i] = v;                                                                      \
        }                                                                                                      \
    double* bmax = (double*)calloc((size_t)n, sizeof(double));                                                 \
    for (int64_t j = 0; j < n; ++j) { /* col_abs_max :33-43 */                                                 \
        double v = 0.0;                                                                                        \
        for (int64_t i = 0; i < k; ++i) {                                                                      \
            const double x = fabs((double)b[i + j * k]);                                                       \
            v = v > x ? v : x;                                                                                 \
        }                                                                                                      \
        bmax[j] = v;                                                                                           \
    }                                                                                                          \
    for (int64_t i = 0; i < m; ++i) mu_exp[i] = 0;                                                             \
    for (int64_t j = 0; j < n; ++j) nu_exp[j] = 0;                                                             \
    if (mode == 0) {                                                                                           \
        /* scale_fast_impl :58-99 */                                                                           \
        int* g = (int*)calloc((size_t)m, sizeof(int));                                                         \
        double* sums = (double*)calloc((size_t)m, sizeof(double));                                             \
        for (int64_t i = 0; i < m; ++i)                                                                        \
            if (amax[i] != 0.0) g[i] = ilogb(amax[i]);                                                         \
        for (int64_t j = 0; j < k; ++j)                                                                        \
            for (int64_t i = 0; i < m; ++i) {                                                                  \
                if (amax[i] == 0.0) continue;                                                                  \
                const double nh = ldexp((double)a[i + j * m], -g[i]);                                          \
                sums[i] += nh * nh;                                                                            \
            }                                                                                                  \
        for (int64_t i = 0; i < m; ++i)                                                                        \
            if (amax[i] != 0.0) mu_exp[i] = fast_exponent(sum_upper_bound(sums[i], k), g[i], c);               \
        for (int64_t j = 0; j < n; ++j) {                                                                      \
            if (bmax[j] == 0.0) continue;                                                                      \
            const int gb = ilogb(bmax[j]);                                                                     \
            double sum = 0.0;                                                                                  \
            for (int64_t i = 0; i < k; ++i) {                                                                  \
                const double nh = ldexp((double)b[i + j * k], -gb);                                            \
                sum += nh * nh;                                                                                \
            }                                                                                                  \
            nu_exp[j] = fast_exponent(sum_upper_bound(sum, k), gb, c);                                         \
        }                                                                                                      \
        free(g);                                                                                               \
        free(sums);                                                                                            \
    } else {                                                                                                   \
        /* scale_accurate_impl :101-167 */                                                                     \
        int* ma = (int*)calloc((size_t)m, sizeof(int));                                                        \
        int* nb = (int*)calloc((size_t)n, sizeof(int));                                                        \
        for (int64_t i = 0; i < m; ++i)                                                                        \
            if (amax[i] != 0.0) ma[i] = 5 - ilogb(amax[i]);                                                    \
        for (int64_t j = 0; j < n; ++j)                                                                        \
            if (bmax[j] != 0.0) nb[j] = 5 - ilogb(bmax[j]);                                                    \
        int8_t* abar = (int8_t*)malloc((size_t)(m * k));                                                       \
        int8_t* bbar = (int8_t*)malloc((size_t)(k * n));                                                       \
        for (int64_t j = 0; j < k; ++j) /* :119-126 */                                                         \
            for (int64_t i = 0; i < m; ++i)                                                                    \
                abar[i + j * m] = (int8_t)ceil(ldexp(fabs((double)a[i + j * m]), ma[i]));                      \
        for (int64_t j = 0; j < n; ++j) /* :127-133 */                                                         \
            for (int64_t i = 0; i < k; ++i)                                                                    \
                bbar[i + j * k] = (int8_t)ceil(ldexp(fabs((double)b[i + j * k]), nb[j]));                      \
        /* Cbar = Abar*Bbar (:137-149). Entries are in [0,64], so every k-block                             \
         * product (<= 2^12 * 2^17) is exact in int32 and the int64 total does                                \
         * not depend on block_k; it is summed directly in int64 here. */                                     \
        (void)block_k;                                                                                         \
        int64_t* rowmax = (int64_t*)calloc((size_t)m, sizeof(int64_t));                                        \
        int64_t* colmax = (int64_t*)calloc((size_t)n, sizeof(int64_t));                                        \
        int64_t* acc = (int64_t*)malloc((size_t)m * sizeof(int64_t));                                         \
        for (int64_t j = 0; j < n; ++j) {                                                                      \
            for (int64_t i = 0; i < m; ++i) acc[i] = 0;                                                        \
            for (int64_t h = 0; h < k; ++h) {                                                                  \
                const int64_t bv = bbar[h + j * k];                                                            \
                if (!bv) continue;                                                                             \
                const int8_t* acol = abar + h * m;                                                             \
                for (int64_t i = 0; i < m; ++i) acc[i] += (int64_t)acol[i] * bv;                               \
            }                                                                                                  \
            for (int64_t i = 0; i < m; ++i) {                                                                  \
                if (acc[i] > rowmax[i]) rowmax[i] = acc[i];                                                    \
                if (acc[i] > colmax[j]) colmax[j] = acc[i];                                                    \
            }                                                                                                  \
        }                                                                                                      \
        const int cap = magnitude_cap(prec) - 6; /* :151-161 */                                                \
        const int cl = exponent_clamp(prec);                                                                   \
        for (int64_t i = 0; i < m; ++i) {                                                                      \
            if (amax[i] == 0.0) continue;                                                                      \
            int e = 0;                                                                                         \
            if (rowmax[i] > 0) {                                                                               \
                e = (int)floor((double)c->pp_accu - 0.51 * log2((double)rowmax[i]));                           \
                if (e > cap) e = cap;                                                                          \
            }                                                                                                  \
            mu_exp[i] = clampi(ma[i] + e, -cl, cl);                                                            \
        }                                                                                                      \
        for (int64_t j = 0; j < n; ++j) {                                                                      \
            if (bmax[j] == 0.0) continue;                                                                      \
            int e = 0;                                                                                         \
            if (colmax[j] > 0) {                                                                               \
                e = (int)floor((double)c->pp_accu - 0.51 * log2((double)colmax[j]));                           \
                if (e > cap) e = cap;                                                                          \
            }                                                                                                  \
            nu_exp[j] = clampi(nb[j] + e, -cl, cl);                                                            \
        }                                                                                                      \
        free(ma);                                                                                              \
        free(nb);                                                                                              \
        free(abar);                                                                                            \
        free(bbar);                                                                                            \
        free(rowmax);                                                                                          \
        free(colmax);                                                                                          \
        free(acc);                                                                                             \
    }                                                                                                          \
    free(amax);                                                                                                \
    free(bmax);                                                                                                \
    return 0;

int ozo_scale_f64(const double* a, const double* b, int64_t m, int64_t n, int64_t k, const ozo_constants* c,
                  int mode, int64_t block_k, int32_t* mu_exp, int32_t* nu_exp) {
    SCALE_BODY(double)
}

int ozo_scale_f32(const float* a, const float* b, int64_t m, int64_t n, int64_t k, const ozo_constants* c, int mode,
                  int64_t block_k, int32_t* mu_exp, int32_t* nu_exp) {
    SCALE_BODY(float)
}

/* ---------------------------------------------------------------------------
 * stage 1b: truncation and residues (residue.cpp, residue.hpp)
 * ------------------------------------------------------------------------- */
/* truncate_scale_impl, residue.cpp:7-22 (scale = 2^exp; (T)scale is exact) */
void ozo_truncate_f64(const double* x, int64_t rows, int64_t cols, const int32_t* scale_exp, int side, double* out) {
    for (int64_t j = 0; j < cols; ++j)
        for (int64_t i = 0; i < rows; ++i) {
            const double s = ldexp(1.0, side == 0 ? scale_exp[i] : scale_exp[j]);
            out[i + j * rows] = trunc(x[i + j * rows] * s);
        }
}

void ozo_truncate_f32(const float* x, int64_t rows, int64_t cols, const int32_t* scale_exp, int side, float* out) {
    for (int64_t j = 0; j < cols; ++j)
        for (int64_t i = 0; i < rows; ++i) {
            const float s = (float)ldexp(1.0, side == 0 ? scale_exp[i] : scale_exp[j]);
            out[i + j * rows] = truncf(x[i + j * rows] * s);
        }
}

/* rmod_fast fp64, residue.hpp:39-45; refinement thresholds :17-20 */
int8_t ozo_rmod_fast_f64(double x, int p, double pinv64, float pinv32, int n_moduli) {
    float y = (float)fma(nearbyint(x * pinv64), -(double)p, x);
    const float pf = (float)p;
    if (n_moduli >= 13) y = fmaf(nearbyintf(y * pinv32), -pf, y);
    if (n_moduli >= 19) y = fmaf(nearbyintf(y * pinv32), -pf, y);
    return (int8_t)(int32_t)y;
}

/* rmod_fast fp32, residue.hpp:47-53 */
int8_t ozo_rmod_fast_f32(float x, int p, float pinv32, int n_moduli) {
    const float pf = (float)p;
    float y = fmaf(nearbyintf(x * pinv32), -pf, x);
    if (n_moduli >= 5) y = fmaf(nearbyintf(y * pinv32), -pf, y);
    if (n_moduli >= 11) y = fmaf(nearbyintf(y * pinv32), -pf, y);
    return (int8_t)(int32_t)y;
}

/* to_residue_slices_impl, residue.cpp:24-42 */
void ozo_residues_f64(const double* xp, int64_t count, const ozo_constants* c, int8_t* planes) {
    for (int i = 0; i < c->n_moduli; ++i)
        for (int64_t e = 0; e < count; ++e)
            planes[i * count + e] = ozo_rmod_fast_f64(xp[e], c->moduli[i], c->pinv64[i], c->pinv32[i], c->n_moduli);
}

void ozo_residues_f32(const float* xp, int64_t count, const ozo_constants* c, int8_t* planes) {
    for (int i = 0; i < c->n_moduli; ++i)
        for (int64_t e = 0; e < count; ++e)
            planes[i * count + e] = ozo_rmod_fast_f32(xp[e], c->moduli[i], c->pinv32[i], c->n_moduli);
}

/* ---------------------------------------------------------------------------
 * stage 2 (int8_engine.cpp) and the mod epilogue (reconstruct.hpp:31-37)
 * ------------------------------------------------------------------------- */
/* int8_gemm / gemm_columns, int8_engine.cpp:15-38: uint32 wrapping sum (the
 * pairwise grouping there does not change the value mod 2^32). */
void ozo_int8_gemm(const int8_t* a, const int8_t* b, int64_t m, int64_t n, int64_t k, int32_t* c) {
    uint32_t* acc = (uint32_t*)malloc((size_t)m * sizeof(uint32_t));
    for (int64_t j = 0; j < n; ++j) {
        for (int64_t i = 0; i < m; ++i) acc[i] = 0u;
        for (int64_t h = 0; h < k; ++h) {
            const int32_t bv = b[h + j * k];
            const int8_t* acol = a + h * m;
            for (int64_t i = 0; i < m; ++i) acc[i] += (uint32_t)((int32_t)acol[i] * bv);
        }
        for (int64_t i = 0; i < m; ++i) c[i + j * m] = (int32_t)acc[i];
    }
    free(acc);
}

/* mod_u8, reconstruct.hpp:31-37 */
uint8_t ozo_mod_u8(int32_t x, int32_t p, int32_t pinv_mulhi) {
    const int32_t hi = (int32_t)(((int64_t)x * pinv_mulhi) >> 32);
    int64_t y = (int64_t)x - (int64_t)hi * p;
    if (y >= p) y -= p;
    if (y < 0) y += p;
    return (uint8_t)y;
}

/* ---------------------------------------------------------------------------
 * stage 3 (reconstruct.cpp, reconstruct.hpp)
 * ------------------------------------------------------------------------- */
/* accumulate, reconstruct.cpp:22-38 (u: N consecutive count-element planes) */
void ozo_accumulate(const uint8_t* u, int64_t count, const ozo_constants* c, double* c1, double* c2) {
    for (int64_t e = 0; e < count; ++e) c1[e] = c2[e] = 0.0;
    for (int i = 0; i < c->n_moduli; ++i)
        for (int64_t e = 0; e < count; ++e) {
            const double v = (double)u[i * count + e];
            c1[e] += c->s1[i] * v;
            c2[e] += c->s2[i] * v;
        }
}

/* crt_reduce_element, reconstruct.hpp:51-54 */
double ozo_crt_reduce_element(double c1, double c2, const ozo_constants* c) {
    const double q = nearbyint(c->P_inv * c1);
    return fma(-c->P2, q, fma(-c->P1, q, c1) + c2);
}

/* unscale, reconstruct.cpp:49-69 */
void ozo_unscale(const double* cpp, int64_t m, int64_t n, const int32_t* mu_exp, const int32_t* nu_exp, double* out) {
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) out[i + j * m] = ldexp(cpp[i + j * m], -(mu_exp[i] + nu_exp[j]));
}

/* ---------------------------------------------------------------------------
 * pipeline (emulator.cpp)
 * ------------------------------------------------------------------------- */
/* validate_inputs, emulator.cpp:12-23 (threads are not a parameter here) */
#define VALIDATE(T)                                                                                            \
    if (m < 1 || k < 1 || n < 1) return 2;                                                                     \
    if (block_k < 1 || block_k > ((int64_t)1 << 17)) return 1;                                                 \
    for (int64_t e = 0; e < m * k; ++e)                                                                        \
        if (!isfinite(a[e])) return 2;                                                                         \
    for (int64_t e = 0; e < k * n; ++e)                                                                        \
        if (!isfinite(b[e])) return 2;

/* per-modulus product + mod (+ k blocking, emulator.cpp:42-74); writes U_i */
static void products_u8(const int8_t* sa, const int8_t* sb, int64_t m, int64_t n, int64_t k, int64_t block_k,
                        int32_t p, int32_t pinv, uint8_t* u) {
    int32_t* prod = (int32_t*)malloc((size_t)(m * n) * sizeof(int32_t));
    if (k <= block_k) {
        ozo_int8_gemm(sa, sb, m, n, k, prod);
        for (int64_t e = 0; e < m * n; ++e) u[e] = ozo_mod_u8(prod[e], p, pinv);
    } else {
        int32_t* usum = (int32_t*)calloc((size_t)(m * n), sizeof(int32_t));
        int8_t* ablk = (int8_t*)malloc((size_t)(m * block_k));
        int8_t* bblk = (int8_t*)malloc((size_t)(block_k * n));
        for (int64_t h0 = 0; h0 < k; h0 += block_k) {
            const int64_t len = block_k < k - h0 ? block_k : k - h0;
            memcpy(ablk, sa + h0 * m, (size_t)(m * len)); /* column_block, matrix.hpp:35-41 */
            for (int64_t j = 0; j < n; ++j) memcpy(bblk + j * len, sb + h0 + j * k, (size_t)len); /* row_block */
            ozo_int8_gemm(ablk, bblk, m, n, len, prod);
            for (int64_t e = 0; e < m * n; ++e) usum[e] += ozo_mod_u8(prod[e], p, pinv);
        }
        for (int64_t e = 0; e < m * n; ++e) u[e] = ozo_mod_u8(usum[e], p, pinv);
        free(usum);
        free(ablk);
        free(bblk);
    }
    free(prod);
}

#define PIPELINE(T, TRUNC, RESID, SCALE)                                                                       \
    int32_t* mu = (int32_t*)malloc((size_t)m * sizeof(int32_t));                                               \
    int32_t* nu = (int32_t*)malloc((size_t)n * sizeof(int32_t));                                               \
    SCALE(a, b, m, n, k, c, mode, block_k, mu, nu);                                                            \
    T* ap = (T*)malloc((size_t)(m * k) * sizeof(T));                                                           \
    T* bp = (T*)malloc((size_t)(k * n) * sizeof(T));                                                           \
    TRUNC(a, m, k, mu, 0, ap);                                                                                 \
    TRUNC(b, k, n, nu, 1, bp);                                                                                 \
    int8_t* sa = (int8_t*)malloc((size_t)(c->n_moduli * m * k));                                               \
    int8_t* sb = (int8_t*)malloc((size_t)(c->n_moduli * k * n));                                               \
    RESID(ap, m * k, c, sa);                                                                                   \
    RESID(bp, k * n, c, sb);                                                                                   \
    for (int i = 0; i < c->n_moduli; ++i)                                                                      \
        products_u8(sa + i * m * k, sb + i * k * n, m, n, k, block_k, c->moduli[i], c->pinv_mulhi[i],          \
                    u + i * m * n);                                                                            \
    free(ap);                                                                                                  \
    free(bp);                                                                                                  \
    free(sa);                                                                                                  \
    free(sb);

static int run_f64(const double* a, const double* b, int64_t m, int64_t n, int64_t k, const ozo_constants* c,
                   int mode, int64_t block_k, uint8_t* u_out, double* out) {
    VALIDATE(double)
    uint8_t* u = u_out ? u_out : (uint8_t*)malloc((size_t)(c->n_moduli * m * n));
    PIPELINE(double, ozo_truncate_f64, ozo_residues_f64, ozo_scale_f64)
    if (out) {
        double* c1 = (double*)malloc((size_t)(m * n) * sizeof(double));
        double* c2 = (double*)malloc((size_t)(m * n) * sizeof(double));
        ozo_accumulate(u, m * n, c, c1, c2);
        for (int64_t e = 0; e < m * n; ++e) c1[e] = ozo_crt_reduce_element(c1[e], c2[e], c); /* :76 */
        ozo_unscale(c1, m, n, mu, nu, out);                                                  /* :77 */
        free(c1);
        free(c2);
    }
    if (!u_out) free(u);
    free(mu);
    free(nu);
    return 0;
}

static int run_f32(const float* a, const float* b, int64_t m, int64_t n, int64_t k, const ozo_constants* c, int mode,
                   int64_t block_k, double* out) {
    VALIDATE(float)
    uint8_t* u = (uint8_t*)malloc((size_t)(c->n_moduli * m * n));
    PIPELINE(float, ozo_truncate_f32, ozo_residues_f32, ozo_scale_f32)
    double* c1 = (double*)malloc((size_t)(m * n) * sizeof(double));
    double* c2 = (double*)malloc((size_t)(m * n) * sizeof(double));
    ozo_accumulate(u, m * n, c, c1, c2);
    for (int64_t e = 0; e < m * n; ++e) c1[e] = ozo_crt_reduce_element(c1[e], c2[e], c);
    ozo_unscale(c1, m, n, mu, nu, out);
    free(c1);
    free(c2);
    free(u);
    free(mu);
    free(nu);
    return 0;
}

/* the pipeline after scaling with caller-given exponents (emulator.cpp:34-77);
 * used to check column-sharded runs, whose mu comes from an exchange */
int ozo_gemm_f64_scaled(const double* a, const double* b, int64_t m, int64_t n, int64_t k, const ozo_constants* c,
                        const int32_t* mu, const int32_t* nu, int64_t block_k, double* out) {
    double* ap = (double*)malloc((size_t)(m * k) * sizeof(double));
    double* bp = (double*)malloc((size_t)(k * n) * sizeof(double));
    ozo_truncate_f64(a, m, k, mu, 0, ap);
    ozo_truncate_f64(b, k, n, nu, 1, bp);
    int8_t* sa = (int8_t*)malloc((size_t)(c->n_moduli * m * k));
    int8_t* sb = (int8_t*)malloc((size_t)(c->n_moduli * k * n));
    ozo_residues_f64(ap, m * k, c, sa);
    ozo_residues_f64(bp, k * n, c, sb);
    uint8_t* u = (uint8_t*)malloc((size_t)(c->n_moduli * m * n));
    for (int i = 0; i < c->n_moduli; ++i)
        products_u8(sa + i * m * k, sb + i * k * n, m, n, k, block_k, c->moduli[i], c->pinv_mulhi[i], u + i * m * n);
    double* c1 = (double*)malloc((size_t)(m * n) * sizeof(double));
    double* c2 = (double*)malloc((size_t)(m * n) * sizeof(double));
    ozo_accumulate(u, m * n, c, c1, c2);
    for (int64_t e = 0; e < m * n; ++e) c1[e] = ozo_crt_reduce_element(c1[e], c2[e], c);
    ozo_unscale(c1, m, n, mu, nu, out);
    free(ap);
    free(bp);
    free(sa);
    free(sb);
    free(u);
    free(c1);
    free(c2);
    return 0;
}

/* FP32 twin of ozo_gemm_f64_scaled (emulator.cpp:82-93 after scaling) */
int ozo_gemm_f32_scaled(const float* a, const float* b, int64_t m, int64_t n, int64_t k, const ozo_constants* c,
                        const int32_t* mu, const int32_t* nu, int64_t block_k, double* out) {
    float* ap = (float*)malloc((size_t)(m * k) * sizeof(float));
    float* bp = (float*)malloc((size_t)(k * n) * sizeof(float));
    ozo_truncate_f32(a, m, k, mu, 0, ap);
    ozo_truncate_f32(b, k, n, nu, 1, bp);
    int8_t* sa = (int8_t*)malloc((size_t)(c->n_moduli * m * k));
    int8_t* sb = (int8_t*)malloc((size_t)(c->n_moduli * k * n));
    ozo_residues_f32(ap, m * k, c, sa);
    ozo_residues_f32(bp, k * n, c, sb);
    uint8_t* u = (uint8_t*)malloc((size_t)(c->n_moduli * m * n));
    for (int i = 0; i < c->n_moduli; ++i)
        products_u8(sa + i * m * k, sb + i * k * n, m, n, k, block_k, c->moduli[i], c->pinv_mulhi[i], u + i * m * n);
    double* c1 = (double*)malloc((size_t)(m * n) * sizeof(double));
    double* c2 = (double*)malloc((size_t)(m * n) * sizeof(double));
    ozo_accumulate(u, m * n, c, c1, c2);
    for (int64_t e = 0; e < m * n; ++e) c1[e] = ozo_crt_reduce_element(c1[e], c2[e], c);
    ozo_unscale(c1, m, n, mu, nu, out);
    free(ap);
    free(bp);
    free(sa);
    free(sb);
    free(u);
    free(c1);
    free(c2);
    return 0;
}

/* accurate-mode exponent of one line from its bound maximum (scaling.cpp:153-161);
 * base = 5 - ilogb(max|x|), the caller handles zero lines */
int ozo_accurate_exponent(int64_t cmax, int base, const ozo_constants* c) {
    int e = 0;
    if (cmax > 0) {
        e = (int)floor((double)c->pp_accu - 0.51 * log2((double)cmax));
        const int cap = magnitude_cap(c->precision) - 6;
        if (e > cap) e = cap;
    }
    const int cl = exponent_clamp(c->precision);
    return clampi(base + e, -cl, cl);
}

/* gemm_emulated(Matrix<double>...), emulator.cpp:102-104 -> :82-93 */
int ozo_gemm_f64(const double* a, const double* b, int64_t m, int64_t n, int64_t k, int n_moduli, int mode,
                 int64_t block_k, double* c) {
    ozo_constants cs;
    const int st = ozo_build_constants(n_moduli, 0, &cs);
    if (st) return st;
    return run_f64(a, b, m, n, k, &cs, mode, block_k, NULL, c);
}

int ozo_gemm_f64_consts(const double* a, const double* b, int64_t m, int64_t n, int64_t k, const ozo_constants* c,
                        int mode, int64_t block_k, double* out) {
    if (c->precision != 0) return 1;
    return run_f64(a, b, m, n, k, c, mode, block_k, NULL, out);
}

/* gemm_emulated(Matrix<float>...), emulator.cpp:106-108 -> :95-100 */
int ozo_gemm_f32(const float* a, const float* b, int64_t m, int64_t n, int64_t k, int n_moduli, int mode,
                 int64_t block_k, double* c) {
    ozo_constants cs;
    const int st = ozo_build_constants(n_moduli, 1, &cs);
    if (st) return st;
    return run_f32(a, b, m, n, k, &cs, mode, block_k, c);
}

int ozo_products_u8_f64(const double* a, const double* b, int64_t m, int64_t n, int64_t k, int n_moduli, int mode,
                        int64_t block_k, uint8_t* u) {
    ozo_constants cs;
    const int st = ozo_build_constants(n_moduli, 0, &cs);
    if (st) return st;
    return run_f64(a, b, m, n, k, &cs, mode, block_k, u, NULL);
}
