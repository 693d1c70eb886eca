/* Minimal GMP 6.x C declarations so the reference sources compile against the
 * system runtime libgmp.so.10 (its headers are not installed in this image).
 *
 * TEST INFRASTRUCTURE ONLY: used to build oracle/_ref (the unmodified
 * reference, compiled from /root/reference) and never linked into the product.
 * Only the entry points the reference touches (crt_tables.cpp, oracle.cpp) and
 * the mpz_class shim in gmpxx.h need are declared; the struct layout is the
 * public GMP ABI (__mpz_struct = {int alloc; int size; limb* d;}).
 */
#ifndef OZK_ORACLE_SHIM_GMP_H
#define OZK_ORACLE_SHIM_GMP_H

#ifdef __cplusplus
extern "C" {
#endif

typedef unsigned long mp_limb_t;
typedef unsigned long mp_bitcnt_t;
typedef struct {
    int _mp_alloc;
    int _mp_size;
    mp_limb_t* _mp_d;
} __mpz_struct;
typedef __mpz_struct mpz_t[1];
typedef __mpz_struct* mpz_ptr;
typedef const __mpz_struct* mpz_srcptr;

void __gmpz_init(mpz_ptr);
void __gmpz_init_set(mpz_ptr, mpz_srcptr);
void __gmpz_init_set_si(mpz_ptr, long);
void __gmpz_init_set_ui(mpz_ptr, unsigned long);
void __gmpz_init_set_d(mpz_ptr, double);
void __gmpz_clear(mpz_ptr);
void __gmpz_set(mpz_ptr, mpz_srcptr);
void __gmpz_set_si(mpz_ptr, long);
void __gmpz_set_ui(mpz_ptr, unsigned long);
void __gmpz_set_d(mpz_ptr, double);
double __gmpz_get_d(mpz_srcptr);
void __gmpz_add(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_sub(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mul_si(mpz_ptr, mpz_srcptr, long);
void __gmpz_tdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_fdiv_qr(mpz_ptr, mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mul_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_fdiv_q_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_and(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_abs(mpz_ptr, mpz_srcptr);
void __gmpz_neg(mpz_ptr, mpz_srcptr);
int __gmpz_cmp(mpz_srcptr, mpz_srcptr);
int __gmpz_cmp_si(mpz_srcptr, long);
unsigned long __gmpz_sizeinbase(mpz_srcptr, int);
int __gmpz_tstbit(mpz_srcptr, mp_bitcnt_t);
void __gmpz_addmul(mpz_ptr, mpz_srcptr, mpz_srcptr);
char* __gmpz_get_str(char*, int, mpz_srcptr);

#define mpz_sizeinbase __gmpz_sizeinbase
#define mpz_tstbit __gmpz_tstbit
#define mpz_fdiv_qr __gmpz_fdiv_qr
#define mpz_addmul __gmpz_addmul

#ifdef __cplusplus
}
#endif

#endif
