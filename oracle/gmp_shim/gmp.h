/* Minimal GMP 6.x C declarations, written for this repo's test oracle.
 *
 * The image ships the GMP runtime (libgmp.so.10, GMP 6.3.0) but not its
 * development headers. This header declares exactly the ABI subset the
 * reference hot path (proj/src/modmat.cpp) and its tests use, so the
 * unmodified reference sources can be compiled into oracle/_ref/ and linked
 * against the system runtime. Struct layouts follow the documented GMP ABI
 * (x86-64, 64-bit limbs). Test infrastructure only; never shipped. */
#ifndef IRL_GMP_SHIM_H
#define IRL_GMP_SHIM_H

#include <stddef.h>
#include <stdio.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef unsigned long mp_limb_t;
typedef long mp_exp_t;
typedef unsigned long mp_bitcnt_t;
typedef long mp_size_t;

typedef struct {
    int _mp_alloc;
    int _mp_size;
    mp_limb_t* _mp_d;
} __mpz_struct;
typedef __mpz_struct mpz_t[1];
typedef __mpz_struct* mpz_ptr;
typedef const __mpz_struct* mpz_srcptr;

typedef struct {
    int _mp_prec;
    int _mp_size;
    mp_exp_t _mp_exp;
    mp_limb_t* _mp_d;
} __mpf_struct;
typedef __mpf_struct mpf_t[1];
typedef __mpf_struct* mpf_ptr;
typedef const __mpf_struct* mpf_srcptr;

typedef enum { GMP_RAND_ALG_DEFAULT = 0, GMP_RAND_ALG_LC = 0 } gmp_randalg_t;
typedef struct {
    __mpz_struct _mp_seed;
    gmp_randalg_t _mp_alg;
    union {
        void* _mp_lc;
    } _mp_algdata;
} __gmp_randstate_struct;
typedef __gmp_randstate_struct gmp_randstate_t[1];

void __gmpz_init(mpz_ptr);
void __gmpz_init_set(mpz_ptr, mpz_srcptr);
void __gmpz_init_set_ui(mpz_ptr, unsigned long);
void __gmpz_init_set_si(mpz_ptr, long);
int __gmpz_init_set_str(mpz_ptr, const char*, int);
void __gmpz_clear(mpz_ptr);
void __gmpz_set(mpz_ptr, mpz_srcptr);
void __gmpz_set_si(mpz_ptr, long);
void __gmpz_set_ui(mpz_ptr, unsigned long);
void __gmpz_swap(mpz_ptr, mpz_ptr);
void __gmpz_add(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_add_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_sub(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mul_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_mul_si(mpz_ptr, mpz_srcptr, long);
void __gmpz_mul_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_tdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_tdiv_r(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mod(mpz_ptr, mpz_srcptr, mpz_srcptr);
unsigned long __gmpz_fdiv_ui(mpz_srcptr, unsigned long);
int __gmpz_invert(mpz_ptr, mpz_srcptr, mpz_srcptr);
int __gmpz_cmp(mpz_srcptr, mpz_srcptr);
int __gmpz_cmp_si(mpz_srcptr, long);
size_t __gmpz_sizeinbase(mpz_srcptr, int);
unsigned long __gmpz_get_ui(mpz_srcptr);
char* __gmpz_get_str(char*, int, mpz_srcptr);
void* __gmpz_export(void*, size_t*, int, size_t, int, size_t, mpz_srcptr);
void __gmpz_import(mpz_ptr, size_t, int, size_t, int, size_t, const void*);
void __gmpz_urandomm(mpz_ptr, __gmp_randstate_struct*, mpz_srcptr);

void __gmpf_init2(mpf_ptr, mp_bitcnt_t);
void __gmpf_set_z(mpf_ptr, mpz_srcptr);
void __gmpf_clear(mpf_ptr);
double __gmpf_get_d_2exp(long*, mpf_srcptr);

void __gmp_randinit_default(__gmp_randstate_struct*);
void __gmp_randseed_ui(__gmp_randstate_struct*, unsigned long);
void __gmp_randclear(__gmp_randstate_struct*);

#define mpz_init __gmpz_init
#define mpz_clear __gmpz_clear
#define mpz_fdiv_ui __gmpz_fdiv_ui
#define mpz_invert __gmpz_invert
#define mpz_mod __gmpz_mod
#define mpz_sizeinbase __gmpz_sizeinbase
#define mpz_export __gmpz_export
#define mpz_import __gmpz_import
#define mpz_urandomm __gmpz_urandomm
#define mpf_get_d_2exp __gmpf_get_d_2exp
#define gmp_randinit_default __gmp_randinit_default
#define gmp_randseed_ui __gmp_randseed_ui
#define gmp_randclear __gmp_randclear

#ifdef __cplusplus
}
#endif

#endif /* IRL_GMP_SHIM_H */
