/* irl_oracle — CPU restatement of the reference hot path, TEST INFRASTRUCTURE.
 *
 * This library is the parity checker for the B200 engine. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it; the product (paper_2601_17561_b200) never links or calls it.
 *
 * Each function restates one reference function (file:line relative to
 * /root/reference/proj) in plain C with fixed-width integers instead of GMP.
 * Parity of this restatement is pinned against (1) the reference's own
 * known-answer tests (tests/test_modmat.cpp, tests/acceptance.cpp:96-120),
 * committed as JSON fixtures under tests/golden/ by oracle/gen_golden.py, and (2) the
 * unmodified reference compiled into oracle/_ref/ (oracle/Makefile).
 *
 * Status codes are the ones of include/irl_capi.h. */
#ifndef IRL_ORACLE_H
#define IRL_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* --- RNS basis (modmat.cpp:8-63) -------------------------------------- */
size_t orc_primes_in_range(uint32_t lo, uint32_t hi, uint32_t* out, size_t cap);
size_t orc_paper_basis(uint32_t* primes, uint32_t* exps, size_t cap); /* 24 x (p, 2) */
double orc_log2_Q(const uint32_t* primes, const uint32_t* exps, size_t n);
double orc_max_int8_rns_capacity(void);
size_t orc_pure_rns_plane_count(void);
/* Q = prod p^e as little-endian bytes; returns the byte width ceil(log256 Q). */
size_t orc_basis_Q_bytes(const uint32_t* primes, const uint32_t* exps, size_t n, uint8_t* out,
                         size_t cap);

/* --- digits and small GEMMs (modmat.cpp:86-160) ------------------------ */
int orc_digit_decompose(const int32_t* m, size_t count, uint32_t p, int32_t* d0, int32_t* d1);
void orc_digit_recompose(const int32_t* d0, const int32_t* d1, size_t count, uint32_t p,
                         int32_t* out);
/* Returns IRL_ERR_ACCUMULATION_OVERFLOW_RISK (bound in *bound) when
 * K*max|A|*max|B| >= 2^31, exactly as small_gemm's precheck (:122-129). */
int orc_small_gemm(const int32_t* a, const int32_t* b, int32_t* c, size_t m, size_t k, size_t n,
                   int64_t* bound);
int orc_gemm_mod_psq(const int32_t* a, const int32_t* b, int32_t* c, size_t m, size_t k,
                     size_t n, uint32_t p);

/* --- mod-Q path (modmat.cpp:162-212) ------------------------------------
 * Big matrices are row-major arrays of fixed-width little-endian entries of
 * `width` bytes (the reference's on-disk entry format, modmat.cpp:216-231). */
int orc_gemm_mod_Q(const uint8_t* a, const uint8_t* b, uint8_t* c, size_t m, size_t k, size_t n,
                   size_t width, const uint32_t* primes, const uint32_t* exps, size_t nmod);
int orc_oracle_gemm_mod_Q(const uint8_t* a, const uint8_t* b, uint8_t* c, size_t m, size_t k,
                          size_t n, size_t width, const uint32_t* primes, const uint32_t* exps,
                          size_t nmod);

/* --- PPMM over residue planes (CCMM building block; no reference code) ---
 * out[n][r] = sum_k a[r][k] * bt[n][k] mod m for the listed rows, by
 * schoolbook int64 accumulation (the test_modmat.cpp:110-122 check). */
void orc_ppmm_rows_direct(const uint16_t* a, size_t lda, const uint16_t* bt, size_t ldb,
                          const uint32_t* rows, size_t nrows, size_t N, size_t K, uint32_t m,
                          uint16_t* out /* [nrows][N] */);

/* --- counter-based synthetic residues (shared with the product's generator)
 * uniform in [0, m) keyed by (seed, stream, plane, row, col). */
uint32_t orc_synth_residue(uint64_t seed, uint32_t stream, uint32_t plane, uint32_t row,
                           uint32_t col, uint32_t m);
/* Emulator::ccmm_twin's product (emulator.cpp:411-421): i-k-j loop over
 * row-major doubles, zero database entries skipped, each multiply and add
 * rounded (no contraction); written transposed, out[j*d1 + i], which is
 * ccmm_twin's message order. */
void orc_ccmm_twin_product(const double* db, const double* qry, size_t d1, size_t d2, size_t d3, double* out);

void orc_synth_block(uint64_t seed, uint32_t stream, uint32_t plane, uint32_t row0,
                     uint32_t nrows, uint32_t col0, uint32_t ncols, uint32_t m,
                     uint16_t* out /* [nrows][ncols] */);

/* ---- plaintext iris scoring (iris_core.cpp:28-59, 65-76; pipeline.cpp:78-82) ----
 * db / query templates as unpacked {0,1} bytes [n][d]; query column c =
 * e*rho + r is rotate(q_e, r). inner/overlap: int32 [n_eyes*rho][n_db]. */
void orc_iris_inner_overlap(const uint8_t* db_code, const uint8_t* db_mask, size_t n_db, const uint8_t* q_code,
                            const uint8_t* q_mask, size_t n_eyes, size_t rho, size_t d, int32_t* inner,
                            int32_t* overlap);

/* ---- Alg. 2 fold stage, message level (pipeline.cpp:359-408, 538-633) ----
 * Same contract as irl_fold_stage (include/irl_capi.h): normalize, the
 * folding polynomial, the Rot alignment and group sums (folded, may be NULL),
 * the fold chain and the refold over groups (refolded, may be NULL), the
 * folding-assumption check. Polynomials follow ps_execute (poly.hpp:91-119)
 * operation by operation in IEEE double (built with -ffp-contract=off). */
double orc_ps_execute(const double* coeffs, size_t n, double x);
int orc_fold_stage(size_t batch, size_t rho, size_t n_db, size_t d, size_t fold_k, const double* fold_c,
                   size_t fold_len, size_t nstages, const double* centers, const size_t* lens,
                   const double* chain_c, double neg_lo, double neg_hi, const int32_t* inner,
                   const int32_t* overlap, double* folded, double* refolded, int32_t* assumption_ok);

#ifdef __cplusplus
}
#endif

#endif
