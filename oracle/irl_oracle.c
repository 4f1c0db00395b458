/* irl_oracle.c — CPU restatement of the reference hot path. TEST
 * INFRASTRUCTURE ONLY (see irl_oracle.h): the product never links this.
 *
 * Reference line numbers are relative to /root/reference/proj. Big integers
 * are little-endian arrays of 32-bit limbs; no GMP. */
#include "irl_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "../include/irl_capi.h"

/* ---------------------------------------------------------------------------
 * RNS basis — modmat.cpp:8-63
 * ------------------------------------------------------------------------- */

/* primes_in_range (modmat.cpp:8-21): trial division, n from max(lo,2). */
size_t orc_primes_in_range(uint32_t lo, uint32_t hi, uint32_t* out, size_t cap) {
    size_t cnt = 0;
    for (uint32_t n = lo > 2 ? lo : 2; n <= hi; ++n) {
        int prime = 1;
        for (uint32_t q = 2; q * q <= n; ++q) {
            if (n % q == 0) {
                prime = 0;
                break;
            }
        }
        if (prime) {
            if (out && cnt < cap) out[cnt] = n;
            ++cnt;
        }
    }
    return cnt;
}

/* build_paper_basis (modmat.cpp:37-45): every prime 127..253 squared. */
size_t orc_paper_basis(uint32_t* primes, uint32_t* exps, size_t cap) {
    uint32_t ps[64];
    const size_t n = orc_primes_in_range(127, 253, ps, 64);
    for (size_t i = 0; i < n && i < cap; ++i) {
        primes[i] = ps[i];
        exps[i] = 2;
    }
    return n;
}

/* RnsBasis::log2_Q (modmat.cpp:29-35) computes log2 of the exact product
 * through mpf; the sum of e*log2(p) is the same quantity (test_modmat.cpp:38-40
 * pins the equality to 1e-9). */
double orc_log2_Q(const uint32_t* primes, const uint32_t* exps, size_t n) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += (double)exps[i] * log2((double)primes[i]);
    return s;
}

/* max_int8_rns_capacity (modmat.cpp:47-59). */
double orc_max_int8_rns_capacity(void) {
    uint32_t ps[64];
    const size_t n = orc_primes_in_range(3, 253, ps, 64);
    double total = 0.0;
    for (size_t i = 0; i < n; ++i) {
        uint32_t e = 0;
        uint64_t pw = 1;
        while (pw * ps[i] < 256) {
            pw *= ps[i];
            ++e;
        }
        total += e * log2((double)ps[i]);
    }
    return total;
}

/* pure_rns_plane_count (modmat.cpp:61-63). */
size_t orc_pure_rns_plane_count(void) { return orc_primes_in_range(3, 253, NULL, 0); }

/* ---------------------------------------------------------------------------
 * Little-endian 32-bit-limb big integers
 * ------------------------------------------------------------------------- */

#define BN_MAX 96

static void bn_from_le(const uint8_t* b, size_t w, uint32_t* x, size_t L) {
    memset(x, 0, L * sizeof(uint32_t));
    for (size_t i = 0; i < w && i / 4 < L; ++i) x[i / 4] |= (uint32_t)b[i] << (8 * (i % 4));
}

static void bn_to_le(const uint32_t* x, size_t L, uint8_t* b, size_t w) {
    for (size_t i = 0; i < w; ++i) b[i] = i / 4 < L ? (uint8_t)(x[i / 4] >> (8 * (i % 4))) : 0;
}

static uint32_t bn_mod_small(const uint32_t* x, size_t L, uint32_t m) {
    uint64_t r = 0;
    for (size_t i = L; i-- > 0;) r = ((r << 32) | x[i]) % m;
    return (uint32_t)r;
}

/* x /= m in place, returns the remainder. */
static uint32_t bn_divmod_small(uint32_t* x, size_t L, uint32_t m) {
    uint64_t r = 0;
    for (size_t i = L; i-- > 0;) {
        const uint64_t cur = (r << 32) | x[i];
        x[i] = (uint32_t)(cur / m);
        r = cur % m;
    }
    return (uint32_t)r;
}

static int bn_cmp(const uint32_t* a, const uint32_t* b, size_t L) {
    for (size_t i = L; i-- > 0;) {
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    }
    return 0;
}

static uint32_t bn_sub(uint32_t* a, const uint32_t* b, size_t L) {
    uint64_t borrow = 0;
    for (size_t i = 0; i < L; ++i) {
        const uint64_t t = (uint64_t)a[i] - b[i] - borrow;
        a[i] = (uint32_t)t;
        borrow = (t >> 63) & 1;
    }
    return (uint32_t)borrow;
}

/* acc += x * s (acc has L limbs; x has Lx <= L limbs). */
static void bn_addmul_small(uint32_t* acc, size_t L, const uint32_t* x, size_t Lx, uint32_t s) {
    uint64_t carry = 0;
    for (size_t i = 0; i < L; ++i) {
        const uint64_t xi = i < Lx ? x[i] : 0;
        const uint64_t t = (uint64_t)acc[i] + xi * s + carry;
        acc[i] = (uint32_t)t;
        carry = t >> 32;
        if (i >= Lx && carry == 0) break;
    }
}

/* acc (La limbs) += a (L) * b (L). */
static void bn_addmul(uint32_t* acc, size_t La, const uint32_t* a, const uint32_t* b, size_t L) {
    for (size_t i = 0; i < L; ++i) {
        if (a[i] == 0) continue;
        uint64_t carry = 0;
        size_t j = 0;
        for (; j < L; ++j) {
            const uint64_t t = (uint64_t)acc[i + j] + (uint64_t)a[i] * b[j] + carry;
            acc[i + j] = (uint32_t)t;
            carry = t >> 32;
        }
        for (size_t t = i + j; carry && t < La; ++t) {
            const uint64_t s = (uint64_t)acc[t] + carry;
            acc[t] = (uint32_t)s;
            carry = s >> 32;
        }
    }
}

/* r (LQ limbs) = x (Lx limbs) mod Q (LQ limbs) by binary long division. */
static void bn_mod(const uint32_t* x, size_t Lx, const uint32_t* Q, size_t LQ, uint32_t* r) {
    uint32_t cur[BN_MAX + 1];
    memset(cur, 0, sizeof(cur));
    for (size_t bit = Lx * 32; bit-- > 0;) {
        /* cur = 2 cur + bit */
        uint32_t c = (x[bit / 32] >> (bit % 32)) & 1u;
        for (size_t i = 0; i <= LQ; ++i) {
            const uint32_t nc = cur[i] >> 31;
            cur[i] = (cur[i] << 1) | c;
            c = nc;
        }
        uint32_t qx[BN_MAX + 1];
        memcpy(qx, Q, LQ * sizeof(uint32_t));
        qx[LQ] = 0;
        if (bn_cmp(cur, qx, LQ + 1) >= 0) bn_sub(cur, qx, LQ + 1);
    }
    memcpy(r, cur, LQ * sizeof(uint32_t));
}

static size_t basis_Q_limbs(const uint32_t* primes, const uint32_t* exps, size_t n, uint32_t* Q) {
    memset(Q, 0, BN_MAX * sizeof(uint32_t));
    Q[0] = 1;
    for (size_t i = 0; i < n; ++i) {
        for (uint32_t e = 0; e < exps[i]; ++e) {
            uint32_t tmp[BN_MAX] = {0};
            bn_addmul_small(tmp, BN_MAX, Q, BN_MAX, primes[i]);
            memcpy(Q, tmp, sizeof(tmp));
        }
    }
    size_t L = BN_MAX;
    while (L > 1 && Q[L - 1] == 0) --L;
    return L;
}

static size_t bn_byte_width(const uint32_t* x, size_t L) {
    size_t bits = 0;
    for (size_t i = L; i-- > 0;) {
        if (x[i]) {
            uint32_t v = x[i];
            size_t b = 0;
            while (v) {
                ++b;
                v >>= 1;
            }
            bits = i * 32 + b;
            break;
        }
    }
    return bits ? (bits + 7) / 8 : 1;
}

size_t orc_basis_Q_bytes(const uint32_t* primes, const uint32_t* exps, size_t n, uint8_t* out,
                         size_t cap) {
    uint32_t Q[BN_MAX];
    const size_t L = basis_Q_limbs(primes, exps, n, Q);
    const size_t w = bn_byte_width(Q, L);
    if (out) bn_to_le(Q, L, out, w < cap ? w : cap);
    return w;
}

/* ---------------------------------------------------------------------------
 * Digits and small GEMMs — modmat.cpp:86-160
 * ------------------------------------------------------------------------- */

/* digit_decompose (modmat.cpp:86-106). */
int orc_digit_decompose(const int32_t* m, size_t count, uint32_t p, int32_t* d0, int32_t* d1) {
    if (p >= 256) return IRL_ERR_MODULUS_TOO_LARGE; /* :87 */
    const int32_t psq = (int32_t)(p * p);
    const int32_t half = (int32_t)((p - 1) / 2);
    for (size_t i = 0; i < count; ++i) {
        int32_t v = m[i] % psq;
        if (v < 0) v += psq;
        int32_t a = v % (int32_t)p;
        if (a > half) a -= (int32_t)p;
        int32_t b = ((v - a) / (int32_t)p) % (int32_t)p;
        if (b > half) b -= (int32_t)p;
        d0[i] = a;
        d1[i] = b;
    }
    return IRL_OK;
}

/* digit_recompose (modmat.cpp:108-118). */
void orc_digit_recompose(const int32_t* d0, const int32_t* d1, size_t count, uint32_t p,
                         int32_t* out) {
    const int32_t pp = (int32_t)p, psq = pp * pp;
    for (size_t i = 0; i < count; ++i) {
        int32_t v = (d0[i] + pp * d1[i]) % psq;
        if (v < 0) v += psq;
        out[i] = v;
    }
}

static int64_t max_abs(const int32_t* x, size_t n) {
    int64_t m = 0;
    for (size_t i = 0; i < n; ++i) {
        const int64_t v = x[i] < 0 ? -(int64_t)x[i] : x[i];
        if (v > m) m = v;
    }
    return m;
}

/* small_gemm (modmat.cpp:120-141): precheck, then i-k-j int32 accumulation
 * (wrap-free by the precheck). */
int orc_small_gemm(const int32_t* a, const int32_t* b, int32_t* c, size_t m, size_t k, size_t n,
                   int64_t* bound) {
    const int64_t bnd = (int64_t)k * max_abs(a, m * k) * max_abs(b, k * n);
    if (bound) *bound = bnd;
    if (bnd >= ((int64_t)1 << 31)) return IRL_ERR_ACCUMULATION_OVERFLOW_RISK;
    memset(c, 0, m * n * sizeof(int32_t));
    for (size_t i = 0; i < m; ++i) {
        int32_t* crow = c + i * n;
        for (size_t kk = 0; kk < k; ++kk) {
            const int32_t aik = a[i * k + kk];
            if (aik == 0) continue;
            const int32_t* brow = b + kk * n;
            for (size_t j = 0; j < n; ++j) crow[j] += aik * brow[j];
        }
    }
    return IRL_OK;
}

/* gemm_mod_psq (modmat.cpp:143-160): A0B0, A0B1, A1B0 then
 * (t00 + p (t01 + t10)) mod p^2 in int64. */
int orc_gemm_mod_psq(const int32_t* a, const int32_t* b, int32_t* c, size_t m, size_t k, size_t n,
                     uint32_t p) {
    int st = IRL_OK;
    int32_t *a0 = malloc(m * k * 4 + 1), *a1 = malloc(m * k * 4 + 1);
    int32_t *b0 = malloc(k * n * 4 + 1), *b1 = malloc(k * n * 4 + 1);
    int32_t *t00 = malloc(m * n * 4 + 1), *t01 = malloc(m * n * 4 + 1), *t10 = malloc(m * n * 4 + 1);
    if ((st = orc_digit_decompose(a, m * k, p, a0, a1)) != IRL_OK) goto done;
    if ((st = orc_digit_decompose(b, k * n, p, b0, b1)) != IRL_OK) goto done;
    if ((st = orc_small_gemm(a0, b0, t00, m, k, n, NULL)) != IRL_OK) goto done;
    if ((st = orc_small_gemm(a0, b1, t01, m, k, n, NULL)) != IRL_OK) goto done;
    if ((st = orc_small_gemm(a1, b0, t10, m, k, n, NULL)) != IRL_OK) goto done;
    {
        const int64_t psq = (int64_t)p * p;
        for (size_t i = 0; i < m * n; ++i) {
            int64_t v = ((int64_t)t00[i] + (int64_t)p * ((int64_t)t01[i] + t10[i])) % psq;
            if (v < 0) v += psq;
            c[i] = (int32_t)v;
        }
    }
done:
    free(a0);
    free(a1);
    free(b0);
    free(b1);
    free(t00);
    free(t01);
    free(t10);
    return st;
}

/* ---------------------------------------------------------------------------
 * mod-Q path — modmat.cpp:162-212
 * ------------------------------------------------------------------------- */

static uint32_t inv_mod(uint32_t a, uint32_t m, int* ok) {
    int64_t t = 0, nt = 1, r = m, nr = a % m;
    while (nr) {
        const int64_t q = r / nr, tt = t - q * nt, rr = r - q * nr;
        t = nt;
        nt = tt;
        r = nr;
        nr = rr;
    }
    *ok = (r == 1) || (m == 1);
    if (t < 0) t += m;
    return (uint32_t)t;
}

/* gemm_mod_Q (modmat.cpp:162-195): per modulus (in basis order) residues
 * via x mod m (:168-176), gemm_mod_psq or small_gemm (:177-178), CRT lift
 * c += (Q/m) * ((Q/m)^-1 r mod m) (:180-191), final reduce (:193). */
int orc_gemm_mod_Q(const uint8_t* a, const uint8_t* b, uint8_t* c, size_t m, size_t k, size_t n,
                   size_t width, const uint32_t* primes, const uint32_t* exps, size_t nmod) {
    uint32_t Q[BN_MAX];
    const size_t LQ = basis_Q_limbs(primes, exps, nmod, Q);
    const size_t Lw = (width + 3) / 4 > LQ ? (width + 3) / 4 : LQ;
    const size_t Lc = LQ + 2;
    int st = IRL_OK;
    uint32_t* A = calloc(m * k * Lw + 1, 4);
    uint32_t* B = calloc(k * n * Lw + 1, 4);
    uint32_t* C = calloc(m * n * Lc + 1, 4);
    int32_t* ra = malloc(m * k * 4 + 1);
    int32_t* rb = malloc(k * n * 4 + 1);
    int32_t* rc = malloc(m * n * 4 + 1);
    for (size_t i = 0; i < m * k; ++i) bn_from_le(a + i * width, width, A + i * Lw, Lw);
    for (size_t i = 0; i < k * n; ++i) bn_from_le(b + i * width, width, B + i * Lw, Lw);
    for (size_t t = 0; t < nmod; ++t) {
        const uint32_t mod = exps[t] == 2 ? primes[t] * primes[t] : primes[t];
        for (size_t i = 0; i < m * k; ++i) ra[i] = (int32_t)bn_mod_small(A + i * Lw, Lw, mod);
        for (size_t i = 0; i < k * n; ++i) rb[i] = (int32_t)bn_mod_small(B + i * Lw, Lw, mod);
        st = exps[t] == 2 ? orc_gemm_mod_psq(ra, rb, rc, m, k, n, primes[t])
                          : orc_small_gemm(ra, rb, rc, m, k, n, NULL);
        if (st != IRL_OK) goto done;
        uint32_t qi[BN_MAX];
        memcpy(qi, Q, sizeof(qi));
        bn_divmod_small(qi, LQ, mod);
        int ok = 0;
        const uint32_t inv = inv_mod(bn_mod_small(qi, LQ, mod), mod, &ok);
        if (!ok) {
            st = IRL_ERR_NOT_COPRIME;
            goto done;
        }
        for (size_t i = 0; i < m * n; ++i) {
            uint64_t r = (uint64_t)(uint32_t)rc[i] % mod;
            r = (r * inv) % mod;
            bn_addmul_small(C + i * Lc, Lc, qi, LQ, (uint32_t)r);
        }
    }
    for (size_t i = 0; i < m * n; ++i) {
        uint32_t r[BN_MAX];
        bn_mod(C + i * Lc, Lc, Q, LQ, r);
        bn_to_le(r, LQ, c + i * width, width);
    }
done:
    free(A);
    free(B);
    free(C);
    free(ra);
    free(rb);
    free(rc);
    return st;
}

/* oracle_gemm_mod_Q (modmat.cpp:197-212): schoolbook sum then mod Q. */
int orc_oracle_gemm_mod_Q(const uint8_t* a, const uint8_t* b, uint8_t* c, size_t m, size_t k,
                          size_t n, size_t width, const uint32_t* primes, const uint32_t* exps,
                          size_t nmod) {
    uint32_t Q[BN_MAX];
    const size_t LQ = basis_Q_limbs(primes, exps, nmod, Q);
    const size_t Lw = (width + 3) / 4 > LQ ? (width + 3) / 4 : LQ;
    const size_t La = 2 * Lw + 2;
    if (La > BN_MAX) return IRL_ERR_INVALID_ARGUMENT;
    uint32_t* A = calloc(m * k * Lw + 1, 4);
    uint32_t* B = calloc(k * n * Lw + 1, 4);
    for (size_t i = 0; i < m * k; ++i) bn_from_le(a + i * width, width, A + i * Lw, Lw);
    for (size_t i = 0; i < k * n; ++i) bn_from_le(b + i * width, width, B + i * Lw, Lw);
    for (size_t i = 0; i < m; ++i) {
        for (size_t j = 0; j < n; ++j) {
            uint32_t acc[BN_MAX];
            memset(acc, 0, sizeof(acc));
            for (size_t kk = 0; kk < k; ++kk) bn_addmul(acc, La, A + (i * k + kk) * Lw, B + (kk * n + j) * Lw, Lw);
            uint32_t r[BN_MAX];
            bn_mod(acc, La, Q, LQ, r);
            bn_to_le(r, LQ, c + (i * n + j) * width, width);
        }
    }
    free(A);
    free(B);
    return IRL_OK;
}

/* ---------------------------------------------------------------------------
 * PPMM over residues (CCMM building block)
 * ------------------------------------------------------------------------- */

struct ppmm_job {
    const uint16_t *a, *bt;
    size_t lda, ldb, nrows, N, K;
    const uint32_t* rows;
    uint32_t m;
    uint16_t* out;
    size_t next; /* shared work counter (guarded by mu) */
    pthread_mutex_t mu;
};

static void* ppmm_worker(void* arg) {
    struct ppmm_job* j = (struct ppmm_job*)arg;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        const size_t ri = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (ri >= j->nrows) break;
        const uint16_t* ar = j->a + (size_t)j->rows[ri] * j->lda;
        for (size_t nn = 0; nn < j->N; ++nn) {
            const uint16_t* br = j->bt + nn * j->ldb;
            uint64_t acc = 0;
            for (size_t kk = 0; kk < j->K; ++kk) acc += (uint64_t)ar[kk] * br[kk];
            j->out[ri * j->N + nn] = (uint16_t)(acc % j->m);
        }
    }
    return NULL;
}

/* Schoolbook: every product < 2^32, K < 2^31 terms fit uint64. Rows are
 * spread over the host cores with pthreads. */
void orc_ppmm_rows_direct(const uint16_t* a, size_t lda, const uint16_t* bt, size_t ldb,
                          const uint32_t* rows, size_t nrows, size_t N, size_t K, uint32_t m,
                          uint16_t* out) {
    struct ppmm_job j = {a, bt, lda, ldb, nrows, N, K, rows, m, out, 0, PTHREAD_MUTEX_INITIALIZER};
    long nt = sysconf(_SC_NPROCESSORS_ONLN);
    if (nt < 1) nt = 1;
    if ((size_t)nt > nrows) nt = (long)(nrows ? nrows : 1);
    pthread_t th[256];
    if (nt > 256) nt = 256;
    for (long t = 0; t < nt; ++t) pthread_create(&th[t], NULL, ppmm_worker, &j);
    for (long t = 0; t < nt; ++t) pthread_join(th[t], NULL);
}

/* ---------------------------------------------------------------------------
 * Counter-based synthetic residues
 * ------------------------------------------------------------------------- */

static uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint32_t orc_synth_residue(uint64_t seed, uint32_t stream, uint32_t plane, uint32_t row,
                           uint32_t col, uint32_t m) {
    const uint64_t key = ((uint64_t)(stream & 0xFF) << 56) | ((uint64_t)(plane & 0xFF) << 48) |
                         ((uint64_t)(row & 0xFFFFFF) << 24) | (uint64_t)(col & 0xFFFFFF);
    const uint64_t x = mix64(key ^ mix64(seed));
    return (uint32_t)(((x >> 32) * (uint64_t)m) >> 32);
}

/* emulator.cpp:411-421 (built with -ffp-contract=off, like the reference's
 * baseline x86-64 build: a * q and the += round separately). */
void orc_ccmm_twin_product(const double* db, const double* qry, size_t d1, size_t d2, size_t d3, double* out) {
    double* prow = (double*)malloc((d3 ? d3 : 1) * sizeof(double));
    for (size_t i = 0; i < d1; ++i) {
        for (size_t j = 0; j < d3; ++j) prow[j] = 0.0;
        for (size_t k = 0; k < d2; ++k) {
            const double a = db[i * d2 + k];
            if (a == 0.0) continue;
            const double* qrow = qry + k * d3;
            for (size_t j = 0; j < d3; ++j) prow[j] += a * qrow[j];
        }
        for (size_t j = 0; j < d3; ++j) out[j * d1 + i] = prow[j];
    }
    free(prow);
}

void orc_synth_block(uint64_t seed, uint32_t stream, uint32_t plane, uint32_t row0,
                     uint32_t nrows, uint32_t col0, uint32_t ncols, uint32_t m, uint16_t* out) {
    for (uint32_t r = 0; r < nrows; ++r)
        for (uint32_t c = 0; c < ncols; ++c)
            out[(size_t)r * ncols + c] =
                (uint16_t)orc_synth_residue(seed, stream, plane, row0 + r, col0 + c, m);
}

/* ---- plaintext iris scoring ------------------------------------------------
 * inner_and_overlap (iris_core.cpp:37-51): av = m - 2 (c & m) per entry
 * (to_masked, :28-35), inner = sum av*bv, overlap = sum (m_a & m_b) =
 * overlap_count of the packed masks (pipeline.cpp:78-82). The query column
 * c = e*rho + r is rotate(q_e, r) (iris_core.cpp:65-76): out[(i + r) % d] =
 * t[i], i.e. entry k of the rotated template is t[(k - r) mod d]. */
void orc_iris_inner_overlap(const uint8_t* db_code, const uint8_t* db_mask, size_t n_db, const uint8_t* q_code,
                            const uint8_t* q_mask, size_t n_eyes, size_t rho, size_t d, int32_t* inner,
                            int32_t* overlap) {
    for (size_t e = 0; e < n_eyes; ++e)
        for (size_t r = 0; r < rho; ++r) {
            const size_t c = e * rho + r, rr = d ? r % d : 0;
            for (size_t j = 0; j < n_db; ++j) {
                long in = 0, ov = 0;
                const uint8_t* ac = db_code + j * d;
                const uint8_t* am = db_mask + j * d;
                for (size_t k = 0; k < d; ++k) {
                    const size_t i = k >= rr ? k - rr : k + d - rr;
                    const int bc = q_code[e * d + i], bm = q_mask[e * d + i];
                    const int av = am[k] - 2 * (ac[k] & am[k]);
                    const int bv = bm - 2 * (bc & bm);
                    in += av * bv;
                    ov += am[k] & bm;
                }
                inner[c * n_db + j] = (int32_t)in;
                overlap[c * n_db + j] = (int32_t)ov;
            }
        }
}

/* ---- Alg. 2 fold stage ------------------------------------------------------ */

/* Polynomial::degree (poly.cpp:10-15): index of the last nonzero coefficient */
static int orc_poly_degree(const double* c, size_t n) {
    for (size_t i = n; i-- > 0;)
        if (c[i] != 0.0) return (int)i;
    return 0;
}

/* CtRing::axpb (pipeline.cpp:41-43): pmult_const(x, a), then add_const(b) */
static double orc_axpb(double a, double x, double b) {
    const double t = x * a;
    return t + b;
}

/* detail::ps_eval_range (poly.hpp:62-86) */
static double orc_ps_range(const double* c, size_t lo, size_t hi, const double* baby, const double* giant,
                           size_t m) {
    const size_t n = hi - lo;
    if (n <= m) {
        double acc = orc_axpb(0.0, baby[0], c[lo]);
        for (size_t i = 1; i < n; ++i) acc = acc + orc_axpb(c[lo + i], baby[i - 1], 0.0);
        return acc;
    }
    size_t split = m, g = 0;
    while (split * 2 < n) {
        split *= 2;
        ++g;
    }
    const double low = orc_ps_range(c, lo, lo + split, baby, giant, m);
    const double high = orc_ps_range(c, lo + split, hi, baby, giant, m);
    return high * giant[g] + low;
}

/* ps_execute (poly.hpp:91-119) */
double orc_ps_execute(const double* coeffs, size_t n, double x) {
    const int d = orc_poly_degree(coeffs, n);
    double c[64];
    if (d >= 64) return NAN;
    for (int i = 0; i <= d; ++i) c[i] = (size_t)i < n ? coeffs[i] : 0.0;
    if (d == 0) return orc_axpb(0.0, x, c[0]);
    int k = 0; /* ps_depth (poly.hpp:50-54) */
    while ((1 << k) < d + 1) ++k;
    const size_t m = (size_t)1 << ((k + 1) / 2); /* ps_baby_m */
    double baby[64], giant[8];
    baby[0] = x;
    const size_t nb = m < (size_t)d ? m : (size_t)d;
    for (size_t j = 2; j <= nb; ++j) baby[j - 1] = baby[(j + 1) / 2 - 1] * baby[j / 2 - 1];
    size_t ng = 0;
    if ((size_t)d + 1 > m) {
        giant[ng++] = baby[m - 1];
        size_t pw = m;
        while (pw * 2 < (size_t)d + 1) {
            giant[ng] = giant[ng - 1] * giant[ng - 1];
            ++ng;
            pw *= 2;
        }
    }
    return orc_ps_range(c, 0, (size_t)d + 1, baby, giant, m);
}

int orc_fold_stage(size_t batch, size_t rho, size_t n_db, size_t d, size_t fold_k, const double* fold_c,
                   size_t fold_len, size_t nstages, const double* centers, const size_t* lens,
                   const double* chain_c, double neg_lo, double neg_hi, const int32_t* inner,
                   const int32_t* overlap, double* folded, double* refolded, int32_t* assumption_ok) {
    /* PipelineConfig::validate (pipeline.cpp:232-243) */
    if (rho < 1 || batch < 1) return IRL_ERR_CONFIG;
    if (fold_k < 1 || fold_k > rho) return IRL_ERR_CONFIG;
    if (d < 2 || (d & (d - 1)) != 0) return IRL_ERR_CONFIG;
    if (n_db < d || n_db % d != 0) return IRL_ERR_CONFIG;
    if (refolded && nstages == 0) return IRL_ERR_CONFIG; /* eval_chain_ct: empty chain */
    const size_t blocks = n_db / d, groups = (rho + fold_k - 1) / fold_k;
    int ok = 1, empty = 0;
    double* t = (double*)malloc(d * sizeof(double));
    double* acc = (double*)malloc(d * sizeof(double));
    double* refold = (double*)malloc(d * sizeof(double));
    for (size_t e = 0; e < batch; ++e)
        for (size_t b = 0; b < blocks; ++b) {
            for (size_t g = 0; g < groups; ++g) {
                const size_t r_end = (g + 1) * fold_k < rho ? (g + 1) * fold_k : rho;
                /* folding-assumption shadow check (pipeline.cpp:565-590) */
                for (size_t i = 0; i < d; ++i) {
                    int non_d = 0;
                    for (size_t r = g * fold_k; r < r_end; ++r) {
                        const size_t j = (i + r) % d, off = (e * rho + r) * n_db + b * d + j;
                        const double raw = (double)inner[off], ov = (double)overlap[off];
                        if (ov == 0.0 || !(raw / ov >= neg_lo && raw / ov <= neg_hi)) ++non_d;
                    }
                    if (non_d > 1) ok = 0;
                }
                /* fold_group(normalize(scored[idx]) for the group's r) (pipeline.cpp:391-408) */
                for (size_t r = g * fold_k; r < r_end; ++r) {
                    const size_t row = (e * rho + r) * n_db + b * d;
                    for (size_t j = 0; j < d; ++j) {
                        const double ov = (double)overlap[row + j];
                        if (ov == 0.0) empty = 1;
                        const double inv = 1.0 / ov; /* normalize (pipeline.cpp:364-369) */
                        t[j] = orc_ps_execute(fold_c, fold_len, (double)inner[row + j] * inv);
                    }
                    for (size_t i = 0; i < d; ++i) { /* rot by r (emulator.cpp:232-245), then add */
                        const double v = t[(i + r) % d];
                        acc[i] = r == g * fold_k ? v : acc[i] + v;
                    }
                }
                if (folded) memcpy(folded + ((e * blocks + b) * groups + g) * d, acc, d * sizeof(double));
                if (refolded) {
                    for (size_t i = 0; i < d; ++i) {
                        double cls = acc[i];
                        size_t off = 0;
                        for (size_t s = 0; s < nstages; ++s) { /* eval_chain_ct (pipeline.cpp:379-389) */
                            cls = orc_ps_execute(chain_c + off, lens[s], cls + -centers[s]);
                            off += lens[s];
                        }
                        refold[i] = g == 0 ? cls : refold[i] + cls;
                    }
                }
            }
            if (refolded) memcpy(refolded + (e * blocks + b) * d, refold, d * sizeof(double));
        }
    free(t);
    free(acc);
    free(refold);
    if (assumption_ok) *assumption_ok = ok;
    return empty ? IRL_ERR_ZERO_OVERLAP : IRL_OK;
}
