// extern "C" wrappers around the UNMODIFIED reference hot path
// (/root/reference/proj/src/modmat.cpp, iris_core.cpp, and for the Alg. 2
// fold stage emulator.cpp, pipeline.cpp, poly.cpp), compiled together
// into oracle/_ref/libirl_ref.so by oracle/Makefile. TEST INFRASTRUCTURE:
// used by tests/ (parity pinning, golden-vector generation) and by bench.py's
// CPU-baseline / --impl reference leg. Never linked by the product.
//
// Big matrices cross this boundary as fixed-width little-endian entries
// (the reference's own file format, modmat.cpp:216-231).
#include <cstdint>
#include <atomic>
#include <cstring>
#include <exception>
#include <limits>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "irislab/errors.hpp"
#include "irislab/iris_core.hpp"
#include "irislab/modmat.hpp"
#include "irislab/pipeline.hpp"

using namespace irislab;
using modmat::BigMatrix;
using modmat::SmallMatrix;

namespace {

thread_local std::string g_err;

int map_exception() {
    try {
        throw;
    } catch (const ShapeMismatch& e) {
        g_err = e.what();
        return 1;
    } catch (const ModulusTooLarge& e) {
        g_err = e.what();
        return 2;
    } catch (const AccumulationOverflowRisk& e) {
        g_err = e.what();
        return 3;
    } catch (const ModulusBudget& e) {
        g_err = e.what();
        return 5;
    } catch (const ZeroOverlap& e) {
        g_err = e.what();
        return 11;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 13;
    } catch (const Error& e) {
        g_err = e.what();
        return std::string(e.what()).find("coprime") != std::string::npos ? 4 : 6;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 6;
    }
}

SmallMatrix to_small(const int32_t* p, size_t r, size_t c) {
    SmallMatrix m{r, c, std::vector<int32_t>(r * c)};
    if (r * c) std::memcpy(m.a.data(), p, r * c * 4);
    return m;
}

void to_big(BigMatrix& m, const uint8_t* p, size_t width) {
    for (size_t i = 0; i < m.a.size(); ++i)
        mpz_import(m.a[i].get_mpz_t(), width, -1, 1, -1, 0, p + i * width);
}

void from_big(const BigMatrix& m, uint8_t* p, size_t width) {
    for (size_t i = 0; i < m.a.size(); ++i) {
        std::memset(p + i * width, 0, width);
        size_t count = 0;
        mpz_export(p + i * width, &count, -1, 1, -1, 0, m.a[i].get_mpz_t());
    }
}

modmat::RnsBasis make_basis(const uint32_t* primes, const uint32_t* exps, size_t n) {
    modmat::RnsBasis b;
    b.Q = 1;
    for (size_t i = 0; i < n; ++i) {
        b.moduli.push_back({primes[i], exps[i]});
        b.Q *= mpz_class(b.moduli.back().value());
    }
    return b;
}

// Acceptance criterion 2 stream (acceptance.cpp:96-120), replayed.
struct Crit2 {
    modmat::RnsBasis basis = modmat::build_paper_basis();
    gmp_randclass rng{gmp_randinit_default};
    std::mt19937_64 dims{2};
    std::uniform_int_distribution<int> dim{1, 64};
    Crit2() { rng.seed(2); }
};
Crit2* g_crit2 = nullptr;

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

size_t ref_paper_basis(uint32_t* primes, uint32_t* exps, size_t cap) {
    auto b = modmat::build_paper_basis();
    for (size_t i = 0; i < b.moduli.size() && i < cap; ++i) {
        primes[i] = b.moduli[i].p;
        exps[i] = b.moduli[i].e;
    }
    return b.moduli.size();
}
size_t ref_digit_planes() { return modmat::build_paper_basis().digit_planes(); }
double ref_log2_Q() { return modmat::build_paper_basis().log2_Q(); }
double ref_max_int8_rns_capacity() { return modmat::max_int8_rns_capacity(); }
size_t ref_pure_rns_plane_count() { return modmat::pure_rns_plane_count(); }
size_t ref_paper_Q_bytes(uint8_t* out, size_t cap) {
    auto b = modmat::build_paper_basis();
    const size_t w = (mpz_sizeinbase(b.Q.get_mpz_t(), 2) + 7) / 8;
    if (out && cap >= w) {
        size_t count = 0;
        std::memset(out, 0, w);
        mpz_export(out, &count, -1, 1, -1, 0, b.Q.get_mpz_t());
    }
    return w;
}

int ref_digit_decompose(const int32_t* m, size_t rows, size_t cols, uint32_t p, int32_t* d0,
                        int32_t* d1) {
    try {
        auto d = modmat::digit_decompose(to_small(m, rows, cols), p);
        if (rows * cols) {
            std::memcpy(d0, d.m0.a.data(), rows * cols * 4);
            std::memcpy(d1, d.m1.a.data(), rows * cols * 4);
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ref_digit_recompose(const int32_t* d0, const int32_t* d1, size_t rows, size_t cols,
                        uint32_t p, int32_t* out) {
    try {
        modmat::DigitMatrices d{p, to_small(d0, rows, cols), to_small(d1, rows, cols)};
        auto m = modmat::digit_recompose(d);
        if (rows * cols) std::memcpy(out, m.a.data(), rows * cols * 4);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ref_small_gemm(const int32_t* a, const int32_t* b, int32_t* c, size_t m, size_t k, size_t n) {
    try {
        auto r = modmat::small_gemm(to_small(a, m, k), to_small(b, k, n));
        if (m * n) std::memcpy(c, r.a.data(), m * n * 4);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ref_gemm_mod_psq(const int32_t* a, const int32_t* b, int32_t* c, size_t m, size_t k, size_t n,
                     uint32_t p) {
    try {
        auto r = modmat::gemm_mod_psq(to_small(a, m, k), to_small(b, k, n), p);
        if (m * n) std::memcpy(c, r.a.data(), m * n * 4);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// Multi-threaded driver for the CPU baseline: independent gemm_mod_psq calls
// (one per task), each task = (a_i, b_i, c_i, p_i); the function is pure
// (SPEC.md:214-215), so tasks run on `threads` host threads.
int ref_gemm_mod_psq_batch(const int32_t* const* a, const int32_t* const* b, int32_t* const* c,
                           const uint32_t* p, size_t ntasks, size_t m, size_t k, size_t n,
                           int threads) {
    std::vector<int> st(ntasks, 0);
    std::vector<std::thread> pool;
    std::atomic<size_t> next{0};
    const int nt = threads > 0 ? threads : 1;
    for (int t = 0; t < nt; ++t) {
        pool.emplace_back([&] {
            for (size_t i; (i = next.fetch_add(1)) < ntasks;) {
                st[i] = ref_gemm_mod_psq(a[i], b[i], c[i], m, k, n, p[i]);
            }
        });
    }
    for (auto& th : pool) th.join();
    for (int s : st)
        if (s) return s;
    return 0;
}

int ref_gemm_mod_Q(const uint8_t* a, const uint8_t* b, uint8_t* c, size_t m, size_t k, size_t n,
                   size_t width, const uint32_t* primes, const uint32_t* exps, size_t nmod) {
    try {
        auto basis = make_basis(primes, exps, nmod);
        BigMatrix A = BigMatrix::zeros(m, k), B = BigMatrix::zeros(k, n);
        to_big(A, a, width);
        to_big(B, b, width);
        auto C = modmat::gemm_mod_Q(A, B, basis);
        from_big(C, c, width);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ref_oracle_gemm_mod_Q(const uint8_t* a, const uint8_t* b, uint8_t* c, size_t m, size_t k,
                          size_t n, size_t width, const uint32_t* primes, const uint32_t* exps,
                          size_t nmod) {
    try {
        auto basis = make_basis(primes, exps, nmod);
        BigMatrix A = BigMatrix::zeros(m, k), B = BigMatrix::zeros(k, n);
        to_big(A, a, width);
        to_big(B, b, width);
        auto C = modmat::oracle_gemm_mod_Q(A, B, basis.Q);
        from_big(C, c, width);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// Replays acceptance criterion 2's input stream. ref_crit2_reset() then
// repeated ref_crit2_next(): writes dims, then (if buffers are large enough:
// 64*64*width each) the entries of A (m x k) and B (k x n).
void ref_crit2_reset() {
    delete g_crit2;
    g_crit2 = new Crit2();
}
int ref_crit2_next(size_t* m, size_t* k, size_t* n, uint8_t* a, uint8_t* b, size_t width) {
    if (!g_crit2) ref_crit2_reset();
    Crit2& s = *g_crit2;
    *m = static_cast<size_t>(s.dim(s.dims));
    *k = static_cast<size_t>(s.dim(s.dims));
    *n = static_cast<size_t>(s.dim(s.dims));
    BigMatrix A = BigMatrix::zeros(*m, *k), B = BigMatrix::zeros(*k, *n);
    for (auto& v : A.a) v = s.rng.get_z_range(s.basis.Q);
    for (auto& v : B.a) v = s.rng.get_z_range(s.basis.Q);
    from_big(A, a, width);
    from_big(B, b, width);
    return 0;
}

// test_modmat.cpp:12-22 random_big with mt19937_64(seed): rows*cols entries.
void ref_random_big(uint64_t seed, size_t skip, size_t rows, size_t cols, uint8_t* out,
                    size_t width) {
    auto basis = modmat::build_paper_basis();
    std::mt19937_64 rng(seed);
    for (size_t s = 0; s < skip; ++s) rng();
    BigMatrix m = BigMatrix::zeros(rows, cols);
    for (auto& v : m.a) {
        mpz_class x = 0;
        for (int w = 0; w < 6; ++w)
            x = (x << 32) + static_cast<unsigned long>(rng() & 0xffffffffULL);
        v = x % basis.Q;
    }
    from_big(m, out, width);
}

int ref_save_load_roundtrip(const char* path, const uint8_t* entries, size_t rows, size_t cols,
                            size_t width, uint8_t* back) {
    try {
        auto basis = modmat::build_paper_basis();
        BigMatrix m = BigMatrix::zeros(rows, cols);
        to_big(m, entries, width);
        modmat::save_big_matrix(path, m, basis.Q);
        mpz_class q;
        auto r = modmat::load_big_matrix(path, &q);
        from_big(r, back, width);
        return q == basis.Q ? 0 : 6;
    } catch (...) {
        return map_exception();
    }
}

// iris_core.cpp:92-112 synth_db + :28-35 to_masked: ternary values
// out[t*d + i] in {-1, 0, 1} for n templates of dimension d.
int ref_synth_masked(size_t n, size_t d, double mask_density, uint64_t seed, int8_t* out) {
    try {
        auto db = iris::synth_db(n, d, mask_density, seed);
        for (size_t t = 0; t < n; ++t) {
            auto mv = iris::to_masked(db[t]);
            std::memcpy(out + t * d, mv.values.data(), d);
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// iris_core.cpp:65-76 rotate followed by to_masked.
int ref_synth_masked_rotated(size_t n, size_t d, double mask_density, uint64_t seed, size_t rot,
                             int8_t* out) {
    try {
        auto db = iris::synth_db(n, d, mask_density, seed);
        for (size_t t = 0; t < n; ++t) {
            auto mv = iris::to_masked(iris::rotate(db[t], rot));
            std::memcpy(out + t * d, mv.values.data(), d);
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// Raw synth_db templates (iris_core.cpp:92-112): code / mask bits [n][d].
int ref_synth_templates(size_t n, size_t d, double mask_density, uint64_t seed, uint8_t* code, uint8_t* mask) {
    try {
        auto db = iris::synth_db(n, d, mask_density, seed);
        for (size_t t = 0; t < n; ++t) {
            std::memcpy(code + t * d, db[t].code.data(), d);
            std::memcpy(mask + t * d, db[t].mask.data(), d);
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

namespace {
std::vector<iris::IrisTemplate> to_templates(const uint8_t* code, const uint8_t* mask, size_t n, size_t d) {
    std::vector<iris::IrisTemplate> ts(n);
    for (size_t t = 0; t < n; ++t) {
        ts[t].code.assign(code + t * d, code + (t + 1) * d);
        ts[t].mask.assign(mask + t * d, mask + (t + 1) * d);
    }
    return ts;
}
}  // namespace

// iris::score (iris_core.cpp:55-59) for every (query c, template j):
// out[c * n_db + j]; NaN where it throws ZeroOverlap. Returns 0.
int ref_iris_scores(const uint8_t* q_code, const uint8_t* q_mask, size_t nq, const uint8_t* db_code,
                    const uint8_t* db_mask, size_t n_db, size_t d, double* out) {
    try {
        auto q = to_templates(q_code, q_mask, nq, d);
        auto db = to_templates(db_code, db_mask, n_db, d);
        for (size_t c = 0; c < nq; ++c)
            for (size_t j = 0; j < n_db; ++j) {
                try {
                    out[c * n_db + j] = iris::score(q[c], db[j]);
                } catch (const ZeroOverlap&) {
                    out[c * n_db + j] = std::numeric_limits<double>::quiet_NaN();
                }
            }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// iris::rotate (iris_core.cpp:65-76) of one template.
void ref_iris_rotate(const uint8_t* code, const uint8_t* mask, size_t d, size_t r, uint8_t* out_code,
                     uint8_t* out_mask) {
    auto t = to_templates(code, mask, 1, d);
    auto o = iris::rotate(t[0], r);
    std::memcpy(out_code, o.code.data(), d);
    std::memcpy(out_mask, o.mask.data(), d);
}

// iris::save_templates (iris_core.cpp:183-196) of n templates [n][d].
int ref_save_templates(const char* path, const uint8_t* code, const uint8_t* mask, size_t n, size_t d) {
    try {
        iris::save_templates(path, to_templates(code, mask, n, d));
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// iris::match_db_reference (iris_core.cpp:78-90): *out = 0/1; status 11 on ZeroOverlap.
int ref_match_db_reference(const uint8_t* q_code, const uint8_t* q_mask, size_t nq, const uint8_t* db_code,
                           const uint8_t* db_mask, size_t n_db, size_t d, double n_lo, double n_hi,
                           double p_lo, double p_hi, int* out) {
    try {
        auto q = to_templates(q_code, q_mask, nq, d);
        auto db = to_templates(db_code, db_mask, n_db, d);
        *out = iris::match_db_reference(q, db, iris::Interval{n_lo, n_hi}, iris::Interval{p_lo, p_hi}) ? 1 : 0;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// Alg. 2 fold stage through the reference's own pipe::normalize,
// pipe::fold_group and pipe::eval_chain_ct on a noise-free emulator
// (Emulator(default_emulator_config()), inject_noise = false), in run_alg2's
// loop order (pipeline.cpp:594-627). The bootstrap between fold_group and the
// chain (boot(bts_fold_pre)) only moves levels, so it is left out. inner /
// overlap: int32 [batch*rho][n_db] (prepare's product and overlaps). The
// score ciphertexts enter at the top level, as CI slots of ring degree d.
int ref_fold_stage(size_t batch, size_t rho, size_t n_db, size_t d, size_t fold_k, const double* fold_c,
                   size_t fold_len, size_t nstages, const double* centers, const size_t* lens,
                   const double* chain_c, const int32_t* inner, const int32_t* overlap, double* folded,
                   double* refolded) {
    try {
        pipe::PipelineConfig cfg;
        cfg.rho = static_cast<int>(rho);
        cfg.batch = static_cast<int>(batch);
        cfg.n_db = static_cast<long>(n_db);
        cfg.d = static_cast<long>(d);
        cfg.fold_k = static_cast<int>(fold_k);
        cfg.emu_cfg = pipe::default_emulator_config();
        cfg.validate();
        emu::Emulator em(cfg.emu_cfg);
        const polydes::Polynomial fpoly(std::vector<double>(fold_c, fold_c + fold_len));
        polydes::ClassifierChain chain;
        size_t off = 0;
        for (size_t s = 0; s < nstages; ++s) {
            polydes::ClassifierChain::Stage st;
            st.poly = polydes::Polynomial(std::vector<double>(chain_c + off, chain_c + off + lens[s]));
            st.center = centers[s];
            chain.stages.push_back(st);
            off += lens[s];
        }
        int logn = 0;
        while ((size_t{1} << logn) < d) ++logn;
        const int top = cfg.emu_cfg.chain.top_level();
        const size_t blocks = n_db / d, groups = (rho + fold_k - 1) / fold_k;
        for (size_t e = 0; e < batch; ++e)
            for (size_t b = 0; b < blocks; ++b) {
                emu::EmulatedCiphertext refold;
                for (size_t g = 0; g < groups; ++g) {
                    std::vector<emu::EmulatedCiphertext> group;
                    const size_t r_end = std::min(rho, (g + 1) * fold_k);
                    for (size_t r = g * fold_k; r < r_end; ++r) {
                        const size_t row = (e * rho + r) * n_db + b * d;
                        std::vector<std::complex<double>> msg(d);
                        std::vector<double> ov(d);
                        for (size_t j = 0; j < d; ++j) {
                            msg[j] = {static_cast<double>(inner[row + j]), 0.0};
                            ov[j] = static_cast<double>(overlap[row + j]);
                        }
                        const auto ct = em.ecd(msg, emu::Encoding::Slot, true, logn, cfg.scale_bits, top);
                        group.push_back(pipe::normalize(em, ct, ov, cfg.scale_bits));
                    }
                    const auto f = pipe::fold_group(em, group, fpoly, cfg.scale_bits, static_cast<long>(g * fold_k));
                    if (folded)
                        for (size_t i = 0; i < d; ++i) folded[((e * blocks + b) * groups + g) * d + i] = f.message[i].real();
                    if (refolded) {
                        auto cls = pipe::eval_chain_ct(em, chain, f, cfg.scale_bits);
                        if (g == 0) {
                            refold = std::move(cls);
                        } else {
                            const int lv = std::min(refold.level, cls.level);
                            refold = em.add(em.mod_switch(refold, lv), em.mod_switch(cls, lv));
                        }
                    }
                }
                if (refolded)
                    for (size_t i = 0; i < d; ++i) refolded[(e * blocks + b) * d + i] = refold.message[i].real();
                em.clear_trace();
            }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// Emulator::ccmm_twin (emulator.cpp:389-447) itself, noise-free default
// emulator: msgs receives its outputs' real parts in output order
// (d1*d3/n_db ciphertexts of n_db slots). top_level = the chain's top level.
int ref_ccmm_twin(long d1, long d2, long d3, long n_db, long n_qry, double db_bits, double q_bits,
                  double scale_bits, int out_level, int out_slot, int out_ci, const double* db,
                  const double* qry, double* msgs, int* top_level) {
    try {
        emu::Emulator em(pipe::default_emulator_config());
        *top_level = em.config().chain.top_level();
        emu::CcmmSpec spec;
        spec.d1 = d1;
        spec.d2 = d2;
        spec.d3 = d3;
        spec.n_db = n_db;
        spec.n_qry = n_qry;
        spec.db_modulus_bits = db_bits;
        spec.qry_modulus_bits = q_bits;
        spec.scale_bits = scale_bits;
        spec.out_level = out_level;
        spec.out_encoding = out_slot ? emu::Encoding::Slot : emu::Encoding::Coeff;
        spec.out_ci = out_ci != 0;
        const std::vector<double> a(db, db + (d1 > 0 && d2 > 0 ? d1 * d2 : 0));
        const std::vector<double> b(qry, qry + (d2 > 0 && d3 > 0 ? d2 * d3 : 0));
        const auto out = em.ccmm_twin(spec, a, b);
        size_t k = 0;
        for (const auto& ct : out)
            for (const auto& m : ct.message) msgs[k++] = m.real();
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// ps_execute on scalars through the emulator's ring (one slot), for the
// polynomial unit checks.
int ref_ps_execute(const double* coeffs, size_t n, double x, double* out) {
    try {
        emu::Emulator em(pipe::default_emulator_config());
        const auto ct = em.ecd({{x, 0.0}, {0.0, 0.0}}, emu::Encoding::Slot, true, 1, 23.0, 24);
        polydes::ClassifierChain chain;
        polydes::ClassifierChain::Stage st;
        st.poly = polydes::Polynomial(std::vector<double>(coeffs, coeffs + n));
        chain.stages.push_back(st);
        *out = pipe::eval_chain_ct(em, chain, ct, 23.0).message[0].real();
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// run_alg2's folding-assumption flag (pipeline.cpp:565-590) from the
// reference's own run, on templates (prepare computes the products and
// overlaps). The fold chain is the caller's; the post chain is a fixed
// smooth step (the flag is computed before either is used).
int ref_alg2_assumption(const uint8_t* q_code, const uint8_t* q_mask, size_t batch, const uint8_t* db_code,
                        const uint8_t* db_mask, size_t n_db, size_t d, size_t rho, size_t fold_k,
                        const double* fold_c, size_t fold_len, size_t nstages, const double* centers,
                        const size_t* lens, const double* chain_c, double neg_lo, double neg_hi, int* ok) {
    try {
        pipe::PipelineConfig cfg;
        cfg.rho = static_cast<int>(rho);
        cfg.batch = static_cast<int>(batch);
        cfg.n_db = static_cast<long>(n_db);
        cfg.d = static_cast<long>(d);
        cfg.fold_k = static_cast<int>(fold_k);
        cfg.emu_cfg = pipe::default_emulator_config();
        cfg.model.negative = {neg_lo, neg_hi};
        cfg.model.positive = {0.4, 0.475};
        cfg.fold_poly = polydes::Polynomial(std::vector<double>(fold_c, fold_c + fold_len));
        size_t off = 0;
        for (size_t s = 0; s < nstages; ++s) {
            polydes::ClassifierChain::Stage st;
            st.poly = polydes::Polynomial(std::vector<double>(chain_c + off, chain_c + off + lens[s]));
            st.center = centers[s];
            cfg.fold_chain.stages.push_back(st);
            off += lens[s];
        }
        cfg.alg1_chain = cfg.fold_chain;
        polydes::ClassifierChain::Stage step;  // (3y - y^3) / 2 around 1/2
        step.poly = polydes::Polynomial(std::vector<double>{0.5, 0.75, 0.0, -0.5});
        step.center = 0.5;
        cfg.post_chain.stages = {step, step};
        cfg.post_chain.eps_schedule = {1e-3};
        auto q = to_templates(q_code, q_mask, batch, d);
        auto db = to_templates(db_code, db_mask, n_db, d);
        emu::Emulator em(cfg.emu_cfg);
        *ok = pipe::run_alg2(em, cfg, q, db).folding_assumption_ok ? 1 : 0;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

}  // extern "C"
