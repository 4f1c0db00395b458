// The reference's ccmm_twin unit case (proj/tests/test_emulator.cpp:215-270)
// restated against the C++ host mirror (irislab_b200/ccmm.hpp), plus the
// device-resident CCMM engine against the plain-C oracle (test
// infrastructure). Needs a B200.
#include <cmath>
#include <cstdio>
#include <vector>

#include "irislab_b200/ccmm.hpp"
#include "../../oracle/irl_oracle.h"

using namespace irislab;

static int g_checks = 0, g_fail = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        ++g_checks;                                                           \
        if (!(c)) {                                                           \
            ++g_fail;                                                         \
            std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
        }                                                                     \
    } while (0)
#define CHECK_THROWS_AS(expr, T)       \
    do {                               \
        bool thrown_ = false;          \
        try {                          \
            (void)(expr);              \
        } catch (const T&) {           \
            thrown_ = true;            \
        } catch (...) {                \
        }                              \
        CHECK(thrown_ && #T);          \
    } while (0)

namespace {

void ccmm_twin_case() {  // test_emulator.cpp:215-270
    emu::CcmmSpec spec;
    spec.d1 = 4;
    spec.d2 = 3;
    spec.d3 = 2;
    spec.n_db = 2;
    spec.n_qry = 3;
    spec.qry_modulus_bits = 36.0;
    spec.scale_bits = 23.0;
    spec.db_modulus_bits = 2 * 36.0 - 23.0;
    const std::vector<double> db = {1, 0, 2, 0, 1, 0, 3, 0, 0, 0, 0, 1};
    const std::vector<double> qry = {1, 2, 3, 4, 5, 6};
    const int top = 10;
    auto out = emu::ccmm_twin_product(spec, db, qry, top);
    CHECK(out.size() == static_cast<size_t>(spec.d1 / spec.n_db * spec.d3));
    CHECK(out[0][0] == 11.0 && out[0][1] == 3.0);
    CHECK(out[1][0] == 3.0 && out[1][1] == 5.0);
    CHECK(out[2][0] == 14.0 && out[2][1] == 4.0);
    CHECK(out[3][0] == 6.0 && out[3][1] == 6.0);
    spec.db_modulus_bits = 36.0;
    CHECK_THROWS_AS(emu::ccmm_twin_product(spec, db, qry, top), ModulusBudget);
    spec.db_modulus_bits = 2 * 36.0 - 23.0;
    spec.out_level = 99;
    CHECK_THROWS_AS(emu::ccmm_twin_product(spec, db, qry, top), ModulusBudget);
    spec.out_level = 0;
    spec.out_encoding = emu::Encoding::Slot;  // slot output requires ci
    CHECK_THROWS_AS(emu::ccmm_twin_product(spec, db, qry, top), ShapeMismatch);
    spec.out_encoding = emu::Encoding::Coeff;
    spec.d1 = 5;  // not a multiple of n_db
    CHECK_THROWS_AS(emu::ccmm_twin_product(spec, db, qry, top), ShapeMismatch);
    spec.d1 = 4;
    spec.out_level = 5;
    spec.out_encoding = emu::Encoding::Slot;
    spec.out_ci = true;
    auto raised = emu::ccmm_twin_product(spec, db, qry, top);
    CHECK(raised[0][0] == 11.0);
}

void engine_vs_oracle() {
    // 3 parts of 300 x 700 against a 70-column query batch, all 24 moduli
    const size_t parts = 3, m = 300, k = 700, n = 70;
    const auto basis = modmat::build_paper_basis();
    b200::CcmmEngine eng(parts, m, k, n, basis);
    eng.synth_db(1);
    const size_t nmod = eng.moduli();
    std::vector<uint16_t> q(nmod * k * n);
    for (size_t i = 0; i < nmod; ++i)
        orc_synth_block(2, 0xFF, static_cast<uint32_t>(i), 0, static_cast<uint32_t>(k), 0,
                        static_cast<uint32_t>(n), basis.moduli[i].value(), q.data() + i * k * n);
    const auto out = eng.run(q, n);
    const std::vector<uint32_t> rows = {0, 1, 150, 299};
    for (size_t g = 0; g < parts; ++g)
        for (size_t i = 0; i < nmod; ++i) {
            const uint32_t mod = basis.moduli[i].value();
            std::vector<uint16_t> a(m * k), qt(n * k), want(rows.size() * n);
            orc_synth_block(1, static_cast<uint32_t>(g), static_cast<uint32_t>(i), 0, static_cast<uint32_t>(m), 0,
                            static_cast<uint32_t>(k), mod, a.data());
            for (size_t kk = 0; kk < k; ++kk)
                for (size_t c = 0; c < n; ++c) qt[c * k + kk] = q[i * k * n + kk * n + c];
            orc_ppmm_rows_direct(a.data(), k, qt.data(), k, rows.data(), rows.size(), n, k, mod, want.data());
            bool ok = true;
            for (size_t r = 0; r < rows.size(); ++r)
                for (size_t c = 0; c < n; ++c)
                    ok = ok && out[((g * nmod + i) * n + c) * m + rows[r]] == want[r * n + c];
            CHECK(ok);
        }
    // load_part equals the synthetic part it restates
    std::vector<uint16_t> res(nmod * m * k);
    for (size_t i = 0; i < nmod; ++i)
        orc_synth_block(1, 0, static_cast<uint32_t>(i), 0, static_cast<uint32_t>(m), 0, static_cast<uint32_t>(k),
                        basis.moduli[i].value(), res.data() + i * m * k);
    b200::CcmmEngine one(1, m, k, n, basis);
    one.load_part(0, res);
    const auto out1 = one.run(q, n);
    bool same = true;
    for (size_t x = 0; x < out1.size(); ++x) same = same && out1[x] == out[x];
    CHECK(same);
    CHECK_THROWS_AS(one.load_part(0, std::vector<uint16_t>(3)), ShapeMismatch);

    // the same database over a group of two ranks (both on device 0 here):
    // parts dealt 2 + 1, outputs in global order equal to the one engine's,
    // with the query copied whole per rank and sharded with a peer all-gather
    b200::CcmmGroup grp({0, 0}, parts, m, k, n, basis);
    CHECK(grp.ranks() == 2 && grp.first_part(0) == 0 && grp.rank_parts(0) == 2 && grp.first_part(1) == 2 &&
          grp.rank_parts(1) == 1);
    grp.synth_db(1);
    for (int shard : {0, 1}) {
        grp.set_query_shard(shard);
        const auto outg = grp.run(q, n);
        bool eq = outg.size() == out.size();
        for (size_t x = 0; eq && x < out.size(); ++x) eq = outg[x] == out[x];
        CHECK(eq);
    }
    CHECK_THROWS_AS(b200::CcmmGroup({0, 0, 0, 0}, parts, m, k, n, basis), ShapeMismatch);
}

}  // namespace

int main() {
    try {
        ccmm_twin_case();
        engine_vs_oracle();
    } catch (const std::exception& e) {
        std::printf("uncaught exception: %s\n", e.what());
        return 2;
    }
    std::printf("%d checks, %d failed; %llu kernel launches\n", g_checks, g_fail,
                static_cast<unsigned long long>(b200::kernel_launches()));
    return g_fail ? 1 : 0;
}
