// The reference's sizing suite (proj/tests/test_costmodel.cpp:10-72) restated
// against the B200 host mirror irislab_b200/costmodel.hpp, plus the B200
// residency plan. Header-only arithmetic: runs on CPU.
#include <cstdio>

#include "irislab_b200/costmodel.hpp"

using namespace irislab;
using namespace irislab::cost;

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

int main() {
    // database sizes (test_costmodel.cpp:10-23)
    CHECK(db_size_bits(1, 48) == 3LL * 2 * (1LL << 27) * 48);
    CHECK(db_size_bits(1, 8) == db_size_bytes_int8(1, 1) * 8);
    CHECK(db_size_bytes_int8(1, 48) == 36LL * GiB);
    CHECK(db_size_bytes_int8(1, 48) - a_part_bytes_int8(48) == 18LL * GiB);
    CHECK(a_part_bytes_int8(48) == 18LL * GiB);
    CHECK_THROWS_AS(db_size_bits(-1, 48), ConfigError);
    CHECK_THROWS_AS(db_size_bytes_int8(1, 0), ConfigError);
    // query sizes (:25-31)
    CHECK(query_size_bytes(16, 16, 2) == 512 * KiB);
    CHECK(query_size_bytes(16, 16, 1) == 256 * KiB);
    CHECK_THROWS_AS(query_size_bytes(16, 0, 2), ConfigError);
    // packed query ciphertext count (:33-39)
    CHECK(packed_query_ct_count(31, 4, 32, 1L << 14, 16) == 62);
    CHECK(packed_query_ct_count(1, 1, 1, 10, 3) == 2);
    CHECK_THROWS_AS(packed_query_ct_count(0, 4, 32, 1L << 14, 16), ConfigError);
    // gpu distribution plan (:60-72)
    auto plan = gpu_distribution_plan(1L << 19, 1L << 16, 8, 48);
    CHECK(plan.slices == 8);
    CHECK(plan.a_slice_bytes == 18LL * GiB);
    CHECK(plan.b_slice_bytes == 18LL * GiB / 7);
    CHECK(plan.clusters == 2);
    auto big = gpu_distribution_plan(1L << 22, 1L << 14, 8, 48);
    CHECK(big.clusters == 37);
    CHECK_THROWS_AS(gpu_distribution_plan(0, 1, 8, 48), ConfigError);
    CHECK_THROWS_AS(gpu_distribution_plan(100, 10, 1, 48), ConfigError);

    // B200 residency: one 8-part cluster at the paper's slice (2^14 rows,
    // K = 2^14 + 2^13, 992 query columns, 48 planes) fits one 180 GB GPU, so
    // the 2^22-entry database needs 37 GPUs rather than 37 x 8
    auto b = b200_plan(1L << 22, 1L << 14, 8, 48, (1L << 14) + (1L << 13), 992);
    CHECK(b.clusters == 37);
    CHECK(b.parts_per_gpu == 8 && b.cluster_per_gpu);
    CHECK(b.gpus == 37);
    CHECK(b.part_bytes == 18LL * GiB);  // 48 planes x 2^14 rows x 24576 = a_part_bytes_int8(48)
    CHECK(b.gpu_bytes < 180LL * 1000 * 1000 * 1000);
    // c5 slices (2^17 rows, 144 GiB of planes each): one part per GPU
    auto c5 = b200_plan(1L << 22, 1L << 17, 8, 48, (1L << 14) + (1L << 13), 992);
    CHECK(c5.parts_per_gpu == 1 && c5.gpus == 5 * 8);
    CHECK_THROWS_AS(b200_plan(1, 1L << 14, 8, 48, 0, 992), ConfigError);

    std::printf("costmodel mirror: %d checks, %d failed\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
