// irislab::cost on the B200 host side: the reference's database / query
// sizing and GPU distribution plan (reference proj/src/costmodel.cpp:10-73,
// include/irislab/costmodel.hpp:15-66; same names, arguments and ConfigError
// conditions), plus the plan this engine actually runs (b200_plan).
//
// The reference plans one database slice per GPU: a cluster is one a-slice
// GPU and slices-1 b-slice GPUs, and ceil(n_db / ((slices-1) n_per_slice))
// clusters cover the database (2^22 entries of 2^14-entry slices: 37 clusters
// of 8 GPUs). A B200 holds 180 GB of HBM, so a whole 8-slice cluster at
// 48 digit planes (144 GiB of planes + query / output staging) fits one GPU;
// b200_plan packs slices per GPU by HBM capacity, so the same database needs
// 37 GPUs instead of 296, each running the cluster's CCMM on its own.
#pragma once

#include <cstdint>
#include <string>

#include "iris.hpp"  // irislab::ConfigError

namespace irislab::cost {

inline constexpr long long KiB = 1LL << 10;
inline constexpr long long MiB = 1LL << 20;
inline constexpr long long GiB = 1LL << 30;

/// Encrypted database size in bits: 3 (ell+1) 2^27 log_Q (costmodel.cpp:10-13).
inline long long db_size_bits(int ell, long long log_q) {
    if (ell < 0 || log_q <= 0) throw ConfigError("db_size_bits: bad parameters");
    return 3LL * (ell + 1) * (1LL << 27) * log_q;
}

/// Digit-plane database bytes: planes * 3 * (ell+1) * 2^27 (costmodel.cpp:15-18).
inline long long db_size_bytes_int8(int ell, int planes) {
    if (ell < 0 || planes <= 0) throw ConfigError("db_size_bytes_int8: bad parameters");
    return static_cast<long long>(planes) * 3 * (ell + 1) * (1LL << 27);
}

/// The a-part: half of the ell = 1 layout (costmodel.cpp:20-23).
inline long long a_part_bytes_int8(int planes) { return db_size_bytes_int8(1, planes) / 2; }

/// cts_per_query (a, b) pairs of degree-2^log_n ring elements (costmodel.cpp:25-32).
inline long long query_size_bytes(int log_n, long long q_bits, int cts_per_query) {
    if (log_n < 0 || q_bits <= 0 || cts_per_query <= 0) throw ConfigError("query_size_bytes: bad parameters");
    return cts_per_query * 2LL * (1LL << log_n) * q_bits / 8;
}

/// ceil(batch * rho * d / (beta 2^log_n)) (costmodel.cpp:34-43).
inline long long packed_query_ct_count(int rho, int beta, int batch, long d, int log_n) {
    if (rho < 1 || beta < 1 || batch < 1 || d < 1) throw ConfigError("packed_query_ct_count: bad parameters");
    const long long values = static_cast<long long>(batch) * rho * d;
    const long long per_ct = static_cast<long long>(beta) * (1LL << log_n);
    return (values + per_ct - 1) / per_ct;
}

struct GpuPlan {
    int slices = 0;
    long entries_per_slice = 0;
    long long a_slice_bytes = 0;
    long long b_slice_bytes = 0;
    long clusters = 0;  // number of such plans to cover n_db
};

/// costmodel.cpp:59-73: one A-slice GPU plus (slices-1) B-part GPUs.
inline GpuPlan gpu_distribution_plan(long n_db, long n_per_slice, int slices, int planes) {
    if (n_db < 1 || n_per_slice < 1 || slices < 2) throw ConfigError("gpu_distribution_plan: bad parameters");
    GpuPlan plan;
    plan.slices = slices;
    plan.entries_per_slice = n_per_slice;
    plan.a_slice_bytes = a_part_bytes_int8(planes);
    plan.b_slice_bytes = (db_size_bytes_int8(1, planes) - plan.a_slice_bytes) / (slices - 1);
    const long per_cluster = static_cast<long>(slices - 1) * n_per_slice;
    plan.clusters = (n_db + per_cluster - 1) / per_cluster;
    return plan;
}

/// The plan this engine runs. One part = one slice of n_per_slice rows with
/// K = d2 + n_qry columns of `planes` int8 digit planes (the engine's
/// [part][modulus][digit][row][K] layout, K rounded up to 16). Each GPU also
/// stages the query residues and planes ([nmod][K][N] uint16 + int8 planes) and
/// the outputs ([parts][nmod][N][M] uint16) next to its parts.
struct B200Plan {
    long clusters = 0;            // reference clusters (a-slice + slices-1 b-slices)
    int parts_per_gpu = 0;        // parts resident per GPU
    long gpus = 0;                // GPUs to hold every cluster resident
    long long part_bytes = 0;     // digit planes of one part
    long long gpu_bytes = 0;      // planes + staging on a full GPU
    bool cluster_per_gpu = false; // a whole cluster fits one GPU (no a-part exchange)
};

inline B200Plan b200_plan(long n_db, long n_per_slice, int slices, int planes, long k, long query_cols,
                          long long hbm_bytes = 180LL * 1000 * 1000 * 1000, long long reserve_bytes = 4LL * GiB) {
    if (k < 1 || query_cols < 1 || hbm_bytes <= reserve_bytes) throw ConfigError("b200_plan: bad parameters");
    const GpuPlan ref = gpu_distribution_plan(n_db, n_per_slice, slices, planes);
    B200Plan p;
    p.clusters = ref.clusters;
    const long long ldk = (k + 15) / 16 * 16;
    const long long nmod = planes / 2;
    p.part_bytes = static_cast<long long>(planes) * n_per_slice * ldk;
    const long long query = nmod * k * query_cols * 2 + static_cast<long long>(planes) * query_cols * ldk;
    const long long out_per_part = nmod * query_cols * n_per_slice * 2;
    const long long budget = hbm_bytes - reserve_bytes - query;
    int fit = static_cast<int>(budget / (p.part_bytes + out_per_part));
    if (fit < 1) throw ConfigError("b200_plan: one part does not fit the GPU");
    if (fit > slices) fit = slices;
    p.parts_per_gpu = fit;
    p.cluster_per_gpu = fit == slices;
    const long per_cluster_gpus = (slices + fit - 1) / fit;
    p.gpus = p.clusters * per_cluster_gpus;
    p.gpu_bytes = query + fit * (p.part_bytes + out_per_part);
    return p;
}

}  // namespace irislab::cost
