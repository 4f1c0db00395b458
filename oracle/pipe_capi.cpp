// extern "C" drivers for the reference's END-TO-END tests, linked against the
// UNMODIFIED reference pipeline (emulator.cpp, pipeline.cpp, poly.cpp,
// poly_design.cpp, iris_core.cpp compiled where they lie). TEST
// INFRASTRUCTURE ONLY.
//
// Two libraries are built from the same objects (oracle/Makefile `pipe`):
//   _ref/libirl_pipe_ref.so   Emulator::ccmm_twin = the reference's own product
//   _ref/libirl_pipe_b200.so  Emulator::ccmm_twin's product from the B200
//                             engine (paper_2601_17561_b200/host/emulator_ccmm_hook.cpp,
//                             interposed with -Wl,--wrap)
// so tests/test_pipeline_b200.py can run the reference's own run_alg1/run_alg2
// both ways and require identical results.
//
// The scenarios restate the reference's test drivers (doctest is absent):
//   pipe_planted_small:  test_pipeline.cpp:254-299 ("end-to-end: both
//                        algorithms match the plaintext oracle")
//   pipe_instances:      acceptance.cpp:187-312 run_instances() for
//                        criteria 6 and 7 (full_config, and the rho = 32 run)
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "irislab/errors.hpp"
#include "irislab/pipeline.hpp"

using namespace irislab;

namespace {

std::string g_err;

const polydes::ClassifierChain& chain(int which) {
    // test_pipeline.cpp:22-38 and acceptance.cpp full_config()
    static const polydes::ClassifierChain core =
        polydes::compose_classifier({-0.25, 0.25}, {0.4, 0.475}, 1e-4, {15, 15});
    static const polydes::ClassifierChain core3 =
        polydes::compose_classifier({-0.25, 0.25}, {0.4, 0.475}, 1e-4, {15, 15, 7});
    static const polydes::ClassifierChain fold =
        polydes::compose_classifier({-0.15, 0.35}, {0.4, 3.8}, 1e-4, {15, 15, 7});
    static const polydes::ClassifierChain post =
        polydes::compose_classifier({-0.414, 0.571}, {0.585, 1.414}, 1e-3, {31, 31});
    switch (which) {
        case 0: return core;
        case 1: return core3;
        case 2: return fold;
        default: return post;
    }
}

pipe::PipelineConfig small_config() {  // test_pipeline.cpp:46-61
    pipe::PipelineConfig cfg;
    cfg.rho = 8;
    cfg.batch = 1;
    cfg.n_db = 1024;
    cfg.d = 1024;
    cfg.fold_k = 4;
    cfg.emu_cfg = pipe::default_emulator_config();
    cfg.model.negative = {-0.25, 0.25};
    cfg.model.positive = {0.4, 0.475};
    cfg.fold_poly = polydes::Polynomial(std::vector<double>{0.004105, -0.173510, -2.528271, 24.347349, 124.161550,
                                                            -412.746212, 376.961251, 106.553952});
    cfg.alg1_chain = chain(0);
    cfg.fold_chain = chain(2);
    cfg.post_chain = chain(3);
    return cfg;
}

pipe::PipelineConfig full_config(const double* fold_c, std::size_t nfold) {  // acceptance.cpp:200-222
    pipe::PipelineConfig cfg;
    cfg.rho = 31;
    cfg.batch = 4;
    cfg.n_db = 4096;
    cfg.d = 1024;
    cfg.fold_k = 16;
    cfg.emu_cfg = pipe::default_emulator_config();
    cfg.model.negative = {-0.25, 0.25};
    cfg.model.positive = {0.4, 0.475};
    // data/fold_poly_appc.json, passed in by the caller (tests/oracle_lib.py)
    cfg.fold_poly = polydes::Polynomial(std::vector<double>(fold_c, fold_c + nfold));
    cfg.alg1_chain = chain(1);
    cfg.fold_chain = chain(2);
    cfg.post_chain = chain(3);
    return cfg;
}

// A rotated copy of `q` with `flips` code bits flipped at the first positions
// of a shuffle of [0, d) drawn from `rng`: the planted near-match.
iris::IrisTemplate planted(const iris::IrisTemplate& q, std::size_t rot, std::mt19937_64& rng, int flips) {
    iris::IrisTemplate t = iris::rotate(q, rot);
    std::vector<int> idx(t.code.size());
    for (std::size_t i = 0; i < idx.size(); ++i) idx[i] = static_cast<int>(i);
    std::shuffle(idx.begin(), idx.end(), rng);
    for (int i = 0; i < flips; ++i) t.code[static_cast<std::size_t>(idx[static_cast<std::size_t>(i)])] ^= 1;
    return t;
}

// Result record: [agrees, folding_ok, bts_pre, bts_post, bts_acc, total_ops,
// batch, match_bits[batch], oracle_bits[batch]] in int64s.
constexpr int kHead = 7;
std::size_t put(const pipe::PipelineResult& r, int64_t* out) {
    out[0] = r.agrees_with_oracle();
    out[1] = r.folding_assumption_ok;
    out[2] = r.bts_pre;
    out[3] = r.bts_post;
    out[4] = r.bts_acc;
    out[5] = r.total_ops;
    out[6] = static_cast<int64_t>(r.match_bits.size());
    std::size_t k = kHead;
    for (int b : r.match_bits) out[k++] = b;
    for (int b : r.oracle_bits) out[k++] = b;
    return k;
}

}  // namespace

extern "C" {

const char* pipe_last_error() { return g_err.c_str(); }

// test_pipeline.cpp:254-299. out: three records (r1 = run_alg1, r2 =
// run_alg2 on the planted query, r3 = run_alg1 on a clean query), 16 int64
// each, plus out[48] = whether the planted score lies in P.
int pipe_planted_small(int64_t* out) {
    try {
        pipe::PipelineConfig cfg = small_config();
        auto db = iris::synth_db(static_cast<std::size_t>(cfg.n_db), static_cast<std::size_t>(cfg.d), 1.0, 42);
        auto queries = iris::synth_db(1, static_cast<std::size_t>(cfg.d), 1.0, 4242);
        {
            std::mt19937_64 rng(7);
            db[777] = planted(queries[0], 5, rng, 292);
            const double s = iris::score(iris::rotate(queries[0], 5), db[777]);
            out[48] = cfg.model.positive.contains(s);
        }
        emu::Emulator em(cfg.emu_cfg);
        put(pipe::run_alg1(em, cfg, queries, db), out);
        put(pipe::run_alg2(em, cfg, queries, db), out + 16);
        auto clean_q = iris::synth_db(1, static_cast<std::size_t>(cfg.d), 1.0, 999);
        put(pipe::run_alg1(em, cfg, clean_q, db), out + 32);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// acceptance.cpp:227-275 run_instances(): `instances` instances from seed0
// (criterion 6: full_config, 100 instances from 60000; criterion 7's exact
// run: rho = 32, batch 1, n_db 1024, seed 70000). Each instance writes two
// records (run_alg1, run_alg2) of `stride` int64s.
int pipe_instances(int rho, int batch, long n_db, int instances, uint64_t seed0, const double* fold_c,
                   std::size_t nfold, int64_t* out, std::size_t stride) {
    try {
        pipe::PipelineConfig cfg = full_config(fold_c, nfold);
        cfg.rho = rho;
        cfg.batch = batch;
        cfg.n_db = n_db;
        if (stride < static_cast<std::size_t>(kHead + 2 * batch)) throw Error("pipe_instances: stride too small");
        for (int inst = 0; inst < instances; ++inst) {
            const uint64_t s = seed0 + static_cast<uint64_t>(inst) * 1000;
            auto db = iris::synth_db(static_cast<std::size_t>(cfg.n_db), static_cast<std::size_t>(cfg.d), 1.0, s);
            auto queries =
                iris::synth_db(static_cast<std::size_t>(cfg.batch), static_cast<std::size_t>(cfg.d), 1.0, s + 1);
            std::mt19937_64 rng(s + 2);
            std::uniform_int_distribution<int> rot(0, cfg.rho - 1);
            std::uniform_int_distribution<long> slot(0, cfg.n_db - 1);
            for (int e = 0; e < cfg.batch; ++e) {
                if ((rng() & 1) == 0) continue;
                const auto r = static_cast<std::size_t>(rot(rng));
                iris::IrisTemplate t = planted(queries[static_cast<std::size_t>(e)], r, rng, 292);
                db[static_cast<std::size_t>(slot(rng))] = t;
            }
            emu::Emulator em(cfg.emu_cfg);
            put(pipe::run_alg1(em, cfg, queries, db), out + (2 * inst) * stride);
            put(pipe::run_alg2(em, cfg, queries, db), out + (2 * inst + 1) * stride);
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // extern "C"
