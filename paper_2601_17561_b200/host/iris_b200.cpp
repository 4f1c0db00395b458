// irislab::iris on the B200 (see irislab_b200/iris.hpp).
#include "irislab_b200/iris.hpp"

#include <random>
#include <string>

#include "../../include/irl_capi.h"

namespace irislab {
namespace b200 {
irl_ctx* context();  // modmat_b200.cpp
}

namespace iris {
namespace {

void check(int st) {
    if (st == IRL_OK) return;
    const std::string m = irl_last_error(b200::context());
    switch (st) {
        case IRL_ERR_SHAPE_MISMATCH: throw ShapeMismatch(m);
        case IRL_ERR_ZERO_OVERLAP: throw ZeroOverlap();
        case IRL_ERR_CONFIG: throw ConfigError(m);
        case IRL_ERR_CUDA:
        case IRL_ERR_NO_DEVICE:
        case IRL_ERR_OUT_OF_MEMORY: throw DeviceError(m);
        default: throw Error(m);
    }
}

// pack_bits (pipeline.cpp:70-76) of n templates -> code / mask words
void pack(const std::vector<IrisTemplate>& ts, std::size_t d, std::vector<uint64_t>* code,
          std::vector<uint64_t>* mask) {
    const std::size_t words = (d + 63) / 64;
    code->assign(ts.size() * words, 0);
    mask->assign(ts.size() * words, 0);
    for (std::size_t t = 0; t < ts.size(); ++t) {
        if (ts[t].code.size() != d || ts[t].mask.size() != d) throw ShapeMismatch("template lengths differ");
        for (std::size_t i = 0; i < d; ++i) {
            if (ts[t].code[i]) (*code)[t * words + i / 64] |= uint64_t{1} << (i % 64);
            if (ts[t].mask[i]) (*mask)[t * words + i / 64] |= uint64_t{1} << (i % 64);
        }
    }
}

}  // namespace

void IrisTemplate::validate() const {
    if (code.size() != mask.size() || code.empty())
        throw ShapeMismatch("code and mask must have identical nonzero length");
    for (std::size_t i = 0; i < code.size(); ++i)
        if (code[i] > 1 || mask[i] > 1) throw ShapeMismatch("template entries must be bits");
}

MaskedBitvector to_masked(const IrisTemplate& t) {
    MaskedBitvector out;
    out.values.resize(t.size());
    for (std::size_t i = 0; i < t.size(); ++i)
        out.values[i] = static_cast<int8_t>(t.mask[i] ? 1 - 2 * (t.code[i] & 1) : 0);
    return out;
}

IrisTemplate rotate(const IrisTemplate& t, std::size_t r) {
    const std::size_t d = t.size();
    IrisTemplate out;
    out.code.resize(d);
    out.mask.resize(d);
    if (d == 0) return out;
    r %= d;
    for (std::size_t k = 0; k < d; ++k) {  // entry i moves to (i + r) mod d
        const std::size_t src = (k + d - r) % d;
        out.code[k] = t.code[src];
        out.mask[k] = t.mask[src];
    }
    return out;
}

IrisTemplate pad_to(const IrisTemplate& t, std::size_t d_target) {
    if (d_target < t.size()) throw ShapeMismatch("cannot pad to a smaller length");
    IrisTemplate out = t;
    out.code.resize(d_target, 0);
    out.mask.resize(d_target, 0);
    return out;
}

std::vector<IrisTemplate> synth_db(std::size_t n_db, std::size_t d, double mask_density, uint64_t seed) {
    // same generator and draw order as the reference (iris_core.cpp:92-112):
    // codes first, then masks, per template; full masks draw nothing
    if (!(mask_density > 0.0 && mask_density <= 1.0)) throw ConfigError("mask density must be in (0, 1]");
    std::mt19937_64 rng(seed);
    std::bernoulli_distribution code_bit(0.5), mask_bit(mask_density);
    std::vector<IrisTemplate> out(n_db);
    for (auto& t : out) {
        t.code.resize(d);
        t.mask.assign(d, 1);
        for (std::size_t i = 0; i < d; ++i) t.code[i] = code_bit(rng) ? 1 : 0;
        if (mask_density < 1.0)
            for (std::size_t i = 0; i < d; ++i) t.mask[i] = mask_bit(rng) ? 1 : 0;
    }
    return out;
}

void inner_and_overlap(const std::vector<IrisTemplate>& db, const std::vector<IrisTemplate>& eyes,
                       std::size_t rho, std::vector<int32_t>* inner, std::vector<int32_t>* overlap) {
    const std::size_t d = !db.empty() ? db[0].size() : (!eyes.empty() ? eyes[0].size() : 0);
    std::vector<uint64_t> dc, dm, qc, qm;
    pack(db, d, &dc, &dm);
    pack(eyes, d, &qc, &qm);
    const std::size_t n = eyes.size() * rho * db.size();
    if (inner) inner->assign(n, 0);
    if (overlap) overlap->assign(n, 0);
    check(irl_iris_inner_overlap(b200::context(), dc.data(), dm.data(), db.size(), qc.data(), qm.data(),
                                 eyes.size(), rho, d, inner ? inner->data() : nullptr,
                                 overlap ? overlap->data() : nullptr));
}

double score(const IrisTemplate& a, const IrisTemplate& b) {
    if (a.size() != b.size()) throw ShapeMismatch("template lengths differ");
    std::vector<int32_t> in, ov;
    inner_and_overlap({b}, {a}, 1, &in, &ov);
    if (ov[0] == 0) throw ZeroOverlap();
    return static_cast<double>(in[0]) / static_cast<double>(ov[0]);
}

double distance(const IrisTemplate& a, const IrisTemplate& b) { return (1.0 - score(a, b)) / 2.0; }

bool match_db_reference(const std::vector<IrisTemplate>& query, const std::vector<IrisTemplate>& db,
                        const Interval& n_int, const Interval& p_int) {
    (void)n_int;  // scores in N (or the gap) do not set the bit (iris_core.cpp:85-86)
    if (query.empty() || db.empty()) return false;
    const std::size_t d = db[0].size();
    std::vector<uint64_t> dc, dm, qc, qm;
    pack(db, d, &dc, &dm);
    pack(query, d, &qc, &qm);
    // each query template is its own "eye" (rho = 1); the first eye, in query
    // order, whose row has an event decides: a match returns true, an empty
    // overlap before any match throws
    std::vector<int32_t> res(query.size());
    const int st = irl_iris_match(b200::context(), dc.data(), dm.data(), db.size(), qc.data(), qm.data(),
                                  query.size(), 1, d, p_int.lo, p_int.hi, nullptr, res.data(), nullptr);
    if (st != IRL_OK && st != IRL_ERR_ZERO_OVERLAP) check(st);
    for (int32_t r : res) {
        if (r == 1) return true;
        if (r < 0) throw ZeroOverlap();
    }
    return false;
}

}  // namespace iris
namespace pipe {
namespace {

using iris::check;

// irl_fold_params over cfg; the vectors it points into live in the holder.
struct Params {
    irl_fold_params p{};
    std::vector<double> centers, coeffs;
    std::vector<size_t> lens;
    explicit Params(const FoldConfig& cfg) {
        for (const ChainStage& st : cfg.fold_chain) {
            centers.push_back(st.center);
            lens.push_back(st.coeffs.size());
            coeffs.insert(coeffs.end(), st.coeffs.begin(), st.coeffs.end());
        }
        p.batch = cfg.batch < 0 ? 0 : static_cast<size_t>(cfg.batch);
        p.rho = cfg.rho < 0 ? 0 : static_cast<size_t>(cfg.rho);
        p.n_db = cfg.n_db < 0 ? 0 : static_cast<size_t>(cfg.n_db);
        p.d = cfg.d < 0 ? 0 : static_cast<size_t>(cfg.d);
        p.fold_k = cfg.fold_k < 0 ? 0 : static_cast<size_t>(cfg.fold_k);
        p.fold_coeffs = cfg.fold_poly.data();
        p.fold_len = cfg.fold_poly.size();
        p.chain_stages = cfg.fold_chain.size();
        p.chain_centers = centers.data();
        p.chain_lens = lens.data();
        p.chain_coeffs = coeffs.data();
        p.negative_lo = cfg.negative.lo;
        p.negative_hi = cfg.negative.hi;
    }
};

// PipelineConfig::validate (pipeline.cpp:232-243) for the fields the stage
// reads, then eval_chain_ct's empty-chain check; the C ABI repeats them.
void validate(const FoldConfig& cfg, bool want_refolded) {
    if (cfg.rho < 1 || cfg.batch < 1) throw ConfigError("pipeline: rho and batch must be >= 1");
    if (cfg.fold_k < 1 || cfg.fold_k > cfg.rho) throw ConfigError("pipeline: fold_k must satisfy 1 <= k <= rho");
    if (cfg.d < 2 || (cfg.d & (cfg.d - 1)) != 0) throw ConfigError("pipeline: d must be a power of two");
    if (cfg.n_db < cfg.d || cfg.n_db % cfg.d != 0)
        throw ConfigError("pipeline: n_db must be a positive multiple of d");
    if (want_refolded && cfg.fold_chain.empty()) throw ConfigError("eval_chain_ct: empty chain");
}

void size_outputs(const FoldConfig& cfg, bool want_refolded, FoldMessages* out) {
    const bool valid = cfg.d > 0 && cfg.fold_k > 0 && cfg.batch > 0 && cfg.n_db >= cfg.d;
    const size_t blocks = valid ? static_cast<size_t>(cfg.n_db / cfg.d) : 0;
    const size_t groups = valid ? static_cast<size_t>((cfg.rho + cfg.fold_k - 1) / cfg.fold_k) : 0;
    const size_t slots = valid ? static_cast<size_t>(cfg.batch) * blocks * static_cast<size_t>(cfg.d) : 0;
    out->folded.assign(slots * groups, 0.0);
    out->refolded.assign(want_refolded ? slots : 0, 0.0);
}

}  // namespace

FoldMessages fold_stage(const FoldConfig& cfg, const std::vector<int32_t>& inner,
                        const std::vector<int32_t>& overlap, bool want_refolded) {
    Params prm(cfg);
    validate(cfg, want_refolded);
    const size_t need = prm.p.batch * prm.p.rho * prm.p.n_db;
    if (inner.size() < need || overlap.size() < need)
        throw ShapeMismatch("fold_stage: product / overlap smaller than batch * rho * n_db");
    FoldMessages out;
    size_outputs(cfg, want_refolded, &out);
    int32_t ok = 1;
    check(irl_fold_stage(b200::context(), &prm.p, inner.data(), overlap.data(), out.folded.data(),
                         want_refolded ? out.refolded.data() : nullptr, &ok));
    out.folding_assumption_ok = ok != 0;
    return out;
}

FoldMessages fold_stage(const FoldConfig& cfg, const std::vector<iris::IrisTemplate>& queries,
                        const std::vector<iris::IrisTemplate>& db, bool want_refolded) {
    Params prm(cfg);
    validate(cfg, want_refolded);  // run_alg2: cfg.validate() before prepare
    // prepare (pipeline.cpp:100-118)
    if (static_cast<long>(db.size()) != cfg.n_db) throw ShapeMismatch("pipeline: database size does not match config");
    if (static_cast<int>(queries.size()) != cfg.batch) throw ShapeMismatch("pipeline: query count does not match batch");
    for (const iris::IrisTemplate& t : db)
        if (static_cast<long>(t.size()) != cfg.d) throw ShapeMismatch("pipeline: database template dimension mismatch");
    for (const iris::IrisTemplate& q : queries)
        if (static_cast<long>(q.size()) != cfg.d) throw ShapeMismatch("pipeline: query template dimension mismatch");
    const size_t d = static_cast<size_t>(cfg.d);
    std::vector<uint64_t> dc, dm, qc, qm;
    iris::pack(db, d, &dc, &dm);
    iris::pack(queries, d, &qc, &qm);
    irl_iris_db* h = nullptr;
    check(irl_iris_db_create(b200::context(), dc.data(), dm.data(), db.size(), d,
                             queries.size() * static_cast<size_t>(cfg.rho), &h));
    FoldMessages out;
    size_outputs(cfg, want_refolded, &out);
    int32_t ok = 1;
    const int st = irl_iris_db_fold(h, qc.data(), qm.data(), &prm.p, out.folded.data(),
                                    want_refolded ? out.refolded.data() : nullptr, &ok);
    irl_iris_db_destroy(h);
    check(st);
    out.folding_assumption_ok = ok != 0;
    return out;
}

}  // namespace pipe
}  // namespace irislab
