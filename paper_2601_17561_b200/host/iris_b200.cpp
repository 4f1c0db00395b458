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
}  // namespace irislab
