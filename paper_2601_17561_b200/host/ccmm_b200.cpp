// irislab::emu::ccmm_twin_product and irislab::b200::CcmmEngine on the B200
// (see irislab_b200/ccmm.hpp).
#include "irislab_b200/ccmm.hpp"

#include <string>

#include "../../include/irl_capi.h"

namespace irislab {
namespace b200 {
irl_ctx* context();  // modmat_b200.cpp
}

namespace {

void check_msg(int st, const std::string& m) {
    switch (st) {
        case IRL_ERR_SHAPE_MISMATCH: throw ShapeMismatch(m);
        case IRL_ERR_MODULUS_TOO_LARGE: throw ModulusTooLarge(m);
        case IRL_ERR_ACCUMULATION_OVERFLOW_RISK: throw AccumulationOverflowRisk(m);
        case IRL_ERR_MODULUS_BUDGET: throw ModulusBudget(m);
        case IRL_ERR_CUDA:
        case IRL_ERR_NO_DEVICE:
        case IRL_ERR_OUT_OF_MEMORY: throw DeviceError(m);
        default: throw Error(m);
    }
}

void check(int st) {
    if (st != IRL_OK) check_msg(st, irl_last_error(b200::context()));
}

}  // namespace

namespace emu {

std::vector<std::vector<double>> ccmm_twin_product(const CcmmSpec& spec, const std::vector<double>& db,
                                                   const std::vector<double>& qry, int top_level) {
    // sizes are validated by the C ABI in ccmm_twin's order (emulator.cpp:392-410);
    // the buffers must at least hold what the shapes promise
    if (spec.d1 > 0 && spec.d2 > 0 && spec.d3 > 0 &&
        (db.size() != static_cast<std::size_t>(spec.d1 * spec.d2) ||
         qry.size() != static_cast<std::size_t>(spec.d2 * spec.d3)))
        throw ShapeMismatch("ccmm: operand sizes do not match the spec");
    const long total = spec.d1 > 0 && spec.d3 > 0 ? spec.d1 * spec.d3 : 0;
    std::vector<double> flat(static_cast<std::size_t>(total > 0 ? total : 1));
    check(irl_ccmm_twin(b200::context(), spec.d1, spec.d2, spec.d3, spec.n_db, spec.n_qry, spec.db_modulus_bits,
                        spec.qry_modulus_bits, spec.scale_bits, spec.out_level, top_level,
                        spec.out_encoding == Encoding::Slot ? 1 : 0, spec.out_ci ? 1 : 0, db.data(), qry.data(),
                        flat.data()));
    std::vector<std::vector<double>> out(static_cast<std::size_t>(total / spec.n_db));
    for (std::size_t k = 0; k < out.size(); ++k)
        out[k].assign(flat.begin() + static_cast<long>(k * spec.n_db),
                      flat.begin() + static_cast<long>((k + 1) * spec.n_db));
    return out;
}

}  // namespace emu

namespace b200 {

CcmmEngine::CcmmEngine(std::size_t parts, std::size_t m, std::size_t k, std::size_t max_n,
                       const modmat::RnsBasis& basis)
    : parts_(parts), m_(m), k_(k), max_n_(max_n), nmod_(basis.moduli.size()) {
    std::vector<uint32_t> ps, es;
    for (const auto& md : basis.moduli) {
        ps.push_back(md.p);
        es.push_back(md.e);
    }
    check(irl_ccmm_create(context(), parts, m, k, max_n, ps.data(), es.data(), ps.size(), &e_));
}

CcmmEngine::~CcmmEngine() { irl_ccmm_destroy(e_); }

void CcmmEngine::load_part(std::size_t part, const std::vector<uint16_t>& residues) {
    if (residues.size() != nmod_ * m_ * k_) throw ShapeMismatch("ccmm: part residues must be nmod x m x k");
    check(irl_ccmm_load_part(e_, part, residues.data(), 0));
}

void CcmmEngine::load_part_bigint(std::size_t part, const modmat::BigMatrix& entries) {
    if (entries.rows != m_ || entries.cols != k_) throw ShapeMismatch("ccmm: part must be m x k");
    check(irl_ccmm_load_part_bigint(e_, part, entries.a.data(), entries.width));
}

void CcmmEngine::load_part_file(std::size_t part, const std::string& path) {
    check(irl_ccmm_load_part_file(e_, part, path.c_str()));
}

void CcmmEngine::synth_db(uint64_t seed, uint32_t first_part) { check(irl_ccmm_synth_db(e_, seed, first_part)); }

void CcmmEngine::run(const uint16_t* q_res, std::size_t n, uint16_t* out) { check(irl_ccmm_run(e_, q_res, n, out)); }

std::vector<uint16_t> CcmmEngine::run(const std::vector<uint16_t>& q_res, std::size_t n) {
    if (n == 0 || q_res.size() != nmod_ * k_ * n) throw ShapeMismatch("ccmm: query residues must be nmod x k x n");
    std::vector<uint16_t> out(parts_ * nmod_ * n * m_);
    run(q_res.data(), n, out.data());
    return out;
}

uint64_t CcmmEngine::device_bytes() const { return irl_ccmm_device_bytes(e_); }

CcmmGroup::CcmmGroup(const std::vector<int>& devices, std::size_t parts, std::size_t m, std::size_t k,
                     std::size_t max_n, const modmat::RnsBasis& basis)
    : ranks_(devices.size()), parts_(parts), m_(m), k_(k), max_n_(max_n), nmod_(basis.moduli.size()) {
    std::vector<uint32_t> ps, es;
    for (const auto& md : basis.moduli) {
        ps.push_back(md.p);
        es.push_back(md.e);
    }
    const int st = irl_ccmm_group_create(devices.data(), devices.size(), parts, m, k, max_n, ps.data(), es.data(),
                                         ps.size(), &g_);
    if (st == IRL_ERR_SHAPE_MISMATCH) throw ShapeMismatch("ccmm group: more devices than parts");
    if (st != IRL_OK) check_msg(st, "ccmm group: create failed (status " + std::to_string(st) + ")");
}

CcmmGroup::~CcmmGroup() { irl_ccmm_group_destroy(g_); }

void CcmmGroup::check(int st) const {
    if (st != IRL_OK) check_msg(st, irl_last_error(irl_ccmm_group_ctx(g_, 0)));
}

std::size_t CcmmGroup::first_part(std::size_t rank) const {
    size_t first = 0;
    check(irl_ccmm_group_engine(g_, rank, nullptr, &first, nullptr));
    return first;
}

std::size_t CcmmGroup::rank_parts(std::size_t rank) const {
    size_t count = 0;
    check(irl_ccmm_group_engine(g_, rank, nullptr, nullptr, &count));
    return count;
}

void CcmmGroup::synth_db(uint64_t seed) {
    for (std::size_t r = 0; r < ranks_; ++r) {
        irl_ccmm* e = nullptr;
        size_t first = 0;
        check(irl_ccmm_group_engine(g_, r, &e, &first, nullptr));
        const int st = irl_ccmm_synth_db(e, seed, static_cast<uint32_t>(first));
        if (st != IRL_OK) check_msg(st, irl_last_error(irl_ccmm_group_ctx(g_, r)));
    }
}

void CcmmGroup::load_part_file(std::size_t part, const std::string& path) {
    if (part >= parts_) throw ShapeMismatch("ccmm: part index out of range");
    for (std::size_t r = 0; r < ranks_; ++r) {
        irl_ccmm* e = nullptr;
        size_t first = 0, count = 0;
        check(irl_ccmm_group_engine(g_, r, &e, &first, &count));
        if (part < first || part >= first + count) continue;
        const int st = irl_ccmm_load_part_file(e, part - first, path.c_str());
        if (st != IRL_OK) check_msg(st, irl_last_error(irl_ccmm_group_ctx(g_, r)));
        return;
    }
}

void CcmmGroup::set_exchange(int mode) { check(irl_ccmm_group_set_exchange(g_, mode)); }

void CcmmGroup::set_query_shard(int mode) { check(irl_ccmm_group_set_query_shard(g_, mode)); }

int CcmmGroup::run(const uint16_t* q_res, std::size_t n, uint16_t* out, void** a_out) {
    int mode = 0;
    check(irl_ccmm_full(g_, q_res, n, out, a_out, &mode));
    return mode;
}

std::vector<uint16_t> CcmmGroup::run(const std::vector<uint16_t>& q_res, std::size_t n) {
    if (n == 0 || q_res.size() != nmod_ * k_ * n) throw ShapeMismatch("ccmm: query residues must be nmod x k x n");
    std::vector<uint16_t> out(parts_ * nmod_ * n * m_);
    run(q_res.data(), n, out.data());
    return out;
}

}  // namespace b200
}  // namespace irislab
