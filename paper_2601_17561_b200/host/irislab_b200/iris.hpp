// C++ host mirror of the reference's irislab::iris scoring API
// (/root/reference/proj/include/irislab/iris_core.hpp) with every score
// computed on the B200: the inner products <a', b'> and mask overlaps of a
// whole query batch are two exact GEMMs on the FP4 tensor cores (C ABI
// irl_iris_inner_overlap / irl_iris_match, csrc/iris.cu). Template handling
// (to_masked, rotate, synth_db, pad_to) is host bookkeeping, as in the
// reference. Same names, value semantics and exception types.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "modmat.hpp"  // irislab::Error, ShapeMismatch, DeviceError

namespace irislab {

// errors.hpp:18-20
struct ZeroOverlap : Error {
    ZeroOverlap() : Error("mask overlap is empty, score undefined") {}
};
struct ConfigError : Error {
    using Error::Error;
};

namespace iris {

/// Binary iris code plus validity mask, both of length d (iris_core.hpp:12-18).
struct IrisTemplate {
    std::vector<uint8_t> code;
    std::vector<uint8_t> mask;

    std::size_t size() const { return code.size(); }
    void validate() const;
};

/// c' = m - 2 (c & m) in {-1, 0, 1} (iris_core.hpp:20-25).
struct MaskedBitvector {
    std::vector<int8_t> values;
    std::size_t size() const { return values.size(); }
};

struct Interval {
    double lo = 0.0;
    double hi = 0.0;
    bool contains(double x) const { return x >= lo && x <= hi; }
    double width() const { return hi - lo; }
};

MaskedBitvector to_masked(const IrisTemplate& t);
IrisTemplate rotate(const IrisTemplate& t, std::size_t r);
IrisTemplate pad_to(const IrisTemplate& t, std::size_t d_target);
std::vector<IrisTemplate> synth_db(std::size_t n_db, std::size_t d, double mask_density, uint64_t seed);

/// Score <a', b'> / |m_a & m_b| on the device; ZeroOverlap if the masks do not meet.
double score(const IrisTemplate& a, const IrisTemplate& b);
double distance(const IrisTemplate& a, const IrisTemplate& b);

/// Plaintext ground truth (iris_core.cpp:78-90): one batched device pass over
/// every (query, entry) pair, then the reference's loop-order semantics.
bool match_db_reference(const std::vector<IrisTemplate>& query, const std::vector<IrisTemplate>& db,
                        const Interval& n_int, const Interval& p_int);

/// Batched form used by the server pipeline (pipeline.cpp:92-153): for query
/// column c = e * rho + r = rotate(eyes[e], r) and template j,
/// inner[c * db.size() + j] and overlap[c * db.size() + j].
void inner_and_overlap(const std::vector<IrisTemplate>& db, const std::vector<IrisTemplate>& eyes,
                       std::size_t rho, std::vector<int32_t>* inner, std::vector<int32_t>* overlap);

}  // namespace iris

namespace pipe {

/// ClassifierChain::Stage (poly_design.hpp:66-72): poly in y = x - center.
struct ChainStage {
    std::vector<double> coeffs;
    double center = 0.0;
};

/// The PipelineConfig fields Alg. 2's fold stage reads (pipeline.hpp:16-45).
struct FoldConfig {
    int rho = 31;
    int batch = 4;
    long n_db = 4096;
    long d = 1024;
    int fold_k = 16;
    std::vector<double> fold_poly;         // cfg.fold_poly.coeffs
    std::vector<ChainStage> fold_chain;    // cfg.fold_chain.stages
    iris::Interval negative{-0.25, 0.25};  // cfg.model.negative
};

/// Messages of run_alg2's post-CCMM stage (pipeline.cpp:594-627), equal bit
/// for bit to the noise-free emulator's:
///   folded[((e * blocks + b) * groups + g) * d + i]  = fold_group(normalize(...)) message
///   refolded[(e * blocks + b) * d + i]              = sum over g of eval_chain_ct(folded_g)
/// plus PipelineResult::folding_assumption_ok (pipeline.cpp:565-590).
struct FoldMessages {
    std::vector<double> folded;
    std::vector<double> refolded;  // empty unless requested
    bool folding_assumption_ok = true;
};

/// From the CCMM product and the overlaps, int32 [batch * rho][n_db] (the
/// layout of iris::inner_and_overlap). Throws ConfigError
/// (PipelineConfig::validate, "eval_chain_ct: empty chain") and ZeroOverlap
/// (normalize) as the reference does.
FoldMessages fold_stage(const FoldConfig& cfg, const std::vector<int32_t>& inner,
                        const std::vector<int32_t>& overlap, bool want_refolded = true);

/// From templates: prepare's products and overlaps as tensor-core GEMMs, then the
/// fold stage, without leaving the device (irl_iris_db_fold).
FoldMessages fold_stage(const FoldConfig& cfg, const std::vector<iris::IrisTemplate>& queries,
                        const std::vector<iris::IrisTemplate>& db, bool want_refolded = true);

}  // namespace pipe
}  // namespace irislab
