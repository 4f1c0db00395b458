// Alg. 2 fold stage at message level: normalize by the mask
// overlaps, the folding polynomial, the Rot alignment and the group sums, then
// the fold classifier chain and the refold across groups, plus the
// folding-assumption shadow check (reference pipeline.cpp:359-408, 538-633).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/irl_capi.h"

struct irl_ctx;

namespace irl {

constexpr int kFoldMaxDegree = 31;  // Paterson-Stockmeyer plans up to degree 31 (baby step 8)
constexpr int kFoldMaxStages = 8;

// Kernel parameters (passed by value: the coefficients sit in the constant
// bank, every thread reads the same address).
struct FoldArgs {
    double fold_c[kFoldMaxDegree + 1];
    double chain_c[kFoldMaxStages][kFoldMaxDegree + 1];
    double center[kFoldMaxStages];
    int stage_deg[kFoldMaxStages];
    int fold_deg = 0;
    int nstages = 0;
    double neg_lo = 0.0, neg_hi = 0.0;
    double lo_in = 0.0, lo_out = 0.0, hi_in = 0.0, hi_out = 0.0;  // shadow-check bands (fold.cu)
    bool fast = false;                 // no -0.0 coefficient: the reduced evaluation (fold.cu)
    const double* rcp = nullptr;       // rcp[k] = RN(1 / k), k <= rcp_max
    uint32_t rcp_max = 0;
    uint32_t batch = 0, rho = 0, blocks = 0, d = 0, fold_k = 0, groups = 0;
    unsigned long long n_db = 0;  // row length of inner / overlap
    const int32_t* inner = nullptr;    // [batch * rho][n_db]
    const int32_t* overlap = nullptr;  // [batch * rho][n_db]
    double* folded = nullptr;          // [batch][blocks][groups][d] or null
    double* refolded = nullptr;        // [batch][blocks][d] or null
    uint32_t* flags = nullptr;         // [0] folding assumption violated, [1] empty overlap
};

// Validates p in PipelineConfig::validate's order (pipeline.cpp:232-243) and
// fills everything but the buffer pointers. want_refold: the caller asked for
// the refolded output, which runs the chain (eval_chain_ct rejects an empty
// one, pipeline.cpp:382).
int fold_prepare(irl_ctx* ctx, const irl_fold_params* p, bool want_refold, FoldArgs* a);
// Fills the context's reciprocal table up to a.d (once, synchronously) and
// launches the fold kernel on s. Counts its launches in ctx.
int launch_fold_stage(irl_ctx* ctx, FoldArgs& a, cudaStream_t s);

}  // namespace irl
