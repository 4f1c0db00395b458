// Alg. 2 fold stage on the device, message level: see the
// contract in include/irl_capi.h (irl_fold_stage) and fold.cuh.
//
// One thread per output slot (eye e, DB block b, slot i). It walks the
// rotation groups; for each rotation r of a group it reads the product and
// the overlap at column c = e*rho + r, template b*d + (i + r) mod d (for a
// fixed r the threads of a warp read consecutive templates, so the int32
// rows stream coalesced), normalizes, runs the folding polynomial and sums
// the group; the fold chain and the refold across groups follow in
// registers. Every (column, template) pair is read exactly once, so the
// kernel moves 8 B per pair plus the outputs: HBM-bound at paper scale
// (992 x 114688 pairs = 0.91 GB).
//
// Bit parity with the reference's noise-free emulator: each ring operation is
// one IEEE double operation in the reference's order -- __dmul_rn / __dadd_rn
// / __ddiv_rn keep nvcc from contracting a multiply and an add into an FMA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/irl_capi.h"
#include "ctx_internal.h"
#include "fold.cuh"

namespace irl {

namespace {

// ---- Paterson-Stockmeyer plan of poly.hpp:46-119, resolved at compile time --

__host__ __device__ constexpr int ps_depth(int degree) {  // poly.hpp:50-54
    int k = 0;
    while ((1 << k) < degree + 1) ++k;
    return k;
}
__host__ __device__ constexpr int ps_baby_m(int degree) {  // poly.hpp:56-60
    return degree == 0 ? 1 : 1 << ((ps_depth(degree) + 1) / 2);
}
__host__ __device__ constexpr int ps_giants(int degree) {  // giant powers x^m, x^2m, ... (poly.hpp:103-111)
    const int m = ps_baby_m(degree);
    if (degree + 1 <= m) return 0;
    int n = 1, pw = m;
    while (pw * 2 < degree + 1) {
        ++n;
        pw *= 2;
    }
    return n;
}
__host__ __device__ constexpr int ps_split(int n, int m) {  // largest m * 2^t < n (poly.hpp:76-81)
    int split = m;
    while (split * 2 < n) split *= 2;
    return split;
}
__host__ __device__ constexpr int ps_giant_index(int n, int m) {
    int split = m, g = 0;
    while (split * 2 < n) {
        split *= 2;
        ++g;
    }
    return g;
}

// CtRing::axpb (pipeline.cpp:41-43): pmult_const(x, a) then add_const(b)
__device__ __forceinline__ double ring_axpb(double a, double x, double b) {
    return __dadd_rn(__dmul_rn(x, a), b);
}

// detail::ps_eval_range (poly.hpp:62-86): sum_{i in [LO, HI)} c[i] x^(i-LO)
template <int LO, int HI, int M>
__device__ __forceinline__ double ps_range(const double* c, const double* baby, const double* giant) {
    constexpr int N = HI - LO;
    if constexpr (N <= M) {
        double acc = ring_axpb(0.0, baby[0], c[LO]);
#pragma unroll
        for (int i = 1; i < N; ++i) acc = __dadd_rn(acc, ring_axpb(c[LO + i], baby[i - 1], 0.0));
        return acc;
    } else {
        constexpr int S = ps_split(N, M);
        constexpr int G = ps_giant_index(N, M);
        const double low = ps_range<LO, LO + S, M>(c, baby, giant);
        const double high = ps_range<LO + S, HI, M>(c, baby, giant);
        return __dadd_rn(__dmul_rn(high, giant[G]), low);
    }
}

// ps_execute (poly.hpp:91-119) for a polynomial of degree D (c has D + 1 entries)
template <int D>
__device__ __forceinline__ double ps_eval(const double* c, double x) {
    if constexpr (D == 0) {
        return ring_axpb(0.0, x, c[0]);
    } else {
        constexpr int M = ps_baby_m(D);
        constexpr int NB = M < D ? M : D;
        constexpr int NG = ps_giants(D);
        double baby[NB];
        baby[0] = x;
#pragma unroll
        for (int j = 2; j <= NB; ++j) baby[j - 1] = __dmul_rn(baby[(j + 1) / 2 - 1], baby[j / 2 - 1]);
        double giant[NG > 0 ? NG : 1];
        if constexpr (NG > 0) {
            giant[0] = baby[M - 1];
#pragma unroll
            for (int g = 1; g < NG; ++g) giant[g] = __dmul_rn(giant[g - 1], giant[g - 1]);
        }
        return ps_range<0, D + 1, M>(c, baby, giant);
    }
}

template <int D>
__device__ __forceinline__ double ps_dispatch_from(int deg, const double* c, double x) {
    if constexpr (D > kFoldMaxDegree) {
        return 0.0;  // unreachable: fold_prepare bounds the degree
    } else {
        if (deg == D) return ps_eval<D>(c, x);
        return ps_dispatch_from<D + 1>(deg, c, x);
    }
}

__device__ __forceinline__ double ps_dispatch(int deg, const double* c, double x) {
    switch (deg) {  // the common degrees first (fold poly 7, classifier stages 15 / 31)
        case 7: return ps_eval<7>(c, x);
        case 15: return ps_eval<15>(c, x);
        case 31: return ps_eval<31>(c, x);
        default: return ps_dispatch_from<0>(deg, c, x);
    }
}

__global__ void __launch_bounds__(256) fold_stage_kernel(const FoldArgs a) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.d) return;
    const uint32_t b = blockIdx.y, e = blockIdx.z;
    const uint32_t dmask = a.d - 1;
    const size_t base = static_cast<size_t>(b) * a.d;
    double refold = 0.0;
    bool violated = false, empty = false;
    for (uint32_t g = 0; g < a.groups; ++g) {
        const uint32_t r0 = g * a.fold_k;
        const uint32_t r_end = min(a.rho, r0 + a.fold_k);
        double acc = 0.0;
        int non_d = 0;
        for (uint32_t r = r0; r < r_end; ++r) {
            const size_t c = static_cast<size_t>(e) * a.rho + r;
            const size_t off = c * a.n_db + base + ((i + r) & dmask);
            const double raw = static_cast<double>(__ldcs(a.inner + off));
            const double ov = static_cast<double>(__ldcs(a.overlap + off));
            // folding-assumption shadow check (pipeline.cpp:574-583)
            if (ov == 0.0) {
                empty = true;
                ++non_d;
            } else {
                const double q = __ddiv_rn(raw, ov);
                if (!(q >= a.neg_lo && q <= a.neg_hi)) ++non_d;
            }
            // normalize: message * (1.0 / overlap) (pipeline.cpp:364-369)
            const double x = __dmul_rn(raw, __ddiv_rn(1.0, ov));
            const double t = ps_dispatch(a.fold_deg, a.fold_c, x);
            acc = r == r0 ? t : __dadd_rn(acc, t);  // fold_group's running sum (pipeline.cpp:397-406)
        }
        if (non_d > 1) violated = true;
        const size_t eb = static_cast<size_t>(e) * a.blocks + b;
        if (a.folded) a.folded[(eb * a.groups + g) * a.d + i] = acc;
        if (a.refolded) {
            double cls = acc;
            for (int s = 0; s < a.nstages; ++s)  // eval_chain_ct (pipeline.cpp:383-388)
                cls = ps_dispatch(a.stage_deg[s], a.chain_c[s], __dadd_rn(cls, -a.center[s]));
            refold = g == 0 ? cls : __dadd_rn(refold, cls);  // refold (pipeline.cpp:620-626)
        }
    }
    if (a.refolded) a.refolded[(static_cast<size_t>(e) * a.blocks + b) * a.d + i] = refold;
    if (violated) atomicOr(a.flags, 1u);
    if (empty) atomicOr(a.flags + 1, 1u);
}

int degree_of(const double* c, size_t n) {  // Polynomial::degree (poly.cpp:10-15)
    for (size_t i = n; i-- > 0;)
        if (c[i] != 0.0) return static_cast<int>(i);
    return 0;
}

}  // namespace

int fold_prepare(irl_ctx* ctx, const irl_fold_params* p, bool want_refold, FoldArgs* a) {
    if (!p || !a) return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "fold: null parameters");
    // PipelineConfig::validate (pipeline.cpp:232-243), same order and messages
    if (p->rho < 1 || p->batch < 1) return set_err(ctx, IRL_ERR_CONFIG, "pipeline: rho and batch must be >= 1");
    if (p->fold_k < 1 || p->fold_k > p->rho)
        return set_err(ctx, IRL_ERR_CONFIG, "pipeline: fold_k must satisfy 1 <= k <= rho");
    if (p->d < 2 || (p->d & (p->d - 1)) != 0) return set_err(ctx, IRL_ERR_CONFIG, "pipeline: d must be a power of two");
    if (p->n_db < p->d || p->n_db % p->d != 0)
        return set_err(ctx, IRL_ERR_CONFIG, "pipeline: n_db must be a positive multiple of d");
    if (want_refold && p->chain_stages == 0) return set_err(ctx, IRL_ERR_CONFIG, "eval_chain_ct: empty chain");
    if (p->chain_stages > static_cast<size_t>(kFoldMaxStages))
        return set_err(ctx, IRL_ERR_UNSUPPORTED, "fold: at most 8 chain stages");
    if ((p->fold_len && !p->fold_coeffs) ||
        (p->chain_stages && (!p->chain_centers || !p->chain_lens)))
        return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "fold: null coefficient buffer");
    const size_t blocks = p->n_db / p->d;
    const size_t cols = p->batch * p->rho;
    if (p->d > (size_t{1} << 30) || blocks > 65535 || p->batch > 65535 || cols * p->n_db >= (size_t{1} << 40))
        return set_err(ctx, IRL_ERR_UNSUPPORTED, "fold: dimensions too large");
    std::memset(a->fold_c, 0, sizeof(a->fold_c));
    std::memset(a->chain_c, 0, sizeof(a->chain_c));
    std::memset(a->center, 0, sizeof(a->center));
    std::memset(a->stage_deg, 0, sizeof(a->stage_deg));
    a->fold_deg = degree_of(p->fold_coeffs, p->fold_len);
    if (a->fold_deg > kFoldMaxDegree) return set_err(ctx, IRL_ERR_UNSUPPORTED, "fold: polynomial degree above 31");
    for (int k = 0; k <= a->fold_deg; ++k) a->fold_c[k] = p->fold_coeffs[k];
    size_t off = 0;
    a->nstages = static_cast<int>(p->chain_stages);
    for (size_t s = 0; s < p->chain_stages; ++s) {
        const size_t n = p->chain_lens[s];
        if (n && !p->chain_coeffs) return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "fold: null coefficient buffer");
        const int deg = degree_of(p->chain_coeffs + off, n);
        if (deg > kFoldMaxDegree) return set_err(ctx, IRL_ERR_UNSUPPORTED, "fold: polynomial degree above 31");
        a->stage_deg[s] = deg;
        a->center[s] = p->chain_centers[s];
        for (int k = 0; k <= deg && static_cast<size_t>(k) < n; ++k) a->chain_c[s][k] = p->chain_coeffs[off + k];
        off += n;
    }
    a->neg_lo = p->negative_lo;
    a->neg_hi = p->negative_hi;
    a->batch = static_cast<uint32_t>(p->batch);
    a->rho = static_cast<uint32_t>(p->rho);
    a->blocks = static_cast<uint32_t>(blocks);
    a->d = static_cast<uint32_t>(p->d);
    a->fold_k = static_cast<uint32_t>(p->fold_k);
    a->groups = static_cast<uint32_t>((p->rho + p->fold_k - 1) / p->fold_k);
    a->n_db = p->n_db;
    return IRL_OK;
}

cudaError_t launch_fold_stage(const FoldArgs& a, cudaStream_t s) {
    const dim3 grid((a.d + 255) / 256, a.blocks, a.batch);
    fold_stage_kernel<<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace irl

using namespace irl;

extern "C" {

int irl_fold_stage_device(irl_ctx* ctx, const irl_fold_params* p, const int32_t* inner, const int32_t* overlap,
                          double* folded, double* refolded, uint32_t* flags, void* stream) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx);
    FoldArgs a;
    if (int st = fold_prepare(ctx, p, refolded != nullptr, &a)) return st;
    if (!inner || !overlap || !flags) return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "fold: null buffer");
    a.inner = inner;
    a.overlap = overlap;
    a.folded = folded;
    a.refolded = refolded;
    a.flags = flags;
    IRL_LAUNCH(ctx, launch_fold_stage(a, pick_stream(ctx, stream)));
    return IRL_OK;
}

int irl_fold_stage(irl_ctx* ctx, const irl_fold_params* p, const int32_t* inner, const int32_t* overlap,
                   double* folded, double* refolded, int32_t* assumption_ok) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx);
    FoldArgs a;
    if (int st = fold_prepare(ctx, p, refolded != nullptr, &a)) return st;
    if (!inner || !overlap) return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "fold: null buffer");
    cudaStream_t s = ctx->stream;
    const size_t cols = p->batch * p->rho, in_bytes = cols * p->n_db * sizeof(int32_t);
    const size_t fold_elems = size_t(a.batch) * a.blocks * a.groups * a.d;
    const size_t refold_elems = size_t(a.batch) * a.blocks * a.d;
    const size_t off_f = 0, off_r = off_f + (folded ? fold_elems * 8 : 0), off_flags = off_r + (refolded ? refold_elems * 8 : 0);
    IRL_CK(ctx, ctx->ws[3].ensure(2 * in_bytes));
    IRL_CK(ctx, ctx->ws[5].ensure(off_flags + 16));
    auto* din = ctx->ws[3].as<int32_t>();
    auto* dov = reinterpret_cast<int32_t*>(ctx->ws[3].as<uint8_t>() + in_bytes);
    uint8_t* out = ctx->ws[5].as<uint8_t>();
    auto* dflags = reinterpret_cast<uint32_t*>(out + off_flags);
    IRL_CK(ctx, copy_h2d(ctx, din, inner, in_bytes, s));
    IRL_CK(ctx, copy_h2d(ctx, dov, overlap, in_bytes, s));
    IRL_CK(ctx, cudaMemsetAsync(dflags, 0, 8, s));
    a.inner = din;
    a.overlap = dov;
    a.folded = folded ? reinterpret_cast<double*>(out + off_f) : nullptr;
    a.refolded = refolded ? reinterpret_cast<double*>(out + off_r) : nullptr;
    a.flags = dflags;
    IRL_LAUNCH(ctx, launch_fold_stage(a, s));
    if (folded) IRL_CK(ctx, copy_d2h(ctx, folded, a.folded, fold_elems * 8, s));
    if (refolded) IRL_CK(ctx, copy_d2h(ctx, refolded, a.refolded, refold_elems * 8, s));
    uint32_t hf[2] = {0, 0};
    IRL_CK(ctx, cudaMemcpyAsync(hf, dflags, 8, cudaMemcpyDeviceToHost, s));
    IRL_CK(ctx, cudaStreamSynchronize(s));
    if (assumption_ok) *assumption_ok = hf[0] ? 0 : 1;
    if (hf[1]) return set_err(ctx, IRL_ERR_ZERO_OVERLAP, "mask overlap is empty, score undefined");
    return IRL_OK;
}

}  // extern "C"
