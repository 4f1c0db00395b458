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
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/irl_capi.h"
#include "ctx_internal.h"
#include "fold.cuh"

#ifndef IRL_FOLD_PREFETCH
#define IRL_FOLD_PREFETCH 1  // 0: the r07 loop (A/B variant builds)
#endif

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

// Two evaluation modes with identical results:
//  * exact (kFast = false): every ring operation of the reference, including
//    the axpb(0, x, c) leaf starts and the "+ 0.0" of axpb(c, x, 0);
//  * fast (kFast = true), valid when no coefficient is -0.0 (fold_prepare
//    checks): a leaf's running sum never becomes -0 (it starts at
//    RN(RN(x * 0) + c), which is -0 only for c = -0, and RN(a + b) is -0 only
//    for a = b = -0), so RN(acc + RN(RN(b * c) + 0)) = RN(acc + RN(b * c)):
//    the "+ 0.0" only turns a -0 product into +0, which no acc != -0 can see.
//    That drops 6 of the 27 double operations of a degree-7 evaluation.

// detail::ps_eval_range (poly.hpp:62-86): sum_{i in [LO, HI)} c[i] x^(i-LO)
template <bool kFast, int LO, int HI, int M>
__device__ __forceinline__ double ps_range(const double* c, const double* baby, const double* giant) {
    constexpr int N = HI - LO;
    if constexpr (N <= M) {
        double acc;
        if constexpr (kFast) {
            acc = ring_axpb(0.0, baby[0], c[LO]);
#pragma unroll
            for (int i = 1; i < N; ++i) acc = __dadd_rn(acc, __dmul_rn(baby[i - 1], c[LO + i]));
        } else {
            acc = ring_axpb(0.0, baby[0], c[LO]);
#pragma unroll
            for (int i = 1; i < N; ++i) acc = __dadd_rn(acc, ring_axpb(c[LO + i], baby[i - 1], 0.0));
        }
        return acc;
    } else {
        constexpr int S = ps_split(N, M);
        constexpr int G = ps_giant_index(N, M);
        const double low = ps_range<kFast, LO, LO + S, M>(c, baby, giant);
        const double high = ps_range<kFast, LO + S, HI, M>(c, baby, giant);
        return __dadd_rn(__dmul_rn(high, giant[G]), low);
    }
}

// ps_execute (poly.hpp:91-119) for a polynomial of degree D (c has D + 1 entries)
template <bool kFast, int D>
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
        return ps_range<kFast, 0, D + 1, M>(c, baby, giant);
    }
}

template <bool kFast, int D>
__device__ __forceinline__ double ps_dispatch_from(int deg, const double* c, double x) {
    if constexpr (D > kFoldMaxDegree) {
        return 0.0;  // unreachable: fold_prepare bounds the degree
    } else {
        if (deg == D) return ps_eval<kFast, D>(c, x);
        return ps_dispatch_from<kFast, D + 1>(deg, c, x);
    }
}

template <bool kFast>
__device__ __forceinline__ double ps_dispatch(int deg, const double* c, double x) {
    switch (deg) {  // the common degrees first (fold poly 7, classifier stages 15 / 31)
        case 7: return ps_eval<kFast, 7>(c, x);
        case 15: return ps_eval<kFast, 15>(c, x);
        case 31: return ps_eval<kFast, 31>(c, x);
        default: return ps_dispatch_from<kFast, 0>(deg, c, x);
    }
}

// Folding polynomial of a compile-time degree (kFoldDeg >= 0: the reference's
// degree-7 polynomial takes this path) or any degree <= 31 (kFoldDeg < 0).
template <bool kFast, int kFoldDeg>
__device__ __forceinline__ double fold_poly(const FoldArgs& a, const double* fc, double x) {
    if constexpr (kFoldDeg >= 0) {
        return ps_eval<kFast, kFoldDeg>(fc, x);  // coefficients held in registers
    } else {
        return ps_dispatch<kFast>(a.fold_deg, a.fold_c, x);
    }
}

// !negative.contains(raw / ov) for ov != 0 (pipeline.cpp:580). x = raw *
// RN(1 / ov) is within 2^-51 |q| of the IEEE quotient q, so outside the
// bands [lo_out, lo_in] and [hi_in, hi_out] (2^-48 |bound| wide, fold_prepare)
// x decides; inside a band the quotient is formed.
__device__ __forceinline__ bool outside_negative(const FoldArgs& a, int32_t raw, int32_t ov, double x) {
    if (x >= a.lo_in && x <= a.hi_in) return false;
    if (x < a.lo_out || x > a.hi_out) return true;
    const double q = __ddiv_rn(static_cast<double>(raw), static_cast<double>(ov));
    return !(q >= a.neg_lo && q <= a.neg_hi);
}

template <bool kFast, int kFoldDeg>
__global__ void __launch_bounds__(256, 8) fold_stage_kernel(const FoldArgs a) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.d) return;
    const uint32_t b = blockIdx.y, e = blockIdx.z;
    const uint32_t dmask = a.d - 1;
    const int32_t* inner = a.inner + static_cast<size_t>(e) * a.rho * a.n_db + static_cast<size_t>(b) * a.d;
    const int32_t* overlap = a.overlap + static_cast<size_t>(e) * a.rho * a.n_db + static_cast<size_t>(b) * a.d;
    double fc[kFoldDeg >= 0 ? kFoldDeg + 1 : 1];
#pragma unroll
    for (int k = 0; k < (kFoldDeg >= 0 ? kFoldDeg + 1 : 1); ++k) fc[k] = a.fold_c[k];
    double refold = 0.0;
    bool violated = false, empty = false;
    for (uint32_t g = 0; g < a.groups; ++g) {
        const uint32_t r0 = g * a.fold_k;
        const uint32_t r_end = min(a.rho, r0 + a.fold_k);
        double acc = 0.0;
        int non_d = 0;
        const int32_t* in_row = inner + static_cast<size_t>(r0) * a.n_db;
        const int32_t* ov_row = overlap + static_cast<size_t>(r0) * a.n_db;
        uint32_t j = (i + r0) & dmask;
#if IRL_FOLD_PREFETCH
        // Software-pipelined: the next rotation's product and overlap are
        // loaded while this one is evaluated (its row is the current one again
        // on the group's last rotation, so no load leaves the group's rows),
        // and the shadow check is predicated, with the exact quotient behind
        // one rarely taken branch.
        int32_t raw_n = __ldcs(in_row + j), ov_n = __ldcs(ov_row + j);
        for (uint32_t r = r0; r < r_end; ++r) {
            const int32_t raw = raw_n, ov = ov_n;
            const size_t step = r + 1 < r_end ? a.n_db : 0;
            in_row += step;
            ov_row += step;
            j = step ? (j + 1) & dmask : j;
            raw_n = __ldcs(in_row + j);
            ov_n = __ldcs(ov_row + j);
            // normalize: message * (1.0 / overlap) (pipeline.cpp:364-369);
            // rcp[k] = RN(1 / k) for the overlaps a template can have
            const double inv = static_cast<uint32_t>(ov) <= a.rcp_max ? __ldg(a.rcp + ov)
                                                                      : __drcp_rn(static_cast<double>(ov));
            const double x = __dmul_rn(static_cast<double>(raw), inv);
            // folding-assumption shadow check (pipeline.cpp:574-583): x decides
            // outside the bands around the interval ends (see outside_negative)
            const bool zero = ov == 0;
            const bool sure_in = x >= a.lo_in && x <= a.hi_in;
            const bool sure_out = x < a.lo_out || x > a.hi_out;
            bool outside = sure_out;
            if (!zero && !sure_in && !sure_out) {
                const double q = __ddiv_rn(static_cast<double>(raw), static_cast<double>(ov));
                outside = !(q >= a.neg_lo && q <= a.neg_hi);
            }
            non_d += (zero || outside) ? 1 : 0;
            empty = empty || zero;
            const double t = fold_poly<kFast, kFoldDeg>(a, fc, x);
            acc = r == r0 ? t : __dadd_rn(acc, t);  // fold_group's running sum (pipeline.cpp:397-406)
        }
#else
        for (uint32_t r = r0; r < r_end; ++r, in_row += a.n_db, ov_row += a.n_db, j = (j + 1) & dmask) {
            const int32_t raw = __ldcs(in_row + j);
            const int32_t ov = __ldcs(ov_row + j);
            const double inv = static_cast<uint32_t>(ov) <= a.rcp_max ? __ldg(a.rcp + ov)
                                                                      : __drcp_rn(static_cast<double>(ov));
            const double x = __dmul_rn(static_cast<double>(raw), inv);
            if (ov == 0) {
                empty = true;
                ++non_d;
            } else if (outside_negative(a, raw, ov, x)) {
                ++non_d;
            }
            const double t = fold_poly<kFast, kFoldDeg>(a, fc, x);
            acc = r == r0 ? t : __dadd_rn(acc, t);  // fold_group's running sum (pipeline.cpp:397-406)
        }
#endif
        if (non_d > 1) violated = true;
        const size_t eb = static_cast<size_t>(e) * a.blocks + b;
        if (a.folded) a.folded[(eb * a.groups + g) * a.d + i] = acc;
        if (a.refolded) {
            double cls = acc;
            for (int s = 0; s < a.nstages; ++s)  // eval_chain_ct (pipeline.cpp:383-388)
                cls = ps_dispatch<kFast>(a.stage_deg[s], a.chain_c[s], __dadd_rn(cls, -a.center[s]));
            refold = g == 0 ? cls : __dadd_rn(refold, cls);  // refold (pipeline.cpp:620-626)
        }
    }
    if (a.refolded) a.refolded[(static_cast<size_t>(e) * a.blocks + b) * a.d + i] = refold;
    if (violated) atomicOr(a.flags, 1u);
    if (empty) atomicOr(a.flags + 1, 1u);
}

__global__ void rcp_table_kernel(double* rcp, uint32_t n) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) rcp[k] = __drcp_rn(static_cast<double>(k));  // correctly rounded 1.0 / k
}

bool has_negative_zero(const double* c, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (c[i] == 0.0 && std::signbit(c[i])) return true;
    return false;
}

// Band edges around an interval end v: |x - q| <= 2^-51 |q| near v.
void band(double v, double* in_side, double* out_side, double dir) {
    if (!std::isfinite(v)) {
        *in_side = *out_side = v;
        return;
    }
    const double w = std::fabs(v) * 0x1p-48 + 0x1p-1000;
    *in_side = v + dir * w;
    *out_side = v - dir * w;
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
    for (int k = 0; k <= a->fold_deg && static_cast<size_t>(k) < p->fold_len; ++k) a->fold_c[k] = p->fold_coeffs[k];
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
    band(a->neg_lo, &a->lo_in, &a->lo_out, 1.0);
    band(a->neg_hi, &a->hi_in, &a->hi_out, -1.0);
    a->fast = !has_negative_zero(a->fold_c, kFoldMaxDegree + 1);
    for (int s = 0; s < a->nstages; ++s) a->fast = a->fast && !has_negative_zero(a->chain_c[s], kFoldMaxDegree + 1);
    a->batch = static_cast<uint32_t>(p->batch);
    a->rho = static_cast<uint32_t>(p->rho);
    a->blocks = static_cast<uint32_t>(blocks);
    a->d = static_cast<uint32_t>(p->d);
    a->fold_k = static_cast<uint32_t>(p->fold_k);
    a->groups = static_cast<uint32_t>((p->rho + p->fold_k - 1) / p->fold_k);
    a->n_db = p->n_db;
    return IRL_OK;
}

int launch_fold_stage(irl_ctx* ctx, FoldArgs& a, cudaStream_t s) {
    const uint32_t need = a.d + 1;  // an overlap never exceeds the template length d
    if (ctx->rcp_n < need) {
        IRL_CK(ctx, ctx->rcp.ensure(size_t(need) * sizeof(double)));
        rcp_table_kernel<<<(need + 255) / 256, 256, 0, s>>>(ctx->rcp.as<double>(), need);
        IRL_LAUNCH(ctx, cudaGetLastError());
        IRL_CK(ctx, cudaStreamSynchronize(s));  // later calls may read it from other streams
        ctx->rcp_n = need;
    }
    a.rcp = ctx->rcp.as<double>();
    a.rcp_max = ctx->rcp_n - 1;
    const dim3 grid((a.d + 255) / 256, a.blocks, a.batch);
    if (a.fast && a.fold_deg == 7)
        fold_stage_kernel<true, 7><<<grid, 256, 0, s>>>(a);
    else if (a.fast)
        fold_stage_kernel<true, -1><<<grid, 256, 0, s>>>(a);
    else
        fold_stage_kernel<false, -1><<<grid, 256, 0, s>>>(a);
    IRL_LAUNCH(ctx, cudaGetLastError());
    return IRL_OK;
}

}  // namespace irl

using namespace irl;

extern "C" {

int irl_fold_stage_device(irl_ctx* ctx, const irl_fold_params* p, const int32_t* inner, const int32_t* overlap,
                          double* folded, double* refolded, uint32_t* flags, void* stream) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx, __func__);
    FoldArgs a;
    if (int st = fold_prepare(ctx, p, refolded != nullptr, &a)) return st;
    if (!inner || !overlap || !flags) return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "fold: null buffer");
    a.inner = inner;
    a.overlap = overlap;
    a.folded = folded;
    a.refolded = refolded;
    a.flags = flags;
    return launch_fold_stage(ctx, a, pick_stream(ctx, stream));
}

int irl_fold_stage(irl_ctx* ctx, const irl_fold_params* p, const int32_t* inner, const int32_t* overlap,
                   double* folded, double* refolded, int32_t* assumption_ok) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx, __func__);
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
    if (int st = launch_fold_stage(ctx, a, s)) return st;
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
