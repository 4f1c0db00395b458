// Plaintext iris scoring stage on the tensor cores.
//
// The server-side plaintext work around the encrypted CCMM in the reference:
//   * mask overlaps |m_db(j) AND m_qry(c)| for every (query column, template)
//     (pipeline.cpp:140-151, overlap_count :78-82, pack_bits :70-76), the
//     plaintext vector `normalize` divides by (pipeline.cpp:359-371);
//   * the ternary inner products <a', b'> and scores inner / overlap
//     (iris_core.cpp:37-59), and the plaintext ground-truth matcher
//     match_db_reference (iris_core.cpp:78-90) with its early-exit and
//     ZeroOverlap semantics.
//
// Both integer sums are int8 GEMMs over K = d: acc1 = X0 Y0 with X0/Y0 the
// ternary planes c' = m - 2 (c & m) (to_masked, iris_core.cpp:28-35), and
// acc2 = X1 Y1 with X1/Y1 the 0/1 mask planes. They run through the PPMM
// kernel in kModeInner (two products per K step, raw int32 epilogue).
// Query column c = e * rho + r holds rotate(q_e, r) (iris_core.cpp:65-76),
// built on the device from the packed eye templates.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "ctx_internal.h"

using namespace irl;

namespace {

// Packed templates (little-endian bit order, `words` uint64 per template) ->
// K-major int8 planes: planes[0][c][ldk] = to_masked(rotate(t_e, r)),
// planes[1][c][ldk] = its mask, for column c = e * rho + r. Entries k >= d are 0.
// One thread writes 16 consecutive k of one column to each plane.
__global__ void iris_planes_kernel(const uint64_t* __restrict__ code, const uint64_t* __restrict__ mask,
                                   uint32_t words, uint32_t d, uint32_t rho, uint32_t cols, uint32_t ldk,
                                   int8_t* __restrict__ planes) {
    const uint32_t chunks = ldk / 16;
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= static_cast<size_t>(cols) * chunks) return;
    const uint32_t c = static_cast<uint32_t>(tid / chunks);
    const uint32_t k0 = static_cast<uint32_t>(tid % chunks) * 16;
    const uint32_t e = c / rho, r = c % rho % d;
    const uint64_t* cw = code + static_cast<size_t>(e) * words;
    const uint64_t* mw = mask + static_cast<size_t>(e) * words;
    uint32_t v[4] = {0, 0, 0, 0}, w[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t k = k0 + j;
        if (k >= d) break;
        // rotate: out[(i + r) % d] = t[i]  =>  out[k] = t[(k - r) mod d]
        const uint32_t i = k >= r ? k - r : k + d - r;
        const uint32_t cb = static_cast<uint32_t>((__ldg(cw + (i >> 6)) >> (i & 63)) & 1u);
        const uint32_t mb = static_cast<uint32_t>((__ldg(mw + (i >> 6)) >> (i & 63)) & 1u);
        const int32_t t = static_cast<int32_t>(mb) - 2 * static_cast<int32_t>(cb & mb);
        v[j / 4] |= (static_cast<uint32_t>(t) & 0xFFu) << (8 * (j % 4));
        w[j / 4] |= mb << (8 * (j % 4));
    }
    const size_t o = static_cast<size_t>(c) * ldk + k0;
    *reinterpret_cast<uint4*>(planes + o) = make_uint4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<uint4*>(planes + static_cast<size_t>(cols) * ldk + o) = make_uint4(w[0], w[1], w[2], w[3]);
}

// inner / overlap [cols][n_db] -> per-(eye, template) match bits (OR over the
// eye's rho rotations of score in [lo, hi]), optional scores, and per eye the
// first match / first empty overlap in match_db_reference's iteration order
// (rotation-major, then template: linear index r * n_db + j).
__global__ void iris_match_kernel(const int32_t* __restrict__ inner, const int32_t* __restrict__ overlap,
                                  uint32_t n_db, uint32_t n_eyes, uint32_t rho, double lo, double hi,
                                  uint8_t* __restrict__ bits, double* __restrict__ scores,
                                  unsigned long long* __restrict__ first /* [n_eyes][2] */) {
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= static_cast<size_t>(n_eyes) * n_db) return;
    const uint32_t e = static_cast<uint32_t>(tid / n_db), j = static_cast<uint32_t>(tid % n_db);
    unsigned long long fm = ~0ull, fz = ~0ull;
    uint8_t any = 0;
    for (uint32_t r = 0; r < rho; ++r) {
        const size_t idx = static_cast<size_t>(e * rho + r) * n_db + j;
        const int32_t ov = overlap[idx];
        const unsigned long long lin = static_cast<unsigned long long>(r) * n_db + j;
        if (ov == 0) {
            if (scores) scores[idx] = __longlong_as_double(0x7FF8000000000000ll);  // undefined (ZeroOverlap)
            fz = min(fz, lin);
            continue;
        }
        // iris_core.cpp:58: static_cast<double>(inner) / static_cast<double>(overlap), IEEE division
        const double s = __ddiv_rn(static_cast<double>(inner[idx]), static_cast<double>(ov));
        if (scores) scores[idx] = s;
        if (s >= lo && s <= hi) {  // Interval::contains (iris_core.hpp)
            any = 1;
            fm = min(fm, lin);
        }
    }
    if (bits) bits[tid] = any;
    if (fm != ~0ull) atomicMin(first + 2 * e, fm);
    if (fz != ~0ull) atomicMin(first + 2 * e + 1, fz);
}

size_t round16(size_t x) { return (x + 15) / 16 * 16; }

// Shared front half: planes for the DB and the rotated queries, and the
// kModeInner GEMM into device inner / overlap [cols][n_db].
int inner_overlap_device(irl_ctx* ctx, const uint64_t* db_code, const uint64_t* db_mask, size_t n_db,
                         const uint64_t* q_code, const uint64_t* q_mask, size_t n_eyes, size_t rho, size_t d,
                         int32_t** d_inner, int32_t** d_overlap) {
    cudaStream_t s = ctx->stream;
    const size_t words = (d + 63) / 64, ldk = round16(d), cols = n_eyes * rho;
    if (d > (1u << 30) || n_db >= (1u << 29) || cols >= (1u << 29))
        return set_err(ctx, IRL_ERR_UNSUPPORTED, "iris: dimensions too large");
    const size_t db_bits = n_db * words * 8, q_bits = n_eyes * words * 8;
    const size_t db_planes = 2 * n_db * ldk, q_planes = 2 * cols * ldk, outs = cols * n_db * 4;
    IRL_CK(ctx, ctx->ws[0].ensure(2 * db_bits + 2 * q_bits));
    IRL_CK(ctx, ctx->ws[1].ensure(db_planes));
    IRL_CK(ctx, ctx->ws[2].ensure(q_planes));
    IRL_CK(ctx, ctx->ws[3].ensure(2 * outs));
    uint8_t* bitbuf = ctx->ws[0].as<uint8_t>();
    uint64_t* dc = reinterpret_cast<uint64_t*>(bitbuf);
    uint64_t* dm = reinterpret_cast<uint64_t*>(bitbuf + db_bits);
    uint64_t* qc = reinterpret_cast<uint64_t*>(bitbuf + 2 * db_bits);
    uint64_t* qm = reinterpret_cast<uint64_t*>(bitbuf + 2 * db_bits + q_bits);
    IRL_CK(ctx, cudaMemcpyAsync(dc, db_code, db_bits, cudaMemcpyHostToDevice, s));
    IRL_CK(ctx, cudaMemcpyAsync(dm, db_mask, db_bits, cudaMemcpyHostToDevice, s));
    IRL_CK(ctx, cudaMemcpyAsync(qc, q_code, q_bits, cudaMemcpyHostToDevice, s));
    IRL_CK(ctx, cudaMemcpyAsync(qm, q_mask, q_bits, cudaMemcpyHostToDevice, s));
    int8_t* xp = ctx->ws[1].as<int8_t>();
    int8_t* yp = ctx->ws[2].as<int8_t>();
    const uint32_t T = 256;
    {
        const size_t n = n_db * (ldk / 16);
        iris_planes_kernel<<<static_cast<unsigned>((n + T - 1) / T), T, 0, s>>>(
            dc, dm, static_cast<uint32_t>(words), static_cast<uint32_t>(d), 1u, static_cast<uint32_t>(n_db),
            static_cast<uint32_t>(ldk), xp);
        IRL_LAUNCH(ctx, cudaGetLastError());
    }
    {
        const size_t n = cols * (ldk / 16);
        iris_planes_kernel<<<static_cast<unsigned>((n + T - 1) / T), T, 0, s>>>(
            qc, qm, static_cast<uint32_t>(words), static_cast<uint32_t>(d), static_cast<uint32_t>(rho),
            static_cast<uint32_t>(cols), static_cast<uint32_t>(ldk), yp);
        IRL_LAUNCH(ctx, cudaGetLastError());
    }
    int32_t* inner = ctx->ws[3].as<int32_t>();
    int32_t* ovl = inner + cols * n_db;
    PpmmLaunch L;
    L.mode = kModeInner;
    L.a_planes = xp;
    L.b_planes = yp;
    L.out_i32[0] = inner;
    L.out_i32[1] = ovl;
    L.M = static_cast<uint32_t>(n_db);
    L.N = static_cast<uint32_t>(cols);
    L.K = static_cast<uint32_t>(d);
    L.ldk = static_cast<uint32_t>(ldk);
    L.parts = 1;
    L.nprimes = 1;
    L.mc[0] = make_modconst(2, 1);  // unused by kModeInner
    L.progress = ctx->d_progress;
    IRL_LAUNCH(ctx, launch_ppmm_planes(L, s));
    *d_inner = inner;
    *d_overlap = ovl;
    return IRL_OK;
}

int check_args(irl_ctx* ctx, const void* dbc, const void* dbm, size_t n_db, const void* qc, const void* qm,
               size_t n_eyes, size_t d) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    // IrisTemplate::validate (iris_core.cpp:10-19): nonzero length
    if (d == 0) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "code and mask must have identical nonzero length");
    if ((n_db && (!dbc || !dbm)) || (n_eyes && (!qc || !qm)))
        return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "iris: null template buffer");
    return IRL_OK;
}

}  // namespace

extern "C" {

int irl_iris_inner_overlap(irl_ctx* ctx, const uint64_t* db_code, const uint64_t* db_mask, size_t n_db,
                           const uint64_t* q_code, const uint64_t* q_mask, size_t n_eyes, size_t rho, size_t d,
                           int32_t* inner, int32_t* overlap) {
    if (int st = check_args(ctx, db_code, db_mask, n_db, q_code, q_mask, n_eyes, d)) return st;
    Guard g(ctx);
    const size_t cols = n_eyes * rho;
    if (cols == 0 || n_db == 0) return IRL_OK;
    int32_t *di = nullptr, *dov = nullptr;
    if (int st = inner_overlap_device(ctx, db_code, db_mask, n_db, q_code, q_mask, n_eyes, rho, d, &di, &dov))
        return st;
    const size_t bytes = cols * n_db * sizeof(int32_t);
    if (inner) IRL_CK(ctx, cudaMemcpyAsync(inner, di, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    if (overlap) IRL_CK(ctx, cudaMemcpyAsync(overlap, dov, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return IRL_OK;
}

int irl_iris_match(irl_ctx* ctx, const uint64_t* db_code, const uint64_t* db_mask, size_t n_db,
                   const uint64_t* q_code, const uint64_t* q_mask, size_t n_eyes, size_t rho, size_t d,
                   double p_lo, double p_hi, uint8_t* match_bits, int32_t* eye_result, double* scores) {
    if (int st = check_args(ctx, db_code, db_mask, n_db, q_code, q_mask, n_eyes, d)) return st;
    Guard g(ctx);
    const size_t cols = n_eyes * rho;
    if (cols == 0 || n_db == 0) {
        // match_db_reference over an empty product: no score is evaluated
        if (eye_result) std::memset(eye_result, 0, n_eyes * sizeof(int32_t));
        if (match_bits) std::memset(match_bits, 0, n_eyes * n_db);
        return IRL_OK;
    }
    int32_t *di = nullptr, *dov = nullptr;
    if (int st = inner_overlap_device(ctx, db_code, db_mask, n_db, q_code, q_mask, n_eyes, rho, d, &di, &dov))
        return st;
    cudaStream_t s = ctx->stream;
    const size_t nbits = n_eyes * n_db, nsc = cols * n_db;
    IRL_CK(ctx, ctx->ws[4].ensure(16 * n_eyes + nbits + (scores ? nsc * 8 : 0) + 16));
    auto* first = ctx->ws[4].as<unsigned long long>();
    uint8_t* dbits = reinterpret_cast<uint8_t*>(first + 2 * n_eyes);
    double* dsc = scores ? reinterpret_cast<double*>(ctx->ws[4].as<uint8_t>() + ((16 * n_eyes + nbits + 15) / 16 * 16))
                         : nullptr;
    IRL_CK(ctx, cudaMemsetAsync(first, 0xFF, 16 * n_eyes, s));
    const uint32_t T = 256;
    iris_match_kernel<<<static_cast<unsigned>((nbits + T - 1) / T), T, 0, s>>>(
        di, dov, static_cast<uint32_t>(n_db), static_cast<uint32_t>(n_eyes), static_cast<uint32_t>(rho), p_lo,
        p_hi, dbits, dsc, first);
    IRL_LAUNCH(ctx, cudaGetLastError());
    std::vector<unsigned long long> h(2 * n_eyes);
    IRL_CK(ctx, cudaMemcpyAsync(h.data(), first, 16 * n_eyes, cudaMemcpyDeviceToHost, s));
    if (match_bits) IRL_CK(ctx, cudaMemcpyAsync(match_bits, dbits, nbits, cudaMemcpyDeviceToHost, s));
    if (scores) IRL_CK(ctx, cudaMemcpyAsync(scores, dsc, nsc * 8, cudaMemcpyDeviceToHost, s));
    IRL_CK(ctx, cudaStreamSynchronize(s));
    int status = IRL_OK;
    for (size_t e = 0; e < n_eyes; ++e) {
        const unsigned long long fm = h[2 * e], fz = h[2 * e + 1];
        // match_db_reference: the first evaluated score either matches (return
        // true) or throws ZeroOverlap, whichever comes first in loop order
        const int32_t res = fz < fm ? -1 : (fm != ~0ull ? 1 : 0);
        if (eye_result) eye_result[e] = res;
        if (res < 0 && status == IRL_OK)
            status = set_err(ctx, IRL_ERR_ZERO_OVERLAP, "mask overlap is empty, score undefined");
    }
    return status;
}

}  // extern "C"
