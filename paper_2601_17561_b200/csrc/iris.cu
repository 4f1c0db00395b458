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
// kernel: kModeInner writes the raw int32 sums (irl_iris_inner_overlap);
// kModeIrisMatch scores and matches in the epilogue, so only match bits
// leave the GEMM (irl_iris_match, irl_iris_db_match).
// Query column c = e * rho + r holds rotate(q_e, r) (iris_core.cpp:65-76),
// built on the device from the packed eye templates. By default both run on
// the block-scaled FP4 path (kModeInnerF4 / kModeIrisMatchF4, e2m1 planes);
// the fused match of more than 768 columns puts the query columns on M
// (4x1 clusters, one pass over the database; iris_query_rows).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ctx_internal.h"
#include "fold.cuh"

using namespace irl;

namespace {

// The iris products run on the block-scaled FP4 tensor path unless
// IRL_IRIS_I8 is set: ternary values and mask bits are exact in e2m1, and the
// FP32 accumulators hold every partial sum exactly while |sum| <= d < 2^24,
// at twice the int8 rate with half the plane bytes (profiles/fp4_probe.cu;
// all-ones masks at d = 40000 and d = 2^20 checked against the oracle in
// tests/test_iris.py). Longer templates (d >= 2^24, sums no longer exact in
// FP32) run on the int8 path, whose int32 accumulators are exact to 2^31.
constexpr size_t kF4ExactD = size_t(1) << 24;
bool iris_f4(size_t d) {
    static const bool f4 = std::getenv("IRL_IRIS_I8") == nullptr;
    return f4 && d < kF4ExactD;
}
// Bytes of one plane row holding d entries (int8: one per byte; e2m1: two).
size_t plane_kbytes(size_t d) { return iris_f4(d) ? (d + 1) / 2 : d; }
size_t plane_ldk(size_t d) { return round16(plane_kbytes(d)); }

// Column split of the FP4 query batch. A 1 x 4 cluster covers four 240-column
// tiles (960 columns) per pass over the database; a remainder (992 = 960 + 32
// for the paper's batch) would cost a second, mostly padding pass of the
// whole cluster, so it runs as its own launch on plain pairs. Returns the
// columns of the main launch, 0 = no split.
// The FP4 iris products (the fused match and the raw inner products /
// overlaps) put the query columns on M (IrisMatchOut::query_rows) for batches
// of more than 768 columns: one 4x1-cluster pass over the database covers up
// to 1024 columns (four 256-row blocks), so the query planes are not split.
// Smaller batches would leave blocks of the cluster idle and keep the
// database on M. IRL_IRIS_DB_ON_M=1 / IRL_IRIS_QUERY_ON_M=1 force either layout.
// The raw products (inner = true) default to the database on M: with the
// query on M each thread stores 16 consecutive templates of one column, a
// 64-byte run per row instead of the warp's coalesced 128-byte rows, and the
// launch measured slower (1.78 ms against 1.32 + 0.32 ms at the paper's
// scale, profiles/iris_diag.py --inner); it stays available forced.
bool iris_query_rows(size_t d, size_t cols, bool inner = false) {
    if (!iris_f4(d) || std::getenv("IRL_IRIS_DB_ON_M")) return false;
    if (std::getenv("IRL_IRIS_QUERY_ON_M")) return true;
    return !inner && cols > 3 * 256;
}

size_t col_split(size_t cols, size_t d) {
    if (!iris_f4(d) || std::getenv("IRL_IRIS_NO_SPLIT")) return 0;
    const size_t pass = 4 * kF4TileCols;
    const size_t main = cols / pass * pass;
    return main > 0 && main < cols ? main : 0;
}


// One entry of a plane row into the 16-byte chunk being assembled: int8
// value t / mask mb at position j, or their e2m1 nibbles (+1 = 0x2, -1 = 0xA).
template <bool kF4>
__device__ __forceinline__ void put_entry(uint32_t (&v)[4], uint32_t (&w)[4], int j, int32_t t, uint32_t mb) {
    if constexpr (kF4) {
        const uint32_t tv = t == 0 ? 0u : (t > 0 ? 0x2u : 0xAu);
        v[j / 8] |= tv << (4 * (j % 8));
        w[j / 8] |= (mb ? 0x2u : 0u) << (4 * (j % 8));
    } else {
        v[j / 4] |= (static_cast<uint32_t>(t) & 0xFFu) << (8 * (j % 4));
        w[j / 4] |= mb << (8 * (j % 4));
    }
}

// Packed templates (little-endian bit order, `words` uint64 per template) ->
// K-major planes: planes[0][c][ldk] = to_masked(rotate(t_e, r)),
// planes[1][c][ldk] = its mask, for column c = e * rho + r. Entries k >= d are 0.
// One thread writes one 16-byte chunk of one column to each plane (16 entries
// as int8, 32 as e2m1 nibbles, low nibble first).
template <bool kF4>
__global__ void iris_planes_kernel(const uint64_t* __restrict__ code, const uint64_t* __restrict__ mask,
                                   uint32_t words, uint32_t d, uint32_t rho, uint32_t c0, uint32_t cols,
                                   uint32_t ldk, int8_t* __restrict__ planes) {
    constexpr int kPer = kF4 ? 32 : 16;
    const uint32_t chunks = ldk / 16;
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= static_cast<size_t>(cols) * chunks) return;
    const uint32_t cl = static_cast<uint32_t>(tid / chunks);  // column within [c0, c0 + cols)
    const uint32_t c = c0 + cl;
    const uint32_t chunk = static_cast<uint32_t>(tid % chunks);
    const uint32_t k0 = chunk * kPer;
    const uint32_t e = c / rho, r = c % rho % d;
    const uint64_t* cw = code + static_cast<size_t>(e) * words;
    const uint64_t* mw = mask + static_cast<size_t>(e) * words;
    uint32_t v[4] = {0, 0, 0, 0}, w[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const uint32_t k = k0 + j;
        if (k >= d) break;
        // rotate: out[(i + r) % d] = t[i]  =>  out[k] = t[(k - r) mod d]
        const uint32_t i = k >= r ? k - r : k + d - r;
        const uint32_t cb = static_cast<uint32_t>((__ldg(cw + (i >> 6)) >> (i & 63)) & 1u);
        const uint32_t mb = static_cast<uint32_t>((__ldg(mw + (i >> 6)) >> (i & 63)) & 1u);
        put_entry<kF4>(v, w, j, static_cast<int32_t>(mb) - 2 * static_cast<int32_t>(cb & mb), mb);
    }
    const size_t o = static_cast<size_t>(cl) * ldk + chunk * 16;
    *reinterpret_cast<uint4*>(planes + o) = make_uint4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<uint4*>(planes + static_cast<size_t>(cols) * ldk + o) = make_uint4(w[0], w[1], w[2], w[3]);
}

// The reference's template file planes (save_templates, iris_core.cpp:148-196):
// all templates' bits back to back, little-endian bit order (bit i of byte j
// is element 8 j + i) -- so template t, entry k is global bit t * d + k.
// Same outputs as iris_planes_kernel for rho = 1.
template <bool kF4>
__global__ void iris_file_planes_kernel(const uint8_t* __restrict__ code, const uint8_t* __restrict__ mask,
                                        uint32_t d, uint32_t n, uint32_t ldk, int8_t* __restrict__ planes) {
    constexpr int kPer = kF4 ? 32 : 16;
    const uint32_t chunks = ldk / 16;
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= static_cast<size_t>(n) * chunks) return;
    const uint32_t t = static_cast<uint32_t>(tid / chunks);
    const uint32_t chunk = static_cast<uint32_t>(tid % chunks);
    const uint32_t k0 = chunk * kPer;
    uint32_t v[4] = {0, 0, 0, 0}, w[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const uint32_t k = k0 + j;
        if (k >= d) break;
        const size_t bit = static_cast<size_t>(t) * d + k;
        const uint32_t cb = (__ldg(code + (bit >> 3)) >> (bit & 7)) & 1u;
        const uint32_t mb = (__ldg(mask + (bit >> 3)) >> (bit & 7)) & 1u;
        put_entry<kF4>(v, w, j, static_cast<int32_t>(mb) - 2 * static_cast<int32_t>(cb & mb), mb);
    }
    const size_t o = static_cast<size_t>(t) * ldk + chunk * 16;
    *reinterpret_cast<uint4*>(planes + o) = make_uint4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<uint4*>(planes + static_cast<size_t>(n) * ldk + o) = make_uint4(w[0], w[1], w[2], w[3]);
}

// kModeInner GEMM of device planes x (DB, [2][n_db][ldk]) and y (queries,
// [2][cols][ldk]) into inner / overlap [cols][n_db].
int inner_overlap_gemm(irl_ctx* ctx, const int8_t* xp, const int8_t* yp, size_t n_db, size_t cols, size_t d,
                       size_t ldk, int32_t* inner, int32_t* ovl, uint32_t* progress, cudaStream_t s) {
    if (iris_query_rows(d, cols, true)) {
        // one launch, the query planes on M: the outputs [cols][n_db] are the
        // launch's [M][N], each thread storing 16 consecutive templates
        PpmmLaunch L;
        L.mode = kModeInnerF4;
        L.a_planes = yp;
        L.b_planes = xp;
        L.out_i32[0] = inner;
        L.out_i32[1] = ovl;
        L.M = static_cast<uint32_t>(cols);
        L.N = static_cast<uint32_t>(n_db);
        L.K = static_cast<uint32_t>(plane_kbytes(d));
        L.ldk = static_cast<uint32_t>(ldk);
        L.parts = 1;
        L.nprimes = 1;
        L.mc[0] = make_modconst(2, 1);  // unused by the inner modes
        L.progress = progress;
        L.cluster_pm = 4;
        L.cluster_pn = 1;
        L.b_streamed = 1;
        L.iris.query_rows = 1;
        if (ctx->diag && ctx->d_diag) {
            L.stats = ctx->d_diag;
            IRL_CK(ctx, cudaMemsetAsync(ctx->d_diag, 0, 1024 * kStatSlots * sizeof(uint64_t), s));
        }
        IRL_LAUNCH(ctx, launch_ppmm_planes(L, s));
        ctx->launches += ppmm_kernels_last_launch() > 1 ? ppmm_kernels_last_launch() - 1 : 0;  // + filler
        return IRL_OK;
    }
    // one launch per column range of build_query_planes (see col_split)
    const size_t split = col_split(cols, d);
    const size_t ranges[2][2] = {{0, split ? split : cols}, {split, split ? cols - split : 0}};
    for (const auto& rg : ranges) {
        const size_t c0 = rg[0], nc = rg[1];
        if (nc == 0) continue;
        PpmmLaunch L;
        L.mode = iris_f4(d) ? kModeInnerF4 : kModeInner;
        L.a_planes = xp;
        L.b_planes = yp + 2 * c0 * ldk;
        L.out_i32[0] = inner ? inner + c0 * n_db : nullptr;
        L.out_i32[1] = ovl ? ovl + c0 * n_db : nullptr;
        L.M = static_cast<uint32_t>(n_db);
        L.N = static_cast<uint32_t>(nc);
        L.K = static_cast<uint32_t>(plane_kbytes(d));
        L.ldk = static_cast<uint32_t>(ldk);
        L.parts = 1;
        L.nprimes = 1;
        L.mc[0] = make_modconst(2, 1);  // unused by the inner modes
        L.progress = progress;
        if (c0 > 0) L.cluster_pm = L.cluster_pn = 1;  // the remainder on plain pairs
        if (ctx->diag && ctx->d_diag && c0 == 0) {  // irl_diag_ppmm: counters of the main launch
            L.stats = ctx->d_diag;
            IRL_CK(ctx, cudaMemsetAsync(ctx->d_diag, 0, 1024 * kStatSlots * sizeof(uint64_t), s));
        }
        IRL_LAUNCH(ctx, launch_ppmm_planes(L, s));
        ctx->launches += ppmm_kernels_last_launch() > 1 ? ppmm_kernels_last_launch() - 1 : 0;  // + filler
    }
    return IRL_OK;
}

// Planes [2][ncols][ldk] of query columns [c0, c0 + ncols) (column c =
// e * rho + r is rotate(t_e, r)); the database is the case rho = 1.
int build_planes_range(irl_ctx* ctx, const uint64_t* code, const uint64_t* mask, size_t rho, size_t d, size_t c0,
                       size_t ncols, int8_t* planes, cudaStream_t s) {
    const size_t words = (d + 63) / 64, ldk = plane_ldk(d);
    const size_t total = ncols * (ldk / 16);
    if (total == 0) return IRL_OK;
    auto kern = iris_f4(d) ? iris_planes_kernel<true> : iris_planes_kernel<false>;
    kern<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(
        code, mask, static_cast<uint32_t>(words), static_cast<uint32_t>(d), static_cast<uint32_t>(rho),
        static_cast<uint32_t>(c0), static_cast<uint32_t>(ncols), static_cast<uint32_t>(ldk), planes);
    IRL_LAUNCH(ctx, cudaGetLastError());
    return IRL_OK;
}

int build_planes(irl_ctx* ctx, const uint64_t* code, const uint64_t* mask, size_t n, size_t rho, size_t d,
                 int8_t* planes, cudaStream_t s) {
    return build_planes_range(ctx, code, mask, rho, d, 0, n * rho, planes, s);
}

// Query planes, laid out per launch: [2][main][ldk] then [2][rest][ldk].
int build_query_planes(irl_ctx* ctx, const uint64_t* code, const uint64_t* mask, size_t n_eyes, size_t rho,
                       size_t d, int8_t* planes, cudaStream_t s, bool allow_split = true) {
    const size_t cols = n_eyes * rho, split = allow_split ? col_split(cols, d) : 0;
    if (!split) return build_planes_range(ctx, code, mask, rho, d, 0, cols, planes, s);
    if (int st = build_planes_range(ctx, code, mask, rho, d, 0, split, planes, s)) return st;
    return build_planes_range(ctx, code, mask, rho, d, split, cols - split, planes + 2 * split * plane_ldk(d), s);
}

// Scoring fused into the GEMM (kModeIrisMatch): the epilogue divides,
// matches and folds the first match / first empty overlap per eye; only the
// match bits (and optional scores) leave the device. Blocks. Returns
// IRL_ERR_ZERO_OVERLAP if any eye's first evaluated score had an empty overlap.
int match_fused(irl_ctx* ctx, const int8_t* xp, const int8_t* yp, size_t n_db, size_t n_eyes, size_t rho, size_t d,
                size_t ldk, double p_lo, double p_hi, uint8_t* match_bits, int32_t* eye_result, double* scores,
                irl::DevBuf& ws, uint32_t* progress, cudaStream_t s) {
    const size_t cols = n_eyes * rho, nbits = n_eyes * n_db, nsc = cols * n_db;
    if (static_cast<unsigned long long>(rho) * n_db >= 0xFFFFFFFFull)
        return set_err(ctx, IRL_ERR_UNSUPPORTED, "iris: rho * n_db must stay below 2^32");
    const size_t off_bits = 8 * n_eyes, off_sc = (off_bits + nbits + 15) / 16 * 16;
    IRL_CK(ctx, ws.ensure(off_sc + (scores ? nsc * 8 : 0)));
    auto* first = ws.as<uint32_t>();
    uint8_t* dbits = ws.as<uint8_t>() + off_bits;
    double* dsc = scores ? reinterpret_cast<double*>(ws.as<uint8_t>() + off_sc) : nullptr;
    IRL_CK(ctx, cudaMemsetAsync(first, 0xFF, 8 * n_eyes, s));
    IRL_CK(ctx, cudaMemsetAsync(dbits, 0, nbits, s));
    // Query columns on M (iris_query_rows): one launch, the query planes
    // unsplit. Otherwise one launch per column range of build_query_planes
    // (see col_split); the launches fold into the same first-event indices
    // and match bits.
    const bool qrows = iris_query_rows(d, cols);
    const size_t split = qrows ? 0 : col_split(cols, d);
    const size_t ranges[2][2] = {{0, split ? split : cols}, {split, split ? cols - split : 0}};
    for (const auto& rg : ranges) {
        const size_t c0 = rg[0], nc = rg[1];
        if (nc == 0) continue;
        PpmmLaunch L;
        L.mode = iris_f4(d) ? kModeIrisMatchF4 : kModeIrisMatch;
        if (qrows) {
            // A = the query planes (992 rows), B = the database, streamed once
            // by 4x1 clusters that multicast each database tile to their pairs
            L.a_planes = yp;
            L.b_planes = xp;
            L.M = static_cast<uint32_t>(nc);
            L.N = static_cast<uint32_t>(n_db);
            L.cluster_pm = 4;
            L.cluster_pn = 1;
            L.b_streamed = 1;
            L.iris.query_rows = 1;
        } else {
            L.a_planes = xp;
            L.b_planes = yp + 2 * c0 * ldk;
            L.M = static_cast<uint32_t>(n_db);
            L.N = static_cast<uint32_t>(nc);
        }
        L.K = static_cast<uint32_t>(plane_kbytes(d));
        L.ldk = static_cast<uint32_t>(ldk);
        L.parts = 1;
        L.nprimes = 1;
        L.mc[0] = make_modconst(2, 1);  // unused
        L.progress = progress;
        if (c0 > 0) L.cluster_pm = L.cluster_pn = 1;  // the remainder on plain pairs
        L.iris.lo = p_lo;
        L.iris.hi = p_hi;
        L.iris.rho = static_cast<uint32_t>(rho);
        L.iris.col0 = static_cast<uint32_t>(c0);
        L.iris.bits = dbits;
        L.iris.first = first;
        L.iris.scores = dsc;
        if (ctx->diag && ctx->d_diag && c0 == 0) {  // irl_diag_ppmm: counters of the main launch
            L.stats = ctx->d_diag;
            IRL_CK(ctx, cudaMemsetAsync(ctx->d_diag, 0, 1024 * kStatSlots * sizeof(uint64_t), s));
        }
        IRL_LAUNCH(ctx, launch_ppmm_planes(L, s));
        ctx->launches += ppmm_kernels_last_launch() > 1 ? ppmm_kernels_last_launch() - 1 : 0;  // + filler
    }
    std::vector<uint32_t> h(2 * n_eyes);
    IRL_CK(ctx, cudaMemcpyAsync(h.data(), first, 8 * n_eyes, cudaMemcpyDeviceToHost, s));
    // pageable host outputs go through the context's pinned bounce buffers
    if (match_bits) IRL_CK(ctx, copy_d2h(ctx, match_bits, dbits, nbits, s));
    if (scores) IRL_CK(ctx, copy_d2h(ctx, scores, dsc, nsc * 8, s));
    IRL_CK(ctx, cudaStreamSynchronize(s));
    int status = IRL_OK;
    for (size_t e = 0; e < n_eyes; ++e) {
        const uint32_t fm = h[2 * e], fz = h[2 * e + 1];
        // match_db_reference: the first evaluated score either matches (return
        // true) or throws ZeroOverlap, whichever comes first in loop order
        const int32_t res = fz < fm ? -1 : (fm != 0xFFFFFFFFu ? 1 : 0);
        if (eye_result) eye_result[e] = res;
        if (res < 0 && status == IRL_OK)
            status = set_err(ctx, IRL_ERR_ZERO_OVERLAP, "mask overlap is empty, score undefined");
    }
    return status;
}

int check_dims(irl_ctx* ctx, size_t n_db, size_t cols, size_t d) {
    if (d > (1u << 30) || n_db >= (1u << 29) || cols >= (1u << 29))
        return set_err(ctx, IRL_ERR_UNSUPPORTED, "iris: dimensions too large");
    return IRL_OK;
}

// One-shot path (host templates in, device scratch of the context):
// planes for the DB and the rotated queries, then the kModeInner GEMM into
// device inner / overlap [cols][n_db].
int inner_overlap_device(irl_ctx* ctx, const uint64_t* db_code, const uint64_t* db_mask, size_t n_db,
                         const uint64_t* q_code, const uint64_t* q_mask, size_t n_eyes, size_t rho, size_t d,
                         int32_t** d_inner, int32_t** d_overlap) {
    cudaStream_t s = ctx->stream;
    const size_t words = (d + 63) / 64, ldk = plane_ldk(d), cols = n_eyes * rho;
    if (int st = check_dims(ctx, n_db, cols, d)) return st;
    const size_t db_bits = n_db * words * 8, q_bits = n_eyes * words * 8;
    IRL_CK(ctx, ctx->ws[0].ensure(2 * db_bits + 2 * q_bits));
    IRL_CK(ctx, ctx->ws[1].ensure(2 * n_db * ldk));
    IRL_CK(ctx, ctx->ws[2].ensure(2 * cols * ldk));
    IRL_CK(ctx, ctx->ws[3].ensure(2 * cols * n_db * 4));
    uint8_t* bitbuf = ctx->ws[0].as<uint8_t>();
    auto* dc = reinterpret_cast<uint64_t*>(bitbuf);
    auto* dm = reinterpret_cast<uint64_t*>(bitbuf + db_bits);
    auto* qc = reinterpret_cast<uint64_t*>(bitbuf + 2 * db_bits);
    auto* qm = reinterpret_cast<uint64_t*>(bitbuf + 2 * db_bits + q_bits);
    IRL_CK(ctx, copy_h2d(ctx, dc, db_code, db_bits, s));
    IRL_CK(ctx, copy_h2d(ctx, dm, db_mask, db_bits, s));
    IRL_CK(ctx, copy_h2d(ctx, qc, q_code, q_bits, s));
    IRL_CK(ctx, copy_h2d(ctx, qm, q_mask, q_bits, s));
    int8_t* xp = ctx->ws[1].as<int8_t>();
    int8_t* yp = ctx->ws[2].as<int8_t>();
    if (int st = build_planes(ctx, dc, dm, n_db, 1, d, xp, s)) return st;
    if (int st = build_query_planes(ctx, qc, qm, n_eyes, rho, d, yp, s, !iris_query_rows(d, cols, true))) return st;
    int32_t* inner = ctx->ws[3].as<int32_t>();
    int32_t* ovl = inner + cols * n_db;
    if (int st = inner_overlap_gemm(ctx, xp, yp, n_db, cols, d, ldk, inner, ovl, ctx->d_progress, s)) return st;
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

// Device-resident template database (the server keeps its enrolled templates
// in HBM as int8 planes; each query batch then moves only the eyes' bits).
struct irl_iris_db {
    irl_ctx* ctx = nullptr;
    size_t n_db = 0, d = 0, ldk = 0, max_cols = 0;
    int8_t* planes = nullptr;    // [2][n_db][ldk]
    int8_t* qplanes = nullptr;   // [2][max_cols][ldk]
    uint64_t* qbits = nullptr;   // eyes' code + mask words
    uint32_t* progress = nullptr;
    irl::DevBuf match_ws;
    irl::DevBuf fold_ws;  // inner / overlap [cols][n_db] + fold outputs of irl_iris_db_fold
    cudaStream_t copy_stream = nullptr;   // irl_iris_db_fold: output D2H behind each eye chunk
    std::vector<cudaEvent_t> fold_done;   // per eye chunk: folded on the context stream
};

extern "C" {

int irl_iris_inner_overlap(irl_ctx* ctx, const uint64_t* db_code, const uint64_t* db_mask, size_t n_db,
                           const uint64_t* q_code, const uint64_t* q_mask, size_t n_eyes, size_t rho, size_t d,
                           int32_t* inner, int32_t* overlap) {
    if (int st = check_args(ctx, db_code, db_mask, n_db, q_code, q_mask, n_eyes, d)) return st;
    Guard g(ctx, __func__);
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
    Guard g(ctx, __func__);
    const size_t cols = n_eyes * rho;
    if (cols == 0 || n_db == 0) {
        // match_db_reference over an empty product: no score is evaluated
        if (eye_result) std::memset(eye_result, 0, n_eyes * sizeof(int32_t));
        if (match_bits) std::memset(match_bits, 0, n_eyes * n_db);
        return IRL_OK;
    }
    cudaStream_t s = ctx->stream;
    const size_t words = (d + 63) / 64, ldk = plane_ldk(d);
    if (int st = check_dims(ctx, n_db, cols, d)) return st;
    const size_t db_bits = n_db * words * 8, q_bits = n_eyes * words * 8;
    IRL_CK(ctx, ctx->ws[0].ensure(2 * db_bits + 2 * q_bits));
    IRL_CK(ctx, ctx->ws[1].ensure(2 * n_db * ldk));
    IRL_CK(ctx, ctx->ws[2].ensure(2 * cols * ldk));
    uint8_t* bitbuf = ctx->ws[0].as<uint8_t>();
    auto* dc = reinterpret_cast<uint64_t*>(bitbuf);
    auto* dm = reinterpret_cast<uint64_t*>(bitbuf + db_bits);
    auto* qc = reinterpret_cast<uint64_t*>(bitbuf + 2 * db_bits);
    auto* qm = reinterpret_cast<uint64_t*>(bitbuf + 2 * db_bits + q_bits);
    IRL_CK(ctx, copy_h2d(ctx, dc, db_code, db_bits, s));
    IRL_CK(ctx, copy_h2d(ctx, dm, db_mask, db_bits, s));
    IRL_CK(ctx, copy_h2d(ctx, qc, q_code, q_bits, s));
    IRL_CK(ctx, copy_h2d(ctx, qm, q_mask, q_bits, s));
    if (int st = build_planes(ctx, dc, dm, n_db, 1, d, ctx->ws[1].as<int8_t>(), s)) return st;
    if (int st = build_query_planes(ctx, qc, qm, n_eyes, rho, d, ctx->ws[2].as<int8_t>(), s,
                                    !iris_query_rows(d, n_eyes * rho)))
        return st;
    return match_fused(ctx, ctx->ws[1].as<int8_t>(), ctx->ws[2].as<int8_t>(), n_db, n_eyes, rho, d, ldk, p_lo, p_hi,
                       match_bits, eye_result, scores, ctx->ws[4], ctx->d_progress, s);
}

int irl_iris_db_create(irl_ctx* ctx, const uint64_t* db_code, const uint64_t* db_mask, size_t n_db, size_t d,
                       size_t max_cols, irl_iris_db** out) {
    if (!out) return IRL_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    if (int st = check_args(ctx, db_code, db_mask, n_db, db_code, db_mask, 0, d)) return st;
    Guard g(ctx, __func__);
    if (n_db == 0 || max_cols == 0) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "iris db: empty database or batch");
    if (int st = check_dims(ctx, n_db, max_cols, d)) return st;
    auto* e = new irl_iris_db();
    e->ctx = ctx;
    e->n_db = n_db;
    e->d = d;
    e->ldk = plane_ldk(d);
    e->max_cols = max_cols;
    const size_t words = (d + 63) / 64, db_bits = n_db * words * 8;
    uint64_t* staging = nullptr;
    cudaError_t err = cudaMalloc(&e->planes, 2 * n_db * e->ldk);
    if (err == cudaSuccess) err = cudaMalloc(&e->qplanes, 2 * max_cols * e->ldk);
    if (err == cudaSuccess) err = cudaMalloc(&e->qbits, 2 * max_cols * words * 8);
    if (err == cudaSuccess) err = cudaMalloc(&e->progress, kScheduleScratchBytes);
    if (err == cudaSuccess) err = cudaMalloc(&staging, 2 * db_bits);
    if (err == cudaSuccess) err = copy_h2d(ctx, staging, db_code, db_bits, ctx->stream);
    if (err == cudaSuccess)
        err = copy_h2d(ctx, staging + db_bits / 8, db_mask, db_bits, ctx->stream);
    int st = IRL_OK;
    if (err == cudaSuccess) st = build_planes(ctx, staging, staging + db_bits / 8, n_db, 1, d, e->planes, ctx->stream);
    if (err == cudaSuccess) err = cudaStreamSynchronize(ctx->stream);
    cudaFree(staging);
    if (err != cudaSuccess || st != IRL_OK) {
        irl_iris_db_destroy(e);
        return err != cudaSuccess ? cuda_fail(ctx, err, "irl_iris_db_create") : st;
    }
    *out = e;
    return IRL_OK;
}

int irl_iris_db_create_file(irl_ctx* ctx, const char* path, size_t max_cols, irl_iris_db** out, size_t* n_db_out,
                            size_t* d_out) {
    if (!ctx || !path || !out) return IRL_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    Guard g(ctx, __func__);
    std::FILE* f = std::fopen(path, "rb");
    if (!f) return set_err(ctx, IRL_ERR_IO, std::string("cannot open ") + path);
    struct Closer {
        std::FILE* f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    // header {magic "IRIT", version 1, n_db, d}, little-endian (iris_core.cpp:183-196)
    uint8_t hdr[24];
    if (std::fread(hdr, 1, sizeof(hdr), f) != sizeof(hdr))
        return set_err(ctx, IRL_ERR_IO, std::string("bad template file magic in ") + path);
    auto u32 = [&](int o) { uint32_t v = 0; for (int i = 0; i < 4; ++i) v |= uint32_t(hdr[o + i]) << (8 * i); return v; };
    auto u64 = [&](int o) { uint64_t v = 0; for (int i = 0; i < 8; ++i) v |= uint64_t(hdr[o + i]) << (8 * i); return v; };
    if (u32(0) != 0x49524954u) return set_err(ctx, IRL_ERR_IO, std::string("bad template file magic in ") + path);
    if (u32(4) != 1u) return set_err(ctx, IRL_ERR_IO, "unsupported template file version");
    const uint64_t n = u64(8), d = u64(16);
    if (n == 0 || d == 0) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "iris db: empty template file");
    if (max_cols == 0) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "iris db: empty database or batch");
    if (int st = check_dims(ctx, n, max_cols, d)) return st;
    const size_t plane_bytes = (n * d + 7) / 8;
    uint8_t* host = nullptr;
    IRL_CK(ctx, cudaMallocHost(&host, 2 * plane_bytes));
    struct HostFree {
        uint8_t* p;
        ~HostFree() { cudaFreeHost(p); }
    } hf{host};
    if (std::fread(host, 1, 2 * plane_bytes, f) != 2 * plane_bytes)
        return set_err(ctx, IRL_ERR_IO, std::string("truncated template file ") + path);
    auto* e = new irl_iris_db();
    e->ctx = ctx;
    e->n_db = n;
    e->d = d;
    e->ldk = plane_ldk(d);
    e->max_cols = max_cols;
    const size_t words = (d + 63) / 64;
    uint8_t* staging = nullptr;
    cudaError_t err = cudaMalloc(&e->planes, 2 * n * e->ldk);
    if (err == cudaSuccess) err = cudaMalloc(&e->qplanes, 2 * max_cols * e->ldk);
    if (err == cudaSuccess) err = cudaMalloc(&e->qbits, 2 * max_cols * words * 8);
    if (err == cudaSuccess) err = cudaMalloc(&e->progress, kScheduleScratchBytes);
    if (err == cudaSuccess) err = cudaMalloc(&staging, 2 * plane_bytes);
    if (err == cudaSuccess) err = cudaMemcpyAsync(staging, host, 2 * plane_bytes, cudaMemcpyHostToDevice, ctx->stream);
    if (err == cudaSuccess) {
        const size_t total = n * (e->ldk / 16);
        auto kern = iris_f4(d) ? iris_file_planes_kernel<true> : iris_file_planes_kernel<false>;
        kern<<<static_cast<unsigned>((total + 255) / 256), 256, 0, ctx->stream>>>(
            staging, staging + plane_bytes, static_cast<uint32_t>(d), static_cast<uint32_t>(n),
            static_cast<uint32_t>(e->ldk), e->planes);
        err = cudaGetLastError();
        if (err == cudaSuccess) ++ctx->launches;
    }
    if (err == cudaSuccess) err = cudaStreamSynchronize(ctx->stream);
    cudaFree(staging);
    if (err != cudaSuccess) {
        irl_iris_db_destroy(e);
        return cuda_fail(ctx, err, "irl_iris_db_create_file");
    }
    if (n_db_out) *n_db_out = n;
    if (d_out) *d_out = d;
    *out = e;
    return IRL_OK;
}

int irl_iris_db_destroy(irl_iris_db* e) {
    if (!e) return IRL_OK;
    cudaSetDevice(e->ctx->device);
    cudaStreamSynchronize(e->ctx->stream);
    cudaFree(e->planes);
    cudaFree(e->qplanes);
    cudaFree(e->qbits);
    cudaFree(e->progress);
    e->match_ws.release();
    e->fold_ws.release();
    if (e->copy_stream) {
        cudaStreamSynchronize(e->copy_stream);
        cudaStreamDestroy(e->copy_stream);
    }
    for (cudaEvent_t ev : e->fold_done) cudaEventDestroy(ev);
    delete e;
    return IRL_OK;
}

int irl_iris_db_match(irl_iris_db* e, const uint64_t* q_code, const uint64_t* q_mask, size_t n_eyes, size_t rho,
                      double p_lo, double p_hi, uint8_t* match_bits, int32_t* eye_result, double* scores) {
    if (!e) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* ctx = e->ctx;
    if (int st = check_args(ctx, q_code, q_mask, 0, q_code, q_mask, n_eyes, e->d)) return st;
    Guard g(ctx, __func__);
    const size_t cols = n_eyes * rho;
    if (cols == 0) {
        if (eye_result) std::memset(eye_result, 0, n_eyes * sizeof(int32_t));
        if (match_bits) std::memset(match_bits, 0, n_eyes * e->n_db);
        return IRL_OK;
    }
    if (cols > e->max_cols) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "iris db: query batch wider than max_cols");
    cudaStream_t s = ctx->stream;
    const size_t words = (e->d + 63) / 64, qb = n_eyes * words * 8;
    IRL_CK(ctx, cudaMemcpyAsync(e->qbits, q_code, qb, cudaMemcpyHostToDevice, s));
    IRL_CK(ctx, cudaMemcpyAsync(e->qbits + n_eyes * words, q_mask, qb, cudaMemcpyHostToDevice, s));
    if (int st = build_query_planes(ctx, e->qbits, e->qbits + n_eyes * words, n_eyes, rho, e->d, e->qplanes, s,
                                    !iris_query_rows(e->d, n_eyes * rho)))
        return st;
    return match_fused(ctx, e->planes, e->qplanes, e->n_db, n_eyes, rho, e->d, e->ldk, p_lo, p_hi, match_bits,
                       eye_result, scores, e->match_ws, e->progress, s);
}

int irl_iris_db_fold(irl_iris_db* e, const uint64_t* q_code, const uint64_t* q_mask, const irl_fold_params* p,
                     double* folded, double* refolded, int32_t* assumption_ok) {
    if (!e || !p) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* ctx = e->ctx;
    Guard g(ctx, __func__);
    FoldArgs a;
    if (int st = fold_prepare(ctx, p, refolded != nullptr, &a)) return st;  // run_alg2: cfg.validate() first
    // prepare (pipeline.cpp:100-118)
    if (p->n_db != e->n_db) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "pipeline: database size does not match config");
    if (p->d != e->d)
        return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "pipeline: database template dimension mismatch");
    const size_t n_eyes = p->batch, rho = p->rho, cols = n_eyes * rho;
    if (int st = check_args(ctx, q_code, q_mask, 0, q_code, q_mask, n_eyes, e->d)) return st;
    if (cols > e->max_cols) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "iris db: query batch wider than max_cols");
    cudaStream_t s = ctx->stream;
    const size_t words = (e->d + 63) / 64, qb = n_eyes * words * 8;
    const size_t in_bytes = cols * e->n_db * sizeof(int32_t);
    const size_t fold_elems = size_t(a.batch) * a.blocks * a.groups * a.d;
    const size_t refold_elems = size_t(a.batch) * a.blocks * a.d;
    const size_t off_f = 2 * in_bytes, off_r = off_f + (folded ? fold_elems * 8 : 0);
    const size_t off_flags = off_r + (refolded ? refold_elems * 8 : 0);
    IRL_CK(ctx, e->fold_ws.ensure(off_flags + 16));
    uint8_t* ws = e->fold_ws.as<uint8_t>();
    auto* inner = reinterpret_cast<int32_t*>(ws);
    auto* ovl = reinterpret_cast<int32_t*>(ws + in_bytes);
    auto* dflags = reinterpret_cast<uint32_t*>(ws + off_flags);
    IRL_CK(ctx, cudaMemcpyAsync(e->qbits, q_code, qb, cudaMemcpyHostToDevice, s));
    IRL_CK(ctx, cudaMemcpyAsync(e->qbits + n_eyes * words, q_mask, qb, cudaMemcpyHostToDevice, s));
    if (int st = build_query_planes(ctx, e->qbits, e->qbits + n_eyes * words, n_eyes, rho, e->d, e->qplanes, s,
                                    !iris_query_rows(e->d, cols, true)))
        return st;
    if (int st = inner_overlap_gemm(ctx, e->planes, e->qplanes, e->n_db, cols, e->d, e->ldk, inner, ovl, e->progress, s))
        return st;
    IRL_CK(ctx, cudaMemsetAsync(dflags, 0, 8, s));
    a.inner = inner;
    a.overlap = ovl;
    a.folded = folded ? reinterpret_cast<double*>(ws + off_f) : nullptr;
    a.refolded = refolded ? reinterpret_cast<double*>(ws + off_r) : nullptr;
    a.flags = dflags;
    // The fold runs in eye chunks; each chunk's outputs go to the host on a
    // copy stream while the next chunk folds (the kernel is unchanged: a chunk
    // is the same launch over a sub-batch, its buffers offset to its first eye).
    // Page-locked outputs only: their copies are asynchronous DMA (2.72 ->
    // 2.48 ms at the paper's scale). Pageable outputs go through the bounce
    // buffers in one piece -- chunked, those copies measured slower (3.0 ->
    // 7.2 ms), so they keep a single chunk.
    const bool pinned_out = (!folded || host_pinned(folded)) && (!refolded || host_pinned(refolded));
    const size_t nch = pinned_out ? std::min<size_t>(a.batch, 4) : 1;
    if (!e->copy_stream) IRL_CK(ctx, cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));
    while (e->fold_done.size() < nch) {
        cudaEvent_t ev;
        IRL_CK(ctx, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        e->fold_done.push_back(ev);
    }
    const size_t per_in = size_t(a.rho) * e->n_db, per_f = size_t(a.blocks) * a.groups * a.d,
                 per_r = size_t(a.blocks) * a.d;
    auto e_of = [&](size_t c) { return c * a.batch / nch; };
    for (size_t c = 0; c < nch; ++c) {
        const size_t e0 = e_of(c);
        FoldArgs ac = a;
        ac.batch = static_cast<uint32_t>(e_of(c + 1) - e0);
        ac.inner = inner + e0 * per_in;
        ac.overlap = ovl + e0 * per_in;
        ac.folded = a.folded ? a.folded + e0 * per_f : nullptr;
        ac.refolded = a.refolded ? a.refolded + e0 * per_r : nullptr;
        if (int st = launch_fold_stage(ctx, ac, s)) return st;
        IRL_CK(ctx, cudaEventRecord(e->fold_done[c], s));
    }
    for (size_t c = 0; c < nch; ++c) {
        const size_t e0 = e_of(c), ne = e_of(c + 1) - e0;
        IRL_CK(ctx, cudaStreamWaitEvent(e->copy_stream, e->fold_done[c], 0));
        // page-locked outputs: async DMA; pageable: the bounce buffers (blocks
        // this thread for the chunk while the next chunks fold)
        if (folded) IRL_CK(ctx, copy_d2h(ctx, folded + e0 * per_f, a.folded + e0 * per_f, ne * per_f * 8, e->copy_stream));
        if (refolded)
            IRL_CK(ctx, copy_d2h(ctx, refolded + e0 * per_r, a.refolded + e0 * per_r, ne * per_r * 8, e->copy_stream));
    }
    IRL_CK(ctx, cudaStreamSynchronize(e->copy_stream));
    (void)fold_elems;
    (void)refold_elems;
    uint32_t hf[2] = {0, 0};
    IRL_CK(ctx, cudaMemcpyAsync(hf, dflags, 8, cudaMemcpyDeviceToHost, s));
    IRL_CK(ctx, cudaStreamSynchronize(s));
    if (assumption_ok) *assumption_ok = hf[0] ? 0 : 1;
    if (hf[1]) return set_err(ctx, IRL_ERR_ZERO_OVERLAP, "mask overlap is empty, score undefined");
    return IRL_OK;
}

}  // extern "C"
