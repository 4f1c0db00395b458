// C ABI of the B200 PPMM / RGSW-CCMM engine (include/irl_capi.h).
//
// Host-buffer calls mirror irislab::modmat (reference proj/src/modmat.cpp)
// value-for-value, including its exception taxonomy and messages; all the
// arithmetic runs in this library's sm_100a kernels. There is no CPU compute
// path: validation only reads the split kernels' device-side statistics.
#include <unistd.h>

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/irl_capi.h"
#include "ctx_internal.h"
#include "kernels_aux.cuh"
#include "ppmm.h"

using namespace irl;

// ---------------------------------------------------------------------------
// Context
// ---------------------------------------------------------------------------

struct irl_ccmm {
    irl_ctx* ctx = nullptr;
    size_t parts = 0, M = 0, K = 0, ldk = 0, max_n = 0, nmod = 0;
    ModTable mt{};
    int8_t* db = nullptr;       // [parts][nmod][2][M][ldk]
    int8_t* qplanes = nullptr;  // [nmod][2][max_n][ldk]
    uint16_t* qres = nullptr;   // [nmod][K][max_n]
    uint16_t* out = nullptr;    // [parts][nmod][max_n][M]
    uint32_t kchunk = 0;        // K chunk keeping the fused int32 accumulators exact
    uint32_t* progress = nullptr;  // group-gating scratch of this engine's PPMM launches
    cudaStream_t copy_stream = nullptr;  // device -> host
    cudaStream_t h2d_stream = nullptr;   // host -> device
    std::vector<cudaEvent_t> part_done;  // per modulus chunk: PPMMs done
    std::vector<cudaEvent_t> h2d_done;   // per modulus chunk: query residues landed
    uint64_t bytes = 0;
    // fused a-part exchange: this engine's receive buffer (peers store into it)
    // and the peers' buffers this engine stores into (IPC-mapped or raw)
    uint16_t* recv = nullptr;
    size_t recv_n = 0;
    size_t mirror_part = 0, mirror_n = 0, n_mirror = 0;
    uint16_t* mirror[kMaxMirrors] = {};
    bool mirror_ipc[kMaxMirrors] = {};
    // part-granular D2H in irl_ccmm_run: per (modulus chunk, part) tile
    // counters the epilogue bumps; the copy stream waits on them with stream
    // memory operations (cuStreamWaitValue32) instead of on the whole launch
    uint32_t* part_cnt = nullptr;       // [nmod][parts]
    std::vector<cudaEvent_t> cnt_zeroed;  // per modulus chunk
    bool memops = true;                 // cleared if stream memory ops are unavailable
};

namespace {

const char* kOverflowMsg = "int32 accumulation bound exceeded: K*|A|*|B| = ";

// Reference precheck of small_gemm (modmat.cpp:122-129).
bool overflow(int64_t k, int64_t ma, int64_t mb, int64_t* bound) {
    *bound = k * ma * mb;
    return *bound >= (int64_t{1} << 31);
}

int validate_moduli(irl_ctx* ctx, const uint32_t* primes, const uint32_t* exps, size_t nmod) {
    if (nmod > kMaxModuli) return set_err(ctx, IRL_ERR_UNSUPPORTED, "at most 32 moduli per basis");
    for (size_t i = 0; i < nmod; ++i) {
        if (exps[i] != 1 && exps[i] != 2)
            return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "modulus exponent must be 1 or 2");
        if (primes[i] < 2) return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "modulus base must be >= 2");
        const uint64_t m = exps[i] == 2 ? uint64_t(primes[i]) * primes[i] : primes[i];
        if (m > 65535) return set_err(ctx, IRL_ERR_UNSUPPORTED, "moduli above 2^16 are not supported");
    }
    return IRL_OK;
}

ModTable make_table(const uint32_t* primes, const uint32_t* exps, size_t nmod) {
    ModTable t{};
    t.n = static_cast<uint32_t>(nmod);
    for (size_t i = 0; i < nmod; ++i) t.mc[i] = make_modconst(primes[i], exps[i]);
    return t;
}

PpmmLaunch make_launch(const ModTable& mt) {
    PpmmLaunch L;
    L.nprimes = mt.n;
    for (uint32_t i = 0; i < mt.n; ++i) L.mc[i] = mt.mc[i];
    return L;
}

// K chunk such that acc2 = sum X0 Y1 + X1 Y0 and acc1 = sum X0 Y0 stay
// within |acc| <= 2^31 - 2^17 (the fused epilogue's exact range, see
// combine_psq_fast) for digit maxima (a0, a1, b0, b1); multiple of 128.
uint32_t safe_kchunk(int64_t a0, int64_t a1, int64_t b0, int64_t b1, uint32_t K) {
    const int64_t per = std::max<int64_t>(std::max<int64_t>(a0 * b1 + a1 * b0, a0 * b0), 1);
    int64_t kc = ((int64_t{1} << 31) - (int64_t{1} << 17)) / per;
    if (kc >= K) return K;
    kc = (kc / 128) * 128;
    return static_cast<uint32_t>(std::max<int64_t>(kc, 128));
}

// One PPMM over planes with K chunking (accumulate mode for chunks > 0).
int run_ppmm(irl_ctx* ctx, PpmmLaunch L, uint32_t kchunk, cudaStream_t s) {
    const uint32_t K = L.K;
    if (K == 0) {
        // Empty inner dimension: the product is zero (modmat.cpp:137 never runs).
        const size_t bytes = size_t(L.parts) * L.nprimes * L.N * L.M * sizeof(uint16_t);
        if (!L.accumulate) IRL_CK(ctx, cudaMemsetAsync(L.out, 0, bytes, s));
        return IRL_OK;
    }
    if (kchunk == 0 || kchunk > K) kchunk = K;
    if (!L.progress) L.progress = ctx->d_progress;
    if (const char* gl = std::getenv("IRL_PPMM_GATE")) L.gate_lead = std::atoi(gl);
    if (const char* cl = std::getenv("IRL_PPMM_CLUSTER")) {
        // "PMxPN" (pairs along M x pairs along N) or a CTA count 2/4/8 (1 x count/2)
        int pm = 1, pn = 1;
        if (std::sscanf(cl, "%dx%d", &pm, &pn) != 2) {
            pm = 1;
            pn = std::max(1, std::atoi(cl) / 2);
        }
        L.cluster_pm = pm;
        L.cluster_pn = pn;
    }
    if (ctx->diag && ctx->d_diag) {
        L.stats = ctx->d_diag;
        IRL_CK(ctx, cudaMemsetAsync(ctx->d_diag, 0, 1024 * kStatSlots * sizeof(uint64_t), s));
    }
    const int8_t* a0 = L.a_planes;
    const int8_t* b0 = L.b_planes;
    uint32_t* const part_done = L.part_done;
    for (uint32_t k0 = 0; k0 < K; k0 += kchunk) {
        L.part_done = k0 + kchunk >= K ? part_done : nullptr;  // the final K chunk completes the outputs
        L.a_planes = a0 + k0;
        L.b_planes = b0 + k0;
        L.K = std::min(kchunk, K - k0);
        L.accumulate = (k0 > 0) || L.accumulate;
        IRL_LAUNCH(ctx, launch_ppmm_planes(L, s));
        ctx->launches += ppmm_kernels_last_launch() > 1 ? ppmm_kernels_last_launch() - 1 : 0;  // + filler
    }
    return IRL_OK;
}

size_t round16(size_t x) { return (x + 15) / 16 * 16; }

// Big-integer helpers for CRT constants (host, 32-bit limbs).
using Limbs = std::vector<uint32_t>;

Limbs basis_Q(const uint32_t* primes, const uint32_t* exps, size_t nmod) {
    Limbs q{1};
    for (size_t i = 0; i < nmod; ++i) {
        for (uint32_t e = 0; e < exps[i]; ++e) {
            uint64_t carry = 0;
            for (auto& l : q) {
                const uint64_t t = uint64_t(l) * primes[i] + carry;
                l = uint32_t(t);
                carry = t >> 32;
            }
            if (carry) q.push_back(uint32_t(carry));
        }
    }
    return q;
}

uint32_t divmod_small(Limbs& x, uint32_t m) {
    uint64_t r = 0;
    for (size_t i = x.size(); i-- > 0;) {
        const uint64_t cur = (r << 32) | x[i];
        x[i] = uint32_t(cur / m);
        r = cur % m;
    }
    return uint32_t(r);
}

size_t byte_width(const Limbs& q) {
    size_t bits = 0;
    for (size_t i = q.size(); i-- > 0;) {
        if (q[i]) {
            bits = i * 32 + (32 - __builtin_clz(q[i]));
            break;
        }
    }
    return bits ? (bits + 7) / 8 : 1;
}

bool inv_mod(uint32_t a, uint32_t m, uint32_t* out) {
    int64_t t = 0, nt = 1, r = m, nr = a % m;
    while (nr) {
        const int64_t q = r / nr, tt = t - q * nt, rr = r - q * nr;
        t = nt;
        nt = tt;
        r = nr;
        nr = rr;
    }
    if (r != 1 && m != 1) return false;
    if (t < 0) t += m;
    *out = uint32_t(t);
    return true;
}

}  // namespace

namespace irl {

namespace {
constexpr size_t kBounceBytes = size_t(16) << 20;
constexpr size_t kDirectCopyBytes = size_t(4) << 20;  // below this the driver's own staging is fine
constexpr int kCopyThreads = 8;

cudaError_t ensure_bounce(irl_ctx* ctx) {
    for (int i = 0; i < 2; ++i) {
        if (!ctx->bounce[i]) {
            cudaError_t e = cudaMallocHost(&ctx->bounce[i], kBounceBytes);
            if (e != cudaSuccess) return e;
        }
        if (!ctx->bounce_ev[i]) {
            cudaError_t e = cudaEventCreateWithFlags(&ctx->bounce_ev[i], cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

void parallel_memcpy(void* dst, const void* src, size_t bytes) {
    if (bytes < (size_t(1) << 20)) {
        std::memcpy(dst, src, bytes);
        return;
    }
    std::thread th[kCopyThreads];
    const size_t piece = (bytes + kCopyThreads - 1) / kCopyThreads;
    for (int t = 0; t < kCopyThreads; ++t) {
        const size_t lo = std::min(bytes, t * piece), hi = std::min(bytes, lo + piece);
        th[t] = std::thread([=] {
            if (hi > lo) std::memcpy(static_cast<uint8_t*>(dst) + lo, static_cast<const uint8_t*>(src) + lo, hi - lo);
        });
    }
    for (auto& t : th) t.join();
}
}  // namespace

cudaError_t copy_h2d(irl_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes < kDirectCopyBytes) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
    cudaError_t e = ensure_bounce(ctx);
    if (e != cudaSuccess) return e;
    for (size_t off = 0, i = 0; off < bytes; off += kBounceBytes, ++i) {
        const int b = static_cast<int>(i % 2);
        const size_t len = std::min(kBounceBytes, bytes - off);
        e = cudaEventSynchronize(ctx->bounce_ev[b]);  // its previous DMA has read it
        if (e != cudaSuccess) return e;
        parallel_memcpy(ctx->bounce[b], static_cast<const uint8_t*>(src) + off, len);
        e = cudaMemcpyAsync(static_cast<uint8_t*>(dst) + off, ctx->bounce[b], len, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaEventRecord(ctx->bounce_ev[b], s);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t copy_d2h(irl_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t s) {
    cudaError_t e;
    if (bytes < kDirectCopyBytes) {
        e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
        return e == cudaSuccess ? cudaStreamSynchronize(s) : e;
    }
    e = ensure_bounce(ctx);
    if (e != cudaSuccess) return e;
    // DMA chunk i into bounce i%2 while the host drains chunk i-1
    size_t prev_off = 0, prev_len = 0;
    for (size_t off = 0, i = 0;; off += kBounceBytes, ++i) {
        const int b = static_cast<int>(i % 2);
        const size_t len = off < bytes ? std::min(kBounceBytes, bytes - off) : 0;
        if (len) {
            e = cudaMemcpyAsync(ctx->bounce[b], static_cast<const uint8_t*>(src) + off, len, cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaEventRecord(ctx->bounce_ev[b], s);
            if (e != cudaSuccess) return e;
        }
        if (prev_len) {
            const int pb = 1 - b;
            e = cudaEventSynchronize(ctx->bounce_ev[pb]);
            if (e != cudaSuccess) return e;
            parallel_memcpy(static_cast<uint8_t*>(dst) + prev_off, ctx->bounce[pb], prev_len);
        }
        if (!len) break;
        prev_off = off;
        prev_len = len;
    }
    return cudaStreamSynchronize(s);
}

void release_bounce(irl_ctx* ctx) {
    for (int i = 0; i < 2; ++i) {
        if (ctx->bounce_ev[i]) cudaEventDestroy(ctx->bounce_ev[i]);
        if (ctx->bounce[i]) cudaFreeHost(ctx->bounce[i]);
        ctx->bounce_ev[i] = nullptr;
        ctx->bounce[i] = nullptr;
    }
}

}  // namespace irl

extern "C" {

int irl_abi_version(void) { return IRL_ABI_VERSION; }

const char* irl_status_string(int s) {
    switch (s) {
        case IRL_OK: return "ok";
        case IRL_ERR_SHAPE_MISMATCH: return "ShapeMismatch";
        case IRL_ERR_MODULUS_TOO_LARGE: return "ModulusTooLarge";
        case IRL_ERR_ACCUMULATION_OVERFLOW_RISK: return "AccumulationOverflowRisk";
        case IRL_ERR_NOT_COPRIME: return "Error";
        case IRL_ERR_MODULUS_BUDGET: return "ModulusBudget";
        case IRL_ERR_INVALID_ARGUMENT: return "InvalidArgument";
        case IRL_ERR_CUDA: return "CudaError";
        case IRL_ERR_NO_DEVICE: return "NoDevice";
        case IRL_ERR_OUT_OF_MEMORY: return "OutOfMemory";
        case IRL_ERR_UNSUPPORTED: return "Unsupported";
        case IRL_ERR_ZERO_OVERLAP: return "ZeroOverlap";
        case IRL_ERR_IO: return "Error";
        default: return "unknown";
    }
}

int irl_ctx_create(int device, irl_ctx** out) {
    if (!out) return IRL_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
        cudaGetLastError();
        return IRL_ERR_NO_DEVICE;
    }
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10) {
        return IRL_ERR_NO_DEVICE;  // built for sm_100a only
    }
    auto* ctx = new irl_ctx();
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&ctx->d_stats, sizeof(SplitStats)) != cudaSuccess ||
        cudaMallocHost(&ctx->h_stats, sizeof(SplitStats)) != cudaSuccess ||
        cudaMalloc(&ctx->d_absmax, 2 * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&ctx->d_progress, kScheduleScratchBytes) != cudaSuccess ||
        cudaMallocHost(&ctx->h_absmax, 2 * sizeof(int32_t)) != cudaSuccess) {
        delete ctx;
        return IRL_ERR_CUDA;
    }
    *out = ctx;
    return IRL_OK;
}

int irl_ctx_destroy(irl_ctx* ctx) {
    if (!ctx) return IRL_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& b : ctx->ws) b.release();
    cudaFree(ctx->d_stats);
    cudaFreeHost(ctx->h_stats);
    cudaFree(ctx->d_absmax);
    cudaFreeHost(ctx->h_absmax);
    cudaFree(ctx->d_progress);
    cudaFree(ctx->d_diag);
    release_bounce(ctx);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
    return IRL_OK;
}

const char* irl_last_error(const irl_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

int irl_diag_ppmm(irl_ctx* ctx, int enable, uint64_t* out, size_t cap) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx);
    if (enable && !ctx->d_diag) IRL_CK(ctx, cudaMalloc(&ctx->d_diag, 1024 * kStatSlots * sizeof(uint64_t)));
    if (out && ctx->d_diag) {
        IRL_CK(ctx, cudaDeviceSynchronize());
        IRL_CK(ctx, cudaMemcpy(out, ctx->d_diag, std::min<size_t>(cap, 1024 * kStatSlots) * sizeof(uint64_t),
                               cudaMemcpyDeviceToHost));
    }
    ctx->diag = enable != 0;
    return IRL_OK;
}
uint64_t irl_kernel_launches(const irl_ctx* ctx) { return ctx ? ctx->launches : 0; }
void* irl_ctx_stream(const irl_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

size_t irl_paper_basis(uint32_t* primes, uint32_t* exps, size_t cap) {
    // build_paper_basis (modmat.cpp:37-45): primes in [127, 253], e = 2.
    size_t n = 0;
    for (uint32_t v = 127; v <= 253; ++v) {
        bool prime = true;
        for (uint32_t q = 2; q * q <= v; ++q)
            if (v % q == 0) {
                prime = false;
                break;
            }
        if (!prime) continue;
        if (n < cap) {
            primes[n] = v;
            exps[n] = 2;
        }
        ++n;
    }
    return n;
}

size_t irl_basis_Q_bytes(const uint32_t* primes, const uint32_t* exps, size_t nmod, uint8_t* out,
                         size_t cap) {
    const Limbs q = basis_Q(primes, exps, nmod);
    const size_t w = byte_width(q);
    if (out)
        for (size_t b = 0; b < std::min(w, cap); ++b)
            out[b] = b / 4 < q.size() ? uint8_t(q[b / 4] >> (8 * (b % 4))) : 0;
    return w;
}

uint32_t irl_synth_residue(uint64_t seed, uint32_t stream, uint32_t plane, uint32_t row,
                           uint32_t col, uint32_t m) {
    return synth_residue_host(seed, stream, plane, row, col, m);
}

void irl_synth_residues_host(uint64_t seed, uint32_t stream, uint32_t plane, uint32_t row0,
                             uint32_t nrows, uint32_t col0, uint32_t ncols, uint32_t m,
                             uint16_t* out) {
    for (uint32_t r = 0; r < nrows; ++r)
        for (uint32_t c = 0; c < ncols; ++c)
            out[size_t(r) * ncols + c] =
                uint16_t(synth_residue_host(seed, stream, plane, row0 + r, col0 + c, m));
}

// ---------------------------------------------------------------------------
// digit_decompose / digit_recompose (modmat.cpp:86-118)
// ---------------------------------------------------------------------------

int irl_digit_decompose(irl_ctx* ctx, const int32_t* m, size_t rows, size_t cols, uint32_t p,
                        int32_t* d0, int32_t* d1) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx);
    if (p >= 256) return set_err(ctx, IRL_ERR_MODULUS_TOO_LARGE, "digit base must be < 2^8");
    if (p == 0) return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "digit base must be positive");
    const size_t n = rows * cols;
    if (n == 0) return IRL_OK;
    const size_t bytes = n * sizeof(int32_t);
    IRL_CK(ctx, ctx->ws[0].ensure(3 * bytes));
    int32_t* din = ctx->ws[0].as<int32_t>();
    IRL_CK(ctx, copy_h2d(ctx, din, m, bytes, ctx->stream));
    IRL_LAUNCH(ctx, launch_digit_decompose(din, n, make_modconst(p, 2), din + n, din + 2 * n, ctx->stream));
    IRL_CK(ctx, copy_d2h(ctx, d0, din + n, bytes, ctx->stream));
    IRL_CK(ctx, copy_d2h(ctx, d1, din + 2 * n, bytes, ctx->stream));
    IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return IRL_OK;
}

int irl_digit_recompose(irl_ctx* ctx, const int32_t* d0, const int32_t* d1, size_t rows,
                        size_t cols, uint32_t p, int32_t* out) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx);
    if (p == 0 || p > 46340)
        return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "p^2 must fit a positive int32");
    const size_t n = rows * cols;
    if (n == 0) return IRL_OK;
    const size_t bytes = n * sizeof(int32_t);
    IRL_CK(ctx, ctx->ws[0].ensure(3 * bytes));
    int32_t* b = ctx->ws[0].as<int32_t>();
    IRL_CK(ctx, copy_h2d(ctx, b, d0, bytes, ctx->stream));
    IRL_CK(ctx, copy_h2d(ctx, b + n, d1, bytes, ctx->stream));
    IRL_LAUNCH(ctx, launch_digit_recompose(b, b + n, n, make_modconst(p, 2), b + 2 * n, ctx->stream));
    IRL_CK(ctx, copy_d2h(ctx, out, b + 2 * n, bytes, ctx->stream));
    IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return IRL_OK;
}

// ---------------------------------------------------------------------------
// small_gemm (modmat.cpp:120-141)
// ---------------------------------------------------------------------------

int irl_small_gemm(irl_ctx* ctx, const int32_t* a, const int32_t* b, int32_t* c, size_t m,
                   size_t k, size_t n) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx);
    if (m > UINT32_MAX || k > UINT32_MAX || n > UINT32_MAX)
        return set_err(ctx, IRL_ERR_UNSUPPORTED, "dimension above 2^32");
    const size_t na = m * k, nb = k * n, nc = m * n;
    IRL_CK(ctx, ctx->ws[0].ensure((na + nb + nc + 1) * sizeof(int32_t)));
    int32_t* da = ctx->ws[0].as<int32_t>();
    int32_t* db = da + na;
    int32_t* dc = db + nb;
    if (na) IRL_CK(ctx, copy_h2d(ctx, da, a, na * 4, ctx->stream));
    if (nb) IRL_CK(ctx, copy_h2d(ctx, db, b, nb * 4, ctx->stream));
    IRL_CK(ctx, cudaMemsetAsync(ctx->d_absmax, 0, 2 * sizeof(int32_t), ctx->stream));
    IRL_LAUNCH(ctx, launch_absmax_i32(da, na, ctx->d_absmax, ctx->stream));
    IRL_LAUNCH(ctx, launch_absmax_i32(db, nb, ctx->d_absmax + 1, ctx->stream));
    IRL_CK(ctx, cudaMemcpyAsync(ctx->h_absmax, ctx->d_absmax, 8, cudaMemcpyDeviceToHost, ctx->stream));
    IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));
    int64_t bound = 0;
    if (overflow(int64_t(k), ctx->h_absmax[0], ctx->h_absmax[1], &bound))
        return set_err(ctx, IRL_ERR_ACCUMULATION_OVERFLOW_RISK, kOverflowMsg + std::to_string(bound));
    if (nc == 0) return IRL_OK;
    IRL_LAUNCH(ctx, launch_gemm_i32(da, db, dc, uint32_t(m), uint32_t(k), uint32_t(n), ctx->stream));
    IRL_CK(ctx, copy_d2h(ctx, c, dc, nc * 4, ctx->stream));
    IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return IRL_OK;
}

// ---------------------------------------------------------------------------
// gemm_mod_psq (modmat.cpp:143-160)
// ---------------------------------------------------------------------------

int irl_gemm_mod_psq(irl_ctx* ctx, const int32_t* a, const int32_t* b, int32_t* c, size_t m,
                     size_t k, size_t n, uint32_t p) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx);
    // digit_decompose(a, p) throws first (modmat.cpp:87, :145).
    if (p >= 256) return set_err(ctx, IRL_ERR_MODULUS_TOO_LARGE, "digit base must be < 2^8");
    if (p == 0) return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "digit base must be positive");
    if (m >= (1u << 30) || n >= (1u << 30) || k >= (1u << 30))
        return set_err(ctx, IRL_ERR_UNSUPPORTED, "dimension above 2^30");
    const size_t ldk = round16(std::max<size_t>(k, 1));
    const size_t na = m * k, nb = k * n;
    const size_t pa = 2 * m * ldk, pb = 2 * n * ldk;  // plane bytes
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = (off + bytes + 127) / 128 * 128;  // TMA / 16-byte vector alignment
        return o;
    };
    const size_t off_a = take(na * 4), off_b = take(nb * 4), off_pa = take(pa), off_pb = take(pb),
                 off_o = take(m * n * 2), off_c = take(m * n * 4);
    IRL_CK(ctx, ctx->ws[0].ensure(off + 16));
    uint8_t* base = ctx->ws[0].as<uint8_t>();
    int32_t* da = reinterpret_cast<int32_t*>(base + off_a);
    int32_t* db = reinterpret_cast<int32_t*>(base + off_b);
    int8_t* pla = reinterpret_cast<int8_t*>(base + off_pa);
    int8_t* plb = reinterpret_cast<int8_t*>(base + off_pb);
    uint16_t* dout = reinterpret_cast<uint16_t*>(base + off_o);
    int32_t* dc = reinterpret_cast<int32_t*>(base + off_c);
    if (na) IRL_CK(ctx, copy_h2d(ctx, da, a, na * 4, ctx->stream));
    if (nb) IRL_CK(ctx, copy_h2d(ctx, db, b, nb * 4, ctx->stream));
    ModTable mt{};
    mt.n = 1;
    mt.mc[0] = make_modconst(p, 2);
    IRL_CK(ctx, cudaMemsetAsync(ctx->d_stats, 0, 2 * sizeof(SplitStats::v[0]), ctx->stream));
    SplitStats* sa = ctx->d_stats;
    // B's stats go to slot 1 of the stats table (a second "modulus" row).
    SplitStats* sb = reinterpret_cast<SplitStats*>(reinterpret_cast<int32_t*>(ctx->d_stats) + 3);
    if (k > 0) {
        IRL_LAUNCH(ctx, launch_split_rows<int32_t>(da, k, 0, uint32_t(m), uint32_t(k), mt, pla, ldk, sa, ctx->stream));
        IRL_LAUNCH(ctx, launch_split_cols<int32_t>(db, n, 0, uint32_t(k), uint32_t(n), mt, plb, ldk, sb, ctx->stream));
    }
    IRL_CK(ctx, cudaMemcpyAsync(ctx->h_stats, ctx->d_stats, 6 * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));
    const int64_t a0 = ctx->h_stats->v[0][0], a1 = ctx->h_stats->v[0][1];
    const int64_t b0 = ctx->h_stats->v[1][0], b1 = ctx->h_stats->v[1][1];
    // small_gemm prechecks in the reference's order: A0B0, A0B1, A1B0 (:147-149).
    int64_t bound = 0;
    if (overflow(int64_t(k), a0, b0, &bound) || overflow(int64_t(k), a0, b1, &bound) ||
        overflow(int64_t(k), a1, b0, &bound))
        return set_err(ctx, IRL_ERR_ACCUMULATION_OVERFLOW_RISK, kOverflowMsg + std::to_string(bound));
    if (m == 0 || n == 0) return IRL_OK;
    PpmmLaunch L = make_launch(mt);
    L.a_planes = pla;
    L.b_planes = plb;
    L.out = dout;
    L.M = uint32_t(m);
    L.N = uint32_t(n);
    L.K = uint32_t(k);
    L.ldk = uint32_t(ldk);
    L.parts = 1;
    int st = run_ppmm(ctx, L, safe_kchunk(a0, a1, b0, b1, uint32_t(k)), ctx->stream);
    if (st) return st;
    IRL_LAUNCH(ctx, launch_transpose_u16_to_i32(dout, uint32_t(m), uint32_t(n), dc, ctx->stream));
    IRL_CK(ctx, copy_d2h(ctx, c, dc, m * n * 4, ctx->stream));
    IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return IRL_OK;
}

// ---------------------------------------------------------------------------
// gemm_mod_Q (modmat.cpp:162-195)
// ---------------------------------------------------------------------------

int irl_gemm_mod_Q(irl_ctx* ctx, const uint8_t* a, const uint8_t* b, uint8_t* c, size_t m,
                   size_t k, size_t n, size_t width, const uint32_t* primes, const uint32_t* exps,
                   size_t nmod) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx);
    int st = validate_moduli(ctx, primes, exps, nmod);
    if (st) return st;
    const Limbs Q = basis_Q(primes, exps, nmod);
    if (Q.size() > kMaxQLimbs) return set_err(ctx, IRL_ERR_UNSUPPORTED, "Q above 2^384 is not supported");
    if (width == 0 || width > kMaxWidth || width < byte_width(Q))
        return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "entry width must be ceil(log256 Q) .. 48 bytes");
    if (m >= (1u << 28) || n >= (1u << 28) || k >= (1u << 28))
        return set_err(ctx, IRL_ERR_UNSUPPORTED, "dimension above 2^28");
    const ModTable mt = make_table(primes, exps, nmod);
    const size_t ldk = round16(std::max<size_t>(k, 1));
    const size_t ba = m * k * width, bb = k * n * width;
    const size_t pa = nmod * 2 * m * ldk, pb = nmod * 2 * n * ldk;
    const size_t raw_a = nmod * m * k * 4, raw_b = nmod * k * n * 4, raw_c = m * n * 4;
    const size_t res = nmod * m * n * 2, outb = m * n * width;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = (off + bytes + 127) / 128 * 128;
        return o;
    };
    const size_t o_a = take(ba), o_b = take(bb), o_pa = take(pa), o_pb = take(pb),
                 o_ra = take(raw_a), o_rb = take(raw_b), o_rc = take(raw_c), o_res = take(res),
                 o_out = take(outb);
    IRL_CK(ctx, ctx->ws[0].ensure(off + 16));
    uint8_t* base = ctx->ws[0].as<uint8_t>();
    uint8_t* dA = base + o_a;
    uint8_t* dB = base + o_b;
    int8_t* pla = reinterpret_cast<int8_t*>(base + o_pa);
    int8_t* plb = reinterpret_cast<int8_t*>(base + o_pb);
    int32_t* ra = reinterpret_cast<int32_t*>(base + o_ra);
    int32_t* rb = reinterpret_cast<int32_t*>(base + o_rb);
    int32_t* rc = reinterpret_cast<int32_t*>(base + o_rc);
    uint16_t* dres = reinterpret_cast<uint16_t*>(base + o_res);
    uint8_t* dout = base + o_out;
    if (ba) IRL_CK(ctx, copy_h2d(ctx, dA, a, ba, ctx->stream));
    if (bb) IRL_CK(ctx, copy_h2d(ctx, dB, b, bb, ctx->stream));
    IRL_CK(ctx, cudaMemsetAsync(pla, 0, pa, ctx->stream));
    IRL_CK(ctx, cudaMemsetAsync(plb, 0, pb, ctx->stream));
    // Two stats tables: A in d_stats[0..], B in the workspace tail.
    IRL_CK(ctx, ctx->ws[1].ensure(sizeof(SplitStats)));
    SplitStats* sa = ctx->d_stats;
    SplitStats* sb = ctx->ws[1].as<SplitStats>();
    IRL_CK(ctx, cudaMemsetAsync(sa, 0, sizeof(SplitStats), ctx->stream));
    IRL_CK(ctx, cudaMemsetAsync(sb, 0, sizeof(SplitStats), ctx->stream));
    // Residue extraction (:168-176) fused with the digit split.
    IRL_LAUNCH(ctx, launch_split_bigint(dA, uint32_t(width), uint32_t(m), uint32_t(k), 0, mt, pla, ldk,
                                        uint32_t(m), 0, ra, sa, ctx->stream));
    IRL_LAUNCH(ctx, launch_split_bigint(dB, uint32_t(width), uint32_t(k), uint32_t(n), 1, mt, plb, ldk,
                                        uint32_t(n), 0, rb, sb, ctx->stream));
    std::vector<SplitStats> hs(2);
    IRL_CK(ctx, cudaMemcpyAsync(&hs[0], sa, sizeof(SplitStats), cudaMemcpyDeviceToHost, ctx->stream));
    IRL_CK(ctx, cudaMemcpyAsync(&hs[1], sb, sizeof(SplitStats), cudaMemcpyDeviceToHost, ctx->stream));
    IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));

    // Per-modulus checks in basis order, as the reference loop would raise them.
    int64_t a0m = 1, a1m = 0, b0m = 1, b1m = 0;
    std::vector<uint32_t> inv(nmod);
    for (size_t i = 0; i < nmod; ++i) {
        const uint32_t mod = mt.mc[i].m;
        int64_t bound = 0;
        if (exps[i] == 2) {
            if (primes[i] >= 256)
                return set_err(ctx, IRL_ERR_MODULUS_TOO_LARGE, "digit base must be < 2^8");
            const int64_t A0 = hs[0].v[i][0], A1 = hs[0].v[i][1];
            const int64_t B0 = hs[1].v[i][0], B1 = hs[1].v[i][1];
            if (overflow(int64_t(k), A0, B0, &bound) || overflow(int64_t(k), A0, B1, &bound) ||
                overflow(int64_t(k), A1, B0, &bound))
                return set_err(ctx, IRL_ERR_ACCUMULATION_OVERFLOW_RISK, kOverflowMsg + std::to_string(bound));
            a0m = std::max(a0m, A0);
            a1m = std::max(a1m, A1);
            b0m = std::max(b0m, B0);
            b1m = std::max(b1m, B1);
        } else if (overflow(int64_t(k), hs[0].v[i][2], hs[1].v[i][2], &bound)) {
            return set_err(ctx, IRL_ERR_ACCUMULATION_OVERFLOW_RISK, kOverflowMsg + std::to_string(bound));
        }
        Limbs qi = Q;
        divmod_small(qi, mod);
        Limbs tmp = qi;
        const uint32_t rem = divmod_small(tmp, mod);  // (Q/m) mod m
        if (!inv_mod(rem, mod, &inv[i]))
            return set_err(ctx, IRL_ERR_NOT_COPRIME, "CRT basis is not coprime");
    }
    if (m == 0 || n == 0) return IRL_OK;

    // e = 2 moduli: tcgen05 PPMM over all planes (e = 1 slots are zero planes
    // and are overwritten below by the exact int32 path).
    PpmmLaunch L = make_launch(mt);
    L.a_planes = pla;
    L.b_planes = plb;
    L.out = dres;
    L.M = uint32_t(m);
    L.N = uint32_t(n);
    L.K = uint32_t(k);
    L.ldk = uint32_t(ldk);
    L.parts = 1;
    st = run_ppmm(ctx, L, safe_kchunk(a0m, a1m, b0m, b1m, uint32_t(k)), ctx->stream);
    if (st) return st;
    for (size_t i = 0; i < nmod; ++i) {
        if (exps[i] != 1) continue;
        IRL_LAUNCH(ctx, launch_gemm_i32(ra + i * m * k, rb + i * k * n, rc, uint32_t(m), uint32_t(k),
                                        uint32_t(n), ctx->stream));
        IRL_LAUNCH(ctx, launch_reduce_raw(rc, uint32_t(m), uint32_t(n), uint32_t(i), mt.mc[i], dres, ctx->stream));
    }
    // CRT lift (:180-193).
    CrtTable t{};
    t.nmod = uint32_t(nmod);
    t.limbs = uint32_t(Q.size());
    t.width = uint32_t(width);
    for (size_t i = 0; i < nmod; ++i) {
        t.m[i] = mt.mc[i].m;
        t.inv[i] = inv[i];
        Limbs qi = Q;
        divmod_small(qi, t.m[i]);
        for (size_t j = 0; j < qi.size() && j < kMaxQLimbs; ++j) t.qi[i][j] = qi[j];
    }
    for (int s = 0; s < 5; ++s) {
        const uint32_t mul = 16u >> s;
        uint64_t carry = 0;
        for (size_t j = 0; j <= Q.size(); ++j) {
            const uint64_t v = (j < Q.size() ? uint64_t(Q[j]) * mul : 0) + carry;
            t.qmul[s][j] = uint32_t(v);
            carry = v >> 32;
        }
    }
    IRL_LAUNCH(ctx, launch_crt_lift(dres, uint32_t(m), uint32_t(n), t, dout, ctx->stream));
    IRL_CK(ctx, copy_d2h(ctx, c, dout, outb, ctx->stream));
    IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return IRL_OK;
}

// ---------------------------------------------------------------------------
// Device-level building blocks
// ---------------------------------------------------------------------------

int irl_split_rows_u16(irl_ctx* ctx, const uint16_t* res, size_t ld_res, size_t plane_stride,
                       size_t rows, size_t cols, const uint32_t* primes, const uint32_t* exps,
                       size_t nmod, int8_t* planes, size_t ldk, void* stream) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx);
    int st = validate_moduli(ctx, primes, exps, nmod);
    if (st) return st;
    if (ldk % 16 || ldk < cols) return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "ldk must be >= cols and a multiple of 16");
    IRL_LAUNCH(ctx, launch_split_rows<uint16_t>(res, ld_res, plane_stride, uint32_t(rows), uint32_t(cols),
                                                make_table(primes, exps, nmod), planes, ldk, nullptr,
                                                pick_stream(ctx, stream)));
    return IRL_OK;
}

int irl_split_cols_u16(irl_ctx* ctx, const uint16_t* res, size_t ld_res, size_t plane_stride,
                       size_t k, size_t n, const uint32_t* primes, const uint32_t* exps,
                       size_t nmod, int8_t* planes, size_t ldk, void* stream) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx);
    int st = validate_moduli(ctx, primes, exps, nmod);
    if (st) return st;
    if (ldk % 16 || ldk < k) return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "ldk must be >= k and a multiple of 16");
    IRL_LAUNCH(ctx, launch_split_cols<uint16_t>(res, ld_res, plane_stride, uint32_t(k), uint32_t(n),
                                                make_table(primes, exps, nmod), planes, ldk, nullptr,
                                                pick_stream(ctx, stream)));
    return IRL_OK;
}

int irl_split_bigint(irl_ctx* ctx, const uint8_t* entries, size_t width, size_t rows, size_t cols,
                     int transpose, const uint32_t* primes, const uint32_t* exps, size_t nmod,
                     int8_t* planes, size_t ldk, void* stream) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx);
    int st = validate_moduli(ctx, primes, exps, nmod);
    if (st) return st;
    for (size_t i = 0; i < nmod; ++i)
        if (exps[i] != 2 || primes[i] >= 256)
            return set_err(ctx, IRL_ERR_UNSUPPORTED, "plane split needs e = 2 and p < 256");
    if (width == 0 || width > kMaxWidth) return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "width must be 1..48");
    IRL_LAUNCH(ctx, launch_split_bigint(entries, uint32_t(width), uint32_t(rows), uint32_t(cols), transpose,
                                        make_table(primes, exps, nmod), planes, ldk,
                                        uint32_t(transpose ? cols : rows), 0, nullptr, nullptr,
                                        pick_stream(ctx, stream)));
    return IRL_OK;
}

int irl_ppmm_planes(irl_ctx* ctx, const int8_t* a_planes, const int8_t* b_planes, uint16_t* out,
                    size_t parts, size_t m, size_t n, size_t k, size_t ldk,
                    const uint32_t* primes, const uint32_t* exps, size_t nmod, int accumulate,
                    void* stream) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx);
    int st = validate_moduli(ctx, primes, exps, nmod);
    if (st) return st;
    if (ldk % 16 || ldk < k) return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "ldk must be >= k and a multiple of 16");
    const ModTable mt = make_table(primes, exps, nmod);
    PpmmLaunch L = make_launch(mt);
    L.a_planes = a_planes;
    L.b_planes = b_planes;
    L.out = out;
    L.M = uint32_t(m);
    L.N = uint32_t(n);
    L.K = uint32_t(k);
    L.ldk = uint32_t(ldk);
    L.parts = uint32_t(parts);
    L.accumulate = accumulate;
    int64_t h = 0;
    for (size_t i = 0; i < nmod; ++i) h = std::max<int64_t>(h, (primes[i] - 1) / 2 + (primes[i] % 2 == 0));
    return run_ppmm(ctx, L, safe_kchunk(h, h, h, h, uint32_t(k)), pick_stream(ctx, stream));
}

int irl_crt_lift(irl_ctx* ctx, const uint16_t* res, size_t m, size_t n, uint8_t* out,
                 size_t width, const uint32_t* primes, const uint32_t* exps, size_t nmod,
                 void* stream) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx);
    int st = validate_moduli(ctx, primes, exps, nmod);
    if (st) return st;
    const Limbs Q = basis_Q(primes, exps, nmod);
    if (Q.size() > kMaxQLimbs || width > kMaxWidth || width < byte_width(Q))
        return set_err(ctx, IRL_ERR_UNSUPPORTED, "Q / width out of range");
    CrtTable t{};
    t.nmod = uint32_t(nmod);
    t.limbs = uint32_t(Q.size());
    t.width = uint32_t(width);
    for (size_t i = 0; i < nmod; ++i) {
        t.m[i] = exps[i] == 2 ? primes[i] * primes[i] : primes[i];
        Limbs qi = Q;
        divmod_small(qi, t.m[i]);
        Limbs tmp = qi;
        if (!inv_mod(divmod_small(tmp, t.m[i]), t.m[i], &t.inv[i]))
            return set_err(ctx, IRL_ERR_NOT_COPRIME, "CRT basis is not coprime");
        for (size_t j = 0; j < qi.size() && j < kMaxQLimbs; ++j) t.qi[i][j] = qi[j];
    }
    for (int s = 0; s < 5; ++s) {
        const uint32_t mul = 16u >> s;
        uint64_t carry = 0;
        for (size_t j = 0; j <= Q.size(); ++j) {
            const uint64_t v = (j < Q.size() ? uint64_t(Q[j]) * mul : 0) + carry;
            t.qmul[s][j] = uint32_t(v);
            carry = v >> 32;
        }
    }
    IRL_LAUNCH(ctx, launch_crt_lift(res, uint32_t(m), uint32_t(n), t, out, pick_stream(ctx, stream)));
    return IRL_OK;
}

int irl_rescale_residues(irl_ctx* ctx, const uint16_t* in, size_t ld_in, size_t count, const uint32_t* primes,
                         const uint32_t* exps, size_t nmod, size_t drop, int round, uint16_t* out, size_t ld_out,
                         void* stream) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx);
    int st = validate_moduli(ctx, primes, exps, nmod);
    if (st) return st;
    if (drop == 0 || drop >= nmod) return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "rescale: need 0 < drop < nmod");
    RescaleTable t{};
    t.nmod = uint32_t(nmod);
    t.drop = uint32_t(drop);
    unsigned long long delta = 1;
    for (size_t i = 0; i < nmod; ++i) {
        t.m[i] = exps[i] == 2 ? primes[i] * primes[i] : primes[i];
        t.magic[i] = static_cast<uint32_t>((1ull << 32) / t.m[i]);
        t.c32[i] = static_cast<uint32_t>((1ull << 32) % t.m[i]);
        if (i >= nmod - drop) {
            if (delta >= (1ull << 48) / t.m[i])
                return set_err(ctx, IRL_ERR_UNSUPPORTED, "rescale: Delta must stay below 2^48");
            delta *= t.m[i];
        }
    }
    t.delta = delta;
    auto inv = [](unsigned long long a, uint32_t m, uint32_t* out) {
        uint32_t v = 0;
        if (!inv_mod(static_cast<uint32_t>(a % m), m, &v)) return false;
        *out = v;
        return true;
    };
    for (size_t i = 0; i < nmod; ++i) {
        const uint32_t m = t.m[i];
        t.add[i] = round ? static_cast<uint32_t>((delta / 2) % m) : 0;
        if (i < nmod - drop) {
            if (!inv(delta, m, &t.dinv[i])) return set_err(ctx, IRL_ERR_NOT_COPRIME, "CRT basis is not coprime");
        } else {
            t.cq[i] = delta / m;
            if (!inv(t.cq[i], m, &t.cinv[i])) return set_err(ctx, IRL_ERR_NOT_COPRIME, "CRT basis is not coprime");
        }
    }
    for (size_t jj = 0; jj < drop && jj < 3; ++jj) {
        const size_t j = nmod - drop + jj;
        for (size_t i = 0; i < nmod - drop; ++i) {
            const uint64_t v = (t.cq[j] % t.m[i]) * t.dinv[i] % t.m[i];
            t.w[jj][i] = static_cast<uint32_t>((t.m[i] - v) % t.m[i]);
        }
    }
    IRL_LAUNCH(ctx, launch_rescale(in, ld_in, count, t, out, ld_out, pick_stream(ctx, stream)));
    return IRL_OK;
}

// ---------------------------------------------------------------------------
// RGSW CCMM engine
// ---------------------------------------------------------------------------

int irl_ccmm_create(irl_ctx* ctx, size_t parts, size_t m, size_t k, size_t max_n,
                    const uint32_t* primes, const uint32_t* exps, size_t nmod, irl_ccmm** out) {
    if (!ctx || !out) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx);
    *out = nullptr;
    int st = validate_moduli(ctx, primes, exps, nmod);
    if (st) return st;
    for (size_t i = 0; i < nmod; ++i)
        if (primes[i] >= 256) return set_err(ctx, IRL_ERR_MODULUS_TOO_LARGE, "digit base must be < 2^8");
    if (parts == 0 || m == 0 || k == 0 || max_n == 0 || nmod == 0)
        return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "ccmm: nonpositive dimensions");
    if (m >= (1u << 24) || k >= (1u << 24) || max_n >= (1u << 24) || parts > 255)
        return set_err(ctx, IRL_ERR_UNSUPPORTED, "ccmm: dimension out of range");
    auto* e = new irl_ccmm();
    e->ctx = ctx;
    e->parts = parts;
    e->M = m;
    e->K = k;
    e->ldk = round16(k);
    e->max_n = max_n;
    e->nmod = nmod;
    e->mt = make_table(primes, exps, nmod);
    int64_t h = 0;
    for (size_t i = 0; i < nmod; ++i) h = std::max<int64_t>(h, (primes[i] - 1) / 2 + (primes[i] % 2 == 0));
    e->kchunk = safe_kchunk(h, h, h, h, uint32_t(k));
    const size_t db_b = parts * nmod * 2 * m * e->ldk, qp_b = nmod * 2 * max_n * e->ldk,
                 qr_b = nmod * k * max_n * 2, out_b = parts * nmod * max_n * m * 2;
    cudaError_t err = cudaMalloc(&e->db, db_b);
    if (err == cudaSuccess) err = cudaMalloc(&e->qplanes, qp_b);
    if (err == cudaSuccess) err = cudaMalloc(&e->qres, qr_b);
    if (err == cudaSuccess) err = cudaMalloc(&e->out, out_b);
    if (err == cudaSuccess) err = cudaMalloc(&e->progress, kScheduleScratchBytes);
    if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking);
    if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&e->h2d_stream, cudaStreamNonBlocking);
    if (err == cudaSuccess) err = cudaMemsetAsync(e->db, 0, db_b, ctx->stream);
    if (err == cudaSuccess) err = cudaMalloc(&e->part_cnt, nmod * parts * sizeof(uint32_t));
    e->part_done.resize(nmod);
    e->h2d_done.resize(nmod);
    e->cnt_zeroed.resize(nmod);
    for (size_t i = 0; err == cudaSuccess && i < nmod; ++i) {
        err = cudaEventCreateWithFlags(&e->part_done[i], cudaEventDisableTiming);
        if (err == cudaSuccess) err = cudaEventCreateWithFlags(&e->h2d_done[i], cudaEventDisableTiming);
        if (err == cudaSuccess) err = cudaEventCreateWithFlags(&e->cnt_zeroed[i], cudaEventDisableTiming);
    }
    if (err != cudaSuccess) {
        irl_ccmm_destroy(e);
        return cuda_fail(ctx, err, "irl_ccmm_create");
    }
    e->bytes = db_b + qp_b + qr_b + out_b;
    *out = e;
    return IRL_OK;
}

int irl_ccmm_destroy(irl_ccmm* e) {
    if (!e) return IRL_OK;
    cudaSetDevice(e->ctx->device);
    cudaStreamSynchronize(e->ctx->stream);
    if (e->copy_stream) cudaStreamSynchronize(e->copy_stream);
    if (e->h2d_stream) cudaStreamSynchronize(e->h2d_stream);
    for (auto ev : e->part_done)
        if (ev) cudaEventDestroy(ev);
    for (auto ev : e->h2d_done)
        if (ev) cudaEventDestroy(ev);
    for (auto ev : e->cnt_zeroed)
        if (ev) cudaEventDestroy(ev);
    cudaFree(e->part_cnt);
    if (e->copy_stream) cudaStreamDestroy(e->copy_stream);
    if (e->h2d_stream) cudaStreamDestroy(e->h2d_stream);
    cudaFree(e->db);
    cudaFree(e->qplanes);
    cudaFree(e->qres);
    cudaFree(e->out);
    cudaFree(e->progress);
    for (size_t i = 0; i < e->n_mirror; ++i)
        if (e->mirror_ipc[i]) cudaIpcCloseMemHandle(e->mirror[i]);
    cudaFree(e->recv);
    delete e;
    return IRL_OK;
}

// ---- fused a-part exchange: the a-part PPMM epilogue stores its
// tiles straight into the peers' receive buffers over NVLink ------------------

int irl_ccmm_alloc_recv(irl_ccmm* e, size_t n, void** dev_ptr, uint8_t* ipc_handle) {
    if (!e || !dev_ptr) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* ctx = e->ctx;
    Guard g(ctx);
    if (n == 0 || n > e->max_n) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "ccmm: receive width out of range");
    if (e->recv) cudaFree(e->recv);
    e->recv = nullptr;
    IRL_CK(ctx, cudaMalloc(&e->recv, e->nmod * n * e->M * sizeof(uint16_t)));
    IRL_CK(ctx, cudaMemset(e->recv, 0, e->nmod * n * e->M * sizeof(uint16_t)));
    e->recv_n = n;
    *dev_ptr = e->recv;
    if (ipc_handle) {
        cudaIpcMemHandle_t h;
        IRL_CK(ctx, cudaIpcGetMemHandle(&h, e->recv));
        std::memcpy(ipc_handle, &h, sizeof(h));
    }
    return IRL_OK;
}

static int set_mirrors(irl_ccmm* e, size_t part, size_t n, uint16_t* const* ptrs, const uint8_t* handles,
                       size_t count) {
    irl_ctx* ctx = e->ctx;
    if (count > kMaxMirrors || part >= e->parts || (count && (n == 0 || n > e->max_n)))
        return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "ccmm: bad mirror set");
    for (size_t i = 0; i < e->n_mirror; ++i)
        if (e->mirror_ipc[i]) cudaIpcCloseMemHandle(e->mirror[i]);
    e->n_mirror = 0;
    for (size_t i = 0; i < count; ++i) {
        if (handles) {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, handles + i * sizeof(h), sizeof(h));
            void* p = nullptr;
            const cudaError_t err = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
            if (err != cudaSuccess) {
                for (size_t j = 0; j < i; ++j) cudaIpcCloseMemHandle(e->mirror[j]);
                return cuda_fail(ctx, err, "cudaIpcOpenMemHandle");
            }
            e->mirror[i] = static_cast<uint16_t*>(p);
            e->mirror_ipc[i] = true;
        } else {
            e->mirror[i] = ptrs[i];
            e->mirror_ipc[i] = false;
        }
    }
    e->n_mirror = count;
    e->mirror_part = part;
    e->mirror_n = n;
    return IRL_OK;
}

int irl_ccmm_set_mirrors(irl_ccmm* e, size_t part, size_t n, const uint8_t* ipc_handles, size_t count) {
    if (!e || (count && !ipc_handles)) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(e->ctx);
    return set_mirrors(e, part, n, nullptr, ipc_handles, count);
}

int irl_ccmm_set_mirror_ptrs(irl_ccmm* e, size_t part, size_t n, uint16_t* const* dev_ptrs, size_t count) {
    if (!e || (count && !dev_ptrs)) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(e->ctx);
    return set_mirrors(e, part, n, dev_ptrs, nullptr, count);
}

uint64_t irl_ccmm_device_bytes(const irl_ccmm* e) { return e ? e->bytes : 0; }

int irl_ccmm_buffers(irl_ccmm* e, void** qres, void** out) {
    if (!e) return IRL_ERR_INVALID_ARGUMENT;
    if (qres) *qres = e->qres;
    if (out) *out = e->out;
    return IRL_OK;
}

int irl_ccmm_load_part(irl_ccmm* e, size_t part, const uint16_t* res, int res_on_device) {
    if (!e) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* ctx = e->ctx;
    Guard g(ctx);
    if (part >= e->parts) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "ccmm: part index out of range");
    const size_t plane_elems = e->M * e->K;
    int8_t* dst = e->db + part * e->nmod * 2 * e->M * e->ldk;
    for (size_t i = 0; i < e->nmod; ++i) {
        const uint16_t* src = res + i * plane_elems;
        if (!res_on_device) {
            IRL_CK(ctx, ctx->ws[2].ensure(plane_elems * 2));
            IRL_CK(ctx, copy_h2d(ctx, ctx->ws[2].p, src, plane_elems * 2, ctx->stream));
            src = ctx->ws[2].as<uint16_t>();
        }
        ModTable one{};
        one.n = 1;
        one.mc[0] = e->mt.mc[i];
        IRL_LAUNCH(ctx, launch_split_rows<uint16_t>(src, e->K, 0, uint32_t(e->M), uint32_t(e->K), one,
                                                    dst + i * 2 * e->M * e->ldk, e->ldk, nullptr, ctx->stream));
    }
    IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return IRL_OK;
}

int irl_ccmm_load_part_bigint(irl_ccmm* e, size_t part, const uint8_t* entries, size_t width) {
    if (!e) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* ctx = e->ctx;
    Guard g(ctx);
    if (part >= e->parts) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "ccmm: part index out of range");
    if (width == 0 || width > kMaxWidth) return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "width must be 1..48");
    for (size_t i = 0; i < e->nmod; ++i)
        if (e->mt.mc[i].e != 2) return set_err(ctx, IRL_ERR_UNSUPPORTED, "bigint ingest needs e = 2");
    int8_t* dst = e->db + part * e->nmod * 2 * e->M * e->ldk;
    const size_t row_bytes = e->K * width;
    const size_t chunk = std::max<size_t>(1, std::min<size_t>(e->M, (size_t(256) << 20) / row_bytes));
    IRL_CK(ctx, ctx->ws[2].ensure(chunk * row_bytes));
    for (size_t r0 = 0; r0 < e->M; r0 += chunk) {
        const size_t rows = std::min(chunk, e->M - r0);
        IRL_CK(ctx, copy_h2d(ctx, ctx->ws[2].p, entries + r0 * row_bytes, rows * row_bytes, ctx->stream));
        IRL_LAUNCH(ctx, launch_split_bigint(ctx->ws[2].as<uint8_t>(), uint32_t(width), uint32_t(rows),
                                            uint32_t(e->K), 0, e->mt, dst, e->ldk, uint32_t(e->M),
                                            uint32_t(r0), nullptr, nullptr, ctx->stream));
        IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));
    }
    return IRL_OK;
}

// Streaming ingest of one part from the reference's BigMatrix file
// (save_big_matrix, modmat.cpp:216-231: "rows cols Q\n" then rows*cols
// little-endian entries of ceil(log256 Q) bytes). Double-buffered: the file
// read of chunk i+1 into pinned memory overlaps the H2D and residue/digit
// split of chunk i, so a 2^17-template slice (148 GB of entries) never has to
// sit in host memory.
int irl_ccmm_load_part_file(irl_ccmm* e, size_t part, const char* path) {
    if (!e || !path) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* ctx = e->ctx;
    Guard g(ctx);
    if (part >= e->parts) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "ccmm: part index out of range");
    for (size_t i = 0; i < e->nmod; ++i)
        if (e->mt.mc[i].e != 2) return set_err(ctx, IRL_ERR_UNSUPPORTED, "bigint ingest needs e = 2");
    std::FILE* f = std::fopen(path, "rb");
    if (!f) return set_err(ctx, IRL_ERR_IO, std::string("cannot open ") + path);
    struct Closer {
        std::FILE* f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    unsigned long long rows = 0, cols = 0;
    char qbuf[256];
    if (std::fscanf(f, "%llu %llu %255s", &rows, &cols, qbuf) != 3 || std::fgetc(f) != '\n')
        return set_err(ctx, IRL_ERR_IO, std::string("bad matrix header in ") + path);
    if (rows != e->M || cols != e->K)
        return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "ccmm: file matrix is not M x K for this engine");
    // the file's modulus must be the engine's Q
    std::vector<uint32_t> ps(e->nmod), es(e->nmod);
    for (size_t i = 0; i < e->nmod; ++i) ps[i] = e->mt.mc[i].p, es[i] = e->mt.mc[i].e;
    const Limbs Q = basis_Q(ps.data(), es.data(), e->nmod);
    Limbs fq{0};
    for (const char* c = qbuf; *c; ++c) {
        if (*c < '0' || *c > '9') return set_err(ctx, IRL_ERR_IO, "bad modulus in matrix header");
        uint64_t carry = static_cast<uint64_t>(*c - '0');
        for (auto& limb : fq) {
            const uint64_t v = static_cast<uint64_t>(limb) * 10 + carry;
            limb = static_cast<uint32_t>(v);
            carry = v >> 32;
        }
        if (carry) fq.push_back(static_cast<uint32_t>(carry));
    }
    while (fq.size() > 1 && fq.back() == 0) fq.pop_back();
    if (fq != Q) return set_err(ctx, IRL_ERR_IO, "ccmm: file modulus differs from the engine's basis Q");
    const size_t width = byte_width(Q);
    if (width > kMaxWidth) return set_err(ctx, IRL_ERR_UNSUPPORTED, "Q too wide");
    const long data_off = std::ftell(f);
    const int fd = ::fileno(f);
    int8_t* dst = e->db + part * e->nmod * 2 * e->M * e->ldk;
    const size_t row_bytes = e->K * width;
    const size_t chunk = std::max<size_t>(1, std::min<size_t>(e->M, (size_t(256) << 20) / row_bytes));
    IRL_CK(ctx, ctx->ws[2].ensure(chunk * row_bytes));
    IRL_CK(ctx, ctx->ws[3].ensure(chunk * row_bytes));
    uint8_t* host[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    struct Cleanup {
        uint8_t** h;
        cudaEvent_t* ev;
        ~Cleanup() {
            for (int i = 0; i < 2; ++i) {
                if (ev[i]) cudaEventSynchronize(ev[i]), cudaEventDestroy(ev[i]);
                if (h[i]) cudaFreeHost(h[i]);
            }
        }
    } cleanup{host, done};
    for (int i = 0; i < 2; ++i) {
        IRL_CK(ctx, cudaMallocHost(&host[i], chunk * row_bytes));
        IRL_CK(ctx, cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
    uint8_t* dev[2] = {ctx->ws[2].as<uint8_t>(), ctx->ws[3].as<uint8_t>()};
    size_t ci = 0;
    for (size_t r0 = 0; r0 < e->M; r0 += chunk, ++ci) {
        const size_t b = ci % 2, nrows = std::min(chunk, e->M - r0), bytes = nrows * row_bytes;
        IRL_CK(ctx, cudaEventSynchronize(done[b]));  // buffer b's previous chunk is on the device
        // 4 readers per chunk (pread at disjoint offsets): page-cache copies and
        // NVMe queues both scale with concurrent requests
        {
            constexpr int kReaders = 4;
            bool ok[kReaders];
            std::thread th[kReaders];
            const size_t piece = (bytes + kReaders - 1) / kReaders;
            for (int t = 0; t < kReaders; ++t) {
                th[t] = std::thread([&, t] {
                    const size_t lo = std::min(bytes, t * piece), hi = std::min(bytes, lo + piece);
                    size_t got = 0;
                    while (got < hi - lo) {
                        const ssize_t r = ::pread(fd, host[b] + lo + got, hi - lo - got,
                                                  static_cast<off_t>(data_off + r0 * row_bytes + lo + got));
                        if (r <= 0) break;
                        got += static_cast<size_t>(r);
                    }
                    ok[t] = got == hi - lo;
                });
            }
            bool all = true;
            for (int t = 0; t < kReaders; ++t) th[t].join(), all = all && ok[t];
            if (!all) return set_err(ctx, IRL_ERR_IO, std::string("truncated matrix file ") + path);
        }
        IRL_CK(ctx, cudaMemcpyAsync(dev[b], host[b], bytes, cudaMemcpyHostToDevice, ctx->stream));
        IRL_LAUNCH(ctx, launch_split_bigint(dev[b], uint32_t(width), uint32_t(nrows), uint32_t(e->K), 0, e->mt, dst,
                                            e->ldk, uint32_t(e->M), uint32_t(r0), nullptr, nullptr, ctx->stream));
        IRL_CK(ctx, cudaEventRecord(done[b], ctx->stream));
    }
    IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return IRL_OK;
}

int irl_ccmm_synth_db(irl_ccmm* e, uint64_t seed, uint32_t first_part) {
    if (!e) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* ctx = e->ctx;
    Guard g(ctx);
    for (size_t p = 0; p < e->parts; ++p) {
        IRL_LAUNCH(ctx, launch_synth_planes(seed, first_part + uint32_t(p), 1, uint32_t(e->M), uint32_t(e->K), e->mt,
                                            e->db + p * e->nmod * 2 * e->M * e->ldk, e->ldk, ctx->stream));
    }
    IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return IRL_OK;
}

// PPMMs of parts [part0, part0 + nparts) for moduli [m0, m0 + nm); `out`
// points at the [part0][0][0][0] corner of a [parts][nmod][n][M] tensor.
static int ccmm_parts(irl_ccmm* e, size_t n, size_t part0, size_t nparts, uint16_t* out,
                      cudaStream_t s, size_t m0 = 0, size_t nm = 0, uint32_t* part_done = nullptr) {
    irl_ctx* ctx = e->ctx;
    if (nm == 0) nm = e->nmod;
    ModTable sub{};
    sub.n = uint32_t(nm);
    for (size_t i = 0; i < nm; ++i) sub.mc[i] = e->mt.mc[m0 + i];
    PpmmLaunch L = make_launch(sub);
    L.a_planes = e->db + (part0 * e->nmod + m0) * 2 * e->M * e->ldk;
    L.b_planes = e->qplanes + m0 * 2 * n * e->ldk;
    L.out = out + m0 * n * e->M;
    L.M = uint32_t(e->M);
    L.N = uint32_t(n);
    L.K = uint32_t(e->K);
    L.ldk = uint32_t(e->ldk);
    L.parts = uint32_t(nparts);
    L.a_part_rows = e->nmod * 2 * e->M;
    L.out_part_elems = e->nmod * n * e->M;
    L.progress = e->progress;
    L.part_done = part_done;
    if (e->n_mirror && n == e->mirror_n && e->mirror_part >= part0 && e->mirror_part < part0 + nparts) {
        L.n_mirror = static_cast<uint32_t>(e->n_mirror);
        L.mirror_part = static_cast<uint32_t>(e->mirror_part - part0);
        for (size_t i = 0; i < e->n_mirror; ++i) L.mirror[i] = e->mirror[i] + m0 * n * e->M;
    }
    return run_ppmm(ctx, L, e->kchunk, s);
}

int irl_ccmm_run_device(irl_ccmm* e, const uint16_t* q_res_dev, int q_ready, size_t n,
                        size_t part0, size_t nparts, uint16_t* out_dev, void* stream) {
    if (!e) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* ctx = e->ctx;
    Guard g(ctx);
    if (n == 0 || n > e->max_n) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "ccmm: query width out of range");
    if (part0 + nparts > e->parts) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "ccmm: part range out of range");
    cudaStream_t s = pick_stream(ctx, stream);
    if (!q_res_dev) q_res_dev = e->qres;
    if (!out_dev) out_dev = e->out + part0 * e->nmod * n * e->M;
    if (!q_ready) {
        IRL_LAUNCH(ctx, launch_split_cols<uint16_t>(q_res_dev, n, e->K * n, uint32_t(e->K), uint32_t(n), e->mt,
                                                    e->qplanes, e->ldk, nullptr, s));
    }
    // qplanes rows are laid out with stride n (not max_n): [nmod][2][n][ldk].
    if (nparts == 0) return IRL_OK;  // split only
    return ccmm_parts(e, n, part0, nparts, out_dev, s);
}

// One column chunk [n0, n0 + w) of an e2e run (query columns of the host
// batch of width n), pipelined by modulus chunks: H2D of chunk c+1 and D2H of
// chunk c-1 run on their own streams while chunk c is split and multiplied.
// cuStreamWaitValue32 (driver API, resolved once); nullptr if unavailable.
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static WaitValueFn wait_value_fn() {
    static WaitValueFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return static_cast<WaitValueFn>(nullptr);
        }
        return reinterpret_cast<WaitValueFn>(p);
    }();
    return fn;
}

static int ccmm_run_columns(irl_ccmm* e, const uint16_t* q_res_host, size_t n, size_t n0, size_t w,
                            uint16_t* out_host) {
    irl_ctx* ctx = e->ctx;
    cudaStream_t s = ctx->stream;
    const size_t nmod = e->nmod, K = e->K, M = e->M;
    // Modulus chunks. With stream memory ops (part-granular D2H below) the
    // pipeline is 1, 3, rest: the first GEMM starts after one modulus of H2D,
    // the second chunk's GEMMs cover the H2D of everything else, and the big
    // last launch streams each (modulus, part) block out as soon as its tiles
    // are stored -- three launches, so three launch tails. Without them the
    // chunks are graded 1, 2, 3, ..., 3, 2, 1 (whole-chunk D2H, short tail).
    const bool memops = e->memops && wait_value_fn() != nullptr;
    std::vector<size_t> bounds{0};
    {
        std::vector<size_t> sizes;
        size_t left = nmod;
        // Chunk planner (stream memory ops available): simulate the pipeline
        // with per-modulus GEMM time g (6 M w K parts ops at ~2.9 POPS plus a
        // launch) and H2D time h (2 K w bytes at ~50 GB/s). The first chunk is
        // one modulus; each next chunk takes every modulus whose residues have
        // landed by the time the previous chunk's GEMMs end, so the GEMMs never
        // wait on PCIe when they can help it and launches stay few. c4 on one
        // GPU plans 1, 7, 16; one part per GPU (N = 8, H2D-bound) plans one
        // modulus per chunk; two parts 1, 1, 2, 4, 7, 9.
        if (memops) {
            const double g = 6.0 * double(M) * double(w) * double(K) * double(e->parts) / 2.9e15 + 5e-5;
            const double h = 2.0 * double(K) * double(w) / 50e9;
            double gemm_end = h + g;  // first chunk: one modulus
            size_t assigned = std::min<size_t>(1, nmod);
            sizes.push_back(assigned);
            while (assigned < nmod) {
                size_t landed = static_cast<size_t>(gemm_end / h);
                landed = std::min(nmod, std::max(landed, assigned + 1));
                const size_t c = landed - assigned;
                const double start = std::max(gemm_end, double(landed) * h);
                gemm_end = start + double(c) * g;
                sizes.push_back(c);
                assigned += c;
            }
            left = 0;
        }
        for (size_t g : {1, 2})
            if (left > 2 * g) sizes.push_back(g), left -= g;
        std::vector<size_t> tail;
        for (size_t g : {1, 2})
            if (left > g + 2) tail.push_back(g), left -= g;
        while (left > 0) {
            const size_t g = std::min<size_t>(3, left);
            sizes.push_back(g);
            left -= g;
        }
        sizes.insert(sizes.end(), tail.rbegin(), tail.rend());
        if (const char* env = std::getenv("IRL_E2E_CHUNKS")) {  // experiment knob: "1,2,3,6,..."
            std::vector<size_t> alt;
            size_t sum = 0;
            for (const char* c = env; *c;) {
                char* end = nullptr;
                const long v = std::strtol(c, &end, 10);
                if (end == c || v <= 0) break;
                alt.push_back(static_cast<size_t>(v));
                sum += static_cast<size_t>(v);
                c = *end == ',' ? end + 1 : end;
            }
            if (sum == nmod) sizes = alt;
        }
        for (size_t g : sizes) bounds.push_back(bounds.back() + g);
    }
    // IRL_E2E_TRACE=1: per-chunk H2D / PPMM / D2H completion times on stderr
    static const bool trace = std::getenv("IRL_E2E_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t st) {
        if (!trace) return;
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        cudaEventRecord(ev, st);
        tev.push_back(ev);
    };
    mark(s);
    IRL_CK(ctx, cudaEventRecord(e->part_done[0], s));  // order after prior work on s
    IRL_CK(ctx, cudaStreamWaitEvent(e->h2d_stream, e->part_done[0], 0));
    for (size_t ci = 0; ci + 1 < bounds.size(); ++ci) {
        const size_t c0 = bounds[ci], nc = bounds[ci + 1] - c0;
        // rows (modulus, k) of the host [nmod][K][n] batch, columns [n0, n0 + w)
        // (one linear copy when the batch is a single column chunk: 2-D DMA of
        // short rows runs at a fraction of PCIe bandwidth)
        if (w == n)
            IRL_CK(ctx, cudaMemcpyAsync(e->qres + c0 * K * w, q_res_host + c0 * K * n, nc * K * n * 2,
                                        cudaMemcpyHostToDevice, e->h2d_stream));
        else
            IRL_CK(ctx, cudaMemcpy2DAsync(e->qres + c0 * K * w, w * 2, q_res_host + c0 * K * n + n0, n * 2, w * 2,
                                          nc * K, cudaMemcpyHostToDevice, e->h2d_stream));
        IRL_CK(ctx, cudaEventRecord(e->h2d_done[ci], e->h2d_stream));
        mark(e->h2d_stream);
    }
    for (size_t ci = 0; ci + 1 < bounds.size(); ++ci) {
        const size_t c0 = bounds[ci], nc = bounds[ci + 1] - c0;
        IRL_CK(ctx, cudaStreamWaitEvent(s, e->h2d_done[ci], 0));
        ModTable sub{};
        sub.n = uint32_t(nc);
        for (size_t i = 0; i < nc; ++i) sub.mc[i] = e->mt.mc[c0 + i];
        IRL_LAUNCH(ctx, launch_split_cols<uint16_t>(e->qres + c0 * K * w, w, K * w, uint32_t(K), uint32_t(w), sub,
                                                    e->qplanes + c0 * 2 * w * e->ldk, e->ldk, nullptr, s));
        // part-granular D2H: each part's copy starts once its tiles are stored
        // (epilogue counters + cuStreamWaitValue32 on the copy stream), so the
        // copies overlap the rest of the launch instead of waiting for all of it
        const bool by_part = memops && e->memops;
        uint32_t* cnt = e->part_cnt + c0 * e->parts;
        if (by_part) {
            IRL_CK(ctx, cudaMemsetAsync(cnt, 0, nc * e->parts * sizeof(uint32_t), s));
            IRL_CK(ctx, cudaEventRecord(e->cnt_zeroed[ci], s));
            IRL_CK(ctx, cudaStreamWaitEvent(e->copy_stream, e->cnt_zeroed[ci], 0));
        }
        int st = ccmm_parts(e, w, 0, e->parts, e->out, s, c0, nc, by_part ? cnt : nullptr);
        if (st) return st;
        const uint32_t target = ppmm_last_part_target();
        IRL_CK(ctx, cudaEventRecord(e->part_done[ci], s));
        bool waited = false;
        if (by_part && target > 0) {
            // one (modulus, part) block at a time, in the order the launch
            // completes them (prime-major units)
            waited = true;
            for (size_t i = 0; i < nc && waited; ++i) {
                for (size_t p = 0; p < e->parts; ++p) {
                    const CUresult r = wait_value_fn()(e->copy_stream, reinterpret_cast<CUdeviceptr>(cnt + i * e->parts + p),
                                                       target, CU_STREAM_WAIT_VALUE_GEQ);
                    if (r != CUDA_SUCCESS) {
                        if (i != 0 || p != 0) return set_err(ctx, IRL_ERR_CUDA, "cuStreamWaitValue32 failed mid-chunk");
                        e->memops = false;  // unavailable here: whole-launch events from now on
                        waited = false;
                        break;
                    }
                    const size_t row = p * nmod + c0 + i;  // [part][modulus] block of n x M
                    if (w == n)
                        IRL_CK(ctx, cudaMemcpyAsync(out_host + row * n * M, e->out + row * w * M, n * M * 2,
                                                    cudaMemcpyDeviceToHost, e->copy_stream));
                    else
                        IRL_CK(ctx, cudaMemcpy2DAsync(out_host + (row * n + n0) * M, n * M * 2, e->out + row * w * M,
                                                      w * M * 2, w * M * 2, 1, cudaMemcpyDeviceToHost,
                                                      e->copy_stream));
                }
            }
        }
        if (waited) {
            mark(s);
            mark(e->copy_stream);
            continue;
        }
        IRL_CK(ctx, cudaStreamWaitEvent(e->copy_stream, e->part_done[ci], 0));
        for (size_t p = 0; p < e->parts; ++p) {
            // device [p][i][w][M] -> host [p][i][n][M] at column n0
            if (w == n)
                IRL_CK(ctx, cudaMemcpyAsync(out_host + (p * nmod + c0) * n * M, e->out + (p * nmod + c0) * w * M,
                                            nc * n * M * 2, cudaMemcpyDeviceToHost, e->copy_stream));
            else
                IRL_CK(ctx, cudaMemcpy2DAsync(out_host + ((p * nmod + c0) * n + n0) * M, n * M * 2,
                                              e->out + (p * nmod + c0) * w * M, w * M * 2, w * M * 2, nc,
                                              cudaMemcpyDeviceToHost, e->copy_stream));
        }
        mark(s);
        mark(e->copy_stream);
    }
    IRL_CK(ctx, cudaStreamSynchronize(e->copy_stream));
    IRL_CK(ctx, cudaStreamSynchronize(s));
    if (trace) {
        const size_t nch = bounds.size() - 1;
        std::fprintf(stderr, "[irl e2e] chunks %zu (h2d done | ppmm done | d2h done, ms from start)\n", nch);
        for (size_t ci = 0; ci < nch; ++ci) {
            float th = 0, tp = 0, td = 0;
            cudaEventElapsedTime(&th, tev[0], tev[1 + ci]);
            cudaEventElapsedTime(&tp, tev[0], tev[1 + nch + 2 * ci]);
            cudaEventElapsedTime(&td, tev[0], tev[2 + nch + 2 * ci]);
            std::fprintf(stderr, "[irl e2e] chunk %zu (%zu moduli): %8.2f %8.2f %8.2f\n", ci,
                         bounds[ci + 1] - bounds[ci], th, tp, td);
        }
        for (auto ev : tev) cudaEventDestroy(ev);
    }
    return IRL_OK;
}

int irl_ccmm_run(irl_ccmm* e, const uint16_t* q_res_host, size_t n, uint16_t* out_host) {
    if (!e) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* ctx = e->ctx;
    Guard g(ctx);
    if (n == 0) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "ccmm: query width out of range");
    // Query batches wider than the engine's staging capacity stream through it
    // in column chunks (whole 256-column tiles when max_n allows).
    size_t w = n <= e->max_n ? n : (e->max_n >= 256 ? e->max_n / 256 * 256 : e->max_n);
    for (size_t n0 = 0; n0 < n; n0 += w) {
        int st = ccmm_run_columns(e, q_res_host, n, n0, std::min(w, n - n0), out_host);
        if (st) return st;
    }
    return IRL_OK;
}

int irl_ccmm_run_dq(irl_ccmm* e, const uint16_t* q_res_dev, size_t n, uint16_t* out_host, void* stream) {
    if (!e || !out_host) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* ctx = e->ctx;
    Guard g(ctx);
    if (n == 0 || n > e->max_n) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "ccmm: query width out of range");
    cudaStream_t s = pick_stream(ctx, stream);
    if (!q_res_dev) q_res_dev = e->qres;
    const size_t nmod = e->nmod, K = e->K, M = e->M;
    IRL_LAUNCH(ctx, launch_split_cols<uint16_t>(q_res_dev, n, K * n, uint32_t(K), uint32_t(n), e->mt, e->qplanes,
                                                e->ldk, nullptr, s));
    const bool by_part = e->memops && wait_value_fn() != nullptr;
    uint32_t* cnt = e->part_cnt;
    if (by_part) {
        IRL_CK(ctx, cudaMemsetAsync(cnt, 0, nmod * e->parts * sizeof(uint32_t), s));
        IRL_CK(ctx, cudaEventRecord(e->cnt_zeroed[0], s));
        IRL_CK(ctx, cudaStreamWaitEvent(e->copy_stream, e->cnt_zeroed[0], 0));
    }
    int st = ccmm_parts(e, n, 0, e->parts, e->out, s, 0, nmod, by_part ? cnt : nullptr);
    if (st) return st;
    const uint32_t target = ppmm_last_part_target();
    bool waited = by_part && target > 0;
    for (size_t i = 0; i < nmod && waited; ++i)
        for (size_t p = 0; p < e->parts; ++p) {
            const CUresult r = wait_value_fn()(e->copy_stream, reinterpret_cast<CUdeviceptr>(cnt + i * e->parts + p),
                                               target, CU_STREAM_WAIT_VALUE_GEQ);
            if (r != CUDA_SUCCESS) {
                if (i != 0 || p != 0) return set_err(ctx, IRL_ERR_CUDA, "cuStreamWaitValue32 failed");
                e->memops = false;
                waited = false;
                break;
            }
            const size_t row = p * nmod + i;
            IRL_CK(ctx, cudaMemcpyAsync(out_host + row * n * M, e->out + row * n * M, n * M * 2,
                                        cudaMemcpyDeviceToHost, e->copy_stream));
        }
    if (!waited) {
        IRL_CK(ctx, cudaEventRecord(e->part_done[0], s));
        IRL_CK(ctx, cudaStreamWaitEvent(e->copy_stream, e->part_done[0], 0));
        IRL_CK(ctx, cudaMemcpyAsync(out_host, e->out, e->parts * nmod * n * M * 2, cudaMemcpyDeviceToHost,
                                    e->copy_stream));
    }
    IRL_CK(ctx, cudaStreamSynchronize(e->copy_stream));
    IRL_CK(ctx, cudaStreamSynchronize(s));
    return IRL_OK;
}

int irl_ccmm_rescale(irl_ccmm* e, size_t n, size_t part0, size_t nparts, size_t drop, int round, uint16_t* dst,
                     void* stream) {
    if (!e || !dst) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* ctx = e->ctx;
    Guard g(ctx);
    if (n == 0 || n > e->max_n || part0 + nparts > e->parts)
        return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "ccmm: rescale range out of range");
    std::vector<uint32_t> primes(e->nmod), exps(e->nmod);
    for (size_t i = 0; i < e->nmod; ++i) {
        primes[i] = e->mt.mc[i].p;
        exps[i] = e->mt.mc[i].e;
    }
    const size_t plane = n * e->M;
    for (size_t p = 0; p < nparts; ++p) {
        int st = irl_rescale_residues(ctx, e->out + (part0 + p) * e->nmod * plane, plane, plane, primes.data(),
                                      exps.data(), e->nmod, drop, round, dst + p * (e->nmod - drop) * plane, plane,
                                      stream);
        if (st) return st;
    }
    return IRL_OK;
}

// ---------------------------------------------------------------------------
// CCMM caller drop-in: the exact product behind Emulator::ccmm_twin
// ---------------------------------------------------------------------------

int irl_ccmm_twin(irl_ctx* ctx, long d1, long d2, long d3, long n_db, long n_qry,
                  double db_modulus_bits, double qry_modulus_bits, double scale_bits,
                  int out_level, int top_level, int out_slot_encoding, int out_ci,
                  const double* db, const double* qry, double* msgs) {
    if (!ctx) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx);
    // emulator.cpp:392-410, same order and messages
    if (d1 <= 0 || d2 <= 0 || d3 <= 0) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "ccmm: nonpositive dimensions");
    if (n_db <= 0 || n_qry <= 0 || d1 % n_db != 0 || d2 % n_qry != 0)
        return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "ccmm: d1 must be a multiple of n_db, d2 of n_qry");
    if (db_modulus_bits < 2.0 * qry_modulus_bits - scale_bits)
        return set_err(ctx, IRL_ERR_MODULUS_BUDGET, "ccmm: database modulus below 2q - delta");
    if (out_level < 0 || out_level > top_level)
        return set_err(ctx, IRL_ERR_MODULUS_BUDGET, "ccmm: output level outside the modulus chain");
    if (out_slot_encoding && !out_ci)
        return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "ccmm: slot-encoded output must be conjugate-invariant");
    if (d1 >= (1l << 30) || d2 >= (1l << 30) || d3 >= (1l << 30))
        return set_err(ctx, IRL_ERR_UNSUPPORTED, "ccmm: dimension above 2^30");
    const size_t M = size_t(d1), K = size_t(d2), N = size_t(d3);
    // Device buffers: inputs, residues, planes, output residues, doubles.
    // Paper-basis prefix with Q > 2 * bound, Q < 2^64 (<= 4 moduli).
    uint32_t P[64], E[64];
    irl_paper_basis(P, E, 64);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = (off + bytes + 127) / 128 * 128;
        return o;
    };
    const size_t ldk = round16(K);
    const size_t o_db = take(M * K * 8), o_q = take(K * N * 8), o_ra = take(4 * M * K * 2),
                 o_rb = take(4 * K * N * 2), o_pa = take(4 * 2 * M * ldk), o_pb = take(4 * 2 * N * ldk),
                 o_res = take(4 * N * M * 2), o_out = take(N * M * 8), o_bad = take(16);
    IRL_CK(ctx, ctx->ws[0].ensure(off));
    uint8_t* base = ctx->ws[0].as<uint8_t>();
    double* ddb = reinterpret_cast<double*>(base + o_db);
    double* dq = reinterpret_cast<double*>(base + o_q);
    int* dbad = reinterpret_cast<int*>(base + o_bad);
    IRL_CK(ctx, copy_h2d(ctx, ddb, db, M * K * 8, ctx->stream));
    IRL_CK(ctx, copy_h2d(ctx, dq, qry, K * N * 8, ctx->stream));
    IRL_CK(ctx, cudaMemsetAsync(dbad, 0, 4, ctx->stream));
    // Modulus count: |product| <= K max|db| max|qry| must stay inside the
    // centred range of Q (validation of the host inputs' magnitudes only;
    // integrality is checked on device by the residue kernel).
    ModTable mt{};
    double amax = 0, bmax = 0;
    for (size_t i = 0; i < M * K; ++i) amax = std::max(amax, std::fabs(db[i]));
    for (size_t i = 0; i < K * N; ++i) bmax = std::max(bmax, std::fabs(qry[i]));
    const double bound = double(K) * amax * bmax;
    if (bound >= 4503599627370496.0)  // 2^52: keep the centred result exact in double
        return set_err(ctx, IRL_ERR_UNSUPPORTED, "ccmm: |product| may exceed 2^52");
    uint32_t nm = 1;
    double q = double(P[0]) * P[0];
    while (q <= 2.0 * bound + 1.0 && nm < 4) {
        q *= double(P[nm]) * P[nm];
        ++nm;
    }
    mt.n = nm;
    for (uint32_t i = 0; i < nm; ++i) mt.mc[i] = make_modconst(P[i], 2);
    uint16_t* ra = reinterpret_cast<uint16_t*>(base + o_ra);
    uint16_t* rb = reinterpret_cast<uint16_t*>(base + o_rb);
    IRL_LAUNCH(ctx, launch_double_to_residues(ddb, uint32_t(M), uint32_t(K), mt, ra, dbad, ctx->stream));
    IRL_LAUNCH(ctx, launch_double_to_residues(dq, uint32_t(K), uint32_t(N), mt, rb, dbad, ctx->stream));
    int bad = 0;
    IRL_CK(ctx, cudaMemcpyAsync(&bad, dbad, 4, cudaMemcpyDeviceToHost, ctx->stream));
    IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (bad) return set_err(ctx, IRL_ERR_UNSUPPORTED, "ccmm: messages must be integers below 2^53");
    int8_t* pa = reinterpret_cast<int8_t*>(base + o_pa);
    int8_t* pb = reinterpret_cast<int8_t*>(base + o_pb);
    IRL_LAUNCH(ctx, launch_split_rows<uint16_t>(ra, K, M * K, uint32_t(M), uint32_t(K), mt, pa, ldk, nullptr, ctx->stream));
    IRL_LAUNCH(ctx, launch_split_cols<uint16_t>(rb, N, K * N, uint32_t(K), uint32_t(N), mt, pb, ldk, nullptr, ctx->stream));
    uint16_t* res = reinterpret_cast<uint16_t*>(base + o_res);
    PpmmLaunch L = make_launch(mt);
    L.a_planes = pa;
    L.b_planes = pb;
    L.out = res;
    L.M = uint32_t(M);
    L.N = uint32_t(N);
    L.K = uint32_t(K);
    L.ldk = uint32_t(ldk);
    L.parts = 1;
    int64_t h = 0;
    for (uint32_t i = 0; i < nm; ++i) h = std::max<int64_t>(h, (P[i] - 1) / 2);
    int st = run_ppmm(ctx, L, safe_kchunk(h, h, h, h, uint32_t(K)), ctx->stream);
    if (st) return st;
    Crt64Table t{};
    t.nmod = nm;
    unsigned long long Qv = 1;
    for (uint32_t i = 0; i < nm; ++i) Qv *= uint64_t(P[i]) * P[i];
    t.Q = Qv;
    for (uint32_t i = 0; i < nm; ++i) {
        const uint32_t m = P[i] * P[i];
        t.mc[i] = make_modconst(P[i], 2);
        t.qi[i] = Qv / m;
        if (!inv_mod(uint32_t(t.qi[i] % m), m, &t.inv[i]))
            return set_err(ctx, IRL_ERR_NOT_COPRIME, "CRT basis is not coprime");
    }
    double* dout = reinterpret_cast<double*>(base + o_out);
    IRL_LAUNCH(ctx, launch_crt_centred_double(res, uint32_t(M), uint32_t(N), t, dout, ctx->stream));
    // [N][M] column-major product == ccmm_twin's ciphertext message order
    IRL_CK(ctx, copy_d2h(ctx, msgs, dout, N * M * 8, ctx->stream));
    IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return IRL_OK;
}

}  // extern "C"
