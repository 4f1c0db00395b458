// C ABI of the B200 PPMM / RGSW-CCMM engine (include/irl_capi.h).
//
// Host-buffer calls mirror irislab::modmat (reference proj/src/modmat.cpp)
// value-for-value, including its exception taxonomy and messages; all the
// arithmetic runs in this library's sm_100a kernels. There is no CPU compute
// path: validation only reads the split kernels' device-side statistics.
#include <unistd.h>

#include <cuda.h>
#include <cuda_runtime.h>

#include <pthread.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
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


namespace irl {

static const char* kOverflowMsg = "int32 accumulation bound exceeded: K*|A|*|B| = ";

// Reference precheck of small_gemm (modmat.cpp:122-129).
static bool overflow(int64_t k, int64_t ma, int64_t mb, int64_t* bound) {
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


// Big-integer helpers for CRT constants (host, 32-bit limbs; Limbs in ctx_internal.h).
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

}  // namespace irl
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

// Persistent host copy workers for the bounce-buffer path: a pageable caller
// buffer is copied by kCopyThreads threads at once (one thread cannot saturate
// host memory), without starting threads per 16 MB chunk. One job at a time;
// process-wide, never torn down (the workers only sleep between jobs).
class CopyPool {
public:
    CopyPool() {
        for (int t = 0; t < kCopyThreads; ++t) std::thread([this, t] { work(t); }).detach();
    }
    void run(void* dst, const void* src, size_t bytes) {
        std::lock_guard<std::mutex> job(run_mu_);
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = static_cast<uint8_t*>(dst);
            src_ = static_cast<const uint8_t*>(src);
            bytes_ = bytes;
            piece_ = (bytes + kCopyThreads - 1) / kCopyThreads;
            pending_ = kCopyThreads;
            ++gen_;
        }
        go_.notify_all();
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return pending_ == 0; });
    }

private:
    void work(int t) {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> lk(mu_);
        for (;;) {
            go_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
            uint8_t* d = dst_;
            const uint8_t* s = src_;
            const size_t lo = std::min(bytes_, t * piece_), hi = std::min(bytes_, lo + piece_);
            lk.unlock();
            if (hi > lo) std::memcpy(d + lo, s + lo, hi - lo);
            lk.lock();
            if (--pending_ == 0) done_.notify_one();
        }
    }
    std::mutex run_mu_, mu_;
    std::condition_variable go_, done_;
    uint8_t* dst_ = nullptr;
    const uint8_t* src_ = nullptr;
    size_t bytes_ = 0, piece_ = 0;
    int pending_ = 0;
    uint64_t gen_ = 0;
};

// The pool is intentionally leaked (its detached workers outlive static
// destruction). A forked child has none of the parent's threads, so it drops
// the inherited pool and starts its own on first use.
std::atomic<CopyPool*> g_copy_pool{nullptr};
std::mutex g_copy_pool_mu;

void parallel_memcpy(void* dst, const void* src, size_t bytes) {
    if (bytes < (size_t(1) << 20)) {
        std::memcpy(dst, src, bytes);
        return;
    }
    CopyPool* pool = g_copy_pool.load(std::memory_order_acquire);
    if (!pool) {
        std::lock_guard<std::mutex> lk(g_copy_pool_mu);
        pool = g_copy_pool.load(std::memory_order_relaxed);
        if (!pool) {
            static const bool registered = [] {
                return pthread_atfork(nullptr, nullptr, [] { g_copy_pool.store(nullptr); }) == 0;
            }();
            (void)registered;
            pool = new CopyPool();
            g_copy_pool.store(pool, std::memory_order_release);
        }
    }
    pool->run(dst, src, bytes);
}
}  // namespace

// Page-locked host memory (cudaMallocHost / cudaHostRegister, e.g. a pinned
// torch tensor) is DMA'd directly; pageable memory goes through the bounce
// buffers from kDirectCopyBytes up.
void host_parallel_copy(void* dst, const void* src, size_t bytes) { parallel_memcpy(dst, src, bytes); }

bool host_pinned(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

cudaError_t copy_h2d(irl_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes < kDirectCopyBytes || host_pinned(src)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
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
    if (bytes < kDirectCopyBytes || host_pinned(dst)) {
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
        case IRL_ERR_CONFIG: return "ConfigError";
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
    ctx->rcp.release();
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
    Guard g(ctx, __func__);
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
    Guard g(ctx, __func__);
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
    Guard g(ctx, __func__);
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
    Guard g(ctx, __func__);
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
    Guard g(ctx, __func__);
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
    Guard g(ctx, __func__);
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
    Guard g(ctx, __func__);
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
    Guard g(ctx, __func__);
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
    Guard g(ctx, __func__);
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
    Guard g(ctx, __func__);
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
    Guard g(ctx, __func__);
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
    Guard g(ctx, __func__);
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
            t.dinv_sh[i] = static_cast<uint32_t>((static_cast<unsigned long long>(t.dinv[i]) << 32) / m);
        } else {
            t.cq[i] = delta / m;
            if (!inv(t.cq[i], m, &t.cinv[i])) return set_err(ctx, IRL_ERR_NOT_COPRIME, "CRT basis is not coprime");
            t.cinv_sh[i] = static_cast<uint32_t>((static_cast<unsigned long long>(t.cinv[i]) << 32) / m);
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

}  // extern "C"
