// Internal: the context object behind the C ABI and the error / launch
// helpers shared by the C-ABI translation units (capi.cu, iris.cu).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/irl_capi.h"
#include "kernels_aux.cuh"
#include "ppmm.h"

namespace irl {

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(bytes, 1 << 20);
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct Status {
    int code;
    std::string msg;
};

}  // namespace irl

struct irl_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    uint64_t launches = 0;
    std::recursive_mutex mu;
    irl::DevBuf ws[8];
    irl::DevBuf rcp;       // fold stage: rcp[k] = RN(1 / k) for k < rcp_n (fold.cu)
    uint32_t rcp_n = 0;
    irl::SplitStats* d_stats = nullptr;
    irl::SplitStats* h_stats = nullptr;
    int32_t* d_absmax = nullptr;
    int32_t* h_absmax = nullptr;
    uint32_t* d_progress = nullptr;  // group-gating scratch of the PPMM kernel
    uint64_t* d_diag = nullptr;      // PPMM diagnostics (irl_diag_ppmm), lazily allocated
    bool diag = false;
    // pinned bounce buffers for large copies of caller (pageable) host memory
    uint8_t* bounce[2] = {nullptr, nullptr};
    cudaEvent_t bounce_ev[2] = {nullptr, nullptr};
};


namespace irl {

inline int set_err(irl_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return code;
}

inline int cuda_fail(irl_ctx* ctx, cudaError_t e, const char* where) {
    cudaGetLastError();  // clear sticky non-fatal state
    const int code = e == cudaErrorMemoryAllocation ? IRL_ERR_OUT_OF_MEMORY : IRL_ERR_CUDA;
    return set_err(ctx, code, std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e));
}

#define IRL_CK(ctx, expr)                                              \
    do {                                                               \
        cudaError_t e__ = (expr);                                      \
        if (e__ != cudaSuccess) return cuda_fail((ctx), e__, #expr);   \
    } while (0)

#define IRL_LAUNCH(ctx, expr)                                          \
    do {                                                               \
        cudaError_t e__ = (expr);                                      \
        if (e__ != cudaSuccess) return cuda_fail((ctx), e__, #expr);   \
        ++(ctx)->launches;                                             \
    } while (0)

// Every C-ABI entry point holds one: the context's lock, its device, a cleared
// error string, and an NVTX range named after the entry point (visible to
// ncu --nvtx / Nsight Systems; a no-op without an attached tool).
struct Guard {
    irl_ctx* c;
    std::lock_guard<std::recursive_mutex> lk;
    explicit Guard(irl_ctx* ctx, const char* range = nullptr) : c(ctx), lk(ctx->mu), named(range != nullptr) {
        cudaSetDevice(ctx->device);
        ctx->err.clear();
        if (named) nvtxRangePushA(range);
    }
    ~Guard() {
        if (named) nvtxRangePop();
    }
    Guard(const Guard&) = delete;
    Guard& operator=(const Guard&) = delete;

   private:
    bool named;
};

inline cudaStream_t pick_stream(irl_ctx* ctx, void* s) {
    return s ? static_cast<cudaStream_t>(s) : ctx->stream;
}

// Copies between caller host memory (usually pageable) and the device for the
// blocking host-buffer API. Large copies go through the context's two pinned
// 16 MB bounce buffers; several host threads fill (drain) one buffer while the
// DMA of the other runs, instead of the driver's single-threaded staging.
// h2d is stream-ordered on s; d2h returns once dst holds the data.
cudaError_t copy_h2d(irl_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t s);
cudaError_t copy_d2h(irl_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t s);
// Host memory page-locked for CUDA (cudaMallocHost / cudaHostRegister)?
bool host_pinned(const void* p);
// Host-to-host copy on the process-wide pool of copy workers (capi.cu).
void host_parallel_copy(void* dst, const void* src, size_t bytes);
void release_bounce(irl_ctx* ctx);

// Shared by the modmat entry points (capi.cu) and the CCMM engine
// (ccmm_engine.cu); defined in capi.cu.
int validate_moduli(irl_ctx* ctx, const uint32_t* primes, const uint32_t* exps, size_t nmod);
ModTable make_table(const uint32_t* primes, const uint32_t* exps, size_t nmod);
PpmmLaunch make_launch(const ModTable& mt);
// K chunk keeping the fused int32 accumulators exact for digit maxima (a0, a1, b0, b1)
uint32_t safe_kchunk(int64_t a0, int64_t a1, int64_t b0, int64_t b1, uint32_t K);
// one PPMM over digit planes, K-chunked (accumulate mode for chunks > 0)
int run_ppmm(irl_ctx* ctx, PpmmLaunch L, uint32_t kchunk, cudaStream_t s);
inline size_t round16(size_t x) { return (x + 15) / 16 * 16; }

// host big integers for CRT constants (32-bit limbs, little-endian)
using Limbs = std::vector<uint32_t>;
Limbs basis_Q(const uint32_t* primes, const uint32_t* exps, size_t nmod);
uint32_t divmod_small(Limbs& x, uint32_t m);  // x /= m, returns x mod m
size_t byte_width(const Limbs& q);
bool inv_mod(uint32_t a, uint32_t m, uint32_t* out);

}  // namespace irl
