// RGSW CCMM engine of the C ABI (include/irl_capi.h, irl_ccmm_*): the
// device-resident 8-slice database, the query split + PPMM launches per
// modulus chunk, the host<->device pipeline of irl_ccmm_run, the fused a-part
// exchange (peer mirrors) and the ccmm_twin caller drop-in (irl_ccmm_twin).
// Shared helpers (make_table, run_ppmm, CRT limbs ...) live in capi.cu.
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
    size_t mirror_part = 0, mirror_n = 0, n_mirror = 0, mirror_slot = 0;
    size_t mirror_parts = 1;  // local parts [mirror_part, mirror_part + mirror_parts) are mirrored
    uint16_t* mirror[kMaxMirrors] = {};
    bool mirror_ipc[kMaxMirrors] = {};
    uint16_t* mc_mirror = nullptr;  // NVLS multicast address of the receive buffers (irl_ccmm_set_mirror_multicast)
    // part-granular D2H in irl_ccmm_run: per (modulus chunk, part) tile
    // counters the epilogue bumps; the copy stream waits on them with stream
    // memory operations (cuStreamWaitValue32) instead of on the whole launch
    uint32_t* part_cnt = nullptr;       // [nmod][parts]
    std::vector<cudaEvent_t> cnt_zeroed;  // per modulus chunk
    bool memops = true;                 // cleared if stream memory ops are unavailable
    // irl_ccmm_run with pageable host buffers: page-locked staging of the query
    // and the outputs (allocated on first use), and per-block D2H events the
    // host waits on to copy each landed block out while the launch runs
    uint16_t* hq = nullptr;
    size_t hq_elems = 0;
    uint16_t* hout = nullptr;
    size_t hout_elems = 0;
    std::vector<cudaEvent_t> blk_done;
};

extern "C" {

// ---------------------------------------------------------------------------
// RGSW CCMM engine
// ---------------------------------------------------------------------------

int irl_ccmm_create(irl_ctx* ctx, size_t parts, size_t m, size_t k, size_t max_n,
                    const uint32_t* primes, const uint32_t* exps, size_t nmod, irl_ccmm** out) {
    if (!ctx || !out) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(ctx, __func__);
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
    for (auto ev : e->blk_done)
        if (ev) cudaEventDestroy(ev);
    if (e->hq) cudaFreeHost(e->hq);
    if (e->hout) cudaFreeHost(e->hout);
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
    return irl_ccmm_alloc_recv_parts(e, n, 1, dev_ptr, ipc_handle);
}

int irl_ccmm_alloc_recv_parts(irl_ccmm* e, size_t n, size_t parts, void** dev_ptr, uint8_t* ipc_handle) {
    if (!e || !dev_ptr || parts == 0) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* ctx = e->ctx;
    Guard g(ctx, __func__);
    if (n == 0 || n > e->max_n) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "ccmm: receive width out of range");
    if (e->recv) cudaFree(e->recv);
    e->recv = nullptr;
    const size_t slot_bytes = parts * e->nmod * n * e->M * sizeof(uint16_t);
    IRL_CK(ctx, cudaMalloc(&e->recv, IRL_RECV_SLOTS * slot_bytes));
    IRL_CK(ctx, cudaMemset(e->recv, 0, IRL_RECV_SLOTS * slot_bytes));
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
    e->mirror_parts = 1;
    e->mirror_n = n;
    return IRL_OK;
}

int irl_ccmm_set_mirrors(irl_ccmm* e, size_t part, size_t n, const uint8_t* ipc_handles, size_t count) {
    if (!e || (count && !ipc_handles)) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(e->ctx, __func__);
    return set_mirrors(e, part, n, nullptr, ipc_handles, count);
}

int irl_ccmm_set_mirror_ptrs(irl_ccmm* e, size_t part, size_t n, uint16_t* const* dev_ptrs, size_t count) {
    if (!e || (count && !dev_ptrs)) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(e->ctx, __func__);
    return set_mirrors(e, part, n, dev_ptrs, nullptr, count);
}

int irl_ccmm_set_mirror_parts(irl_ccmm* e, size_t count) {
    if (!e) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(e->ctx, __func__);
    if (count == 0 || e->mirror_part + count > e->parts)
        return set_err(e->ctx, IRL_ERR_INVALID_ARGUMENT, "ccmm: mirrored part range out of range");
    e->mirror_parts = count;
    return IRL_OK;
}

int irl_ccmm_set_mirror_slot(irl_ccmm* e, size_t slot) {
    if (!e) return IRL_ERR_INVALID_ARGUMENT;
    Guard g(e->ctx, __func__);
    if (slot >= IRL_RECV_SLOTS) return set_err(e->ctx, IRL_ERR_INVALID_ARGUMENT, "ccmm: mirror slot out of range");
    e->mirror_slot = slot;
    return IRL_OK;
}

int irl_ccmm_set_mirror_multicast(irl_ccmm* e, size_t part, size_t n, void* mc_addr) {
    if (!e) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* ctx = e->ctx;
    Guard g(ctx, __func__);
    if (mc_addr && (part >= e->parts || n == 0 || n > e->max_n || (e->M & 1) != 0))
        return set_err(ctx, IRL_ERR_INVALID_ARGUMENT, "ccmm: bad multicast mirror (part, width, or odd M)");
    e->mc_mirror = static_cast<uint16_t*>(mc_addr);
    if (mc_addr) {
        e->mirror_part = part;
        e->mirror_n = n;
    }
    return IRL_OK;
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
    Guard g(ctx, __func__);
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
    Guard g(ctx, __func__);
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
    Guard g(ctx, __func__);
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
        // 8 readers per chunk (pread at disjoint offsets): page-cache copies and
        // NVMe queues both scale with concurrent requests (r2, 16-CPU host, one
        // 18.5 GB part from the page cache: 4 readers 9-15 GB/s, 8 readers
        // 15-23 GB/s, 16 readers 17-22 GB/s; profiles/r2_ingest_readers.txt)
        {
            static const int kReaders = [] {
                const char* v = std::getenv("IRL_INGEST_READERS");
                const int n = v ? std::atoi(v) : 8;
                return n < 1 ? 1 : (n > 32 ? 32 : n);
            }();
            std::vector<char> ok(kReaders, 0);
            std::vector<std::thread> th(kReaders);
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
    Guard g(ctx, __func__);
    for (size_t p = 0; p < e->parts; ++p) {
        IRL_LAUNCH(ctx, launch_synth_planes(seed, first_part + uint32_t(p), 1, uint32_t(e->M), uint32_t(e->K), e->mt,
                                            e->db + p * e->nmod * 2 * e->M * e->ldk, e->ldk, ctx->stream));
    }
    IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return IRL_OK;
}

int irl_ccmm_synth_part(irl_ccmm* e, size_t part, uint64_t seed, uint32_t global_part, uint32_t row0) {
    if (!e) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* ctx = e->ctx;
    Guard g(ctx, __func__);
    if (part >= e->parts) return set_err(ctx, IRL_ERR_SHAPE_MISMATCH, "ccmm: part index out of range");
    IRL_LAUNCH(ctx, launch_synth_planes(seed, global_part, 1, uint32_t(e->M), uint32_t(e->K), e->mt,
                                        e->db + part * e->nmod * 2 * e->M * e->ldk, e->ldk, ctx->stream, row0));
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
    const size_t mfirst = std::max(part0, e->mirror_part);
    const size_t mlast = std::min(part0 + nparts, e->mirror_part + e->mirror_parts);
    if ((e->n_mirror || e->mc_mirror) && n == e->mirror_n && mfirst < mlast) {
        L.n_mirror = static_cast<uint32_t>(e->n_mirror);
        L.mirror_part = static_cast<uint32_t>(mfirst - part0);
        L.mirror_parts = static_cast<uint32_t>(mlast - mfirst);
        // peer buffers: [slot][mirrored part][modulus][n][M]
        const size_t at = ((e->mirror_slot * e->mirror_parts + (mfirst - e->mirror_part)) * e->nmod + m0) * n * e->M;
        for (size_t i = 0; i < e->n_mirror; ++i) L.mirror[i] = e->mirror[i] + at;
        if (e->mc_mirror) L.mc_mirror = e->mc_mirror + at;
    }
    return run_ppmm(ctx, L, e->kchunk, s);
}

int irl_ccmm_run_device(irl_ccmm* e, const uint16_t* q_res_dev, int q_ready, size_t n,
                        size_t part0, size_t nparts, uint16_t* out_dev, void* stream) {
    if (!e) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* ctx = e->ctx;
    Guard g(ctx, __func__);
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

// Page-locked staging for a pageable caller buffer of `elems` uint16 (grown on
// demand); false if it cannot be allocated (the caller then copies directly).
static bool ensure_staging(uint16_t** buf, size_t* have, size_t elems) {
    if (*have >= elems) return true;
    if (*buf) cudaFreeHost(*buf);
    *buf = nullptr;
    *have = 0;
    if (cudaMallocHost(reinterpret_cast<void**>(buf), elems * sizeof(uint16_t)) != cudaSuccess) {
        cudaGetLastError();
        *buf = nullptr;
        return false;
    }
    *have = elems;
    return true;
}

static int ccmm_run_columns(irl_ccmm* e, const uint16_t* q_res_host, size_t n, size_t n0, size_t w,
                            uint16_t* out_host) {
    irl_ctx* ctx = e->ctx;
    cudaStream_t s = ctx->stream;
    const size_t nmod = e->nmod, K = e->K, M = e->M;
    // Pageable caller buffers (std::vector storage, plain numpy) would make
    // every async copy a synchronous driver-staged one and serialize the
    // pipeline (c4: 405 ms against 153 ms pinned). Single-chunk batches stage
    // them instead: the query is copied into page-locked memory up front by the
    // host copy workers, the D2H blocks land in page-locked memory, and the
    // host copies each one out as soon as its event fires, during the launch.
    static const bool no_staging = std::getenv("IRL_E2E_NO_STAGING") != nullptr;
    const uint16_t* q_src = q_res_host;
    uint16_t* out_dst = out_host;
    bool stage_out = false;
    if (w == n && !no_staging) {
        if (!host_pinned(q_res_host) && ensure_staging(&e->hq, &e->hq_elems, nmod * K * n)) {
            host_parallel_copy(e->hq, q_res_host, nmod * K * n * sizeof(uint16_t));
            q_src = e->hq;
        }
        if (!host_pinned(out_host) && ensure_staging(&e->hout, &e->hout_elems, e->parts * nmod * n * M)) {
            out_dst = e->hout;
            stage_out = true;
        }
    }
    // staged outputs: (event, element offset, elements) per D2H block, in order
    struct Landed {
        size_t ev, off, elems;
    };
    std::vector<Landed> landed;
    auto staged_block = [&](size_t off, size_t elems) -> cudaError_t {
        if (!stage_out) return cudaSuccess;
        if (landed.size() == e->blk_done.size()) {
            cudaEvent_t ev;
            const cudaError_t er = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
            if (er != cudaSuccess) return er;
            e->blk_done.push_back(ev);
        }
        landed.push_back({landed.size(), off, elems});
        return cudaEventRecord(e->blk_done[landed.back().ev], e->copy_stream);
    };
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
            IRL_CK(ctx, cudaMemcpyAsync(e->qres + c0 * K * w, q_src + c0 * K * n, nc * K * n * 2,
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
                    if (w == n) {
                        IRL_CK(ctx, cudaMemcpyAsync(out_dst + row * n * M, e->out + row * w * M, n * M * 2,
                                                    cudaMemcpyDeviceToHost, e->copy_stream));
                        IRL_CK(ctx, staged_block(row * n * M, n * M));
                    } else
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
            if (w == n) {
                IRL_CK(ctx, cudaMemcpyAsync(out_dst + (p * nmod + c0) * n * M, e->out + (p * nmod + c0) * w * M,
                                            nc * n * M * 2, cudaMemcpyDeviceToHost, e->copy_stream));
                IRL_CK(ctx, staged_block((p * nmod + c0) * n * M, nc * n * M));
            } else
                IRL_CK(ctx, cudaMemcpy2DAsync(out_host + ((p * nmod + c0) * n + n0) * M, n * M * 2,
                                              e->out + (p * nmod + c0) * w * M, w * M * 2, w * M * 2, nc,
                                              cudaMemcpyDeviceToHost, e->copy_stream));
        }
        mark(s);
        mark(e->copy_stream);
    }
    for (const Landed& b : landed) {  // staged outputs: copy each block out as it lands
        IRL_CK(ctx, cudaEventSynchronize(e->blk_done[b.ev]));
        host_parallel_copy(out_host + b.off, e->hout + b.off, b.elems * sizeof(uint16_t));
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
    Guard g(ctx, __func__);
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
    Guard g(ctx, __func__);
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
    // pageable outputs: D2H into page-locked staging, each block copied out by
    // the host workers as its event fires (as irl_ccmm_run does)
    static const bool no_staging = std::getenv("IRL_E2E_NO_STAGING") != nullptr;
    const bool stage_out = !no_staging && !host_pinned(out_host) &&
                           ensure_staging(&e->hout, &e->hout_elems, e->parts * nmod * n * M);
    uint16_t* out_dst = stage_out ? e->hout : out_host;
    std::vector<std::pair<size_t, size_t>> landed;  // (element offset, elements) per staged block
    auto staged_block = [&](size_t off, size_t elems) -> cudaError_t {
        if (!stage_out) return cudaSuccess;
        if (landed.size() == e->blk_done.size()) {
            cudaEvent_t ev;
            const cudaError_t er = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
            if (er != cudaSuccess) return er;
            e->blk_done.push_back(ev);
        }
        landed.push_back({off, elems});
        return cudaEventRecord(e->blk_done[landed.size() - 1], e->copy_stream);
    };
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
            IRL_CK(ctx, cudaMemcpyAsync(out_dst + row * n * M, e->out + row * n * M, n * M * 2,
                                        cudaMemcpyDeviceToHost, e->copy_stream));
            IRL_CK(ctx, staged_block(row * n * M, n * M));
        }
    if (!waited) {
        IRL_CK(ctx, cudaEventRecord(e->part_done[0], s));
        IRL_CK(ctx, cudaStreamWaitEvent(e->copy_stream, e->part_done[0], 0));
        IRL_CK(ctx, cudaMemcpyAsync(out_dst, e->out, e->parts * nmod * n * M * 2, cudaMemcpyDeviceToHost,
                                    e->copy_stream));
        IRL_CK(ctx, staged_block(0, e->parts * nmod * n * M));
    }
    for (size_t j = 0; j < landed.size(); ++j) {
        IRL_CK(ctx, cudaEventSynchronize(e->blk_done[j]));
        host_parallel_copy(out_host + landed[j].first, e->hout + landed[j].first, landed[j].second * sizeof(uint16_t));
    }
    IRL_CK(ctx, cudaStreamSynchronize(e->copy_stream));
    IRL_CK(ctx, cudaStreamSynchronize(s));
    return IRL_OK;
}

int irl_ccmm_rescale(irl_ccmm* e, size_t n, size_t part0, size_t nparts, size_t drop, int round, uint16_t* dst,
                     void* stream) {
    if (!e || !dst) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* ctx = e->ctx;
    Guard g(ctx, __func__);
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
    Guard g(ctx, __func__);
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
    // Route: integer-valued operands whose partial sums stay below 2^52 in
    // magnitude (every partial sum of the reference's double loop is then an
    // exact integer, so its result is the exact product) run on the int8
    // tensor-core PPMM; anything else runs the ordered FP64 kernel, which
    // replays the reference loop's IEEE operations one for one.
    double amax = 0, bmax = 0;
    bool integral = true;
    for (size_t i = 0; i < M * K; ++i) {
        const double v = db[i];
        integral = integral && v == std::nearbyint(v);
        amax = std::max(amax, std::fabs(v));
    }
    for (size_t i = 0; i < K * N; ++i) {
        const double v = qry[i];
        integral = integral && v == std::nearbyint(v);
        bmax = std::max(bmax, std::fabs(v));
    }
    const double bound = double(K) * amax * bmax;
    if (!integral || !(bound < 4503599627370496.0)) {  // 2^52 (NaN / inf land here too)
        size_t off = 0;
        auto take = [&](size_t bytes) {
            const size_t o = off;
            off = (off + bytes + 127) / 128 * 128;
            return o;
        };
        const size_t o_db = take(M * K * 8), o_q = take(K * N * 8), o_out = take(N * M * 8);
        IRL_CK(ctx, ctx->ws[0].ensure(off));
        uint8_t* base = ctx->ws[0].as<uint8_t>();
        double* ddb = reinterpret_cast<double*>(base + o_db);
        double* dq = reinterpret_cast<double*>(base + o_q);
        double* dout = reinterpret_cast<double*>(base + o_out);
        IRL_CK(ctx, copy_h2d(ctx, ddb, db, M * K * 8, ctx->stream));
        IRL_CK(ctx, copy_h2d(ctx, dq, qry, K * N * 8, ctx->stream));
        IRL_LAUNCH(ctx, launch_ordered_dgemm_t(ddb, dq, uint32_t(M), uint32_t(K), uint32_t(N), dout, ctx->stream));
        IRL_CK(ctx, copy_d2h(ctx, msgs, dout, N * M * 8, ctx->stream));
        IRL_CK(ctx, cudaStreamSynchronize(ctx->stream));
        return IRL_OK;
    }
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
    // Modulus count: |product| <= K max|db| max|qry| < 2^52 must stay inside
    // the centred range of Q.
    ModTable mt{};
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
    if (bad) return set_err(ctx, IRL_ERR_CUDA, "ccmm: residue conversion rejected a checked integer entry");
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
