// Single-process multi-GPU CCMM (include/irl_capi.h, irl_ccmm_group_* and
// irl_ccmm_full; SURVEY §8(b)'s irl_ccmm_full).
//
// One context and one engine per device. The parts are dealt in contiguous
// blocks as dist.part_range does (the a-part on rank 0). Every rank runs its
// parts end to end (irl_ccmm_run) on its own host thread, so the devices work
// concurrently. The a-part exchange is fused into rank 0's PPMM epilogue: it
// stores each output tile of part 0 into every other rank's receive buffer
// over peer memory (NVLink) while it computes. Where peer access is not
// available, a cudaMemcpyPeer after the runs takes its place.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "../../include/irl_capi.h"
#include "ctx_internal.h"

using namespace irl;

struct irl_ccmm_group {
    size_t ndev = 0, parts = 0, M = 0, K = 0, max_n = 0, nmod = 0;
    std::vector<int> dev;
    std::vector<irl_ctx*> ctx;
    std::vector<irl_ccmm*> eng;
    std::vector<size_t> first, count;
    std::vector<uint16_t*> recv;  // rank r > 0: receive buffer of the a-part result [nmod][n][M]
    size_t recv_n = 0;            // width the receive buffers and mirrors are set up for
    bool fused = false;           // rank 0's epilogue stores into the peers
};

namespace {

void destroy_group(irl_ccmm_group* g) {
    for (size_t r = 0; r < g->eng.size(); ++r)
        if (g->eng[r]) irl_ccmm_destroy(g->eng[r]);
    for (irl_ctx* c : g->ctx)
        if (c) irl_ctx_destroy(c);
    delete g;
}

// Receive buffers of width n on ranks 1.., peer access from rank 0's device,
// and rank 0's mirror list (or none, for the copy fallback).
int setup_exchange(irl_ccmm_group* g, size_t n) {
    if (g->recv_n == n) return IRL_OK;
    irl_ctx* c0 = g->ctx[0];
    g->recv.assign(g->ndev, nullptr);
    bool peer = true;
    for (size_t r = 1; r < g->ndev; ++r) {
        void* p = nullptr;
        if (int st = irl_ccmm_alloc_recv(g->eng[r], n, &p, nullptr)) {
            set_err(c0, st, std::string("rank ") + std::to_string(r) + ": " + irl_last_error(g->ctx[r]));
            return st;
        }
        g->recv[r] = static_cast<uint16_t*>(p);
        if (g->dev[r] != g->dev[0]) {
            int can = 0;
            cudaSetDevice(g->dev[0]);
            if (cudaDeviceCanAccessPeer(&can, g->dev[0], g->dev[r]) != cudaSuccess || !can) {
                peer = false;
            } else {
                const cudaError_t e = cudaDeviceEnablePeerAccess(g->dev[r], 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) peer = false;
                cudaGetLastError();
            }
        }
    }
    g->fused = peer && g->ndev > 1 && g->ndev - 1 <= static_cast<size_t>(kMaxMirrors);
    std::vector<uint16_t*> peers(g->recv.begin() + (g->ndev > 1 ? 1 : 0), g->recv.end());
    if (int st = irl_ccmm_set_mirror_ptrs(g->eng[0], 0, n, peers.data(), g->fused ? peers.size() : 0)) return st;
    g->recv_n = n;
    return IRL_OK;
}

}  // namespace

extern "C" {

int irl_ccmm_group_create(const int* devices, size_t ndev, size_t parts, size_t m, size_t k, size_t max_n,
                          const uint32_t* primes, const uint32_t* exps, size_t nmod, irl_ccmm_group** out) {
    if (!devices || !out || ndev == 0) return IRL_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    if (ndev > parts) return IRL_ERR_SHAPE_MISMATCH;  // at least one part per device (dist.part_range)
    auto* g = new irl_ccmm_group();
    g->ndev = ndev;
    g->parts = parts;
    g->M = m;
    g->K = k;
    g->max_n = max_n;
    g->nmod = nmod;
    g->dev.assign(devices, devices + ndev);
    g->ctx.assign(ndev, nullptr);
    g->eng.assign(ndev, nullptr);
    const size_t base = parts / ndev, extra = parts % ndev;
    for (size_t r = 0; r < ndev; ++r) {
        g->first.push_back(r * base + std::min(r, extra));
        g->count.push_back(base + (r < extra ? 1 : 0));
        if (int st = irl_ctx_create(g->dev[r], &g->ctx[r])) {
            destroy_group(g);
            return st;
        }
        if (int st = irl_ccmm_create(g->ctx[r], g->count[r], m, k, max_n, primes, exps, nmod, &g->eng[r])) {
            destroy_group(g);
            return st;
        }
    }
    *out = g;
    return IRL_OK;
}

int irl_ccmm_group_destroy(irl_ccmm_group* g) {
    if (g) destroy_group(g);
    return IRL_OK;
}

int irl_ccmm_group_engine(irl_ccmm_group* g, size_t rank, irl_ccmm** e, size_t* first_part, size_t* nparts) {
    if (!g || rank >= g->ndev) return IRL_ERR_INVALID_ARGUMENT;
    if (e) *e = g->eng[rank];
    if (first_part) *first_part = g->first[rank];
    if (nparts) *nparts = g->count[rank];
    return IRL_OK;
}

irl_ctx* irl_ccmm_group_ctx(irl_ccmm_group* g, size_t rank) {
    return g && rank < g->ndev ? g->ctx[rank] : nullptr;
}

int irl_ccmm_full(irl_ccmm_group* g, const uint16_t* q_res_host, size_t n, uint16_t* out_host, void** a_out,
                  int* fused) {
    if (!g || !q_res_host || !out_host) return IRL_ERR_INVALID_ARGUMENT;
    irl_ctx* c0 = g->ctx[0];
    if (n == 0 || n > g->max_n) return set_err(c0, IRL_ERR_SHAPE_MISMATCH, "ccmm group: query width out of range");
    if (int st = setup_exchange(g, n)) return st;
    std::vector<int> st(g->ndev, IRL_OK);
    std::vector<std::thread> th;
    for (size_t r = 0; r < g->ndev; ++r)
        th.emplace_back([&, r] {
            uint16_t* dst = out_host + g->first[r] * g->nmod * n * g->M;
            st[r] = irl_ccmm_run(g->eng[r], q_res_host, n, dst);
        });
    for (auto& t : th) t.join();
    for (size_t r = 0; r < g->ndev; ++r)
        if (st[r] != IRL_OK)
            return set_err(c0, st[r], std::string("rank ") + std::to_string(r) + ": " + irl_last_error(g->ctx[r]));
    void* q0 = nullptr;
    void* out0 = nullptr;
    irl_ccmm_buffers(g->eng[0], &q0, &out0);  // rank 0's outputs; part 0 = the a-part result
    const size_t a_bytes = g->nmod * n * g->M * sizeof(uint16_t);
    if (!g->fused) {  // the exchange as plain peer copies after the runs
        for (size_t r = 1; r < g->ndev; ++r) {
            cudaSetDevice(g->dev[r]);
            const cudaError_t e = cudaMemcpyPeer(g->recv[r], g->dev[r], out0, g->dev[0], a_bytes);
            if (e != cudaSuccess) return cuda_fail(c0, e, "cudaMemcpyPeer (a-part exchange)");
        }
    }
    if (a_out)
        for (size_t r = 0; r < g->ndev; ++r) a_out[r] = r == 0 ? out0 : g->recv[r];
    if (fused) *fused = g->fused ? 1 : 0;
    return IRL_OK;
}

}  // extern "C"
