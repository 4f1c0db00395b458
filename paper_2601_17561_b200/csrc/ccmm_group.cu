// Single-process multi-GPU CCMM (include/irl_capi.h, irl_ccmm_group_* and
// irl_ccmm_full; SURVEY §8(b)'s irl_ccmm_full).
//
// One context and one engine per device. The parts are dealt in contiguous
// blocks as dist.part_range does (the a-part on rank 0). Every rank runs its
// parts end to end (irl_ccmm_run) on its own host thread, so the devices work
// concurrently. The a-part exchange is fused into rank 0's PPMM epilogue: it
// stores each output tile of part 0 into every other rank's receive buffer
// over peer memory (NVLink) while it computes. Where peer access is not
// available, a cudaMemcpyPeer after the runs takes its place. On request, with
// one rank per multicast-capable device (NVSwitch), the epilogue instead
// stores once to an NVLS multicast address and the switch writes every copy.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/irl_capi.h"
#include "ctx_internal.h"

using namespace irl;

namespace {

// Driver entry points of the NVLS multicast path, resolved once at run time
// (the library links only the runtime).
struct McApi {
    CUresult (*GetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
    CUresult (*Create)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
    CUresult (*AddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
    CUresult (*BindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                        unsigned long long) = nullptr;
    CUresult (*Unbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
    CUresult (*AllocGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
    CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) =
        nullptr;
    CUresult (*Release)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*Reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
    CUresult (*Free)(CUdeviceptr, size_t) = nullptr;
    CUresult (*Map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
    CUresult (*Unmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*SetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
    CUresult (*DeviceGet)(CUdevice*, int) = nullptr;
    CUresult (*GetAttribute)(int*, CUdevice_attribute, CUdevice) = nullptr;
    bool ok = false;
};

template <typename F>
bool entry(const char* name, F* fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
        cudaGetLastError();
        return false;
    }
    *fn = reinterpret_cast<F>(p);
    return true;
}

const McApi& mc_api() {
    static const McApi api = [] {
        McApi a;
        a.ok = entry("cuMulticastGetGranularity", &a.GetGranularity) && entry("cuMulticastCreate", &a.Create) &&
               entry("cuMulticastAddDevice", &a.AddDevice) && entry("cuMulticastBindMem", &a.BindMem) &&
               entry("cuMulticastUnbind", &a.Unbind) &&
               entry("cuMemGetAllocationGranularity", &a.AllocGranularity) && entry("cuMemCreate", &a.MemCreate) &&
               entry("cuMemRelease", &a.Release) && entry("cuMemAddressReserve", &a.Reserve) &&
               entry("cuMemAddressFree", &a.Free) && entry("cuMemMap", &a.Map) && entry("cuMemUnmap", &a.Unmap) &&
               entry("cuMemSetAccess", &a.SetAccess) && entry("cuDeviceGet", &a.DeviceGet) &&
               entry("cuDeviceGetAttribute", &a.GetAttribute);
        return a;
    }();
    return api;
}

// One multicast object over the ranks' devices, a physical receive buffer per
// rank bound to it and mapped locally, and the multicast address mapped for
// rank 0 (the a-part owner, whose epilogue stores through it).
struct McExchange {
    CUmemGenericAllocationHandle mc = 0;
    std::vector<CUmemGenericAllocationHandle> phys;
    std::vector<CUdeviceptr> va;
    CUdeviceptr mc_va = 0;
    size_t size = 0;
    std::vector<int> dev;
};

void mc_release(McExchange* x) {
    const McApi& a = mc_api();
    if (!a.ok) return;
    if (x->mc_va) {
        a.Unmap(x->mc_va, x->size);
        a.Free(x->mc_va, x->size);
    }
    for (size_t r = 0; r < x->va.size(); ++r) {
        if (x->va[r]) {
            a.Unmap(x->va[r], x->size);
            a.Free(x->va[r], x->size);
        }
    }
    if (x->mc) {
        for (int d : x->dev) {
            CUdevice cd;
            if (a.DeviceGet(&cd, d) == CUDA_SUCCESS) a.Unbind(x->mc, cd, 0, x->size);
        }
    }
    for (CUmemGenericAllocationHandle h : x->phys)
        if (h) a.Release(h);
    if (x->mc) a.Release(x->mc);
    *x = McExchange();
}

}  // namespace

struct irl_ccmm_group {
    size_t ndev = 0, parts = 0, M = 0, K = 0, max_n = 0, nmod = 0;
    std::vector<int> dev;
    std::vector<irl_ctx*> ctx;
    std::vector<irl_ccmm*> eng;
    std::vector<size_t> first, count;
    std::vector<uint16_t*> recv;  // rank r: receive buffer of the a-part result [nmod][n][M] (r > 0, or all with MC)
    size_t recv_n = 0;            // width the receive buffers and mirrors are set up for
    size_t slot = 0;              // receive slot of the last irl_ccmm_full (alternates per call)
    int requested = IRL_EXCHANGE_AUTO;
    int mode = IRL_EXCHANGE_COPY;  // the exchange in use
    int shard = -1;                // query distribution: -1 auto, 0 every rank copies it all, 1 sharded
    bool peers_enabled = false;    // all-pairs peer access attempted (sharded query)
    McExchange mcx;
    std::mutex mu;  // one irl_ccmm_full / set_exchange at a time
};

namespace {

void destroy_group(irl_ccmm_group* g) {
    if (!g->eng.empty() && g->eng[0]) irl_ccmm_set_mirror_multicast(g->eng[0], 0, 0, nullptr);
    mc_release(&g->mcx);
    for (size_t r = 0; r < g->eng.size(); ++r)
        if (g->eng[r]) irl_ccmm_destroy(g->eng[r]);
    for (irl_ctx* c : g->ctx)
        if (c) irl_ctx_destroy(c);
    delete g;
}

bool mc_supported(const irl_ccmm_group* g) {
    const McApi& a = mc_api();
    if (!a.ok) return false;
    for (size_t r = 0; r < g->ndev; ++r) {
        for (size_t q = 0; q < r; ++q)
            if (g->dev[q] == g->dev[r]) return false;  // one bound buffer per device
        CUdevice cd;
        int v = 0;
        if (a.DeviceGet(&cd, g->dev[r]) != CUDA_SUCCESS ||
            a.GetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cd) != CUDA_SUCCESS || !v)
            return false;
    }
    return true;
}

#define MC_CK(expr)                                                                    \
    do {                                                                               \
        const CUresult r__ = (expr);                                                   \
        if (r__ != CUDA_SUCCESS) {                                                     \
            mc_release(&g->mcx);                                                       \
            return set_err(g->ctx[0], IRL_ERR_CUDA, std::string("multicast: ") + #expr); \
        }                                                                              \
    } while (0)

int mc_setup(irl_ccmm_group* g, size_t bytes) {
    const McApi& a = mc_api();
    McExchange& x = g->mcx;
    x.dev = g->dev;
    CUmulticastObjectProp prop = {};
    prop.numDevices = static_cast<unsigned>(g->ndev);
    prop.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
    prop.size = bytes;
    size_t mg = 0, pg = 0;
    MC_CK(a.GetGranularity(&mg, &prop, CU_MULTICAST_GRANULARITY_MINIMUM));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = g->dev[0];
    MC_CK(a.AllocGranularity(&pg, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
    const size_t gran = std::max(mg, pg);
    x.size = (bytes + gran - 1) / gran * gran;
    prop.size = x.size;
    MC_CK(a.Create(&x.mc, &prop));
    for (size_t r = 0; r < g->ndev; ++r) {
        CUdevice cd;
        MC_CK(a.DeviceGet(&cd, g->dev[r]));
        MC_CK(a.AddDevice(x.mc, cd));
    }
    x.phys.assign(g->ndev, 0);
    x.va.assign(g->ndev, 0);
    for (size_t r = 0; r < g->ndev; ++r) {
        cudaSetDevice(g->dev[r]);
        cudaFree(nullptr);  // the device's primary context is current for the driver calls
        ap.location.id = g->dev[r];
        MC_CK(a.MemCreate(&x.phys[r], x.size, &ap, 0));
        MC_CK(a.BindMem(x.mc, 0, x.phys[r], 0, x.size, 0));
        MC_CK(a.Reserve(&x.va[r], x.size, 0, 0, 0));
        MC_CK(a.Map(x.va[r], x.size, 0, x.phys[r], 0));
        CUmemAccessDesc ad = {};
        ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ad.location.id = g->dev[r];
        ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        MC_CK(a.SetAccess(x.va[r], x.size, &ad, 1));
    }
    cudaSetDevice(g->dev[0]);
    MC_CK(a.Reserve(&x.mc_va, x.size, 0, 0, 0));
    MC_CK(a.Map(x.mc_va, x.size, 0, x.mc, 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = g->dev[0];
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    MC_CK(a.SetAccess(x.mc_va, x.size, &ad, 1));
    return IRL_OK;
}

// The exchange for width n: NVLS multicast (one multimem.st per element pair,
// replicated by the switch into every rank's bound buffer), P2P stores into
// each peer's receive buffer, or a cudaMemcpyPeer after the runs.
int setup_exchange(irl_ccmm_group* g, size_t n) {
    if (g->recv_n == n) return IRL_OK;
    irl_ctx* c0 = g->ctx[0];
    // invalidate first: a rebuild that fails part way must be retried by the
    // next call, never mistaken for a ready exchange of the old width
    g->recv_n = 0;
    g->mode = IRL_EXCHANGE_COPY;
    irl_ccmm_set_mirror_ptrs(g->eng[0], 0, n, nullptr, 0);
    irl_ccmm_set_mirror_multicast(g->eng[0], 0, 0, nullptr);
    mc_release(&g->mcx);
    g->recv.assign(g->ndev, nullptr);
    const size_t bytes = IRL_RECV_SLOTS * g->nmod * n * g->M * sizeof(uint16_t);
    // multicast is opt-in: it could not be exercised where this was built
    // (cuMulticastCreate is refused inside the container), so AUTO stays on
    // the validated P2P stores
    const bool want_mc = g->requested == IRL_EXCHANGE_MULTICAST;
    if (want_mc && (g->M % 2) == 0 && mc_supported(g)) {
        if (mc_setup(g, bytes) != IRL_OK) {
            return set_err(c0, IRL_ERR_UNSUPPORTED,
                           std::string("ccmm group: NVLS multicast refused by the driver (") + irl_last_error(c0) + ")");
        } else {
            for (size_t r = 0; r < g->ndev; ++r) g->recv[r] = reinterpret_cast<uint16_t*>(g->mcx.va[r]);
            if (int st = irl_ccmm_set_mirror_multicast(g->eng[0], 0, n, reinterpret_cast<void*>(g->mcx.mc_va)))
                return st;
            g->mode = IRL_EXCHANGE_MULTICAST;
            g->recv_n = n;
            return IRL_OK;
        }
    } else if (g->requested == IRL_EXCHANGE_MULTICAST) {
        return set_err(c0, IRL_ERR_UNSUPPORTED, "ccmm group: NVLS multicast unavailable (one rank per device, "
                                                "multicast-capable devices and an even M are required)");
    }
    bool peer = g->requested != IRL_EXCHANGE_COPY;
    for (size_t r = 1; r < g->ndev; ++r) {
        void* p = nullptr;
        if (int st = irl_ccmm_alloc_recv(g->eng[r], n, &p, nullptr)) {
            set_err(c0, st, std::string("rank ") + std::to_string(r) + ": " + irl_last_error(g->ctx[r]));
            return st;
        }
        g->recv[r] = static_cast<uint16_t*>(p);
        if (peer && g->dev[r] != g->dev[0]) {
            int can = 0;
            cudaSetDevice(g->dev[0]);
            if (cudaDeviceCanAccessPeer(&can, g->dev[0], g->dev[r]) != cudaSuccess || !can) {
                peer = false;
            } else {
                const cudaError_t e = cudaDeviceEnablePeerAccess(g->dev[r], 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) peer = false;
            }
            cudaGetLastError();
        }
    }
    peer = peer && g->ndev > 1 && g->ndev - 1 <= static_cast<size_t>(kMaxMirrors);
    if (g->requested == IRL_EXCHANGE_P2P && !peer && g->ndev > 1)
        return set_err(c0, IRL_ERR_UNSUPPORTED, "ccmm group: peer access unavailable for P2P stores");
    std::vector<uint16_t*> peers(g->recv.begin() + (g->ndev > 1 ? 1 : 0), g->recv.end());
    if (int st = irl_ccmm_set_mirror_ptrs(g->eng[0], 0, n, peers.data(), peer ? peers.size() : 0)) return st;
    g->mode = peer ? IRL_EXCHANGE_P2P : IRL_EXCHANGE_COPY;
    g->recv_n = n;
    return IRL_OK;
}

// Sharded query distribution (PAPER.md:72's query AllGather): rank r copies
// moduli [lo_r, hi_r) of the host query into its staging buffer, pushes that
// slice into every other rank's staging buffer over peer memory (NVLink), and
// each rank then runs its parts on the staged query (irl_ccmm_run_dq). The
// host sends the query across PCIe once in total instead of once per GPU,
// which pays when a rank's GEMM per modulus is shorter than its H2D (one
// 2^14-row part per GPU: 18 ms of GEMM against 21.7 ms to copy 1.17 GB).
bool shard_query(const irl_ccmm_group* g) {
    if (g->ndev < 2 || g->shard == 0) return false;
    if (g->shard == 1) return true;
    size_t most = 0;
    for (size_t c : g->count) most = std::max(most, c);
    return most * g->M < 20000;  // about one paper-size part per rank (bench.py uses the same rule)
}

void enable_all_peers(irl_ccmm_group* g) {
    if (g->peers_enabled) return;
    for (size_t a = 0; a < g->ndev; ++a)
        for (size_t b = 0; b < g->ndev; ++b) {
            if (g->dev[a] == g->dev[b]) continue;
            int can = 0;
            cudaSetDevice(g->dev[a]);
            if (cudaDeviceCanAccessPeer(&can, g->dev[a], g->dev[b]) == cudaSuccess && can)
                cudaDeviceEnablePeerAccess(g->dev[b], 0);  // AlreadyEnabled is fine
            cudaGetLastError();
        }
    g->peers_enabled = true;
}

// Runs f(r) on one host thread per rank; the first failing rank's status.
template <typename F>
int on_ranks(irl_ccmm_group* g, F f) {
    std::vector<int> st(g->ndev, IRL_OK);
    std::vector<std::thread> th;
    for (size_t r = 0; r < g->ndev; ++r) th.emplace_back([&, r] { st[r] = f(r); });
    for (auto& t : th) t.join();
    for (size_t r = 0; r < g->ndev; ++r)
        if (st[r] != IRL_OK)
            return set_err(g->ctx[0], st[r], std::string("rank ") + std::to_string(r) + ": " + irl_last_error(g->ctx[r]));
    return IRL_OK;
}

int run_sharded(irl_ccmm_group* g, const uint16_t* q_res_host, size_t n, uint16_t* out_host) {
    enable_all_peers(g);
    const size_t slice = g->K * n;  // elements of one modulus' query [K][n]
    std::vector<uint16_t*> q(g->ndev);
    for (size_t r = 0; r < g->ndev; ++r) {
        void* p = nullptr;
        irl_ccmm_buffers(g->eng[r], &p, nullptr);
        q[r] = static_cast<uint16_t*>(p);
    }
    auto lo = [&](size_t r) { return r * g->nmod / g->ndev; };
    // 1. each rank's share of the moduli, host -> its own staging buffer
    if (int st = on_ranks(g, [&](size_t r) -> int {
            irl_ctx* c = g->ctx[r];
            Guard gd(c, "irl_ccmm_full: query shard H2D");
            const size_t off = lo(r) * slice, elems = (lo(r + 1) - lo(r)) * slice;
            IRL_CK(c, copy_h2d(c, q[r] + off, q_res_host + off, elems * 2, c->stream));
            IRL_CK(c, cudaStreamSynchronize(c->stream));
            return IRL_OK;
        }))
        return st;
    // 2. all-gather: every rank pushes its share into the other ranks' buffers
    if (int st = on_ranks(g, [&](size_t r) -> int {
            irl_ctx* c = g->ctx[r];
            Guard gd(c, "irl_ccmm_full: query all-gather");
            const size_t off = lo(r) * slice, bytes = (lo(r + 1) - lo(r)) * slice * 2;
            for (size_t t = 0; t < g->ndev; ++t)
                if (t != r && bytes)
                    IRL_CK(c, cudaMemcpyPeerAsync(q[t] + off, g->dev[t], q[r] + off, g->dev[r], bytes, c->stream));
            IRL_CK(c, cudaStreamSynchronize(c->stream));
            return IRL_OK;
        }))
        return st;
    // 3. every rank's parts on the staged query
    return on_ranks(g, [&](size_t r) -> int {
        return irl_ccmm_run_dq(g->eng[r], nullptr, n, out_host + g->first[r] * g->nmod * n * g->M, nullptr);
    });
}

}  // namespace

extern "C" {

int irl_ccmm_group_set_query_shard(irl_ccmm_group* g, int mode) {
    if (!g || mode < -1 || mode > 1) return IRL_ERR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(g->mu);
    g->shard = mode;
    return IRL_OK;
}

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

int irl_ccmm_group_set_exchange(irl_ccmm_group* g, int mode) {
    if (!g || mode < IRL_EXCHANGE_AUTO || mode > IRL_EXCHANGE_COPY) return IRL_ERR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(g->mu);
    g->requested = mode;
    g->recv_n = 0;  // set up again on the next run
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
                  int* mode) {
    if (!g || !q_res_host || !out_host) return IRL_ERR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(g->mu);
    irl_ctx* c0 = g->ctx[0];
    if (n == 0 || n > g->max_n) return set_err(c0, IRL_ERR_SHAPE_MISMATCH, "ccmm group: query width out of range");
    if (int st = setup_exchange(g, n)) return st;
    // double-buffered receive: this call stores into the other slot, so a
    // consumer still reading the previous call's a-part is never overwritten
    g->slot = (g->slot + 1) % IRL_RECV_SLOTS;
    if (int st = irl_ccmm_set_mirror_slot(g->eng[0], g->slot)) return st;
    if (shard_query(g)) {
        if (int st = run_sharded(g, q_res_host, n, out_host)) return st;
    } else if (int st = on_ranks(g, [&](size_t r) -> int {
                   return irl_ccmm_run(g->eng[r], q_res_host, n, out_host + g->first[r] * g->nmod * n * g->M);
               })) {
        return st;
    }
    void* q0 = nullptr;
    void* out0 = nullptr;
    irl_ccmm_buffers(g->eng[0], &q0, &out0);  // rank 0's outputs; part 0 = the a-part result
    const size_t a_elems = g->nmod * n * g->M, a_bytes = a_elems * sizeof(uint16_t);
    if (g->mode == IRL_EXCHANGE_COPY) {  // the exchange as plain peer copies after the runs
        for (size_t r = 1; r < g->ndev; ++r) {
            cudaSetDevice(g->dev[r]);
            const cudaError_t e = cudaMemcpyPeer(g->recv[r] + g->slot * a_elems, g->dev[r], out0, g->dev[0], a_bytes);
            if (e != cudaSuccess) return cuda_fail(c0, e, "cudaMemcpyPeer (a-part exchange)");
        }
    }
    if (a_out)
        for (size_t r = 0; r < g->ndev; ++r)
            a_out[r] = g->recv[r] ? static_cast<void*>(g->recv[r] + g->slot * a_elems) : out0;
    if (mode) *mode = g->mode;
    return IRL_OK;
}

}  // extern "C"
