// Probe: how many bytes per clock can TMA deliver into one SM's shared memory
// on B200, with and without cluster multicast? Both PPMM-engine kernels fill a
// 64 KB stage per CTA per K block (DB tile + query tile), so this rate bounds
// them independently of the tensor cores:
//   * int8 PPMM (kModePsq): 64 KB per 12 MMAs (3 products x 4 k-steps of 32),
//     1488 clk at the int8 rate  ->  43 B/clk/SM needed at 100% tensor;
//   * FP4 iris (kModeIrisMatchF4): 62 KB per 8 MMAs (2 products x 4 k-steps of
//     64), 960 clk at the FP4 rate  ->  65 B/clk/SM needed at 100% tensor.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_probe profiles/tma_ingest_probe.cu
//   ./tma_probe            (one JSON line per variant)
//
// Each CTA runs a 3 x 64 KB ring like the engine (producer thread + consumer
// thread, mbarriers, no MMA). A stage is two 32 KB halves: "A" (shared by gA
// CTAs of the cluster: each loads 1/gA and multicasts it to the others) and
// "B" (shared by gB CTAs). A slot is refilled only when every CTA of the
// cluster consumed it (the engine's lock-step). Sources: A streams from a
// 4 GiB buffer (DRAM, like the DB tiles), B cycles through 16 MB (L2-resident,
// like the query planes); a second pass keeps A in a 32 MB L2-resident buffer
// too, which isolates the L2 -> SM delivery cap. Reported: bytes landed in shared memory per SM clock
// (delivered) and global bytes requested per SM clock (delivered / multicast).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

namespace {

constexpr uint32_t kMaxStages = 12;
constexpr uint32_t kRingBytes = 3 * 65536;    // the engine's ring: 3 x 64 KB
constexpr int kThreads = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tLAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LAB_WAIT;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void bulk_mc(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "h"(mask)
        : "memory");
}

// group of `g` CTAs sharing a half: ranks with the same (rank % (C / g)), index rank / (C / g)
// each CTA's share is issued as copies of at most `piece` bytes
__device__ __forceinline__ void load_half(uint32_t dst, const uint8_t* src, uint32_t kHalf, uint32_t g, uint32_t C,
                                          uint32_t rank, uint32_t bar, uint32_t piece) {
    if (g == 1) {
        for (uint32_t o = 0; o < kHalf; o += piece) bulk(dst + o, src + o, min(piece, kHalf - o), bar);
        return;
    }
    const uint32_t stride = C / g, idx = rank / stride, base = rank % stride;
    uint16_t mask = 0;
    for (uint32_t j = 0; j < g; ++j) mask |= 1u << (base + j * stride);
    const uint32_t sub = kHalf / g;
    for (uint32_t o = 0; o < sub; o += piece)
        bulk_mc(dst + idx * sub + o, src + idx * sub + o, min(piece, sub - o), bar, mask);
}

__global__ void __launch_bounds__(kThreads, 1)
    probe_kernel(const uint8_t* __restrict__ a_src, size_t a_bytes, const uint8_t* __restrict__ b_src,
                 size_t b_bytes, uint32_t gA, uint32_t gB, uint32_t iters, uint32_t kStages, uint32_t kHalf,
                 uint32_t hold, uint32_t piece, unsigned long long* cycles) {
    const uint32_t kStage = 2 * kHalf;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRingBytes);
    uint64_t* empty = full + kStages;
    const uint32_t rank = ctarank(), C = nctarank();
    const uint32_t cluster = blockIdx.x / C, nclusters = gridDim.x / C;
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < kStages; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), C);  // every CTA of the cluster releases the slot
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_sync();
    const long long t0 = clock64();
    if (threadIdx.x == 0) {
        // producer: A half from the streaming buffer (distinct per A group and
        // iteration), B half from the L2-resident buffer
        const uint32_t a_groups = C / gA, b_groups = C / gB;
        const size_t a_units = a_bytes / kHalf, b_units = b_bytes / kHalf;
        for (uint32_t it = 0; it < iters; ++it) {
            const uint32_t s = it % kStages, ph = (it / kStages) & 1;
            wait(smem_u32(&empty[s]), ph ^ 1);
            const uint32_t fb = smem_u32(&full[s]);
            expect_tx(fb, kStage);
            const size_t au = (static_cast<size_t>(it) * nclusters * a_groups + cluster * a_groups + rank % a_groups) % a_units;
            const size_t bu = (static_cast<size_t>(it) * 7 + cluster * b_groups + rank % b_groups) % b_units;
            const uint32_t dst = smem_u32(smem + s * kStage);
            load_half(dst, a_src + au * kHalf, kHalf, gA, C, rank, fb, piece);
            load_half(dst + kHalf, b_src + bu * kHalf, kHalf, gB, C, rank, fb, piece);
        }
    } else if (threadIdx.x >= 32) {
        // consumer warp: wait for the stage, then lane r releases it in CTA r
        // of the cluster (all remote arrives in parallel)
        const uint32_t lane = threadIdx.x - 32;
        for (uint32_t it = 0; it < iters; ++it) {
            const uint32_t s = it % kStages, ph = (it / kStages) & 1;
            wait(smem_u32(&full[s]), ph);
            if (hold) {  // emulate the MMAs consuming the stage
                const long long h0 = clock64();
                while (clock64() - h0 < hold) {
                }
            }
            __syncwarp();
            if (lane < C) arrive_remote(mapa(smem_u32(&empty[s]), lane));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = static_cast<unsigned long long>(clock64() - t0);
    cluster_sync();
}

}  // namespace

int main() {
    int dev = 0, sms = 0;
    cudaSetDevice(dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t a_bytes = size_t(4) << 30, b_bytes = size_t(16) << 20;
    uint8_t *a = nullptr, *b = nullptr;
    if (cudaMalloc(&a, a_bytes) != cudaSuccess || cudaMalloc(&b, b_bytes) != cudaSuccess) {
        std::printf("{\"error\": \"alloc\"}\n");
        return 1;
    }
    cudaMemset(a, 1, a_bytes);
    cudaMemset(b, 2, b_bytes);
    unsigned long long* cyc = nullptr;
    cudaMalloc(&cyc, sizeof(unsigned long long) * 1024);
    const size_t smem = kRingBytes + 1024 + 2 * kMaxStages * 8;
    cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    struct V {
        const char* name;
        uint32_t C, gA, gB;
    } vs[] = {{"unicast (1 CTA clusters)", 1, 1, 1},       {"8-CTA cluster, unicast", 8, 1, 1},
              {"int8 PPMM 1x4: A mc 4", 8, 4, 1},         {"2x2: A mc 2, B mc 2", 8, 2, 2},
              {"2x4: A mc 4, B mc 2 (16 CTAs)", 16, 4, 2}, {"A mc 8, B mc 8", 8, 8, 8},
              {"A mc 2 (4-CTA clusters)", 4, 2, 1}, {"unicast, 74 CTAs (half the SMs)", 1, 1, 1}};
    struct Ring {
        uint32_t stages, half;
    } rings[] = {{3, 32768}, {2, 32768}, {4, 16384}, {6, 16384}, {12, 8192}};
    const uint32_t iters_bytes = 3000u * 65536u;  // per CTA
    auto run = [&](const V& v, int src, Ring rg, uint32_t hold_per_kb, uint32_t piece = 1u << 20) {
        // src 0: both halves L2-resident (the delivery cap); src 1: A streams from DRAM
        const size_t a_use = src == 0 ? (size_t(32) << 20) : a_bytes;
        const uint32_t stage = 2 * rg.half, iters = iters_bytes / stage;
        const uint32_t hold = hold_per_kb * (stage / 1024);
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = v.C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(v.C);
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, probe_kernel, &cfg) != cudaSuccess || ncl == 0) {
            cudaGetLastError();
            std::printf("{\"variant\": \"%s\", \"error\": \"no occupancy\"}\n", v.name);
            return;
        }
        uint32_t ctas = static_cast<uint32_t>(ncl) * v.C;
        if (std::string(v.name).find("74 CTAs") != std::string::npos) ctas = 74;
        cfg.gridDim = dim3(ctas);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best_ms = 1e30f;
        std::vector<unsigned long long> h(ctas);
        double best_bpc = 0;
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(e0);
            cudaLaunchKernelEx(&cfg, probe_kernel, (const uint8_t*)a, a_use, (const uint8_t*)b, b_bytes, v.gA,
                               v.gB, iters, rg.stages, rg.half, hold, piece, cyc);
            cudaEventRecord(e1);
            if (cudaEventSynchronize(e1) != cudaSuccess) {
                std::printf("{\"variant\": \"%s\", \"error\": \"%s\"}\n", v.name,
                            cudaGetErrorString(cudaGetLastError()));
                std::exit(1);
            }
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaMemcpy(h.data(), cyc, sizeof(unsigned long long) * ctas, cudaMemcpyDeviceToHost);
            unsigned long long mx = 0;
            for (auto c : h) mx = c > mx ? c : mx;
            const double bpc = double(iters) * stage / double(mx);
            if (ms < best_ms) {
                best_ms = ms;
                best_bpc = bpc;
            }
        }
        const double delivered = double(iters) * stage * ctas;
        const double req_frac = (rg.half / double(v.gA) + rg.half / double(v.gB)) / stage;
        std::printf(
            "{\"variant\": \"%s\", \"a_source\": \"%s\", \"ring\": \"%u x %u KB\", \"hold_clk_per_KB\": %u, \"piece\": %u, "
            "\"cluster\": %u, \"ctas\": %u, \"sms\": %d, \"ms\": %.4f, "
            "\"delivered_TBps\": %.3f, \"requested_TBps\": %.3f, \"delivered_B_per_clk_per_sm\": %.2f, "
            "\"requested_B_per_clk_per_sm\": %.2f, \"sm_clock_GHz\": %.3f}\n",
            v.name, src == 0 ? "L2 (32 MB)" : "DRAM (4 GiB stream)", rg.stages, stage / 1024, hold_per_kb, piece, v.C, ctas,
            sms, best_ms, delivered / (best_ms * 1e-3) / 1e12, delivered * req_frac / (best_ms * 1e-3) / 1e12, best_bpc,
            best_bpc * req_frac, delivered / ctas / best_bpc / (best_ms * 1e-3) / 1e9);
        std::fflush(stdout);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    };
    // 1. delivery cap by cluster shape (the engine's 3 x 64 KB ring, no consumer work)
    for (int src = 0; src < 2; ++src)
        for (const V& v : vs) run(v, src, rings[0], 0);
    // 2. ring depth / granularity for the 1x4 shape, with the consumer holding
    //    each stage as long as the MMAs would: 15 clk/KB (FP4 iris: 960 clk per
    //    64 KB) and 23 clk/KB (int8 PPMM: 1488 clk per 64 KB); 0 = no hold
    for (int src = 0; src < 2; ++src)
        for (uint32_t hold : {0u, 15u, 23u})
            for (const Ring& rg : rings) run(vs[2], src, rg, hold);
    // 3. copy granularity: the engine issues 2-D tensor copies of 128-row boxes
    //    (16 KB, or 4 KB per multicast quarter); here each share is cut into
    //    copies of `piece` bytes
    for (int src = 0; src < 2; ++src)
        for (uint32_t hold : {0u, 15u, 23u})
            for (uint32_t piece : {16384u, 4096u, 1024u}) run(vs[2], src, rings[0], hold, piece);
    return 0;
}
