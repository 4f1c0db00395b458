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

#ifndef RELAXED_ARRIVE
#define RELAXED_ARRIVE 1
#endif

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
// relaxed: a release.cluster arrive here measured the ring at ~42 B/clk per SM
// whatever its depth (the release serialises the consumer behind the copies in
// flight); the engine releases stages with tcgen05.commit instead
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
    if (RELAXED_ARRIVE)
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
    else
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

// Mixed load paths, no clusters: thread 0 streams 64 KB stages by TMA into a
// 2 x 64 KB ring (warp 1 releases them), while `lsu_warps` warps copy 16-byte
// chunks with cp.async (LDGSTS) into a separate 64 KB region, both from the
// L2-resident buffer, for `budget` cycles. Does the LSU path add to the TMA's
// per-SM delivery, or share its port?
__global__ void __launch_bounds__(64 + 32 * 16, 1)
    mixed_kernel(const uint8_t* __restrict__ src, size_t src_bytes, uint32_t tma_on, uint32_t lsu_warps,
                 long long budget, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr uint32_t kSt = 65536, kNs = 2;
    uint8_t* lsu_region = smem + kNs * kSt;
    uint64_t* full = reinterpret_cast<uint64_t*>(lsu_region + 65536);
    uint64_t* empty = full + kNs;
    __shared__ unsigned long long lsu_total;
    __shared__ uint32_t stages_done;
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < kNs; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        lsu_total = 0;
        stages_done = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long t0 = clock64();
    const size_t units = src_bytes / kSt;
    if (warp == 0) {
        if (lane == 0 && tma_on) {
            uint32_t it = 0;
            for (; clock64() - t0 < budget; ++it) {
                const uint32_t s = it % kNs, ph = (it / kNs) & 1;
                wait(smem_u32(&empty[s]), ph ^ 1);
                const uint32_t fb = smem_u32(&full[s]);
                expect_tx(fb, kSt);
                if (tma_on == 1) {
                    const uint8_t* g = src + ((static_cast<size_t>(it) * gridDim.x + blockIdx.x) % units) * kSt;
                    for (uint32_t o = 0; o < kSt; o += 16384) bulk(smem_u32(smem + s * kSt) + o, g + o, 16384, fb);
                } else {
                    // probe_kernel's pattern: two 32 KB halves, A unit it*grid + b, B unit it*7 + b
                    const size_t hu = src_bytes / 32768;
                    const uint8_t* ga = src + ((static_cast<size_t>(it) * gridDim.x + blockIdx.x) % hu) * 32768;
                    const uint8_t* gb = src + ((static_cast<size_t>(it) * 7 + blockIdx.x) % hu) * 32768;
                    const uint32_t pc = tma_on == 2 ? 16384u : 32768u;
                    for (uint32_t o = 0; o < 32768; o += pc) bulk(smem_u32(smem + s * kSt) + o, ga + o, pc, fb);
                    for (uint32_t o = 0; o < 32768; o += pc) bulk(smem_u32(smem + s * kSt) + 32768 + o, gb + o, pc, fb);
                }
            }
            stages_done = it;  // the consumer drains them all
        }
    } else if (warp == 1) {
        if (tma_on) {
            for (uint32_t it = 0;; ++it) {
                // stop once the producer has published its count and we consumed them
                const uint32_t n = *reinterpret_cast<volatile uint32_t*>(&stages_done);
                if (n != 0 && it >= n) break;
                if (n == 0 && clock64() - t0 > 4 * budget) break;  // safety
                const uint32_t s = it % kNs, ph = (it / kNs) & 1;
                // try until the stage lands or the producer has stopped before it
                bool landed = false;
                while (true) {
                    uint32_t ok;
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                        "selp.u32 %0, 1, 0, p;\n\t}"
                        : "=r"(ok)
                        : "r"(smem_u32(&full[s])), "r"(ph)
                        : "memory");
                    if (ok) {
                        landed = true;
                        break;
                    }
                    const uint32_t m = *reinterpret_cast<volatile uint32_t*>(&stages_done);
                    if (m != 0 && it >= m) break;
                }
                if (!landed) break;
                if (lane == 0)
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
                __syncwarp();
            }
        }
    } else if (warp - 2 < lsu_warps) {
        const uint32_t t = threadIdx.x - 64, nt = lsu_warps * 32;
        unsigned long long bytes = 0;
        uint32_t it = 0;
        const uint32_t dst0 = smem_u32(lsu_region);
        while (clock64() - t0 < budget) {
            // 16 x 16 B per thread per batch, coalesced across the warp
            const uint8_t* g = src + ((static_cast<size_t>(it) * gridDim.x + blockIdx.x) % units) * kSt;
#pragma unroll
            for (uint32_t j = 0; j < 16; ++j) {
                const uint32_t off = ((j * nt + t) * 16u) % 65536u;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst0 + off), "l"(g + off) : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_group 3;" ::: "memory");
            bytes += 256;
            ++it;
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        atomicAdd(&lsu_total, bytes);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const long long cyc = clock64() - t0;
        out[3 * blockIdx.x] = static_cast<unsigned long long>(stages_done) * kSt;
        out[3 * blockIdx.x + 1] = lsu_total;
        out[3 * blockIdx.x + 2] = static_cast<unsigned long long>(cyc);
    }
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
        const size_t a_use = src == 0 ? (size_t(32) << 20) : src == 1 ? a_bytes : b_bytes;
        const uint8_t* a_ptr = src == 2 ? b : a;
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
        if (v.C == 1 && std::getenv("PROBE_NOCLUSTER")) cfg.numAttrs = 0;  // plain launch
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best_ms = 1e30f;
        std::vector<unsigned long long> h(ctas);
        double best_bpc = 0;
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(e0);
            cudaLaunchKernelEx(&cfg, probe_kernel, a_ptr, a_use, (const uint8_t*)b, b_bytes, v.gA,
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
            v.name, src == 0 ? "L2 (32 MB)" : src == 1 ? "DRAM (4 GiB stream)" : "L2 (the B buffer, 16 MB)", rg.stages, stage / 1024, hold_per_kb, piece, v.C, ctas,
            sms, best_ms, delivered / (best_ms * 1e-3) / 1e12, delivered * req_frac / (best_ms * 1e-3) / 1e12, best_bpc,
            best_bpc * req_frac, delivered / ctas / best_bpc / (best_ms * 1e-3) / 1e9);
        std::fflush(stdout);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    };
    const bool only5 = std::getenv("PROBE_ONLY_5") != nullptr;
    // 1. delivery cap by cluster shape (the engine's 3 x 64 KB ring, no consumer work)
    for (int src = 0; src < 2 && !only5; ++src)
        for (const V& v : vs) run(v, src, rings[0], 0);
    // 2. ring depth / granularity for the 1x4 shape, with the consumer holding
    //    each stage as long as the MMAs would: 15 clk/KB (FP4 iris: 960 clk per
    //    64 KB) and 23 clk/KB (int8 PPMM: 1488 clk per 64 KB); 0 = no hold
    for (int src = 0; src < 2 && !only5; ++src)
        for (uint32_t hold : {0u, 15u, 23u})
            for (const Ring& rg : rings) run(vs[2], src, rg, hold);
    // 3. copy granularity: the engine issues 2-D tensor copies of 128-row boxes
    //    (16 KB, or 4 KB per multicast quarter); here each share is cut into
    //    copies of `piece` bytes
    for (int src = 0; src < 2 && !only5; ++src)
        for (uint32_t hold : {0u, 15u, 23u})
            for (uint32_t piece : {16384u, 4096u, 1024u}) run(vs[2], src, rings[0], hold, piece);
    // 5. why does the mixed kernel's TMA-only leg deliver more? same ring and
    //    pieces in probe_kernel, one-CTA clusters
    if (std::getenv("PROBE_ONLY_5")) {
        for (int src : {0, 2})
            for (Ring rg : {Ring{2, 32768}, Ring{3, 32768}})
                for (uint32_t piece : {16384u, 32768u}) run(vs[0], src, rg, 0, piece);
    }
    // 4. mixed paths: TMA ring + cp.async warps on one SM (148 CTAs, no clusters)
    {
        const size_t msmem = 3 * 65536 + 1024 + 64;
        cudaFuncSetAttribute(mixed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(msmem));
        unsigned long long* mo = nullptr;
        cudaMalloc(&mo, sizeof(unsigned long long) * 3 * 1024);
        std::vector<unsigned long long> hm(3 * sms);
        for (uint32_t tma_on : {1u, 2u, 3u, 0u})
            for (uint32_t lw : {0u, 4u, 8u, 16u}) {
                if (!tma_on && lw == 0) continue;
                if (tma_on > 1 && lw > 0) continue;
                mixed_kernel<<<sms, 64 + 32 * 16, msmem>>>(b, b_bytes, tma_on, lw, 4000000LL, mo);
                mixed_kernel<<<sms, 64 + 32 * 16, msmem>>>(b, b_bytes, tma_on, lw, 4000000LL, mo);
                if (cudaDeviceSynchronize() != cudaSuccess) {
                    std::printf("{\"mixed\": \"error %s\"}\n", cudaGetErrorString(cudaGetLastError()));
                    break;
                }
                cudaMemcpy(hm.data(), mo, sizeof(unsigned long long) * 3 * sms, cudaMemcpyDeviceToHost);
                double tb = 0, lb = 0, cy = 0;
                for (int i = 0; i < sms; ++i) {
                    tb += hm[3 * i];
                    lb += hm[3 * i + 1];
                    cy += hm[3 * i + 2];
                }
                cy /= sms;
                std::printf("{\"mixed\": true, \"tma\": %u, \"lsu_warps\": %u, \"tma_B_per_clk_per_sm\": %.2f, "
                            "\"lsu_B_per_clk_per_sm\": %.2f, \"total_B_per_clk_per_sm\": %.2f}\n",
                            tma_on, lw, tb / sms / cy, lb / sms / cy, (tb + lb) / sms / cy);
                std::fflush(stdout);
            }
    }
    return 0;
}
