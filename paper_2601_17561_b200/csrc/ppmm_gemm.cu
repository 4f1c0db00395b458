// Persistent tcgen05 int8 GEMM with the fused mod-p^2 epilogue.
//
// Computes, for every (part g, prime i) of a batch,
//     out[g][i][n][m] = ( X0 Y0 + p (X0 Y1 + X1 Y0) ) mod p^2          (m < M, n < N)
// where X0/X1 are the centred digit planes of the database part (M x K,
// K-major) and Y0/Y1 those of the query (N x K, K-major). This is
// `gemm_mod_psq` (reference proj/src/modmat.cpp:143-160) with the three
// small_gemm calls (:147-149) fused into one pass over K and the int64
// recombination (:150-158) applied to the TMEM accumulators in registers,
// so no int32 partial ever reaches HBM.
//
// Execution model (sm_100a):
//   * a CTA pair owns a 256 x n_tile output tile (n_tile <= 256):
//     tcgen05.mma.cta_group::2.kind::i8 with M = 256, issued by one thread of
//     the leader CTA; TMEM holds acc1 = X0 Y0 in columns [0, 256) and
//     acc2 = X0 Y1 + X1 Y0 in [256, 512); X0 stays in the A collector for the
//     second product (collector::a fill / lastuse);
//   * warp 0 = TMA producer (both CTAs load their half of A and B),
//     warp 1 = MMA issuer (leader CTA) + TMEM owner, warps 2.. = epilogue
//     (kEpiWarps / 4 warps per TMEM lane quarter, interleaved over 16-column chunks);
//   * 3-stage smem ring of 128-byte K blocks, 128B-swizzled, mbarrier-paced;
//   * clusters of kPM x kPN pairs: the kPN pairs sharing an m-block receive
//     each DB tile by TMA multicast (loaded L2 evict-first when they are its
//     only reader), the kPM pairs sharing an n-tile each query tile; the
//     default 1x4 covers all of N = 992 so every DB tile leaves L2 once;
//   * persistent dynamic schedule: "units" (m-blocks x one n-chunk of one
//     (prime, part); prime-major, m fastest) come from one atomic counter
//     shared with a 1x1 filler launch on the SMs the clusters strand. A unit's
//     n-tiles run on a group of clusters at once whose TMA producers stay
//     within gate_lead K blocks of each other (bounded spin), so a DB tile is
//     re-read from L2 by its peers;
//   * epilogue: (acc1 + p (acc2 mod p)) mod p^2 with exact Barrett steps,
//     uint16 stores; optional per-(prime, part) completion counters (the e2e
//     pipeline starts each block's D2H from them) and mirror stores into peer
//     GPUs' buffers (the fused a-part exchange);
//   * kModeInner / kModeIrisMatch reuse the pipeline for two independent
//     products (iris inner products and mask overlaps), raw or scored.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "modarith.cuh"
#include "ppmm.h"
#include "sm100_ptx.cuh"

namespace irl {

namespace {

constexpr int kRowsPerCta = 128;   // M rows per CTA (256 per pair)
constexpr int kMaxTileN = 256;     // N columns per tile (pair-wide)
constexpr int kBlockK = 128;       // K bytes per pipeline stage (one 128B-swizzle row)
constexpr int kStages = 3;         // 3 x 64 KB ring (SW128 is the fast UMMA layout; a 7 x 32 KB
                                   // SW64 ring measured 30% slower)
constexpr int kUmmaK = 32;         // K per tcgen05.mma for 8-bit inputs
constexpr int kPlaneTileBytes = kRowsPerCta * kBlockK;          // 16 KB
constexpr int kStageBytes = 4 * kPlaneTileBytes;                // X0 X1 Y0 Y1
#ifndef IRL_A_REUSE
#define IRL_A_REUSE 1  // reuse X0 from the tensor core's A collector (tcgen05 collector::a)
#endif
#ifndef IRL_SPLIT_SLOTS
#define IRL_SPLIT_SLOTS 0  // 1: two-product modes use one 32 KB ring slot per product (6 slots; measured slower)
#endif
#ifndef IRL_EPI_WARPS
#define IRL_EPI_WARPS 16
#endif
constexpr int kEpiWarps = IRL_EPI_WARPS;  // multiple of 4: kEpiWarps / 4 warps per TMEM lane quarter
constexpr int kEpiGroups = kEpiWarps / 4;
constexpr int kNumThreads = 64 + 32 * kEpiWarps;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kAcc2Col = 256;
constexpr uint32_t kF4TileN = kF4TileCols;  // FP4 modes: accumulator columns 0..239 and 256..495
constexpr uint32_t kF4SfaCol = 240;  // unit scale factors (0x7F bytes) for A ...
constexpr uint32_t kF4SfbCol = 248;  // ... and B, in both CTAs' TMEM
constexpr size_t kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
constexpr uint32_t kGateLead = 48;                // max K blocks a pair may lead its group (swept: 6..96)
constexpr long long kGateSpinCycles = 200000;     // then proceed ungated (forward progress)
constexpr uint32_t kProgressWords = 1024;        // per-pair progress counters

struct __align__(64) GemmArgs {
    uint32_t M, N, K;
    uint32_t parts, nprimes;
    uint32_t m_blocks, n_blocks, units;
    uint32_t n_chunks, chunk_tiles;   // a unit covers chunk_tiles n-tiles; n_chunks of them span N
    uint32_t unit_mblocks;            // 256-row blocks per unit (the main launch's cluster_pm)
    uint32_t m_units;                 // units per (prime, part) = ceil(m_blocks / unit_mblocks)
    // group schedule (see group_of): G = clusters per full group
    uint32_t G, F, L, active_clusters;
    uint32_t mail_slots;              // per-group mailbox ring (units + 1 when the scratch allows, so a
                                      // member started late never finds its slot overwritten)
    uint32_t gate_lead;               // max K blocks a pair may lead its group (0: no gating)
    uint32_t a_evict_first;           // DB tiles read exactly once from L2 (G == 1): evict-first policy
    uint32_t b_evict_first;           // B is the streamed operand (PpmmLaunch::b_streamed): B evict-first, A evict-last
    uint32_t accumulate;
    uint32_t a_part_rows;             // plane rows between consecutive parts of A
    unsigned long long out_part;      // output elements between consecutive parts
    uint16_t* out;
    int32_t* out_i32[2];              // kMode == kModeInner: acc1 / acc2 as int32 [n][m] (nullable)
    IrisMatchOut iris;                // kMode == kModeIrisMatch
    uint16_t* mirror[kMaxMirrors];    // peer copies of part mirror_part's outputs (see PpmmLaunch)
    uint32_t n_mirror, mirror_part, mirror_parts;
    uint16_t* mc_mirror;              // multicast address of part mirror_part's copies (see PpmmLaunch)
    uint32_t* part_done;              // optional [nprimes][parts] count of (epilogue warp, tile) completions
    uint32_t* progress;               // [clusters] K blocks issued by each pair's leader producer
    uint32_t* counter;                // next unit to hand out (shared by the main and filler launches)
    unsigned long long* mailbox;      // [groups][mail_slots] ((seq+1) << 32 | unit) published per group
    unsigned long long* stats;        // optional [clusters][kStatSlots] diagnostics (see ppmm.h)
    ModConst mc[kMaxPrimesPerLaunch];
};

constexpr int kRing = 4;              // tile-descriptor ring (producer -> MMA / epilogue)
constexpr uint32_t kMinMail = 64;
constexpr uint64_t kSmallLaunchBlocks = 256;  // below this many (m-block, part, prime) units: plain pairs     // mailbox slots per group (at least; see GemmArgs::mail_slots)
constexpr uint32_t kEnd = 0xFFFFFFFFu;

// Diagnostics: wait on a barrier and add the cycles spent to *acc.
__device__ __forceinline__ void timed_wait(uint64_t* bar, uint32_t parity, bool on,
                                           unsigned long long& acc) {
    if (!on) {
        ptx::mbar_wait(bar, parity);
        return;
    }
    const long long t0 = clock64();
    ptx::mbar_wait(bar, parity);
    acc += static_cast<unsigned long long>(clock64() - t0);
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct TileCoord {
    uint32_t prime, part, m0, n0, n_size;
};

// A unit is `unit_mblocks` consecutive 256-row blocks x one n-chunk
// (chunk_tiles n-tiles) of one (prime, part). Units are ordered prime, part,
// n-chunk, m-block (fastest): the units in flight at once share one n-chunk
// of a prime's query planes, which stays L2-resident while the database
// streams through once per n-chunk. A tile is (unit, m-block within the unit,
// n-tile within the chunk). Tiles past N (padding of the last chunk) get
// n_size 32 and store nothing.
template <uint32_t kTileN = kMaxTileN, uint32_t kNAlign = 32>
__device__ __forceinline__ TileCoord decode(const GemmArgs& a, uint32_t unit, uint32_t mb_sub,
                                            uint32_t nb) {
    TileCoord t;
    const uint32_t mu = unit % a.m_units;
    uint32_t rest = unit / a.m_units;
    const uint32_t nc = rest % a.n_chunks;
    rest /= a.n_chunks;
    t.part = rest % a.parts;
    t.prime = rest / a.parts;
    t.m0 = (mu * a.unit_mblocks + mb_sub) * 2 * kRowsPerCta;
    t.n0 = (nc * a.chunk_tiles + nb) * kTileN;
    const uint32_t rem = a.N > t.n0 ? a.N - t.n0 : 1u;
    const uint32_t ns = rem < kTileN ? rem : kTileN;
    t.n_size = (ns + kNAlign - 1) & ~(kNAlign - 1);  // cta_group::2: kind::i8 N % 32, kind::mxf4 N % 16
    return t;
}

// Groups (cluster granularity): each cluster holds P CTA pairs. F full groups
// of Gc = G / P clusters split a unit's G = n_blocks n-tiles (pair p of group
// member c computes n-tile c*P + p of every unit the group takes, in
// lock-step); then L solo clusters that sweep a unit's n-tiles in G / P passes.
struct GroupInfo {
    uint32_t id, first, size, member;
    bool solo;
};
__device__ __forceinline__ GroupInfo group_of(const GemmArgs& a, uint32_t c) {
    GroupInfo g;
    if (c < a.F * a.G) {  // here a.G = clusters per full group
        g.id = c / a.G;
        g.first = g.id * a.G;
        g.size = a.G;
        g.member = c % a.G;
        g.solo = a.G == 1;
    } else {
        g.id = a.F + (c - a.F * a.G);
        g.first = c;
        g.size = 1;
        g.member = 0;
        g.solo = true;
    }
    return g;
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Cluster = kPM x kPN CTA pairs; pair index = pm * kPN + pn, CTA rank =
// 2 * pair + half. The kPN pairs with the same pm compute the same m-block
// (different n-tiles): each of their CTAs loads 1/kPN of its 128-row A block
// and multicasts it to the same-role CTAs of those pairs. Likewise the kPM
// pairs with the same pn share each B (query) tile. Every stage is released
// only when all pairs of the cluster have consumed it (commit multicast), so
// the cluster runs in lock-step over K.
template <int kPM, int kPN, int kMode>
__global__ void __launch_bounds__(kNumThreads, 1)
    ppmm_i8_sm100_kernel(const __grid_constant__ CUtensorMap tmap_a,
                         const __grid_constant__ CUtensorMap tmap_b,
                         const __grid_constant__ GemmArgs args) {
    constexpr uint32_t kPairs = kPM * kPN;
    constexpr int kCtas = 2 * kPairs;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    constexpr bool kF4 = kMode == kModeInnerF4 || kMode == kModeIrisMatchF4;
    constexpr bool kInner = kMode == kModeInner || kMode == kModeInnerF4;
    constexpr bool kMatch = kMode == kModeIrisMatch || kMode == kModeIrisMatchF4;
    // The modes with two independent products (acc1 = X0 Y0, acc2 = X1 Y1)
    // give each product of a K block its own ring slot (X_p, Y_p: 32 KB), so
    // the same 192 KB ring holds six slots and the MMAs hold only one sixth of
    // it while five slots are in flight (three 64 KB stages left two). The
    // psq products share X0 and Y0, so they keep whole-K-block stages.
    constexpr bool kSplitSlots = IRL_SPLIT_SLOTS && kMode != kModePsq;
    constexpr uint32_t kSlots = kSplitSlots ? 2 * kStages : kStages;
    constexpr uint32_t kSlotBytes = kSplitSlots ? kStageBytes / 2 : kStageBytes;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty_bar = full_bar + kSlots;
    uint64_t* tmem_full_bar = empty_bar + kSlots;
    uint64_t* tmem_empty_bar = tmem_full_bar + 1;
    uint64_t* ring_full = tmem_empty_bar + 1;
    uint64_t* ring_empty = ring_full + kRing;
    uint32_t* ring_tile = reinterpret_cast<uint32_t*>(ring_empty + kRing);  // [kRing][2]
    uint32_t* tmem_base_slot = ring_tile + 2 * kRing;

    constexpr uint32_t kTileN = kF4 ? kF4TileN : kMaxTileN;
    constexpr uint32_t kNAlign = kF4 ? 16u : 32u;
    const uint32_t warp = threadIdx.x / 32;
    const uint32_t lane = threadIdx.x % 32;
    const uint32_t rank = ptx::cluster_ctarank();
    const uint32_t pair = rank >> 1;          // pair within the cluster
    const uint32_t pm = pair / kPN, pn = pair % kPN;
    const uint32_t half_rank = rank & 1;      // CTA within the pair
    const bool leader = half_rank == 0;       // pair leader (issues the MMAs)
    const uint32_t cluster_id = blockIdx.x / kCtas;
    // The filler launch (same stream, programmatic stream serialization) may
    // start on the SMs this grid leaves free as soon as every CTA got here.
    ptx::griddep_launch_dependents();

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmap_a);
        ptx::prefetch_tmap(&tmap_b);
        for (uint32_t s = 0; s < kSlots; ++s) {
            ptx::mbar_init(&full_bar[s], 1);
            ptx::mbar_init(&empty_bar[s], kPairs);  // one commit per pair reading this stage
        }
        ptx::mbar_init(tmem_full_bar, 1);
        ptx::mbar_init(tmem_empty_bar, 2 * kEpiWarps);
        for (int s = 0; s < kRing; ++s) {
            ptx::mbar_init(&ring_full[s], 1);
            ptx::mbar_init(&ring_empty[s], (leader ? 1 : 0) + kEpiWarps);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 1) {
        ptx::tmem_alloc_pair(ptx::smem_u32(tmem_base_slot), kTmemCols);
    }
    if constexpr (kF4) {
        // every byte of the scale-factor columns = 2^0 (UE8M0 127): one
        // epilogue warp per TMEM lane quarter writes them after the alloc
        ptx::tc_fence_before();
        __syncthreads();
        ptx::tc_fence_after();
        if (warp >= 2 && warp < 6) {
            const uint32_t lb = *tmem_base_slot + (((warp % 4) * 32u) << 16);
            for (uint32_t c = kF4SfaCol; c < kAcc2Col; c += 4) ptx::tmem_st_32x32b_x4(lb + c, 0x7F7F7F7Fu);
            for (uint32_t c = kAcc2Col + kF4TileN; c < kTmemCols; c += 4) ptx::tmem_st_32x32b_x4(lb + c, 0x7F7F7F7Fu);
            ptx::tmem_st_wait();
        }
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_base_slot;

    if (warp == 0) {
        // ---------------- TMA producer + scheduler (both CTAs) ----------------
        if (lane == 0) {
            const uint32_t num_kb = (args.K + kBlockK - 1) / kBlockK;
            const GroupInfo grp = group_of(args, cluster_id);
            const bool gate = rank == 0 && grp.size > 1 && args.gate_lead > 0;
            const uint32_t lead = args.gate_lead;
            const bool writer = rank == 0 && grp.member == 0;  // takes units for the group
            unsigned long long* mbox = args.mailbox + static_cast<size_t>(grp.id) * args.mail_slots;
            const uint32_t tiles_per_unit = grp.solo ? args.chunk_tiles / kPN : 1;
            const uint32_t m_passes = args.unit_mblocks / kPM;
            uint32_t issued = 0;  // cumulative K blocks (comparable across the group)
            uint32_t seen = 0;    // last observed minimum of the peers' counters
            uint32_t stage = 0, phase = 0, tile_i = 0;
            const bool diag = args.stats != nullptr && leader;
            unsigned long long w_empty = 0, w_gate = 0;

            auto grab = [&]() -> uint32_t {
                if (grp.solo && grp.size == 1 && args.G > 1) {
                    // a solo cluster needs G tile-times per unit: stop before the
                    // tail so it never finishes last
                    if (ptx::ld_relaxed_gpu(args.counter) + args.G * args.F >= args.units) return kEnd;
                }
                const uint32_t u = atomicAdd(args.counter, 1u);
                return u < args.units ? u : kEnd;
            };
            auto publish = [&](uint32_t seq, uint32_t u) {
                // tag = seq + 1 so the zeroed mailbox never matches
                st_relaxed_u64(mbox + seq % args.mail_slots,
                               (static_cast<unsigned long long>(seq + 1) << 32) | u);
            };
            auto push_tile = [&](uint32_t u, uint32_t mb_sub, uint32_t nb) {
                const uint32_t slot = tile_i % kRing;
                ptx::mbar_wait(&ring_empty[slot], ((tile_i / kRing) & 1) ^ 1);
                ring_tile[2 * slot] = u;
                ring_tile[2 * slot + 1] = nb | (mb_sub << 16);
                asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                                 ptx::smem_u32(&ring_full[slot]))
                             : "memory");
                ++tile_i;
            };

            uint32_t u_next = 0;
            if (writer) {
                u_next = grab();
                publish(0, u_next);
            }
            for (uint32_t seq = 0;; ++seq) {
                uint32_t u;
                if (writer) {
                    u = u_next;
                    if (u != kEnd) {
                        u_next = grab();  // prefetch: members never wait at a unit boundary
                        publish(seq + 1, u_next);
                    }
                } else {
                    unsigned long long v;
                    while (((v = ld_relaxed_u64(mbox + seq % args.mail_slots)) >> 32) != seq + 1) {
                        __nanosleep(64);
                    }
                    u = static_cast<uint32_t>(v);
                }
                if (u == kEnd) {
                    push_tile(kEnd, 0, 0);
                    break;
                }
                for (uint32_t t = 0; t < m_passes * tiles_per_unit; ++t) {
                    const uint32_t r = t % tiles_per_unit;
                    const uint32_t mb_sub = (t / tiles_per_unit) * kPM + pm;
                    const uint32_t nb = (grp.solo ? r : grp.member) * kPN + pn;
                    push_tile(u, mb_sub, nb);
                    const TileCoord tc = decode<kTileN, kNAlign>(args, u, mb_sub, nb);
                    const uint32_t a_row0 = tc.part * args.a_part_rows + tc.prime * 2 * args.M +
                                            tc.m0 + half_rank * kRowsPerCta;
                    const uint32_t half_n = tc.n_size / 2;
                    const uint32_t b_row0 = (tc.prime * 2) * args.N + tc.n0 + half_rank * half_n;
                    // one plane tile of A (this CTA's 128 DB rows; with kPN > 1 a 1/kPN
                    // share, multicast to the same-role CTAs of the pairs sharing pm)
                    auto load_a = [&](uint32_t dst, uint32_t row, uint32_t bar, int32_t k0) {
                        if constexpr (kPN == 1) {
                            if (args.b_evict_first)
                                ptx::tma_load_2d_pair_hint(dst, &tmap_a, bar, k0, static_cast<int32_t>(row),
                                                           ptx::kL2EvictLast);
                            else
                                ptx::tma_load_2d_pair(dst, &tmap_a, bar, k0, static_cast<int32_t>(row));
                        } else {
                            constexpr uint32_t kSubA = kRowsPerCta / kPN;
                            uint16_t mask = 0;
#pragma unroll
                            for (uint32_t j = 0; j < kPN; ++j) mask |= 1u << (2 * (pm * kPN + j) + half_rank);
                            const uint32_t sub = pn * kSubA * kBlockK;
                            if (args.a_evict_first)
                                ptx::tma_load_2d_pair_mcast_hint(dst + sub, &tmap_a, bar, k0,
                                                                 static_cast<int32_t>(row + pn * kSubA), mask,
                                                                 ptx::kL2EvictFirst);
                            else
                                ptx::tma_load_2d_pair_mcast(dst + sub, &tmap_a, bar, k0,
                                                            static_cast<int32_t>(row + pn * kSubA), mask);
                        }
                    };
                    // one plane tile of B (this CTA's half of the n-tile; with kPM > 1
                    // a 1/kPM share, multicast to the pairs sharing pn)
                    auto load_b = [&](uint32_t dst, uint32_t row, uint32_t bar, int32_t k0) {
                        if constexpr (kPM == 1) {
                            ptx::tma_load_2d_pair_hint(dst, &tmap_b, bar, k0, static_cast<int32_t>(row),
                                                       ptx::kL2EvictLast);
                        } else {
                            constexpr uint32_t kSubB = kRowsPerCta / kPM;
                            uint16_t mask = 0;
#pragma unroll
                            for (uint32_t j = 0; j < kPM; ++j) mask |= 1u << (2 * (j * kPN + pn) + half_rank);
                            const uint32_t sub = pm * kSubB * kBlockK;
                            if (args.b_evict_first)
                                ptx::tma_load_2d_pair_mcast_hint(dst + sub, &tmap_b, bar, k0,
                                                                 static_cast<int32_t>(row + pm * kSubB), mask,
                                                                 ptx::kL2EvictFirst);
                            else
                                ptx::tma_load_2d_pair_mcast(dst + sub, &tmap_b, bar, k0,
                                                            static_cast<int32_t>(row + pm * kSubB), mask);
                        }
                    };
                    for (uint32_t kb = 0; kb < num_kb; ++kb, ++issued) {
#pragma unroll
                        for (uint32_t prod = 0; prod < kSlots / kStages; ++prod) {
                            timed_wait(&empty_bar[stage], phase ^ 1, diag, w_empty);
                            if (prod == 0 && gate && issued > seen + lead) {
                                // Stay within kGateLead K blocks of the slowest group peer.
                                // `seen` caches the last observed minimum, so the L2
                                // round trip is paid about once per kGateLead blocks.
                                const long long t0 = clock64();
                                for (;;) {
                                    uint32_t lo = 0xFFFFFFFFu;
                                    for (uint32_t p = grp.first; p < grp.first + grp.size; ++p)
                                        if (p != cluster_id)
                                            lo = min(lo, ptx::ld_relaxed_gpu(args.progress + p));
                                    seen = lo;
                                    if (lo + lead >= issued) break;
                                    if (clock64() - t0 > kGateSpinCycles) {
                                        seen = issued;  // give up for kGateLead blocks (forward progress)
                                        break;
                                    }
                                    __nanosleep(32);
                                }
                                if (diag) w_gate += static_cast<unsigned long long>(clock64() - t0);
                            }
                            // completion bytes land on the pair leader's barrier
                            const uint32_t leader_full = ptx::smem_u32(&full_bar[stage]) & 0xFEFFFFFFu;
                            if (leader) ptx::mbar_arrive_expect_tx(&full_bar[stage], 2 * kSlotBytes);
                            const uint32_t st = ptx::smem_u32(smem + stage * kSlotBytes);
                            const int32_t k0 = static_cast<int32_t>(kb * kBlockK);
                            if constexpr (kSplitSlots) {
                                // slot = product `prod` of this K block: X_prod, then Y_prod
                                load_a(st, a_row0 + prod * args.M, leader_full, k0);
                                load_b(st + kPlaneTileBytes, b_row0 + prod * args.N, leader_full, k0);
                            } else {
                                // stage = X0 X1 Y0 Y1 of this K block
                                load_a(st, a_row0, leader_full, k0);
                                load_a(st + kPlaneTileBytes, a_row0 + args.M, leader_full, k0);
                                load_b(st + 2 * kPlaneTileBytes, b_row0, leader_full, k0);
                                load_b(st + 3 * kPlaneTileBytes, b_row0 + args.N, leader_full, k0);
                            }
                            if (++stage == kSlots) {
                                stage = 0;
                                phase ^= 1;
                            }
                        }
                        if (gate) ptx::st_relaxed_gpu(args.progress + cluster_id, issued + 1);
                    }
                }
            }
            if (diag) {
                unsigned long long* st = args.stats + (blockIdx.x >> 1) * kStatSlots;
                st[0] = w_empty;
                st[1] = w_gate;
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (leader CTA only) ----------------
        if (leader && lane == 0) {
            const uint32_t num_kb = (args.K + kBlockK - 1) / kBlockK;
            const uint32_t acc1 = tmem_base;
            const uint32_t acc2 = tmem_base + kAcc2Col;
            uint32_t stage = 0, phase = 0;
            const bool diag = args.stats != nullptr;
            unsigned long long w_full = 0, w_tmem = 0;
            const long long c_start = clock64();
            const unsigned long long g_start = diag ? globaltimer() : 0;
            uint32_t j = 0;
            for (;; ++j) {
                const uint32_t slot = j % kRing;
                ptx::mbar_wait(&ring_full[slot], (j / kRing) & 1);
                const uint32_t u = ring_tile[2 * slot], nbm = ring_tile[2 * slot + 1];
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                                 ptx::smem_u32(&ring_empty[slot]))
                             : "memory");
                if (u == kEnd) break;
                const TileCoord tc = decode<kTileN, kNAlign>(args, u, nbm >> 16, nbm & 0xFFFFu);
                const uint32_t idesc = kF4 ? ptx::idesc_mxf4(2 * kRowsPerCta, tc.n_size)
                                           : ptx::idesc_i8(2 * kRowsPerCta, tc.n_size);
                // Wait until the epilogue of the previous tile drained TMEM.
                timed_wait(tmem_empty_bar, (j & 1) ^ 1, diag, w_tmem);
                ptx::tc_fence_after();
                for (uint32_t kb = 0; kb < num_kb; ++kb) {
                    if constexpr (kSplitSlots) {
                        // two independent products, one slot each: acc1 = X0 Y0, acc2 = X1 Y1
#pragma unroll
                        for (uint32_t prod = 0; prod < 2; ++prod) {
                            timed_wait(&full_bar[stage], phase, diag, w_full);
                            ptx::tc_fence_after();
                            const uint32_t st = ptx::smem_u32(smem + stage * kSlotBytes);
                            const uint32_t acc = prod ? acc2 : acc1;
#pragma unroll
                            for (int k = 0; k < kBlockK / kUmmaK; ++k) {
                                const uint32_t koff = k * kUmmaK;
                                const uint64_t dx = ptx::smem_desc_k_sw128(st + koff);
                                const uint64_t dy = ptx::smem_desc_k_sw128(st + kPlaneTileBytes + koff);
                                const uint32_t accum = (kb | k) != 0;
                                if constexpr (kF4)  // packed e2m1 operands, 64 k per 32 B
                                    ptx::mma_mxf4_pair(acc, dx, dy, idesc, accum, tmem_base + kF4SfaCol,
                                                       tmem_base + kF4SfbCol);
                                else
                                    ptx::mma_i8_pair(acc, dx, dy, idesc, accum);
                            }
                            ptx::mma_commit_pair(&empty_bar[stage], static_cast<uint16_t>((1u << kCtas) - 1));
                            if (++stage == kSlots) {
                                stage = 0;
                                phase ^= 1;
                            }
                        }
                        continue;
                    }
                    timed_wait(&full_bar[stage], phase, diag, w_full);
                    ptx::tc_fence_after();
                    const uint32_t st = ptx::smem_u32(smem + stage * kStageBytes);
#pragma unroll
                    for (int k = 0; k < kBlockK / kUmmaK; ++k) {
                        const uint32_t koff = k * kUmmaK;
                        const uint64_t dx0 = ptx::smem_desc_k_sw128(st + koff);
                        const uint64_t dx1 = ptx::smem_desc_k_sw128(st + kPlaneTileBytes + koff);
                        const uint64_t dy0 =
                            ptx::smem_desc_k_sw128(st + 2 * kPlaneTileBytes + koff);
                        const uint64_t dy1 =
                            ptx::smem_desc_k_sw128(st + 3 * kPlaneTileBytes + koff);
                        const uint32_t accum = (kb | k) != 0;
                        if constexpr (kF4) {  // IRL_SPLIT_SLOTS=0: both products from one stage
                            ptx::mma_mxf4_pair(acc1, dx0, dy0, idesc, accum, tmem_base + kF4SfaCol,
                                               tmem_base + kF4SfbCol);
                            ptx::mma_mxf4_pair(acc2, dx1, dy1, idesc, accum, tmem_base + kF4SfaCol,
                                               tmem_base + kF4SfbCol);
                            continue;
                        } else if constexpr (kMode != kModePsq) {
                            ptx::mma_i8_pair(acc1, dx0, dy0, idesc, accum);
                            ptx::mma_i8_pair(acc2, dx1, dy1, idesc, accum);
                            continue;
                        }
#if IRL_A_REUSE
                        // X0 stays in the A collector for the second product
                        ptx::mma_i8_pair_ca<ptx::CollectorA::kFill>(acc1, dx0, dy0, idesc, accum);     // X0 Y0
                        ptx::mma_i8_pair_ca<ptx::CollectorA::kLastUse>(acc2, dx0, dy1, idesc, accum);  // X0 Y1
#else
                        ptx::mma_i8_pair(acc1, dx0, dy0, idesc, accum);  // X0 Y0
                        ptx::mma_i8_pair(acc2, dx0, dy1, idesc, accum);  // X0 Y1
#endif
                        ptx::mma_i8_pair(acc2, dx1, dy0, idesc, 1u);     // + X1 Y0
                    }
                    // release the stage in every CTA that wrote into it
                    ptx::mma_commit_pair(&empty_bar[stage], static_cast<uint16_t>((1u << kCtas) - 1));
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::mma_commit_pair(tmem_full_bar, static_cast<uint16_t>(0x3u << (2 * pair)));
            }
            if (diag) {
                // wait for the last tile's drain so the end stamps cover it
                if (j > 0) timed_wait(tmem_empty_bar, (j & 1) ^ 1, false, w_tmem);
                unsigned long long* st = args.stats + (blockIdx.x >> 1) * kStatSlots;
                st[2] = w_full;
                st[3] = w_tmem;
                st[4] = static_cast<unsigned long long>(clock64() - c_start);
                st[7] = g_start;
                st[8] = globaltimer();
                st[11] = j;
                unsigned smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                st[12] = smid;
            }
        }
    } else {
        // ---------------- Epilogue (both CTAs, 8 warps) ----------------
        const uint32_t quarter = warp % 4;        // TMEM lane quarter this warp may access
        const uint32_t cgrp = (warp - 2) / 4;     // which 16-column chunks of the tile (interleaved)
        const uint32_t leader_tmem_empty = ptx::mapa_shared(ptx::smem_u32(tmem_empty_bar), rank & ~1u);
        const bool diag = args.stats != nullptr && leader && warp == 2 && lane == 0;
        unsigned long long w_epi = 0, busy_epi = 0;
        for (uint32_t j = 0;; ++j) {
            const uint32_t slot = j % kRing;
            ptx::mbar_wait(&ring_full[slot], (j / kRing) & 1);
            const uint32_t u = ring_tile[2 * slot], nbm = ring_tile[2 * slot + 1];
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                                 ptx::smem_u32(&ring_empty[slot]))
                             : "memory");
            if (u == kEnd) break;
            const TileCoord tc = decode<kTileN, kNAlign>(args, u, nbm >> 16, nbm & 0xFFFFu);
            const ModConst mc = args.mc[tc.prime];
            timed_wait(tmem_full_bar, j & 1, diag, w_epi);
            const long long e0 = clock64();
            ptx::tc_fence_after();
            const uint32_t row = half_rank * kRowsPerCta + quarter * 32 + lane;
            const uint32_t m = tc.m0 + row;
            const bool row_ok = m < args.M;
            uint16_t* out = args.out + tc.part * args.out_part +
                            static_cast<size_t>(tc.prime) * args.N * args.M +
                            m;
            // parts [mirror_part, mirror_part + mirror_parts) are mirrored; the
            // peers' buffers hold them back to back in the output layout
            const bool mirror_tile = (args.n_mirror != 0 || args.mc_mirror != nullptr) &&
                                     tc.part - args.mirror_part < args.mirror_parts;
            const bool mc_tile = args.mc_mirror != nullptr && mirror_tile;
            const uint32_t lane_base = tmem_base + ((quarter * 32u) << 16);
            for (uint32_t c = cgrp * 16; c < tc.n_size; c += 16 * kEpiGroups) {
                uint32_t a1[16], a2[16];
                ptx::tmem_ld_32x32b_x16(lane_base + c, a1);
                ptx::tmem_ld_32x32b_x16(lane_base + kAcc2Col + c, a2);
                ptx::tmem_ld_wait();
                if constexpr (kMatch) {
                    // Screen first: almost every (column, template) score misses the
                    // interval by far. A miss is decided exactly from the products
                    // (inner < lo_out * ov or inner > hi_out * ov, ov > 0; see the
                    // launcher's margins), with no division. Everything else (a
                    // possible match, an empty overlap, and every element when the
                    // scores are requested) takes the exact path below, once per
                    // warp per chunk that has one.
                    const IrisMatchOut& io = args.iris;
                    uint32_t ev = 0;
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        float fi, fo;  // exact integers (|value| <= d < 2^24)
                        if constexpr (kF4) {
                            fi = __uint_as_float(a1[jj]);
                            fo = __uint_as_float(a2[jj]);
                        } else {
                            fi = static_cast<float>(static_cast<int32_t>(a1[jj]));
                            fo = static_cast<float>(static_cast<int32_t>(a2[jj]));
                        }
                        const bool miss = fo > 0.0f && (fi < io.lo_out * fo || fi > io.hi_out * fo);
                        if (!miss || io.scores) ev |= 1u << jj;
                    }
                    if (!row_ok) ev = 0;
                    if (tc.n0 + c + 16 > args.N) ev &= (1u << (args.N > tc.n0 + c ? args.N - tc.n0 - c : 0u)) - 1u;
                    if (!__any_sync(0xFFFFFFFFu, ev != 0)) continue;
                    if (io.query_rows) {
                        // this thread's row is query column m (one eye, one
                        // rotation); its 16 columns are templates. Events are
                        // rare: each thread folds its own into the per-eye minima.
                        const uint32_t gcol = m + io.col0;
                        const uint32_t eye = gcol / io.rho, rot = gcol % io.rho;
                        uint32_t cm = 0xFFFFFFFFu, cz = 0xFFFFFFFFu;
                        for (int jj = 0; jj < 16; ++jj) {
                            if (!((ev >> jj) & 1u)) continue;
                            const uint32_t t = tc.n0 + c + jj;
                            int32_t inner, ov;
                            if constexpr (kF4) {
                                inner = __float2int_rn(__uint_as_float(a1[jj]));
                                ov = __float2int_rn(__uint_as_float(a2[jj]));
                            } else {
                                inner = static_cast<int32_t>(a1[jj]);
                                ov = static_cast<int32_t>(a2[jj]);
                            }
                            const uint32_t lin = rot * args.N + t;
                            double* sc_out = io.scores ? io.scores + static_cast<size_t>(gcol) * args.N + t : nullptr;
                            if (ov == 0) {
                                cz = min(cz, lin);
                                if (sc_out) *sc_out = __longlong_as_double(0x7FF8000000000000ll);
                                continue;
                            }
                            bool hit;  // iris_core.cpp:58; the screens as below
                            const float q = __fdividef(static_cast<float>(inner), static_cast<float>(ov));
                            if (!sc_out && q >= io.lo_in && q <= io.hi_in) {
                                hit = true;
                            } else if (!sc_out && (q < io.lo_out || q > io.hi_out)) {
                                hit = false;
                            } else {
                                const double sc = __ddiv_rn(static_cast<double>(inner), static_cast<double>(ov));
                                hit = sc >= io.lo && sc <= io.hi;  // Interval::contains
                                if (sc_out) *sc_out = sc;
                            }
                            if (hit) {
                                cm = min(cm, lin);
                                if (io.bits) io.bits[static_cast<size_t>(eye) * args.N + t] = 1;
                            }
                        }
                        if (io.first) {
                            if (cm != 0xFFFFFFFFu) atomicMin(io.first + 2 * eye, cm);
                            if (cz != 0xFFFFFFFFu) atomicMin(io.first + 2 * eye + 1, cz);
                        }
                        continue;
                    }
                    for (int jj = 0; jj < 16; ++jj) {
                        const uint32_t col = tc.n0 + c + jj;
                        if (col >= args.N) break;  // uniform across the warp
                        const uint32_t gcol = col + io.col0;  // global query column
                        const uint32_t eye = gcol / io.rho, rot = gcol % io.rho;
                        int32_t inner, ov;
                        if constexpr (kF4) {
                            inner = __float2int_rn(__uint_as_float(a1[jj]));
                            ov = __float2int_rn(__uint_as_float(a2[jj]));
                        } else {
                            inner = static_cast<int32_t>(a1[jj]);
                            ov = static_cast<int32_t>(a2[jj]);
                        }
                        uint32_t cm = 0xFFFFFFFFu, cz = 0xFFFFFFFFu;
                        if ((ev >> jj) & 1u) {
                            const uint32_t lin = rot * args.M + m;
                            if (ov == 0) {
                                cz = lin;
                                if (io.scores)
                                    io.scores[static_cast<size_t>(gcol) * args.M + m] =
                                        __longlong_as_double(0x7FF8000000000000ll);
                            } else {
                                // iris_core.cpp:58, IEEE double division. A float
                                // quotient (|error| < 1e-6) settles every score
                                // farther than 1e-5 from a bound; the exact
                                // division runs only near the bounds or when the
                                // scores are requested.
                                bool hit;
                                const float q = __fdividef(static_cast<float>(inner), static_cast<float>(ov));
                                if (!io.scores && q >= io.lo_in && q <= io.hi_in) {
                                    hit = true;
                                } else if (!io.scores && (q < io.lo_out || q > io.hi_out)) {
                                    hit = false;
                                } else {
                                    const double sc = __ddiv_rn(static_cast<double>(inner), static_cast<double>(ov));
                                    hit = sc >= io.lo && sc <= io.hi;  // Interval::contains
                                    if (io.scores) io.scores[static_cast<size_t>(gcol) * args.M + m] = sc;
                                }
                                if (hit) {
                                    cm = lin;
                                    if (io.bits) io.bits[static_cast<size_t>(eye) * args.M + m] = 1;
                                }
                            }
                        }
                        // events (a match, an empty overlap) are rare: vote first
                        if (__any_sync(0xFFFFFFFFu, (cm & cz) != 0xFFFFFFFFu) && io.first) {
                            cm = __reduce_min_sync(0xFFFFFFFFu, cm);
                            cz = __reduce_min_sync(0xFFFFFFFFu, cz);
                            if (lane == 0) {
                                if (cm != 0xFFFFFFFFu) atomicMin(io.first + 2 * eye, cm);
                                if (cz != 0xFFFFFFFFu) atomicMin(io.first + 2 * eye + 1, cz);
                            }
                        }
                    }
                    continue;
                }
                if constexpr (kF4) {  // FP32 accumulators of exact integers
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        a1[jj] = static_cast<uint32_t>(__float2int_rn(__uint_as_float(a1[jj])));
                        a2[jj] = static_cast<uint32_t>(__float2int_rn(__uint_as_float(a2[jj])));
                    }
                }
                if (kMode == kModePsq && mc_tile) {
                    // multicast mirror: the whole warp takes part (lanes past M
                    // compute but do not store); even lanes store rows (m, m+1)
                    // as one 32-bit multimem.st, which the switch replicates
                    uint16_t* dst = out + static_cast<size_t>(tc.n0 + c) * args.M;
                    const size_t moff = static_cast<size_t>(tc.part - args.mirror_part) * args.out_part +
                                        static_cast<size_t>(tc.prime) * args.N * args.M +
                                        static_cast<size_t>(tc.n0 + c) * args.M + m;
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        if (tc.n0 + c + jj >= args.N) continue;  // uniform across the warp
                        uint32_t v = combine_psq_fast(static_cast<int32_t>(a1[jj]), static_cast<int32_t>(a2[jj]),
                                                      mc.p, mc.m, mc.magic_p, mc.magic_m, mc.c_p, mc.c_m);
                        uint16_t* d = dst + static_cast<size_t>(jj) * args.M;
                        if (row_ok) {
                            if (args.accumulate) {
                                v += *d;
                                v = min(v, v - mc.m);
                            }
                            *d = static_cast<uint16_t>(v);
                            for (uint32_t mi = 0; mi < args.n_mirror; ++mi)
                                args.mirror[mi][moff + static_cast<size_t>(jj) * args.M] = static_cast<uint16_t>(v);
                        }
                        const uint32_t hi = __shfl_down_sync(0xFFFFFFFFu, v, 1);
                        if (row_ok && (lane & 1u) == 0)
                            ptx::multimem_st_b32(args.mc_mirror + moff + static_cast<size_t>(jj) * args.M,
                                                 (v & 0xFFFFu) | (hi << 16));
                    }
                    __threadfence_system();
                    continue;
                }
                if (!row_ok) continue;
                if constexpr (kInner) {
                    if (args.iris.query_rows) {
                        // outputs [M][N] (query column m, template n): 16
                        // consecutive templates per thread, as 16-byte stores
                        // when the row and chunk are aligned and in range
                        const uint32_t n = tc.n0 + c;
                        const size_t o = static_cast<size_t>(m) * args.N + n;
                        const bool vec = n + 16 <= args.N && (args.N & 3u) == 0;
                        // (the accumulator arrays are passed by reference and
                        // indexed with constants, so they stay in registers)
                        auto store_row = [&](int32_t* dst, const uint32_t (&v)[16]) {
                            if (!dst) return;
                            if (vec) {
                                int4* d4 = reinterpret_cast<int4*>(dst + o);
#pragma unroll
                                for (int q = 0; q < 4; ++q)
                                    d4[q] = make_int4(static_cast<int32_t>(v[4 * q]), static_cast<int32_t>(v[4 * q + 1]),
                                                      static_cast<int32_t>(v[4 * q + 2]), static_cast<int32_t>(v[4 * q + 3]));
                            } else {
#pragma unroll
                                for (int jj = 0; jj < 16; ++jj)
                                    if (n + jj < args.N) dst[o + jj] = static_cast<int32_t>(v[jj]);
                            }
                        };
                        store_row(args.out_i32[0], a1);
                        store_row(args.out_i32[1], a2);
                        continue;
                    }
                    const size_t base = tc.part * args.out_part + static_cast<size_t>(tc.prime) * args.N * args.M +
                                        static_cast<size_t>(tc.n0 + c) * args.M + m;
                    for (int jj = 0; jj < 16; ++jj) {
                        if (tc.n0 + c + jj >= args.N) break;
                        const size_t o = base + static_cast<size_t>(jj) * args.M;
                        if (args.out_i32[0]) args.out_i32[0][o] = static_cast<int32_t>(a1[jj]);
                        if (args.out_i32[1]) args.out_i32[1][o] = static_cast<int32_t>(a2[jj]);
                    }
                    continue;
                }
                uint16_t* dst = out + static_cast<size_t>(tc.n0 + c) * args.M;
                // offset of this chunk inside its part (same in the peers' mirrors)
                const size_t moff = static_cast<size_t>(tc.part - args.mirror_part) * args.out_part +
                                    static_cast<size_t>(tc.prime) * args.N * args.M +
                                    static_cast<size_t>(tc.n0 + c) * args.M + m;
                if (!args.accumulate && tc.n0 + c + 16 <= args.N) {
                    // fast path: whole 16-column chunk in range, overwrite
                    uint16_t vals[16];
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        vals[jj] = static_cast<uint16_t>(
                            combine_psq_fast(static_cast<int32_t>(a1[jj]), static_cast<int32_t>(a2[jj]),
                                             mc.p, mc.m, mc.magic_p, mc.magic_m, mc.c_p, mc.c_m));
                        dst[static_cast<size_t>(jj) * args.M] = vals[jj];
                    }
                    if (mirror_tile) {
                        for (uint32_t mi = 0; mi < args.n_mirror; ++mi) {
                            uint16_t* md = args.mirror[mi] + moff;
#pragma unroll
                            for (int jj = 0; jj < 16; ++jj) md[static_cast<size_t>(jj) * args.M] = vals[jj];
                        }
                    }
                } else {
                    for (int jj = 0; jj < 16; ++jj) {
                        if (tc.n0 + c + jj >= args.N) break;
                        uint32_t v = combine_psq_fast(static_cast<int32_t>(a1[jj]),
                                                      static_cast<int32_t>(a2[jj]), mc.p, mc.m,
                                                      mc.magic_p, mc.magic_m, mc.c_p, mc.c_m);
                        uint16_t* d = dst + static_cast<size_t>(jj) * args.M;
                        if (args.accumulate) {
                            v += *d;
                            v = min(v, v - mc.m);
                        }
                        *d = static_cast<uint16_t>(v);
                        if (mirror_tile)
                            for (uint32_t mi = 0; mi < args.n_mirror; ++mi)
                                args.mirror[mi][moff + static_cast<size_t>(jj) * args.M] = static_cast<uint16_t>(v);
                    }
                }
            }
            if (mirror_tile) __threadfence_system();  // peer stores performed before the tile is released
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(leader_tmem_empty);
            if (args.part_done) {
                // per-part completion count (stream memory ops start that
                // part's D2H as soon as all its tiles are stored)
                __threadfence();
                __syncwarp();
                if (lane == 0) atomicAdd(args.part_done + tc.prime * args.parts + tc.part, 1u);
            }
            if (diag) busy_epi += static_cast<unsigned long long>(clock64() - e0);
        }
        if (diag) {
            unsigned long long* st = args.stats + (blockIdx.x >> 1) * kStatSlots;
            st[5] = w_epi;
            st[6] = busy_epi;
        }
    }

    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_pair(tmem_base, kTmemCols);
    }
    // A filler grid ends only after the main grid it overlapped: the stream's
    // next operation waits for the filler, so it then also follows the main
    // grid (no-op in the main grid, which is an ordinary launch).
    ptx::griddep_wait();
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    return fn;
}

bool make_plane_map(CUtensorMap* map, const void* base, uint64_t k, uint64_t rows, uint64_t ldk,
                    uint32_t box_rows) {
    const cuuint64_t dims[2] = {k, rows};
    const cuuint64_t strides[1] = {ldk};
    const cuuint32_t box[2] = {kBlockK, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return get_encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Kernel variants by cluster shape (pairs along M x pairs along N).
struct Shape {
    int pm, pn;
    int ctas() const { return 2 * pm * pn; }
};
using KernelFn = void (*)(CUtensorMap, CUtensorMap, GemmArgs);
constexpr Shape kShapes[] = {{1, 1}, {1, 2}, {1, 4}, {2, 2}, {2, 4}, {1, 8}, {4, 1}};
constexpr int kShape4x1 = 6;  // the FP4 iris match with the query on M (IrisMatchOut::query_rows)
constexpr int kNumShapes = sizeof(kShapes) / sizeof(kShapes[0]);

int shape_index(int pm, int pn) {
    for (int i = 0; i < kNumShapes; ++i)
        if (kShapes[i].pm == pm && kShapes[i].pn == pn) return i;
    return -1;
}

KernelFn kernel_for(int si, int mode = kModePsq) {
    if (mode == kModeInner) {
        switch (si) {
            case 0: return ppmm_i8_sm100_kernel<1, 1, kModeInner>;
            case 2: return ppmm_i8_sm100_kernel<1, 4, kModeInner>;
        }
        return nullptr;
    }
    if (mode == kModeInnerF4) {
        switch (si) {
            case 0: return ppmm_i8_sm100_kernel<1, 1, kModeInnerF4>;
            case 2: return ppmm_i8_sm100_kernel<1, 4, kModeInnerF4>;
            case kShape4x1: return ppmm_i8_sm100_kernel<4, 1, kModeInnerF4>;
            default: return nullptr;
        }
    }
    if (mode == kModeIrisMatchF4) {
        switch (si) {
            case 0: return ppmm_i8_sm100_kernel<1, 1, kModeIrisMatchF4>;
            case 2: return ppmm_i8_sm100_kernel<1, 4, kModeIrisMatchF4>;
            case kShape4x1: return ppmm_i8_sm100_kernel<4, 1, kModeIrisMatchF4>;
            default: return nullptr;
        }
    }
    if (mode == kModeIrisMatch) {
        switch (si) {
            case 0: return ppmm_i8_sm100_kernel<1, 1, kModeIrisMatch>;
            case 2: return ppmm_i8_sm100_kernel<1, 4, kModeIrisMatch>;
        }
        return nullptr;
    }
    switch (si) {
        case 0: return ppmm_i8_sm100_kernel<1, 1, kModePsq>;
        case 1: return ppmm_i8_sm100_kernel<1, 2, kModePsq>;
        case 2: return ppmm_i8_sm100_kernel<1, 4, kModePsq>;
        case 3: return ppmm_i8_sm100_kernel<2, 2, kModePsq>;
        case 4: return ppmm_i8_sm100_kernel<2, 4, kModePsq>;
        case 5: return ppmm_i8_sm100_kernel<1, 8, kModePsq>;
    }
    return nullptr;
}

// Co-resident clusters of a shape with this kernel's footprint (cached per device).
uint32_t max_active_clusters(int si, int dev, int mode = kModePsq) {
    static std::mutex mu;
    static int cache[64][kNumShapes];
    static bool init = false;
    std::lock_guard<std::mutex> lk(mu);
    if (!init) {
        for (auto& c : cache)
            for (int& v : c) v = -1;
        init = true;
    }
    if (dev < 0 || dev >= 64 || si < 0) return 0;
    if (cache[dev][si] >= 0) return static_cast<uint32_t>(cache[dev][si]);
    const int ctas = kShapes[si].ctas();
    KernelFn kfn = kernel_for(si);  // every mode has the same footprint; psq has the most shapes
    if (!kfn) kfn = kernel_for(si, mode);
    if (!kfn) return 0;
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kSmemBytes)) != cudaSuccess)
        return 0;
    if (ctas > 8 && cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                        cudaSuccess) {
        cudaGetLastError();
        cache[dev][si] = 0;
        return 0;
    }
    cudaLaunchConfig_t q{};
    q.gridDim = dim3(static_cast<unsigned>(ctas) * 8);
    q.blockDim = dim3(kNumThreads);
    q.dynamicSmemBytes = kSmemBytes;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = static_cast<unsigned>(ctas);
    qa[0].val.clusterDim.y = 1;
    qa[0].val.clusterDim.z = 1;
    q.attrs = qa;
    q.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kfn, &q) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    cache[dev][si] = n;
    return static_cast<uint32_t>(n);
}

}  // namespace

size_t ppmm_smem_bytes() { return kSmemBytes; }

namespace {
thread_local uint32_t g_last_kernels = 0;
thread_local uint32_t g_last_part_target = 0;
}
uint32_t ppmm_kernels_last_launch() { return g_last_kernels; }

uint32_t ppmm_last_part_target() { return g_last_part_target; }

cudaError_t launch_ppmm_planes(const PpmmLaunch& L, cudaStream_t stream) {
    g_last_kernels = 0;
    g_last_part_target = 0;
    if (L.nprimes == 0 || L.parts == 0 || L.M == 0 || L.N == 0) return cudaSuccess;
    if (L.nprimes > kMaxPrimesPerLaunch) return cudaErrorInvalidValue;
    if (L.ldk % 16 != 0 || L.ldk < L.K) return cudaErrorInvalidValue;
    const uint64_t a_part_rows = L.a_part_rows ? L.a_part_rows : static_cast<uint64_t>(L.nprimes) * 2 * L.M;
    const uint64_t a_rows = (L.parts - 1) * a_part_rows + static_cast<uint64_t>(L.nprimes) * 2 * L.M;
    const uint64_t b_rows = static_cast<uint64_t>(L.nprimes) * 2 * L.N;
    if (a_rows >= (1ull << 31) || b_rows >= (1ull << 31)) return cudaErrorInvalidValue;

    GemmArgs args;
    std::memset(&args, 0, sizeof(args));
    args.M = L.M;
    args.N = L.N;
    args.K = L.K;
    args.parts = L.parts;
    args.nprimes = L.nprimes;
    args.m_blocks = (L.M + 2 * kRowsPerCta - 1) / (2 * kRowsPerCta);
    const uint32_t tile_n = (L.mode == kModeInnerF4 || L.mode == kModeIrisMatchF4) ? kF4TileN : kMaxTileN;
    args.n_blocks = (L.N + tile_n - 1) / tile_n;

    int dev = 0;
    cudaGetDevice(&dev);
    // cluster shape: a multi-pair shape needs at least pn n-tiles; otherwise
    // the widest shape that divides the n-tiles (1x2 or a plain pair)
    int si = shape_index(L.cluster_pm, L.cluster_pn);
    // the inner / iris modes are built for 1x1 and 1x4 (2x4 measured 40% slower
    // for iris); the FP4 match with the query on M runs on 4x1 (the four pairs
    // share each database tile and cover 1024 query columns)
    const bool query_rows = L.mode != kModePsq && L.iris.query_rows;
    const bool f4 = L.mode == kModeIrisMatchF4 || L.mode == kModeInnerF4;
    if (L.mode != kModePsq && si != 0) si = query_rows && f4 ? kShape4x1 : 2;
    if (si < 0) si = 0;
    // Short launches (a few waves of units) finish sooner on plain pairs: 74
    // workers instead of 15 clusters + a filler whose solo pairs sweep a whole
    // unit alone. Multicast shapes pay off on long launches (DRAM/L2 energy).
    if (si != 0 && L.mode == kModePsq && !std::getenv("IRL_PPMM_CLUSTER") &&
        static_cast<uint64_t>(args.m_blocks) * L.parts * L.nprimes < kSmallLaunchBlocks)
        si = 0;
    if (args.n_blocks < static_cast<uint32_t>(kShapes[si].pn))
        si = (L.mode == kModePsq && args.n_blocks % 2 == 0 && kShapes[si].pm == 1) ? 1 : 0;
    const uint32_t occ2 = max_active_clusters(0, dev);
    uint32_t occ_main = si == 0 ? occ2 : max_active_clusters(si, dev, L.mode);
    if (occ_main == 0) {
        si = 0;
        occ_main = occ2;
    }
    if (occ2 == 0) return cudaErrorInvalidConfiguration;
    const Shape shp = kShapes[si];
    args.unit_mblocks = static_cast<uint32_t>(shp.pm);
    args.m_units = (args.m_blocks + args.unit_mblocks - 1) / args.unit_mblocks;
    // n-chunks: with multi-pair clusters a unit is one cluster-wide n-chunk
    // (pn tiles; the last chunk padded); plain pairs keep the whole N per unit
    // and split it over a gated group of pairs.
    if (si != 0 && !std::getenv("IRL_PPMM_NO_NCHUNK")) {
        args.chunk_tiles = static_cast<uint32_t>(shp.pn);
        args.n_chunks = (args.n_blocks + args.chunk_tiles - 1) / args.chunk_tiles;
    } else {
        args.chunk_tiles = args.n_blocks;
        args.n_chunks = 1;
        if (si != 0 && args.n_blocks % shp.pn != 0) return cudaErrorInvalidValue;
    }
    args.units = args.m_units * args.n_chunks * L.parts * L.nprimes;
    // every tile of a (prime, part) (padding tiles included) is finished by 2 CTAs x kEpiWarps warps
    g_last_part_target = args.m_units * args.unit_mblocks * args.n_chunks * args.chunk_tiles * 2u *
                         static_cast<uint32_t>(kEpiWarps);
    args.accumulate = L.accumulate ? 1u : 0u;
    args.a_part_rows = static_cast<uint32_t>(a_part_rows);
    args.out_part = L.out_part_elems ? L.out_part_elems
                                     : static_cast<unsigned long long>(L.nprimes) * L.N * L.M;
    args.out = L.out;
    if (L.n_mirror > kMaxMirrors || (L.n_mirror && L.mode != kModePsq)) return cudaErrorInvalidValue;
    args.part_done = L.part_done;
    args.n_mirror = L.n_mirror;
    args.mirror_part = L.mirror_part;
    args.mirror_parts = L.mirror_parts;
    args.mc_mirror = L.mc_mirror;
    if (L.mc_mirror && (L.mode != kModePsq || (L.M & 1u) != 0)) return cudaErrorInvalidValue;
    for (uint32_t i = 0; i < L.n_mirror; ++i) args.mirror[i] = L.mirror[i];
    args.out_i32[0] = L.out_i32[0];
    args.out_i32[1] = L.out_i32[1];
    if (L.mode != kModePsq && L.accumulate) return cudaErrorInvalidValue;
    if ((L.mode == kModeIrisMatch || L.mode == kModeIrisMatchF4) &&
        (L.parts != 1 || L.nprimes != 1 || L.iris.rho == 0 ||
         static_cast<uint64_t>(L.iris.rho) * (query_rows ? L.N : L.M) >= 0xFFFFFFFFull))
        return cudaErrorInvalidValue;
    args.iris = L.iris;
    {
        // Float screens with a 1e-5 margin. Scores lie in [-1, 1] (|inner| <=
        // overlap), and inner, overlap are exact in float below 2^24. So the
        // float quotient (error < 1e-6) and the float products lo_out * ov,
        // hi_out * ov (relative error 2^-23 with the bound's own rounding, i.e.
        // below 1e-5 * ov for |bound| < 84; a bound outside that range is
        // never reached by a score or decided the same way) settle every
        // score farther than 1e-5 from a bound. Longer rows (int8 planes with
        // K >= 2^23 bytes) are not exact in float: no screen, every score divides.
        const double eps = 1e-5;
        const float inf = __builtin_huge_valf();
        const bool exact_f32 = L.K < (1u << 23);
        args.iris.lo_in = exact_f32 ? static_cast<float>(L.iris.lo + eps) : inf;
        args.iris.lo_out = exact_f32 ? static_cast<float>(L.iris.lo - eps) : -inf;
        args.iris.hi_in = exact_f32 ? static_cast<float>(L.iris.hi - eps) : -inf;
        args.iris.hi_out = exact_f32 ? static_cast<float>(L.iris.hi + eps) : inf;
    }
    for (uint32_t i = 0; i < L.nprimes; ++i) args.mc[i] = L.mc[i];

    if (!L.progress) return cudaErrorInvalidValue;
    args.gate_lead = L.gate_lead < 0 ? kGateLead : static_cast<uint32_t>(L.gate_lead);
    args.counter = L.progress + kProgressWords;  // shared by every launch of this call

    // Cluster layouts: the main launch uses the requested multi-pair shape;
    // those strand SMs (e.g. 132 of 148 CTAs with 4-CTA clusters on B200), so
    // a 1x1 "filler" launch (same stream, programmatic overlap) takes the remaining SM pairs.
    // Both pull units from the same counter.
    struct Part {
        int si;
        uint32_t clusters, pair0, group0;
    } parts[2];
    int nparts = 0;
    uint32_t pairs_used = 0, groups_used = 0;
    auto plan = [&](int s_idx, uint32_t max_cl) {
        const Shape sh = kShapes[s_idx];
        const uint32_t ppc = static_cast<uint32_t>(sh.pm * sh.pn);
        const uint32_t G = args.chunk_tiles / sh.pn;
        const uint64_t items = static_cast<uint64_t>(args.units) * G;
        uint32_t cl = static_cast<uint32_t>(std::min<uint64_t>(max_cl, items));
        if (L.max_clusters > 0) cl = std::min<uint32_t>(cl, L.max_clusters);
        if (cl == 0) return;
        parts[nparts++] = {s_idx, cl, pairs_used, groups_used};
        pairs_used += cl * ppc;
        groups_used += cl / G + cl % G;
    };
    plan(si, occ_main);
    if (si != 0) {
        const uint32_t ppc = static_cast<uint32_t>(shp.pm * shp.pn);
        const uint32_t spare_pairs = occ2 > ppc * occ_main ? occ2 - ppc * occ_main : 0;
        if (L.max_clusters == 0 && spare_pairs > 0 && !std::getenv("IRL_PPMM_NO_FILLER")) plan(0, spare_pairs);
    }
    if (std::getenv("IRL_PPMM_VERBOSE")) {
        for (int i = 0; i < nparts; ++i)
            std::fprintf(stderr, "[irl] ppmm launch %d: cluster %dx%d pairs, %u clusters (%u CTAs), units %u\n", i,
                         kShapes[parts[i].si].pm, kShapes[parts[i].si].pn, parts[i].clusters,
                         parts[i].clusters * kShapes[parts[i].si].ctas(), args.units);
    }
    const size_t header = (kProgressWords + 32) * 4;
    const size_t fit = groups_used ? (kScheduleScratchBytes - header) / (static_cast<size_t>(groups_used) * 8) : 0;
    const uint32_t mail_slots = static_cast<uint32_t>(std::min<size_t>(static_cast<size_t>(args.units) + 1, fit));
    if (mail_slots < std::min<uint32_t>(kMinMail, args.units + 1) || pairs_used > kProgressWords)
        return cudaErrorInvalidValue;
    args.mail_slots = mail_slots;
    const size_t scratch = header + static_cast<size_t>(groups_used) * mail_slots * 8;
    cudaError_t e = cudaMemsetAsync(L.progress, 0, scratch, stream);
    if (e != cudaSuccess) return e;

    // The filler (parts[1]) goes into the SAME stream right behind the main
    // grid, with programmatic stream serialization: it starts once every main
    // CTA has executed griddepcontrol.launch_dependents (their first
    // instruction), so both grids share the unit counter from the start. No
    // side stream: nothing else queued on the device (copies, other streams
    // aliased onto the same hardware queue) can delay or reorder it.
    for (int i = 0; i < nparts; ++i) {
        const Part& pt = parts[i];
        GemmArgs a = args;
        const Shape sh = kShapes[pt.si];
        a.G = args.chunk_tiles / static_cast<uint32_t>(sh.pn);
        a.F = pt.clusters / a.G;
        a.L = pt.clusters % a.G;
        a.active_clusters = pt.clusters;
        // a cluster that covers a whole n-chunk (G == 1, multi-pair) is the only
        // reader of its DB tile: stream it evict-first so the query stays in L2
        a.a_evict_first = (sh.pn > 1 && a.G == 1 && !std::getenv("IRL_PPMM_A_NORMAL")) ? 1u : 0u;
        // likewise B when the launch streams it through clusters along M
        a.b_evict_first = (L.b_streamed && sh.pm > 1 && sh.pn == 1) ? 1u : 0u;
        a.progress = L.progress + pt.pair0;  // indexed by cluster id (< pairs of this launch)
        a.mailbox = reinterpret_cast<unsigned long long*>(L.progress + kProgressWords + 32) +
                    static_cast<size_t>(pt.group0) * mail_slots;
        a.stats = L.stats ? reinterpret_cast<unsigned long long*>(L.stats) + pt.pair0 * kStatSlots
                          : nullptr;
        CUtensorMap ma, mb;
        if (!make_plane_map(&ma, L.a_planes, L.K, a_rows, L.ldk, kRowsPerCta / sh.pn) ||
            !make_plane_map(&mb, L.b_planes, L.K, b_rows, L.ldk, kRowsPerCta / sh.pm))
            return cudaErrorInvalidValue;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(sh.ctas()) * pt.clusters);
        cfg.blockDim = dim3(kNumThreads);
        cfg.dynamicSmemBytes = kSmemBytes;
        cfg.stream = stream;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = static_cast<unsigned>(sh.ctas());
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = i == 0 ? 1 : 2;
        KernelFn kfn = kernel_for(pt.si, L.mode);
        if (!kfn) return cudaErrorInvalidValue;
        if (L.mode != kModePsq) {
            e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes));
            if (e == cudaSuccess && sh.ctas() > 8)
                e = cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (e != cudaSuccess) return e;
        }
        e = cudaLaunchKernelEx(&cfg, kfn, ma, mb, a);
        if (e != cudaSuccess) return e;
        ++g_last_kernels;
    }
    return e;
}

}  // namespace irl
