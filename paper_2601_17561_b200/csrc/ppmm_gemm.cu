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
//   * a CTA pair (cluster of 2) owns a 256 x n_tile output tile
//     (n_tile <= 256): tcgen05.mma.cta_group::2.kind::i8 with M = 256;
//   * TMEM holds two int32 accumulators per tile: acc1 = X0 Y0 in columns
//     [0, 256) and acc2 = X0 Y1 + X1 Y0 in [256, 512);
//   * warp 0 = TMA producer (both CTAs load their half of A and B),
//     warp 1 = MMA issuer (leader CTA) + TMEM owner, warps 2..5 = epilogue;
//   * 3-stage smem ring of 128-byte K blocks, 128B-swizzled, mbarrier-paced;
//   * persistent static tile scheduler, tiles ordered (prime, part, m, n)
//     so the per-prime query planes stay L2-resident and every database
//     tile is streamed from HBM once.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>

#include "modarith.cuh"
#include "ppmm.h"
#include "sm100_ptx.cuh"

namespace irl {

namespace {

constexpr int kRowsPerCta = 128;   // M rows per CTA (256 per pair)
constexpr int kMaxTileN = 256;     // N columns per tile (pair-wide)
constexpr int kBlockK = 128;       // K bytes per pipeline stage
constexpr int kStages = 3;
constexpr int kUmmaK = 32;         // K per tcgen05.mma for 8-bit inputs
constexpr int kPlaneTileBytes = kRowsPerCta * kBlockK;          // 16 KB
constexpr int kStageBytes = 4 * kPlaneTileBytes;                // X0 X1 Y0 Y1
constexpr int kNumThreads = 192;
constexpr int kEpiWarp0 = 2;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kAcc2Col = 256;
constexpr size_t kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

struct __align__(64) GemmArgs {
    uint32_t M, N, K;
    uint32_t parts, nprimes;
    uint32_t m_blocks, n_blocks, num_tiles;
    uint32_t accumulate;
    uint16_t* out;
    ModConst mc[kMaxPrimesPerLaunch];
};

struct TileCoord {
    uint32_t prime, part, m0, n0, n_size;
};

__device__ __forceinline__ TileCoord decode_tile(const GemmArgs& a, uint32_t t) {
    TileCoord c;
    const uint32_t nb = t % a.n_blocks;
    uint32_t r = t / a.n_blocks;
    const uint32_t mb = r % a.m_blocks;
    r /= a.m_blocks;
    c.part = r % a.parts;
    c.prime = r / a.parts;
    c.m0 = mb * 2 * kRowsPerCta;
    c.n0 = nb * kMaxTileN;
    const uint32_t rem = a.N - c.n0;
    const uint32_t ns = rem < kMaxTileN ? rem : kMaxTileN;
    c.n_size = (ns + 31u) & ~31u;  // cta_group::2 kind::i8 needs N % 32 == 0
    return c;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kNumThreads, 1)
    ppmm_i8_sm100_kernel(const __grid_constant__ CUtensorMap tmap_a,
                         const __grid_constant__ CUtensorMap tmap_b,
                         const __grid_constant__ GemmArgs args) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty_bar = full_bar + kStages;
    uint64_t* tmem_full_bar = empty_bar + kStages;
    uint64_t* tmem_empty_bar = tmem_full_bar + 1;
    uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tmem_empty_bar + 1);

    const uint32_t warp = threadIdx.x / 32;
    const uint32_t lane = threadIdx.x % 32;
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const uint32_t cluster_id = blockIdx.x / 2;
    const uint32_t num_clusters = gridDim.x / 2;

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmap_a);
        ptx::prefetch_tmap(&tmap_b);
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&full_bar[s], 1);
            ptx::mbar_init(&empty_bar[s], 1);
        }
        ptx::mbar_init(tmem_full_bar, 1);
        ptx::mbar_init(tmem_empty_bar, 2 * 4);  // 4 epilogue warps in each CTA
        ptx::fence_barrier_init();
    }
    if (warp == 1) {
        ptx::tmem_alloc_pair(ptx::smem_u32(tmem_base_slot), kTmemCols);
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_base_slot;

    if (warp == 0) {
        // ---------------- TMA producer (both CTAs) ----------------
        if (lane == 0) {
            const uint32_t num_kb = (args.K + kBlockK - 1) / kBlockK;
            uint32_t stage = 0, phase = 0;
            for (uint32_t t = cluster_id; t < args.num_tiles; t += num_clusters) {
                const TileCoord tc = decode_tile(args, t);
                const uint32_t a_row0 =
                    ((tc.part * args.nprimes + tc.prime) * 2) * args.M + tc.m0 + rank * kRowsPerCta;
                const uint32_t half_n = tc.n_size / 2;
                const uint32_t b_row0 = (tc.prime * 2) * args.N + tc.n0 + rank * half_n;
                for (uint32_t kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
                    const uint32_t leader_full =
                        ptx::mapa_shared(ptx::smem_u32(&full_bar[stage]), 0);
                    if (leader) ptx::mbar_arrive_expect_tx(&full_bar[stage], 2 * kStageBytes);
                    uint8_t* st = smem + stage * kStageBytes;
                    const int32_t k0 = static_cast<int32_t>(kb * kBlockK);
                    ptx::tma_load_2d_pair(ptx::smem_u32(st), &tmap_a, leader_full, k0,
                                          static_cast<int32_t>(a_row0));
                    ptx::tma_load_2d_pair(ptx::smem_u32(st + kPlaneTileBytes), &tmap_a,
                                          leader_full, k0,
                                          static_cast<int32_t>(a_row0 + args.M));
                    ptx::tma_load_2d_pair(ptx::smem_u32(st + 2 * kPlaneTileBytes), &tmap_b,
                                          leader_full, k0, static_cast<int32_t>(b_row0));
                    ptx::tma_load_2d_pair(ptx::smem_u32(st + 3 * kPlaneTileBytes), &tmap_b,
                                          leader_full, k0,
                                          static_cast<int32_t>(b_row0 + args.N));
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (leader CTA only) ----------------
        if (leader && lane == 0) {
            const uint32_t num_kb = (args.K + kBlockK - 1) / kBlockK;
            const uint32_t acc1 = tmem_base;
            const uint32_t acc2 = tmem_base + kAcc2Col;
            uint32_t stage = 0, phase = 0, local_tile = 0;
            for (uint32_t t = cluster_id; t < args.num_tiles; t += num_clusters, ++local_tile) {
                const TileCoord tc = decode_tile(args, t);
                const uint32_t idesc = ptx::idesc_i8(2 * kRowsPerCta, tc.n_size);
                // Wait until the epilogue of the previous tile drained TMEM.
                ptx::mbar_wait(tmem_empty_bar, (local_tile & 1) ^ 1);
                ptx::tc_fence_after();
                for (uint32_t kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&full_bar[stage], phase);
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
                        ptx::mma_i8_pair(acc1, dx0, dy0, idesc, accum);  // X0 Y0
                        ptx::mma_i8_pair(acc2, dx0, dy1, idesc, accum);  // X0 Y1
                        ptx::mma_i8_pair(acc2, dx1, dy0, idesc, 1u);     // + X1 Y0
                    }
                    ptx::mma_commit_pair(&empty_bar[stage], 0x3);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::mma_commit_pair(tmem_full_bar, 0x3);
            }
        }
    } else {
        // ---------------- Epilogue (both CTAs) ----------------
        const uint32_t quarter = warp % 4;  // TMEM lane quarter this warp may access
        const uint32_t leader_tmem_empty = ptx::mapa_shared(ptx::smem_u32(tmem_empty_bar), 0);
        uint32_t local_tile = 0;
        for (uint32_t t = cluster_id; t < args.num_tiles; t += num_clusters, ++local_tile) {
            const TileCoord tc = decode_tile(args, t);
            const ModConst mc = args.mc[tc.prime];
            ptx::mbar_wait(tmem_full_bar, local_tile & 1);
            ptx::tc_fence_after();
            const uint32_t row = rank * kRowsPerCta + quarter * 32 + lane;
            const uint32_t m = tc.m0 + row;
            const bool row_ok = m < args.M;
            uint16_t* out = args.out +
                            (static_cast<size_t>(tc.part) * args.nprimes + tc.prime) *
                                static_cast<size_t>(args.N) * args.M +
                            m;
            const uint32_t lane_base = tmem_base + ((quarter * 32u) << 16);
            for (uint32_t c = 0; c < tc.n_size; c += 32) {
                uint32_t a1[32], a2[32];
                ptx::tmem_ld_32x32b_x32(lane_base + c, a1);
                ptx::tmem_ld_32x32b_x32(lane_base + kAcc2Col + c, a2);
                ptx::tmem_ld_wait();
                if (row_ok) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const uint32_t n = tc.n0 + c + j;
                        if (n < args.N) {
                            uint32_t v = combine_psq(static_cast<int32_t>(a1[j]),
                                                     static_cast<int32_t>(a2[j]), mc);
                            uint16_t* dst = out + static_cast<size_t>(n) * args.M;
                            if (args.accumulate) {
                                v += *dst;
                                v = v >= mc.m ? v - mc.m : v;
                            }
                            *dst = static_cast<uint16_t>(v);
                        }
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(leader_tmem_empty);
        }
    }

    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_pair(tmem_base, kTmemCols);
    }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess || p == nullptr) {
            throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
        }
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

void make_plane_map(CUtensorMap* map, const void* base, uint64_t k, uint64_t rows, uint64_t ldk) {
    const cuuint64_t dims[2] = {k, rows};
    const cuuint64_t strides[1] = {ldk};
    const cuuint32_t box[2] = {kBlockK, kRowsPerCta};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = get_encode_fn()(
        map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

}  // namespace

size_t ppmm_smem_bytes() { return kSmemBytes; }

cudaError_t launch_ppmm_planes(const PpmmLaunch& L, cudaStream_t stream) {
    if (L.nprimes == 0 || L.parts == 0 || L.M == 0 || L.N == 0) return cudaSuccess;
    if (L.nprimes > kMaxPrimesPerLaunch) return cudaErrorInvalidValue;
    if (L.ldk % 16 != 0 || L.ldk < L.K) return cudaErrorInvalidValue;
    const uint64_t a_rows = static_cast<uint64_t>(L.parts) * L.nprimes * 2 * L.M;
    const uint64_t b_rows = static_cast<uint64_t>(L.nprimes) * 2 * L.N;
    if (a_rows >= (1ull << 31) || b_rows >= (1ull << 31)) return cudaErrorInvalidValue;

    CUtensorMap ma, mb;
    make_plane_map(&ma, L.a_planes, L.K, a_rows, L.ldk);
    make_plane_map(&mb, L.b_planes, L.K, b_rows, L.ldk);

    GemmArgs args;
    std::memset(&args, 0, sizeof(args));
    args.M = L.M;
    args.N = L.N;
    args.K = L.K;
    args.parts = L.parts;
    args.nprimes = L.nprimes;
    args.m_blocks = (L.M + 2 * kRowsPerCta - 1) / (2 * kRowsPerCta);
    args.n_blocks = (L.N + kMaxTileN - 1) / kMaxTileN;
    args.num_tiles = args.m_blocks * args.n_blocks * L.parts * L.nprimes;
    args.accumulate = L.accumulate ? 1u : 0u;
    args.out = L.out;
    for (uint32_t i = 0; i < L.nprimes; ++i) args.mc[i] = L.mc[i];

    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(ppmm_i8_sm100_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kSmemBytes));
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint32_t clusters = static_cast<uint32_t>(sms / 2);
    if (L.max_clusters > 0) clusters = std::min<uint32_t>(clusters, L.max_clusters);
    clusters = std::min<uint32_t>(clusters, args.num_tiles);

    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(kNumThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, ppmm_i8_sm100_kernel, ma, mb, args);
}

}  // namespace irl
