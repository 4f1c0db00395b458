// Internal (CUDA-side) interface of the PPMM engine kernels. Not part of the
// public C ABI (see include/irl_capi.h).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "modarith.cuh"

namespace irl {

constexpr uint32_t kMaxPrimesPerLaunch = 32;
// Kernel modes: kModePsq = the fused mod-p^2 PPMM (uint16 residues out);
// kModeInner = two independent int8 products acc1 = X0 Y0, acc2 = X1 Y1 with
// raw int32 outputs (mask overlaps and ternary inner products, iris.cu).
constexpr int kModePsq = 0;
constexpr uint32_t kMaxMirrors = 7;
constexpr int kModeInner = 1;
// kModeIrisMatch: the kModeInner products with the plaintext scoring fused
// into the epilogue (score = acc1 / acc2 in IEEE double, match bits and the
// first match / first empty overlap per eye; see IrisMatchOut).
constexpr int kModeIrisMatch = 2;
// The same two modes on the block-scaled FP4 tensor path: planes are packed
// e2m1 nibbles (2 per byte, K in bytes = ceil(d / 2)), tcgen05.mma
// kind::mxf4.block_scale with unit UE8M0 scales, FP32 accumulators (exact for
// the ternary / mask products below 2^24), 240-column tiles (the scale factors
// take TMEM columns 240..255). Twice the int8 rate, half the operand bytes.
constexpr int kModeInnerF4 = 3;
constexpr uint32_t kF4TileCols = 240;  // N of one FP4 tile
constexpr int kModeIrisMatchF4 = 4;

struct IrisMatchOut {
    double lo = 0, hi = 0;      // the P interval
    float lo_in = 0, lo_out = 0, hi_in = 0, hi_out = 0;  // float screens lo +- eps, hi -+ eps (set by the launcher)
    uint32_t rho = 1;           // query column c = eye * rho + rotation
    uint32_t col0 = 0;          // global index of this launch's column 0 (column-split launches)
    uint8_t* bits = nullptr;    // [eyes][M] (zeroed by the caller), nullable
    uint32_t* first = nullptr;  // [eyes][2]: min rotation * M + m of a match / of an empty overlap (0xFF.. init)
    double* scores = nullptr;   // [N][M], NaN where the overlap is empty; nullable
    // 0: A = database templates (M), B = query columns (N), as above.
    // 1: A = query columns (M rows, column c = eye * rho + rotation), B =
    //    database templates (N): bits [eyes][N], first-event index rotation * N
    //    + template, scores [M][N]. A 4x1 cluster then covers up to 1024
    //    columns in one pass over the database (the FP4 tile is 240 wide, so
    //    992 columns on N needed a second, 32-column pass over it).
    uint32_t query_rows = 0;
};
// Diagnostics slots per CTA pair (PpmmLaunch::stats): 0 producer empty-wait
// cycles, 1 producer gate cycles, 2 MMA full-wait cycles, 3 MMA tmem-empty
// wait cycles, 4 MMA thread total cycles, 5 epilogue tmem-full wait cycles,
// 6 epilogue busy cycles, 7/8 globaltimer start/end (ns), 11 tiles.
constexpr uint32_t kStatSlots = 16;
// Device scratch the PPMM launcher needs (progress counters, unit counter,
// per-group unit mailboxes); zeroed by every launch.
constexpr size_t kScheduleScratchBytes = 4 << 20;

// One batched PPMM launch over `parts` database parts and `nprimes` moduli.
//   a_planes: [parts][nprimes][2][M][ldk] int8 centred digits (K-major)
//   b_planes: [nprimes][2][N][ldk]        int8 centred digits (K-major)
//   out:      [parts][nprimes][N][M]      uint16 residues mod p^2
struct PpmmLaunch {
    const int8_t* a_planes = nullptr;
    const int8_t* b_planes = nullptr;
    uint16_t* out = nullptr;
    uint32_t M = 0, N = 0, K = 0, ldk = 0;
    uint32_t parts = 1, nprimes = 0;
    int accumulate = 0;          // out = (out + result) mod p^2
    uint32_t max_clusters = 0;   // 0 = one CTA pair per SM pair
    uint32_t* progress = nullptr;  // kScheduleScratchBytes of device scratch (required)
    uint64_t* stats = nullptr;     // optional [pairs][kStatSlots] diagnostics
    int gate_lead = -1;            // K blocks a pair may lead its group; -1 default, 0 off
    // Part strides for launches over a modulus subset of every part
    // (0 = dense: nprimes * 2 * M rows, nprimes * N * M outputs).
    uint64_t a_part_rows = 0;
    uint64_t out_part_elems = 0;
    // Cluster shape in CTA pairs: cluster_pm pairs along M (sharing each query
    // tile by TMA multicast) x cluster_pn pairs along N (sharing each database
    // tile). 1x1 is a plain CTA pair; SMs a multi-pair shape strands are taken
    // by a 1x1 filler launch pulling from the same unit counter.
    // Mirrors (fused a-part exchange): outputs of part `mirror_part` (relative to
    // this launch) are also stored, same offsets within the part, to each of
    // mirror[0..n_mirror) -- peer GPUs' receive buffers mapped over NVLink.
    uint16_t* mirror[kMaxMirrors] = {};
    uint32_t n_mirror = 0;
    uint32_t mirror_part = 0;
    uint32_t mirror_parts = 1;  // parts [mirror_part, mirror_part + mirror_parts), back to back in the mirrors
    // NVLS multicast mirror: a multicast address (cuMulticastCreate, bound to
    // one receive buffer per GPU); the epilogue stores each pair of output rows
    // once with multimem.st and the switch delivers it to every bound GPU.
    // Needs M even. Used instead of, or with, mirror[].
    uint16_t* mc_mirror = nullptr;
    // Optional [nprimes][parts] completion counters (zeroed by the caller):
    // every epilogue warp adds 1 per finished tile of that (prime, part);
    // ppmm_last_part_target() is the final count of each.
    uint32_t* part_done = nullptr;
    int mode = kModePsq;
    int32_t* out_i32[2] = {nullptr, nullptr};  // kModeInner outputs [parts][nprimes][N][M]
    IrisMatchOut iris;                          // kModeIrisMatch outputs (parts = nprimes = 1)
    int cluster_pm = 1;
    int cluster_pn = 4;
    // B is the operand streamed once (read by one cluster) and A the small one
    // every unit re-reads: load B evict-first, A evict-last (with cluster_pm > 1)
    int b_streamed = 0;
    ModConst mc[kMaxPrimesPerLaunch];
};

cudaError_t launch_ppmm_planes(const PpmmLaunch& L, cudaStream_t stream);
// Value each part_done[prime][part] reaches once every tile of that (prime,
// part) of the calling thread's last launch_ppmm_planes is stored.
uint32_t ppmm_last_part_target();
// Kernels the calling thread's last launch_ppmm_planes issued (main + filler).
uint32_t ppmm_kernels_last_launch();
size_t ppmm_smem_bytes();

}  // namespace irl
