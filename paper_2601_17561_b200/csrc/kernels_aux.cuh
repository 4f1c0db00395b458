// Internal launch interface of the HBM-bound kernels around the PPMM GEMM.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "modarith.cuh"

namespace irl {

constexpr uint32_t kMaxModuli = 32;
constexpr uint32_t kMaxQLimbs = 12;  // Q < 2^384
constexpr uint32_t kMaxWidth = 48;   // bytes per mod-Q entry

// Per-modulus running maxima gathered by the split kernels, used for the
// reference's data-dependent AccumulationOverflowRisk precheck
// (modmat.cpp:122-129): [0] = max|d0|, [1] = max|d1|, [2] = max raw residue.
struct SplitStats {
    int32_t v[kMaxModuli][3];
};

struct ModTable {
    uint32_t n;
    ModConst mc[kMaxModuli];
};

// Residues (or arbitrary int32) -> centred digit planes, no transpose:
// in[i][r][c] (ld_in, plane stride in elements) -> planes[i][d][r][ldk].
template <typename T>
cudaError_t launch_split_rows(const T* in, size_t ld_in, size_t plane_stride, uint32_t rows,
                              uint32_t cols, const ModTable& mt, int8_t* planes, size_t ldk,
                              SplitStats* stats, cudaStream_t s);

// Transposing variant: in[i][k][n] (a K x N matrix) -> planes[i][d][n][ldk].
template <typename T>
cudaError_t launch_split_cols(const T* in, size_t ld_in, size_t plane_stride, uint32_t k,
                              uint32_t n, const ModTable& mt, int8_t* planes, size_t ldk,
                              SplitStats* stats, cudaStream_t s);

// width-byte little-endian mod-Q entries -> residues mod m_i -> digit planes.
// transpose=0: [rows][cols] -> planes[i][d][rows][ldk];
// transpose=1: [rows=K][cols=N] -> planes[i][d][N][ldk].
// Moduli with e == 1 are emitted as raw residues into raw_out[i][rows][cols]
// (int32) instead of planes (nullptr if none).
// dst_rows / dst_row0: row count of each destination plane and the row
// offset this call writes at (lets a large matrix be split in row chunks).
cudaError_t launch_split_bigint(const uint8_t* in, uint32_t width, uint32_t rows, uint32_t cols,
                                int transpose, const ModTable& mt, int8_t* planes, size_t ldk,
                                uint32_t dst_rows, uint32_t dst_row0, int32_t* raw_out,
                                SplitStats* stats, cudaStream_t s);

// max |x| over an int32 array, atomically folded into *dst.
cudaError_t launch_absmax_i32(const int32_t* x, size_t count, int32_t* dst, cudaStream_t s);

// CRT lift: res[i][N][M] (uint16 residues) -> out[m][n] width-byte entries mod Q.
struct CrtTable {
    uint32_t nmod, limbs, width;
    uint32_t m[kMaxModuli];
    uint32_t inv[kMaxModuli];                     // (Q/m_i)^-1 mod m_i
    uint32_t qi[kMaxModuli][kMaxQLimbs];          // Q/m_i
    uint32_t qmul[5][kMaxQLimbs + 1];             // 16Q, 8Q, 4Q, 2Q, Q
};
cudaError_t launch_crt_lift(const uint16_t* res, uint32_t M, uint32_t N, const CrtTable& t,
                            uint8_t* out, cudaStream_t s);

// Exact RNS rescale (ModDown) by Delta = product of the last `drop` moduli:
// residues of x mod Q -> residues of floor((x + add) / Delta) mod Q / Delta
// (add = floor(Delta / 2) rounds). in[i][count] (stride ld_in), out[i][count]
// (stride ld_out) for the nmod - drop kept moduli. Delta < 2^48.
struct RescaleTable {
    uint32_t nmod, drop;
    uint32_t m[kMaxModuli], magic[kMaxModuli];
    uint32_t add[kMaxModuli];      // floor(Delta/2) mod m_i (0: floor)
    uint32_t dinv[kMaxModuli];     // Delta^-1 mod m_i (kept moduli)
    uint32_t c32[kMaxModuli];      // 2^32 mod m_i
    uint32_t cinv[kMaxModuli];     // (Delta/m_j)^-1 mod m_j (dropped moduli)
    unsigned long long cq[kMaxModuli];  // Delta / m_j (dropped moduli)
    unsigned long long delta;
    // folded form: y_i = ((x_i + add_i) dinv_i + sum_j u_j w[j][i] + k) mod m_i with
    // u_j = (x_j + add_j) cinv_j mod m_j, k = floor(sum_j u_j cq_j / Delta),
    // w[j][i] = -(cq_j dinv_i) mod m_i (j indexes the dropped moduli)
    uint32_t w[3][kMaxModuli];
    // Shoup constants floor(c * 2^32 / m) of dinv (kept) and cinv (dropped)
    uint32_t dinv_sh[kMaxModuli], cinv_sh[kMaxModuli];
};
cudaError_t launch_rescale(const uint16_t* in, size_t ld_in, size_t count, const RescaleTable& t, uint16_t* out,
                           size_t ld_out, cudaStream_t s);

// Synthetic database planes: planes[g][i][d][r][ldk] from the counter RNG,
// residue = synth(seed, stream=part0+g, plane=i, row, col, m_i).
// Rows [row0, row0 + rows) of parts part0.. (row0: a row block of a larger part).
cudaError_t launch_synth_planes(uint64_t seed, uint32_t part0, uint32_t parts, uint32_t rows,
                                uint32_t cols, const ModTable& mt, int8_t* planes, size_t ldk,
                                cudaStream_t s, uint32_t row0 = 0);

// int32 GEMM with int32 (wrapping) accumulation, row-major: C = A B.
cudaError_t launch_gemm_i32(const int32_t* a, const int32_t* b, int32_t* c, uint32_t m,
                            uint32_t k, uint32_t n, cudaStream_t s);

// out[r][c] (int32, row-major M x N) = in[c][r] (uint16 [N][M]); optional mod.
cudaError_t launch_transpose_u16_to_i32(const uint16_t* in, uint32_t M, uint32_t N, int32_t* out,
                                        cudaStream_t s);

// res[i][n][m] (uint16) = raw[i][m][n] mod m_i  (int32 raw products of e=1 moduli).
cudaError_t launch_reduce_raw(const int32_t* raw, uint32_t M, uint32_t N, uint32_t mod_index,
                              const ModConst& mc, uint16_t* res, cudaStream_t s);

// Elementwise digit_decompose / digit_recompose on int32 arrays.
cudaError_t launch_digit_decompose(const int32_t* in, size_t count, const ModConst& mc,
                                   int32_t* d0, int32_t* d1, cudaStream_t s);
cudaError_t launch_digit_recompose(const int32_t* d0, const int32_t* d1, size_t count,
                                   const ModConst& mc, int32_t* out, cudaStream_t s);

// Integer-valued doubles -> residues: out[i][r][c] = x[r][c] mod m_i (uint16);
// sets *bad = 1 if any entry is not an integer of magnitude < 2^53.
cudaError_t launch_double_to_residues(const double* x, uint32_t rows, uint32_t cols,
                                      const ModTable& mt, uint16_t* out, int* bad, cudaStream_t s);
// Centred CRT for bases with Q < 2^64: res[i][N][M] -> out[n][m] (double),
// value in (-Q/2, Q/2].
struct Crt64Table {
    uint32_t nmod;
    unsigned long long Q;
    unsigned long long qi[kMaxModuli];   // Q / m_i
    uint32_t inv[kMaxModuli];            // (Q/m_i)^-1 mod m_i
    ModConst mc[kMaxModuli];
};
cudaError_t launch_crt_centred_double(const uint16_t* res, uint32_t M, uint32_t N,
                                      const Crt64Table& t, double* out, cudaStream_t s);

// Emulator::ccmm_twin's product for arbitrary doubles, in the reference's own
// IEEE operation order (emulator.cpp:411-421): for each output (i, j), k runs
// 0..K-1 and acc = RN(acc + RN(a[i][k] * q[k][j])), skipping a[i][k] == 0.0;
// no fused multiply-add. Output transposed, out[j][i] (ccmm_twin's
// column-major message order).
cudaError_t launch_ordered_dgemm_t(const double* a, const double* q, uint32_t M, uint32_t K, uint32_t N,
                                   double* out, cudaStream_t s);

// Host mirror of the device generator.
uint32_t synth_residue_host(uint64_t seed, uint32_t stream, uint32_t plane, uint32_t row,
                            uint32_t col, uint32_t m);

}  // namespace irl
