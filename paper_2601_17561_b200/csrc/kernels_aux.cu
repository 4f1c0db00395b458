// HBM-bound kernels around the PPMM GEMM: residue / digit split (the
// reference's digit_decompose, modmat.cpp:86-106, and residue extraction,
// modmat.cpp:168-176), CRT lift (modmat.cpp:178-193), synthetic planes,
// and small helpers. All kernels are written for sm_100a: 16-byte vector
// accesses where the layout allows, grids sized by the data.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "kernels_aux.cuh"

namespace irl {

namespace {

__device__ __forceinline__ void warp_max_atomic(int32_t v, int32_t* dst) {
    v = __reduce_max_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && dst) atomicMax(dst, v);
}

template <typename T>
__device__ __forceinline__ uint32_t reduce_input(T x, const ModConst& c) {
    if constexpr (sizeof(T) == 4) {
        return mod_s32(static_cast<int32_t>(x), c.m, c.magic_m, c.off_m);
    } else {
        const uint32_t u = static_cast<uint32_t>(x);
        return u < c.m ? u : mod_u32(u, c.m, c.magic_m);
    }
}

// v in [0, m) -> (d0, d1); e == 1 keeps the residue in one centred digit.
__device__ __forceinline__ void split_value(uint32_t v, const ModConst& c, int32_t& d0,
                                            int32_t& d1) {
    if (c.e == 2) {
        digit_split(v, c, d0, d1);
    } else {
        const int32_t half = static_cast<int32_t>((c.p - 1) / 2);
        d0 = static_cast<int32_t>(v) > half ? static_cast<int32_t>(v) - static_cast<int32_t>(c.p)
                                            : static_cast<int32_t>(v);
        d1 = 0;
    }
}

__device__ __forceinline__ uint32_t pack4(int32_t a, int32_t b, int32_t c, int32_t d) {
    return (static_cast<uint32_t>(a) & 0xFF) | ((static_cast<uint32_t>(b) & 0xFF) << 8) |
           ((static_cast<uint32_t>(c) & 0xFF) << 16) | ((static_cast<uint32_t>(d) & 0xFF) << 24);
}

// ---------------------------------------------------------------------------
// Row split: each thread produces 16 consecutive K positions of one row.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) split_rows_kernel(const T* __restrict__ in, size_t ld_in,
                                                         size_t plane_stride, uint32_t rows,
                                                         uint32_t cols, uint32_t groups,
                                                         const __grid_constant__ ModTable mt,
                                                         int8_t* __restrict__ planes,
                                                         size_t ldk, SplitStats* stats) {
    const uint32_t i = blockIdx.y;
    const ModConst c = mt.mc[i];
    const size_t gid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    int32_t m0 = 0, m1 = 0, mr = 0;
    if (gid < static_cast<size_t>(rows) * groups) {
        const uint32_t r = static_cast<uint32_t>(gid / groups);
        const uint32_t c0 = static_cast<uint32_t>(gid % groups) * 16;
        const T* src = in + i * plane_stride + static_cast<size_t>(r) * ld_in;
        int32_t d0[16], d1[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint32_t col = c0 + j;
            if (col < cols) {
                const uint32_t v = reduce_input<T>(src[col], c);
                split_value(v, c, d0[j], d1[j]);
                m0 = max(m0, abs(d0[j]));
                m1 = max(m1, abs(d1[j]));
                mr = max(mr, static_cast<int32_t>(v));
            } else {
                d0[j] = 0;
                d1[j] = 0;
            }
        }
        int8_t* p0 = planes + (static_cast<size_t>(i) * 2 * rows + r) * ldk + c0;
        int8_t* p1 = p0 + static_cast<size_t>(rows) * ldk;
        uint4 w0, w1;
        w0.x = pack4(d0[0], d0[1], d0[2], d0[3]);
        w0.y = pack4(d0[4], d0[5], d0[6], d0[7]);
        w0.z = pack4(d0[8], d0[9], d0[10], d0[11]);
        w0.w = pack4(d0[12], d0[13], d0[14], d0[15]);
        w1.x = pack4(d1[0], d1[1], d1[2], d1[3]);
        w1.y = pack4(d1[4], d1[5], d1[6], d1[7]);
        w1.z = pack4(d1[8], d1[9], d1[10], d1[11]);
        w1.w = pack4(d1[12], d1[13], d1[14], d1[15]);
        *reinterpret_cast<uint4*>(p0) = w0;
        *reinterpret_cast<uint4*>(p1) = w1;
    }
    if (stats) {
        warp_max_atomic(m0, &stats->v[i][0]);
        warp_max_atomic(m1, &stats->v[i][1]);
        warp_max_atomic(mr, &stats->v[i][2]);
    }
}

// ---------------------------------------------------------------------------
// Transposing split of a K x N matrix: 64 (k) x 64 (n) tiles through smem.
// ---------------------------------------------------------------------------
constexpr int kTT = 64;
constexpr int kTStride = 68;  // bytes per n-row in smem (17 words: conflict-free)

template <typename T>
__global__ void __launch_bounds__(256) split_cols_kernel(const T* __restrict__ in, size_t ld_in,
                                                         size_t plane_stride, uint32_t K,
                                                         uint32_t N,
                                                         const __grid_constant__ ModTable mt,
                                                         int8_t* __restrict__ planes,
                                                         size_t ldk, SplitStats* stats) {
    __shared__ __align__(16) int8_t s0[kTT * kTStride];
    __shared__ __align__(16) int8_t s1[kTT * kTStride];
    const uint32_t i = blockIdx.z;
    const ModConst c = mt.mc[i];
    const uint32_t k0 = blockIdx.x * kTT, n0 = blockIdx.y * kTT;
    const uint32_t tn = threadIdx.x % kTT, tk = threadIdx.x / kTT;  // tk in 0..3
    const T* src = in + i * plane_stride;
    int32_t m0 = 0, m1 = 0, mr = 0;
#pragma unroll 4
    for (int kk = 0; kk < 16; ++kk) {
        const uint32_t kl = tk * 16 + kk;
        const uint32_t k = k0 + kl, n = n0 + tn;
        int32_t d0 = 0, d1 = 0;
        if (k < K && n < N) {
            const uint32_t v = reduce_input<T>(src[static_cast<size_t>(k) * ld_in + n], c);
            split_value(v, c, d0, d1);
            m0 = max(m0, abs(d0));
            m1 = max(m1, abs(d1));
            mr = max(mr, static_cast<int32_t>(v));
        }
        s0[tn * kTStride + kl] = static_cast<int8_t>(d0);
        s1[tn * kTStride + kl] = static_cast<int8_t>(d1);
    }
    __syncthreads();
    const uint32_t nl = threadIdx.x / 4, chunk = threadIdx.x % 4;
    const uint32_t n = n0 + nl, k = k0 + chunk * 16;
    if (n < N && k < ldk) {
        const uint32_t* a0 = reinterpret_cast<const uint32_t*>(s0 + nl * kTStride + chunk * 16);
        const uint32_t* a1 = reinterpret_cast<const uint32_t*>(s1 + nl * kTStride + chunk * 16);
        int8_t* p0 = planes + (static_cast<size_t>(i) * 2 * N + n) * ldk + k;
        int8_t* p1 = p0 + static_cast<size_t>(N) * ldk;
        *reinterpret_cast<uint4*>(p0) = make_uint4(a0[0], a0[1], a0[2], a0[3]);
        *reinterpret_cast<uint4*>(p1) = make_uint4(a1[0], a1[1], a1[2], a1[3]);
    }
    if (stats) {
        warp_max_atomic(m0, &stats->v[i][0]);
        warp_max_atomic(m1, &stats->v[i][1]);
        warp_max_atomic(mr, &stats->v[i][2]);
    }
}

// Vectorised transposing split for uint16 residues (the per-step query
// split, the dominant HBM kernel besides the GEMM). Tile 128 (k) x 64 (n):
// each thread loads 4 rows x 8 columns as 16-byte vectors, packs the 4
// k-bytes of every column into one word per plane in shared memory, and the
// block writes 64 rows x 128 bytes per plane as 16-byte stores.
// Needs N, ld_in and plane_stride multiples of 8 and a 16-byte aligned input.

constexpr int kSplitTileDefault = 0;

template <bool kStats, bool kOdd, int kVK, int kVN>
__global__ void __launch_bounds__(256) split_cols_u16_vec_kernel(const uint16_t* __restrict__ in, size_t ld_in,
                                                                 size_t plane_stride, uint32_t K, uint32_t N,
                                                                 const __grid_constant__ ModTable mt,
                                                                 int8_t* __restrict__ planes, size_t ldk,
                                                                 SplitStats* stats) {
    constexpr int kVW = kVK / 4 + 1;  // words per n-row (odd: conflict-light)
    constexpr int kSlots = (kVK / 4) * (kVN / 8) / 256;
    __shared__ uint32_t s0[kVN * kVW], s1[kVN * kVW];
    const uint32_t i = blockIdx.z;
    const ModConst c = mt.mc[i];
    const uint32_t k0 = blockIdx.x * kVK, n0 = blockIdx.y * kVN;
    const uint16_t* src = in + i * plane_stride;
    int32_t m0 = 0, m1 = 0, mr = 0;
    const uint32_t mm1 = c.magic_m + 1u, mp1 = c.magic_p + 1u, h = (c.p - 1) / 2;
#pragma unroll
    for (int sl = 0; sl < kSlots; ++sl) {
    const uint32_t slot = threadIdx.x + 256 * sl;
    const uint32_t kq = slot / (kVN / 8), v = slot % (kVN / 8);
    const uint32_t n = n0 + 8 * v;
    uint32_t w0[8], w1[8];
    uint4 q[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const uint32_t k = k0 + 4 * kq + r;
        q[r] = (k < K && n < N) ? __ldg(reinterpret_cast<const uint4*>(src + static_cast<size_t>(k) * ld_in + n))
                                : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        int32_t d0[4], d1[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t word = j < 2 ? (r == 0 ? q[0].x : r == 1 ? q[1].x : r == 2 ? q[2].x : q[3].x)
                                : j < 4 ? (r == 0 ? q[0].y : r == 1 ? q[1].y : r == 2 ? q[2].y : q[3].y)
                                : j < 6 ? (r == 0 ? q[0].z : r == 1 ? q[1].z : r == 2 ? q[2].z : q[3].z)
                                        : (r == 0 ? q[0].w : r == 1 ? q[1].w : r == 2 ? q[2].w : q[3].w);
            const uint32_t x = (j & 1) ? word >> 16 : word & 0xFFFFu;
            if constexpr (kOdd) {  // every modulus of the launch is p^2 with p odd
                const uint32_t vv = x - c.m * __umulhi(x, mm1);
                digit_split_odd(vv, c.p, h, mp1, d0[r], d1[r]);
            } else {
                digit_split_u16(x, c, d0[r], d1[r]);
            }
            if constexpr (kStats) {
                m0 = max(m0, abs(d0[r]));
                m1 = max(m1, abs(d1[r]));
                mr = max(mr, static_cast<int32_t>(x - c.m * __umulhi(x, mm1)));
            }
        }
        // rows beyond K were zero-filled above and split to digits (0, 0)
        w0[j] = __byte_perm(__byte_perm(d0[0], d0[1], 0x0040), __byte_perm(d0[2], d0[3], 0x0040), 0x5410);
        w1[j] = __byte_perm(__byte_perm(d1[0], d1[1], 0x0040), __byte_perm(d1[2], d1[3], 0x0040), 0x5410);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        s0[(8 * v + j) * kVW + kq] = w0[j];
        s1[(8 * v + j) * kVW + kq] = w1[j];
    }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kVN * (kVK / 16) / 256; ++it) {
        const uint32_t idx = threadIdx.x + 256 * it;
        const uint32_t row = idx / (kVK / 16), ch = idx % (kVK / 16);
        const uint32_t nn = n0 + row, k = k0 + 16 * ch;
        if (nn < N && k < ldk) {
            const uint32_t* a0 = s0 + row * kVW + 4 * ch;
            const uint32_t* a1 = s1 + row * kVW + 4 * ch;
            int8_t* p0 = planes + (static_cast<size_t>(i) * 2 * N + nn) * ldk + k;
            int8_t* p1 = p0 + static_cast<size_t>(N) * ldk;
            *reinterpret_cast<uint4*>(p0) = make_uint4(a0[0], a0[1], a0[2], a0[3]);
            *reinterpret_cast<uint4*>(p1) = make_uint4(a1[0], a1[1], a1[2], a1[3]);
        }
    }
    if constexpr (kStats) {
        warp_max_atomic(m0, &stats->v[i][0]);
        warp_max_atomic(m1, &stats->v[i][1]);
        warp_max_atomic(mr, &stats->v[i][2]);
    }
}

// ---------------------------------------------------------------------------
// RNS rescale by Delta (ModDown, result modulo ~Q/Delta).
// With x' = x + add (residue-wise, mod m_i): r = x' mod Delta from the
// dropped residues by CRT (exact in 64 bits, Delta < 2^48), then for every
// kept modulus y_i = (x'_i - r mod m_i) * Delta^-1 mod m_i, i.e. the residues
// of floor(x' / Delta) (congruent mod Q/Delta even when x + add wraps Q).
// One thread per element; reads nmod x 2 B, writes (nmod - drop) x 2 B.
// ---------------------------------------------------------------------------
// Vectorised rescale: 8 consecutive elements per thread (16-byte loads and
// stores per modulus plane), the CRT correction folded into one 64-bit
// multiply-accumulate chain per kept modulus (RescaleTable::w).
__device__ __forceinline__ uint32_t mod_u35(unsigned long long a, uint32_t m, uint32_t magic, uint32_t c32) {
    // a < 2^35: (hi * (2^32 mod m) + lo) mod m with hi < 8
    const uint32_t t = mod_u32(static_cast<uint32_t>(a), m, magic) + static_cast<uint32_t>(a >> 32) * c32;
    return mod_u32(t, m, magic);
}

__global__ void __launch_bounds__(256) rescale_vec_kernel(const uint16_t* __restrict__ in, size_t ld_in, size_t groups,
                                                          const __grid_constant__ RescaleTable t,
                                                          uint16_t* __restrict__ out, size_t ld_out) {
    const size_t g = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= groups) return;
    const size_t e0 = g * 8;
    const uint32_t keep = t.nmod - t.drop;
    uint32_t u[3][8];
    unsigned long long S[8];
#pragma unroll
    for (int l = 0; l < 8; ++l) S[l] = 0;
#pragma unroll
    for (uint32_t jj = 0; jj < 3; ++jj) {
        if (jj >= t.drop) {
#pragma unroll
            for (int l = 0; l < 8; ++l) u[jj][l] = 0;
            continue;
        }
        const uint32_t j = keep + jj, m = t.m[j];
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(in + j * ld_in + e0));
        const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int l = 0; l < 8; ++l) {
            const uint32_t x = (qw[l / 2] >> (16 * (l % 2))) & 0xFFFFu;
            uint32_t xa = x - m * __umulhi(x, t.magic[j] + 1u) + t.add[j];  // x mod m + add < 2m
            xa = xa >= m ? xa - m : xa;
            u[jj][l] = mod_u32(xa * t.cinv[j], m, t.magic[j]);  // xa, cinv < 2^16
            S[l] += static_cast<unsigned long long>(u[jj][l]) * t.cq[j];
        }
    }
    uint32_t k[8];
#pragma unroll
    for (int l = 0; l < 8; ++l) k[l] = (S[l] >= t.delta) + (S[l] >= 2 * t.delta);
    // kept moduli in groups of 4: the 4 loads are in flight together (one
    // 16-byte load per modulus plane and thread)
    for (uint32_t i0 = 0; i0 < keep; i0 += 4) {
        uint4 q[4];
#pragma unroll
        for (int g = 0; g < 4; ++g)
            q[g] = i0 + g < keep ? __ldg(reinterpret_cast<const uint4*>(in + (i0 + g) * ld_in + e0))
                                 : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const uint32_t i = i0 + g;
            if (i >= keep) break;
            const uint32_t m = t.m[i], mg = t.magic[i], c32 = t.c32[i], dinv = t.dinv[i], ad = t.add[i];
            const uint32_t w0 = t.w[0][i], w1 = t.w[1][i], w2 = t.w[2][i];
            const uint32_t qw[4] = {q[g].x, q[g].y, q[g].z, q[g].w};
            uint32_t y[8];
#pragma unroll
            for (int l = 0; l < 8; ++l) {
                const uint32_t x = (qw[l / 2] >> (16 * (l % 2))) & 0xFFFFu;
                unsigned long long acc = static_cast<unsigned long long>(x + ad) * dinv + k[l];
                acc += static_cast<unsigned long long>(u[0][l]) * w0;
                acc += static_cast<unsigned long long>(u[1][l]) * w1;
                acc += static_cast<unsigned long long>(u[2][l]) * w2;
                y[l] = mod_u35(acc, m, mg, c32);
            }
            *reinterpret_cast<uint4*>(out + i * ld_out + e0) =
                make_uint4(y[0] | (y[1] << 16), y[2] | (y[3] << 16), y[4] | (y[5] << 16), y[6] | (y[7] << 16));
        }
    }
}

// a * w mod m for a constant w < m (Shoup): w_sh = floor(w 2^32 / m), any a <
// 2^32; the result lies in [0, 2m) (one conditional subtraction from reduced).
__device__ __forceinline__ uint32_t shoup_mul(uint32_t a, uint32_t w, uint32_t w_sh, uint32_t m) {
    return a * w - __umulhi(a, w_sh) * m;
}

// Vectorised rescale, all 32-bit: r = x' mod Delta once per element (64-bit,
// from the dropped residues), then per kept modulus r mod m_i from its two
// 32-bit halves (two Barrett reductions) and one Shoup multiplication by
// Delta^-1 -- 8 integer multiplies per output residue instead of four 64-bit
// multiply-accumulates plus a 35-bit reduction.
__global__ void __launch_bounds__(256) rescale_r_kernel(const uint16_t* __restrict__ in, size_t ld_in,
                                                        size_t groups, const __grid_constant__ RescaleTable t,
                                                        uint16_t* __restrict__ out, size_t ld_out) {
    const size_t g = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= groups) return;
    const size_t e0 = g * 8;
    const uint32_t keep = t.nmod - t.drop;
    unsigned long long S[8];
#pragma unroll
    for (int l = 0; l < 8; ++l) S[l] = 0;
    for (uint32_t j = keep; j < t.nmod; ++j) {
        const uint32_t m = t.m[j], ad = t.add[j], ci = t.cinv[j], cs = t.cinv_sh[j];
        const unsigned long long cq = t.cq[j];
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(in + j * ld_in + e0));
        const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int l = 0; l < 8; ++l) {
            uint32_t xa = ((qw[l / 2] >> (16 * (l % 2))) & 0xFFFFu) + ad;  // < 2m
            xa = min(xa, xa - m);
            uint32_t u = shoup_mul(xa, ci, cs, m);
            u = min(u, u - m);
            S[l] += static_cast<unsigned long long>(u) * cq;
        }
    }
    uint32_t rlo[8], rhi[8];
#pragma unroll
    for (int l = 0; l < 8; ++l) {
        const unsigned long long k = (S[l] >= t.delta) + (S[l] >= 2 * t.delta);
        const unsigned long long r = S[l] - k * t.delta;  // x' mod Delta < 2^48
        rlo[l] = static_cast<uint32_t>(r);
        rhi[l] = static_cast<uint32_t>(r >> 32);
    }
    for (uint32_t i0 = 0; i0 < keep; i0 += 4) {
        uint4 q[4];
#pragma unroll
        for (int gg = 0; gg < 4; ++gg)
            q[gg] = i0 + gg < keep ? __ldg(reinterpret_cast<const uint4*>(in + (i0 + gg) * ld_in + e0))
                                   : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int gg = 0; gg < 4; ++gg) {
            const uint32_t i = i0 + gg;
            if (i >= keep) break;
            const uint32_t m = t.m[i], mg = t.magic[i], c32 = t.c32[i], ad = t.add[i];
            const uint32_t dv = t.dinv[i], ds = t.dinv_sh[i];
            const uint32_t qw[4] = {q[gg].x, q[gg].y, q[gg].z, q[gg].w};
            uint32_t y[8];
#pragma unroll
            for (int l = 0; l < 8; ++l) {
                const uint32_t x = (qw[l / 2] >> (16 * (l % 2))) & 0xFFFFu;
                // r mod m_i, left in [0, 2m) by both (unconditioned) Barrett steps:
                // rhi * c32 + [0, 2m) < 2^32 since rhi, c32 < 2^16
                const uint32_t r1 = rlo[l] - __umulhi(rlo[l], mg) * m;
                const uint32_t t = rhi[l] * c32 + r1;
                const uint32_t rm = t - __umulhi(t, mg) * m;
                uint32_t v = shoup_mul(x + ad + 2 * m - rm, dv, ds, m);  // (x' - r) Delta^-1, in [0, 2m)
                y[l] = min(v, v - m);
            }
            *reinterpret_cast<uint4*>(out + i * ld_out + e0) =
                make_uint4(y[0] | (y[1] << 16), y[2] | (y[3] << 16), y[4] | (y[5] << 16), y[6] | (y[7] << 16));
        }
    }
}

__global__ void __launch_bounds__(256) rescale_kernel(const uint16_t* __restrict__ in, size_t ld_in, size_t count,
                                                      const __grid_constant__ RescaleTable t,
                                                      uint16_t* __restrict__ out, size_t ld_out) {
    const size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= count) return;
    const uint32_t keep = t.nmod - t.drop;
    unsigned long long r = 0;
    for (uint32_t j = keep; j < t.nmod; ++j) {
        const uint32_t m = t.m[j];
        uint32_t x = mod_u32(in[j * ld_in + e], m, t.magic[j]) + t.add[j];
        x = x >= m ? x - m : x;
        const uint32_t u = mod_u32(x * t.cinv[j], m, t.magic[j]);  // < 2^32: x, cinv < 2^16
        r += static_cast<unsigned long long>(u) * t.cq[j];            // < drop * Delta < 2^50
    }
    while (r >= t.delta) r -= t.delta;  // at most drop - 1 times
    const uint32_t r_lo = static_cast<uint32_t>(r), r_hi = static_cast<uint32_t>(r >> 32);
    for (uint32_t i = 0; i < keep; ++i) {
        const uint32_t m = t.m[i];
        uint32_t x = mod_u32(in[i * ld_in + e], m, t.magic[i]) + t.add[i];
        x = x >= m ? x - m : x;
        uint32_t rm = mod_u32(r_lo, m, t.magic[i]) + mod_u32(r_hi * t.c32[i], m, t.magic[i]);
        rm = rm >= m ? rm - m : rm;
        const uint32_t d = x >= rm ? x - rm : x + m - rm;
        out[i * ld_out + e] = static_cast<uint16_t>(mod_u32(d * t.dinv[i], m, t.magic[i]));
    }
}

// ---------------------------------------------------------------------------
// Big-integer residue extraction + split.
// x mod m = sum_j b_j (256^j mod m) mod m; the sum stays < 2^30 for
// width <= 48 and m <= 2^16, so one Barrett reduction finishes it.
// ---------------------------------------------------------------------------
struct BigSplitArgs {
    ModTable mt;
    uint32_t coef[kMaxModuli][kMaxWidth / 4];  // 2^(32 k) mod m_i
    uint32_t c32[kMaxModuli];                  // 2^32 mod m_i
};

// Residue of a width-byte little-endian integer held as 32-bit words w[k]:
// sum_k w_k (2^32k mod m) accumulated exactly in 64 bits (< 12 * 2^48), then
// reduced through its two 32-bit halves.
__device__ __forceinline__ uint32_t words_mod(const uint32_t* w, uint32_t nw, const uint32_t* coef, uint32_t m,
                                              uint32_t magic, uint32_t c32) {
    unsigned long long acc = 0;
#pragma unroll
    for (uint32_t k = 0; k < kMaxWidth / 4; ++k)
        if (k < nw) acc += static_cast<unsigned long long>(w[k]) * coef[k];
    const uint32_t hi = mod_u32(static_cast<uint32_t>(acc >> 32), m, magic);  // < m < 2^16
    return mod_u32(hi * c32 + mod_u32(static_cast<uint32_t>(acc), m, magic), m, magic);
}

// Little-endian bytes b[0, width) as 32-bit words, zero above width; every
// index compile-time so the words stay in registers.
__device__ __forceinline__ void load_words(const uint8_t* b, uint32_t width, uint32_t* w) {
#pragma unroll
    for (uint32_t k = 0; k < kMaxWidth / 4; ++k) {
        uint32_t v = 0;
#pragma unroll
        for (uint32_t t = 0; t < 4; ++t)
            if (4 * k + t < width) v |= static_cast<uint32_t>(b[4 * k + t]) << (8 * t);
        w[k] = v;
    }
}

// Entries -> residues -> digit planes, 256 entries per block. The DB layout
// (transpose = 0) stages the block's 256 * width contiguous bytes through
// shared memory with 16-byte loads; each thread then folds its entry as 32-bit
// words (12 wide multiply-adds per modulus for the 46-byte paper width,
// instead of 46 byte multiply-adds). Plane writes are coalesced along K.
__global__ void __launch_bounds__(256) split_bigint_words_kernel(
    const uint8_t* __restrict__ in, uint32_t width, uint32_t rows, uint32_t cols, int transpose,
    const __grid_constant__ BigSplitArgs a, int8_t* __restrict__ planes, size_t ldk,
    uint32_t dst_rows, uint32_t dst_row0, int32_t* __restrict__ raw_out, SplitStats* stats) {
    __shared__ __align__(16) uint8_t stage[256 * kMaxWidth];
    const size_t total = static_cast<size_t>(rows) * cols;
    const size_t base = static_cast<size_t>(blockIdx.x) * 256;
    const size_t gid = base + threadIdx.x;
    const bool ok = gid < total;
    const uint32_t nw = (width + 3) / 4;
    uint32_t w[kMaxWidth / 4];
#pragma unroll
    for (uint32_t k = 0; k < kMaxWidth / 4; ++k) w[k] = 0;
    uint32_t r = 0, cidx = 0;  // (w: registers only -- every index below is compile-time)
    if (!transpose) {
        const size_t nbytes = (total - base < 256 ? total - base : 256) * width;
        const uint8_t* src = in + base * width;
        if ((reinterpret_cast<uintptr_t>(src) & 15) == 0 && nbytes % 16 == 0) {
            for (size_t o = threadIdx.x * 16; o < nbytes; o += 256 * 16)
                *reinterpret_cast<uint4*>(stage + o) = __ldg(reinterpret_cast<const uint4*>(src + o));
        } else {
            for (size_t o = threadIdx.x; o < nbytes; o += 256) stage[o] = src[o];
        }
        __syncthreads();
        if (ok) {
            load_words(stage + threadIdx.x * width, width, w);
            r = static_cast<uint32_t>(gid / cols);
            cidx = static_cast<uint32_t>(gid % cols);
        }
    } else if (ok) {  // K x N query: threads walk k fastest so plane writes stay coalesced
        r = static_cast<uint32_t>(gid % rows);     // k
        cidx = static_cast<uint32_t>(gid / rows);  // n
        load_words(in + (static_cast<size_t>(r) * cols + cidx) * width, width, w);
    }
    const uint32_t prow = (transpose ? cidx : r) + dst_row0;
    const uint32_t pcol = transpose ? r : cidx;
    for (uint32_t i = 0; i < a.mt.n; ++i) {
        const ModConst c = a.mt.mc[i];
        int32_t d0 = 0, d1 = 0, v = 0;
        if (ok) {
            v = static_cast<int32_t>(words_mod(w, nw, a.coef[i], c.m, c.magic_m, a.c32[i]));
            if (c.e == 2) digit_split(static_cast<uint32_t>(v), c, d0, d1);
        }
        if (c.e == 2) {
            if (ok) {
                int8_t* p0 = planes + (static_cast<size_t>(i) * 2 * dst_rows + prow) * ldk + pcol;
                p0[0] = static_cast<int8_t>(d0);
                p0[static_cast<size_t>(dst_rows) * ldk] = static_cast<int8_t>(d1);
            }
            if (stats) {
                warp_max_atomic(abs(d0), &stats->v[i][0]);
                warp_max_atomic(abs(d1), &stats->v[i][1]);
            }
        } else if (raw_out) {
            if (ok) raw_out[static_cast<size_t>(i) * total + static_cast<size_t>(r) * cols + cidx] = v;
        }
        if (stats) warp_max_atomic(v, &stats->v[i][2]);
    }
}

// ---------------------------------------------------------------------------
// CRT lift. acc = sum_i (Q/m_i) * ((Q/m_i)^-1 r_i mod m_i) < nmod * Q <= 32 Q,
// then conditional subtraction of 16Q, 8Q, 4Q, 2Q, Q.
// ---------------------------------------------------------------------------
struct CrtArgs {
    CrtTable t;
    ModConst mc[kMaxModuli];
};

__global__ void __launch_bounds__(256) crt_lift_kernel(const uint16_t* __restrict__ res,
                                                       uint32_t M, uint32_t N,
                                                       const __grid_constant__ CrtArgs a,
                                                       uint8_t* __restrict__ out) {
    const size_t gid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= static_cast<size_t>(M) * N) return;
    const uint32_t m = static_cast<uint32_t>(gid % M), n = static_cast<uint32_t>(gid / M);
    const uint32_t L = a.t.limbs;
    uint32_t acc[kMaxQLimbs + 1];
#pragma unroll
    for (uint32_t j = 0; j <= kMaxQLimbs; ++j) acc[j] = 0;
    for (uint32_t i = 0; i < a.t.nmod; ++i) {
        const ModConst c = a.mc[i];
        uint32_t r = res[(static_cast<size_t>(i) * N + n) * M + m];
        r = r < c.m ? r : mod_u32(r, c.m, c.magic_m);
        const uint32_t t = mod_u32(r * a.t.inv[i], c.m, c.magic_m);
        uint64_t carry = 0;
#pragma unroll
        for (uint32_t j = 0; j < kMaxQLimbs; ++j) {
            if (j < L) {
                const uint64_t s = static_cast<uint64_t>(a.t.qi[i][j]) * t + acc[j] + carry;
                acc[j] = static_cast<uint32_t>(s);
                carry = s >> 32;
            }
        }
        // propagate into the top limb(s); every limb index is compile-time
        // (predicated on L) so acc stays in registers
#pragma unroll
        for (uint32_t j = 0; j <= kMaxQLimbs; ++j) {
            if (j >= L) {
                const uint64_t s = static_cast<uint64_t>(acc[j]) + carry;
                acc[j] = static_cast<uint32_t>(s);
                carry = s >> 32;
            }
        }
    }
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        const uint32_t* q = a.t.qmul[s];
        // compare acc (L+1 limbs) >= q, most significant limb first
        int ge = 1;
        bool decided = false;
#pragma unroll
        for (int j = static_cast<int>(kMaxQLimbs); j >= 0; --j) {
            if (j <= static_cast<int>(L) && !decided && acc[j] != q[j]) {
                ge = acc[j] > q[j];
                decided = true;
            }
        }
        if (ge) {
            uint64_t borrow = 0;
#pragma unroll
            for (uint32_t j = 0; j <= kMaxQLimbs; ++j) {
                if (j <= L) {
                    const uint64_t d = static_cast<uint64_t>(acc[j]) - q[j] - borrow;
                    acc[j] = static_cast<uint32_t>(d);
                    borrow = (d >> 63) & 1;
                }
            }
        }
    }
    uint8_t* dst = out + (static_cast<size_t>(m) * N + n) * a.t.width;
#pragma unroll
    for (uint32_t limb = 0; limb <= kMaxQLimbs; ++limb)
#pragma unroll
        for (uint32_t t = 0; t < 4; ++t)
            if (4 * limb + t < a.t.width) dst[4 * limb + t] = limb <= L ? static_cast<uint8_t>(acc[limb] >> (8 * t)) : 0;
}

// ---------------------------------------------------------------------------
// Counter-based synthetic residues (bit-identical to irl_synth_residue).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint32_t synth_residue(uint64_t seed_mixed, uint32_t stream,
                                                           uint32_t plane, uint32_t row,
                                                           uint32_t col, uint32_t m) {
    const uint64_t key = (static_cast<uint64_t>(stream & 0xFF) << 56) |
                         (static_cast<uint64_t>(plane & 0xFF) << 48) |
                         (static_cast<uint64_t>(row & 0xFFFFFF) << 24) |
                         static_cast<uint64_t>(col & 0xFFFFFF);
    const uint64_t x = mix64(key ^ seed_mixed);
    return static_cast<uint32_t>(((x >> 32) * static_cast<uint64_t>(m)) >> 32);
}

__global__ void __launch_bounds__(256) synth_planes_kernel(uint64_t seed_mixed, uint32_t part0,
                                                           uint32_t row0, uint32_t rows, uint32_t cols,
                                                           uint32_t groups,
                                                           const __grid_constant__ ModTable mt,
                                                           int8_t* __restrict__ planes,
                                                           size_t ldk) {
    const uint32_t i = blockIdx.y, g = blockIdx.z;
    const ModConst c = mt.mc[i];
    const size_t gid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= static_cast<size_t>(rows) * groups) return;
    const uint32_t r = static_cast<uint32_t>(gid / groups);
    const uint32_t c0 = static_cast<uint32_t>(gid % groups) * 16;
    int32_t d0[16], d1[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if (c0 + j < cols) {
            const uint32_t v = synth_residue(seed_mixed, part0 + g, i, row0 + r, c0 + j, c.m);
            split_value(v, c, d0[j], d1[j]);
        } else {
            d0[j] = 0;
            d1[j] = 0;
        }
    }
    int8_t* p0 =
        planes + ((static_cast<size_t>(g) * mt.n + i) * 2 * rows + r) * ldk + c0;
    int8_t* p1 = p0 + static_cast<size_t>(rows) * ldk;
    uint4 w0, w1;
    w0.x = pack4(d0[0], d0[1], d0[2], d0[3]);
    w0.y = pack4(d0[4], d0[5], d0[6], d0[7]);
    w0.z = pack4(d0[8], d0[9], d0[10], d0[11]);
    w0.w = pack4(d0[12], d0[13], d0[14], d0[15]);
    w1.x = pack4(d1[0], d1[1], d1[2], d1[3]);
    w1.y = pack4(d1[4], d1[5], d1[6], d1[7]);
    w1.z = pack4(d1[8], d1[9], d1[10], d1[11]);
    w1.w = pack4(d1[12], d1[13], d1[14], d1[15]);
    *reinterpret_cast<uint4*>(p0) = w0;
    *reinterpret_cast<uint4*>(p1) = w1;
}

// ---------------------------------------------------------------------------
// Small helpers
// ---------------------------------------------------------------------------
__global__ void gemm_i32_kernel(const int32_t* __restrict__ a, const int32_t* __restrict__ b,
                                int32_t* __restrict__ c, uint32_t M, uint32_t K, uint32_t N) {
    __shared__ int32_t sa[16][17], sb[16][17];
    const uint32_t row = blockIdx.y * 16 + threadIdx.y, col = blockIdx.x * 16 + threadIdx.x;
    uint32_t acc = 0;  // wrap-around int32 arithmetic, like the reference's int32 loop
    for (uint32_t k0 = 0; k0 < K; k0 += 16) {
        sa[threadIdx.y][threadIdx.x] =
            (row < M && k0 + threadIdx.x < K) ? a[static_cast<size_t>(row) * K + k0 + threadIdx.x] : 0;
        sb[threadIdx.y][threadIdx.x] =
            (col < N && k0 + threadIdx.y < K) ? b[static_cast<size_t>(k0 + threadIdx.y) * N + col] : 0;
        __syncthreads();
#pragma unroll
        for (int t = 0; t < 16; ++t)
            acc += static_cast<uint32_t>(sa[threadIdx.y][t]) * static_cast<uint32_t>(sb[t][threadIdx.x]);
        __syncthreads();
    }
    if (row < M && col < N) c[static_cast<size_t>(row) * N + col] = static_cast<int32_t>(acc);
}

__global__ void transpose_u16_i32_kernel(const uint16_t* __restrict__ in, uint32_t M, uint32_t N,
                                         int32_t* __restrict__ out) {
    __shared__ uint16_t t[32][33];
    const uint32_t m0 = blockIdx.x * 32, n0 = blockIdx.y * 32;
    for (uint32_t j = threadIdx.y; j < 32; j += 8) {
        const uint32_t n = n0 + j, m = m0 + threadIdx.x;
        t[j][threadIdx.x] = (n < N && m < M) ? in[static_cast<size_t>(n) * M + m] : 0;
    }
    __syncthreads();
    for (uint32_t j = threadIdx.y; j < 32; j += 8) {
        const uint32_t m = m0 + j, n = n0 + threadIdx.x;
        if (m < M && n < N) out[static_cast<size_t>(m) * N + n] = t[threadIdx.x][j];
    }
}

__global__ void reduce_raw_kernel(const int32_t* __restrict__ raw, uint32_t M, uint32_t N,
                                  uint32_t idx, ModConst c, uint16_t* __restrict__ res) {
    const size_t gid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= static_cast<size_t>(M) * N) return;
    const uint32_t m = static_cast<uint32_t>(gid % M), n = static_cast<uint32_t>(gid / M);
    const int32_t v = raw[static_cast<size_t>(m) * N + n];
    res[(static_cast<size_t>(idx) * N + n) * M + m] =
        static_cast<uint16_t>(mod_s32(v, c.m, c.magic_m, c.off_m));
}

__global__ void digit_decompose_kernel(const int32_t* __restrict__ in, size_t count, ModConst c,
                                       int32_t* __restrict__ d0, int32_t* __restrict__ d1) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint32_t v = mod_s32(in[i], c.m, c.magic_m, c.off_m);
    int32_t a, b;
    digit_split(v, c, a, b);
    d0[i] = a;
    d1[i] = b;
}

__global__ void digit_recompose_kernel(const int32_t* __restrict__ d0,
                                       const int32_t* __restrict__ d1, size_t count, ModConst c,
                                       int32_t* __restrict__ out) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    // int32 arithmetic exactly as modmat.cpp:112-116 (wrapping multiply-add,
    // truncating %, then shift into [0, p^2)).
    const int32_t v = static_cast<int32_t>(static_cast<uint32_t>(d0[i]) +
                                           c.p * static_cast<uint32_t>(d1[i]));
    int32_t r = v % static_cast<int32_t>(c.m);
    if (r < 0) r += static_cast<int32_t>(c.m);
    out[i] = static_cast<int32_t>(r);
}

__global__ void absmax_kernel(const int32_t* __restrict__ x, size_t count, int32_t* dst) {
    int32_t m = 0;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int32_t v = x[i];
        // |INT32_MIN| saturates to INT32_MAX: still far beyond any valid bound.
        m = max(m, v == INT32_MIN ? INT32_MAX : abs(v));
    }
    warp_max_atomic(m, dst);
}

__global__ void double_to_residues_kernel(const double* __restrict__ x, size_t count,
                                          const __grid_constant__ ModTable mt,
                                          uint16_t* __restrict__ out, int* bad) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const double v = x[i];
    const bool ok = v == floor(v) && fabs(v) < 9007199254740992.0;  // 2^53
    if (!ok) {
        *bad = 1;
        return;
    }
    const long long iv = static_cast<long long>(v);
    for (uint32_t j = 0; j < mt.n; ++j) {
        long long r = iv % static_cast<long long>(mt.mc[j].m);
        if (r < 0) r += mt.mc[j].m;
        out[static_cast<size_t>(j) * count + i] = static_cast<uint16_t>(r);
    }
}

__global__ void crt_centred_double_kernel(const uint16_t* __restrict__ res, uint32_t M, uint32_t N,
                                          const __grid_constant__ Crt64Table t,
                                          double* __restrict__ out) {
    const size_t gid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= static_cast<size_t>(M) * N) return;
    unsigned __int128 acc = 0;
    for (uint32_t i = 0; i < t.nmod; ++i) {
        const ModConst& c = t.mc[i];
        uint32_t r = res[static_cast<size_t>(i) * M * N + gid];
        r = r < c.m ? r : mod_u32(r, c.m, c.magic_m);
        const uint32_t tt = mod_u32(r * t.inv[i], c.m, c.magic_m);
        acc += static_cast<unsigned __int128>(t.qi[i]) * tt;
    }
    const unsigned long long x = static_cast<unsigned long long>(acc % t.Q);
    const double v = x > t.Q / 2 ? -static_cast<double>(t.Q - x) : static_cast<double>(x);
    out[gid] = v;  // out[n][m] shares the [N][M] indexing of res
}

inline unsigned blocks_for(size_t n, unsigned t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

template <typename T>
cudaError_t launch_split_rows(const T* in, size_t ld_in, size_t plane_stride, uint32_t rows,
                              uint32_t cols, const ModTable& mt, int8_t* planes, size_t ldk,
                              SplitStats* stats, cudaStream_t s) {
    if (rows == 0 || ldk == 0 || mt.n == 0) return cudaSuccess;
    const uint32_t groups = static_cast<uint32_t>(ldk / 16);
    const dim3 grid(blocks_for(static_cast<size_t>(rows) * groups, 256), mt.n);
    split_rows_kernel<T><<<grid, 256, 0, s>>>(in, ld_in, plane_stride, rows, cols, groups, mt,
                                              planes, ldk, stats);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_split_cols(const T* in, size_t ld_in, size_t plane_stride, uint32_t k,
                              uint32_t n, const ModTable& mt, int8_t* planes, size_t ldk,
                              SplitStats* stats, cudaStream_t s) {
    if (n == 0 || ldk == 0 || mt.n == 0) return cudaSuccess;
    if constexpr (sizeof(T) == 2) {
        if (n % 8 == 0 && ld_in % 8 == 0 && plane_stride % 8 == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
            bool odd = true;
            for (uint32_t i = 0; i < mt.n; ++i) odd &= mt.mc[i].e == 2 && (mt.mc[i].p & 1u);
            static const int tile = [] {
                const char* t = std::getenv("IRL_SPLIT_TILE");  // experiment knob: 0 128x64, 1 128x128, 2 256x64
                return t ? std::atoi(t) : kSplitTileDefault;
            }();
            auto pick = [&](auto kvk, auto kvn) {
                constexpr int KT = decltype(kvk)::value, NT = decltype(kvn)::value;
                const dim3 g(blocks_for(ldk, KT), blocks_for(n, NT), mt.n);
                auto kfn = stats ? (odd ? split_cols_u16_vec_kernel<true, true, KT, NT>
                                        : split_cols_u16_vec_kernel<true, false, KT, NT>)
                                 : (odd ? split_cols_u16_vec_kernel<false, true, KT, NT>
                                        : split_cols_u16_vec_kernel<false, false, KT, NT>);
                kfn<<<g, 256, 0, s>>>(in, ld_in, plane_stride, k, n, mt, planes, ldk, stats);
            };
            if (tile == 1)
                pick(std::integral_constant<int, 128>{}, std::integral_constant<int, 128>{});
            else if (tile == 2)
                pick(std::integral_constant<int, 256>{}, std::integral_constant<int, 64>{});
            else
                pick(std::integral_constant<int, 128>{}, std::integral_constant<int, 64>{});
            return cudaGetLastError();
        }
    }
    const dim3 grid(blocks_for(ldk, kTT), blocks_for(n, kTT), mt.n);
    split_cols_kernel<T><<<grid, 256, 0, s>>>(in, ld_in, plane_stride, k, n, mt, planes, ldk, stats);
    return cudaGetLastError();
}

template cudaError_t launch_split_rows<uint16_t>(const uint16_t*, size_t, size_t, uint32_t,
                                                 uint32_t, const ModTable&, int8_t*, size_t,
                                                 SplitStats*, cudaStream_t);
template cudaError_t launch_split_rows<int32_t>(const int32_t*, size_t, size_t, uint32_t, uint32_t,
                                                const ModTable&, int8_t*, size_t, SplitStats*,
                                                cudaStream_t);
template cudaError_t launch_split_cols<uint16_t>(const uint16_t*, size_t, size_t, uint32_t,
                                                 uint32_t, const ModTable&, int8_t*, size_t,
                                                 SplitStats*, cudaStream_t);
template cudaError_t launch_split_cols<int32_t>(const int32_t*, size_t, size_t, uint32_t, uint32_t,
                                                const ModTable&, int8_t*, size_t, SplitStats*,
                                                cudaStream_t);

cudaError_t launch_split_bigint(const uint8_t* in, uint32_t width, uint32_t rows, uint32_t cols,
                                int transpose, const ModTable& mt, int8_t* planes, size_t ldk,
                                uint32_t dst_rows, uint32_t dst_row0, int32_t* raw_out,
                                SplitStats* stats, cudaStream_t s) {
    if (width > kMaxWidth || mt.n > kMaxModuli) return cudaErrorInvalidValue;
    const size_t total = static_cast<size_t>(rows) * cols;
    if (total == 0) return cudaSuccess;
    BigSplitArgs a{};
    a.mt = mt;
    for (uint32_t i = 0; i < mt.n; ++i) {
        const uint64_t m = mt.mc[i].m;
        a.c32[i] = static_cast<uint32_t>((1ull << 32) % m);
        uint64_t pw = 1 % m;
        for (uint32_t k = 0; k < kMaxWidth / 4; ++k) {
            a.coef[i][k] = static_cast<uint32_t>(pw);
            pw = (pw << 32) % m;
        }
    }
    split_bigint_words_kernel<<<blocks_for(total, 256), 256, 0, s>>>(
        in, width, rows, cols, transpose, a, planes, ldk, dst_rows, dst_row0, raw_out, stats);
    return cudaGetLastError();
}

cudaError_t launch_rescale(const uint16_t* in, size_t ld_in, size_t count, const RescaleTable& t, uint16_t* out,
                           size_t ld_out, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    if (count % 8 == 0 && ld_in % 8 == 0 && ld_out % 8 == 0 && t.drop <= 3 &&
        ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
        static const bool r_form = std::getenv("IRL_RESCALE_FOLDED") == nullptr;
        if (r_form)
            rescale_r_kernel<<<blocks_for(count / 8, 256), 256, 0, s>>>(in, ld_in, count / 8, t, out, ld_out);
        else
            rescale_vec_kernel<<<blocks_for(count / 8, 256), 256, 0, s>>>(in, ld_in, count / 8, t, out, ld_out);
        return cudaGetLastError();
    }
    rescale_kernel<<<blocks_for(count, 256), 256, 0, s>>>(in, ld_in, count, t, out, ld_out);
    return cudaGetLastError();
}

cudaError_t launch_crt_lift(const uint16_t* res, uint32_t M, uint32_t N, const CrtTable& t,
                            uint8_t* out, cudaStream_t s) {
    const size_t total = static_cast<size_t>(M) * N;
    if (total == 0) return cudaSuccess;
    CrtArgs a{};
    a.t = t;
    for (uint32_t i = 0; i < t.nmod; ++i) {
        a.mc[i] = make_modconst(t.m[i], 1);
    }
    crt_lift_kernel<<<blocks_for(total, 256), 256, 0, s>>>(res, M, N, a, out);
    return cudaGetLastError();
}

cudaError_t launch_synth_planes(uint64_t seed, uint32_t part0, uint32_t parts, uint32_t rows,
                                uint32_t cols, const ModTable& mt, int8_t* planes, size_t ldk,
                                cudaStream_t s, uint32_t row0) {
    if (rows == 0 || parts == 0 || mt.n == 0) return cudaSuccess;
    const uint32_t groups = static_cast<uint32_t>(ldk / 16);
    const dim3 grid(blocks_for(static_cast<size_t>(rows) * groups, 256), mt.n, parts);
    synth_planes_kernel<<<grid, 256, 0, s>>>(mix64(seed), part0, row0, rows, cols, groups, mt, planes, ldk);
    return cudaGetLastError();
}

cudaError_t launch_gemm_i32(const int32_t* a, const int32_t* b, int32_t* c, uint32_t m, uint32_t k,
                            uint32_t n, cudaStream_t s) {
    if (m == 0 || n == 0) return cudaSuccess;
    const dim3 grid(blocks_for(n, 16), blocks_for(m, 16));
    gemm_i32_kernel<<<grid, dim3(16, 16), 0, s>>>(a, b, c, m, k, n);
    return cudaGetLastError();
}

cudaError_t launch_transpose_u16_to_i32(const uint16_t* in, uint32_t M, uint32_t N, int32_t* out,
                                        cudaStream_t s) {
    if (M == 0 || N == 0) return cudaSuccess;
    const dim3 grid(blocks_for(M, 32), blocks_for(N, 32));
    transpose_u16_i32_kernel<<<grid, dim3(32, 8), 0, s>>>(in, M, N, out);
    return cudaGetLastError();
}

cudaError_t launch_reduce_raw(const int32_t* raw, uint32_t M, uint32_t N, uint32_t mod_index,
                              const ModConst& mc, uint16_t* res, cudaStream_t s) {
    const size_t total = static_cast<size_t>(M) * N;
    if (total == 0) return cudaSuccess;
    reduce_raw_kernel<<<blocks_for(total, 256), 256, 0, s>>>(raw, M, N, mod_index, mc, res);
    return cudaGetLastError();
}

cudaError_t launch_digit_decompose(const int32_t* in, size_t count, const ModConst& mc,
                                   int32_t* d0, int32_t* d1, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    digit_decompose_kernel<<<blocks_for(count, 256), 256, 0, s>>>(in, count, mc, d0, d1);
    return cudaGetLastError();
}

cudaError_t launch_digit_recompose(const int32_t* d0, const int32_t* d1, size_t count,
                                   const ModConst& mc, int32_t* out, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    digit_recompose_kernel<<<blocks_for(count, 256), 256, 0, s>>>(d0, d1, count, mc, out);
    return cudaGetLastError();
}

cudaError_t launch_absmax_i32(const int32_t* x, size_t count, int32_t* dst, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    unsigned b = blocks_for(count, 256);
    if (b > 4096) b = 4096;
    absmax_kernel<<<b, 256, 0, s>>>(x, count, dst);
    return cudaGetLastError();
}

cudaError_t launch_double_to_residues(const double* x, uint32_t rows, uint32_t cols,
                                      const ModTable& mt, uint16_t* out, int* bad, cudaStream_t s) {
    const size_t count = static_cast<size_t>(rows) * cols;
    if (count == 0) return cudaSuccess;
    double_to_residues_kernel<<<blocks_for(count, 256), 256, 0, s>>>(x, count, mt, out, bad);
    return cudaGetLastError();
}

cudaError_t launch_crt_centred_double(const uint16_t* res, uint32_t M, uint32_t N,
                                      const Crt64Table& t, double* out, cudaStream_t s) {
    const size_t count = static_cast<size_t>(M) * N;
    if (count == 0) return cudaSuccess;
    crt_centred_double_kernel<<<blocks_for(count, 256), 256, 0, s>>>(res, M, N, t, out);
    return cudaGetLastError();
}

// 32 rows (one per lane) x 32 columns per block; each thread keeps 4 column
// accumulators. K is walked in 32-wide shared-memory tiles, strictly in order,
// with explicitly rounded multiplies and adds (the reference's loop body
// `prow[j] += a * qrow[j]`, which baseline x86-64 never contracts).
__global__ void __launch_bounds__(256) ordered_dgemm_t_kernel(const double* __restrict__ a,
                                                              const double* __restrict__ q, uint32_t M,
                                                              uint32_t K, uint32_t N, double* __restrict__ out) {
    __shared__ double as[32][33];  // [k][i]
    __shared__ double qs[32][32];  // [k][j]
    const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const uint32_t i = blockIdx.x * 32 + tx;
    const uint32_t j0 = blockIdx.y * 32 + ty * 4;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (uint32_t k0 = 0; k0 < K; k0 += 32) {
        for (uint32_t e = threadIdx.x; e < 32 * 32; e += 256) {
            const uint32_t r = e >> 5, c = e & 31;  // a: row r of the tile, column k0 + c
            const uint32_t gi = blockIdx.x * 32 + r, gk = k0 + c;
            as[c][r] = (gi < M && gk < K) ? a[size_t(gi) * K + gk] : 0.0;
            const uint32_t qk = k0 + r, qj = blockIdx.y * 32 + c;
            qs[r][c] = (qk < K && qj < N) ? q[size_t(qk) * N + qj] : 0.0;
        }
        __syncthreads();
        const uint32_t kn = min(32u, K - k0);
        for (uint32_t kk = 0; kk < kn; ++kk) {
            const double av = as[kk][tx];
            if (!(av == 0.0)) {  // emulator.cpp:415: `if (a == 0.0) continue;`
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[r] = __dadd_rn(acc[r], __dmul_rn(av, qs[kk][ty * 4 + r]));
            }
        }
        __syncthreads();
    }
    if (i < M)
#pragma unroll
        for (int r = 0; r < 4; ++r)
            if (j0 + r < N) out[size_t(j0 + r) * M + i] = acc[r];
}

cudaError_t launch_ordered_dgemm_t(const double* a, const double* q, uint32_t M, uint32_t K, uint32_t N,
                                   double* out, cudaStream_t s) {
    if (M == 0 || N == 0) return cudaSuccess;
    const dim3 grid((M + 31) / 32, (N + 31) / 32);
    ordered_dgemm_t_kernel<<<grid, 256, 0, s>>>(a, q, M, K, N, out);
    return cudaGetLastError();
}

uint32_t synth_residue_host(uint64_t seed, uint32_t stream, uint32_t plane, uint32_t row,
                            uint32_t col, uint32_t m) {
    return synth_residue(mix64(seed), stream, plane, row, col, m);
}

}  // namespace irl
