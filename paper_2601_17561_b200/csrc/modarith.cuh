// Exact small-modulus arithmetic shared by the split, GEMM-epilogue and CRT
// kernels. All reductions are exact for any modulus 2 <= m <= 2^16 (Barrett
// with a 32-bit magic and one correction step).
#pragma once

#include <cstdint>

namespace irl {

// Per-modulus constants handed to kernels by value.
struct ModConst {
    uint32_t p;        // digit base (prime)
    uint32_t m;        // full modulus p^e (e = 1 or 2)
    uint32_t magic_p;  // floor(2^32 / p)
    uint32_t magic_m;  // floor(2^32 / m)
    uint32_t off_p;    // 2^31 mod p
    uint32_t off_m;    // 2^31 mod m
    uint32_t e;        // exponent 1 or 2
    uint32_t pad;
    uint32_t c_p;      // p * ceil(2^31 / p): shifts |x| < 2^31 - 2^17 into [0, 2^32)
    uint32_t c_m;      // m * ceil(2^31 / m)
};

__host__ __device__ inline ModConst make_modconst(uint32_t p, uint32_t e) {
    ModConst c{};
    c.p = p;
    c.e = e;
    c.m = e == 2 ? p * p : p;
    // m = 1 would need 2^32; 0xFFFFFFFF still leaves r in [0, 2m) (exact).
    c.magic_p = p > 1 ? static_cast<uint32_t>((1ull << 32) / p) : 0xFFFFFFFFu;
    c.magic_m = c.m > 1 ? static_cast<uint32_t>((1ull << 32) / c.m) : 0xFFFFFFFFu;
    c.off_p = static_cast<uint32_t>((1ull << 31) % p);
    c.off_m = static_cast<uint32_t>((1ull << 31) % c.m);
    c.c_p = static_cast<uint32_t>(((1ull << 31) + p - 1) / p * p);
    c.c_m = static_cast<uint32_t>(((1ull << 31) + c.m - 1) / c.m * c.m);
    return c;
}

// u mod m for u in [0, 2^32): Barrett quotient (low by at most one), then
// r = min_u32(r, r - m) picks the reduced value (r - m wraps when r < m).
__device__ __forceinline__ uint32_t mod_u32(uint32_t u, uint32_t m, uint32_t magic) {
    const uint32_t q = __umulhi(u, magic);
    const uint32_t r = u - q * m;
    return min(r, r - m);
}

// x mod m in [0, m) for any signed 32-bit x (floor semantics).
__device__ __forceinline__ uint32_t mod_s32(int32_t x, uint32_t m, uint32_t magic, uint32_t off) {
    const uint32_t u = static_cast<uint32_t>(x) + 0x80000000u;  // x + 2^31
    const uint32_t r = mod_u32(u, m, magic);
    return r >= off ? r - off : r + m - off;
}

// Reference epilogue of gemm_mod_psq (modmat.cpp:150-158):
// (t00 + p (t01 + t10)) mod p^2, with acc2 = t01 + t10 already fused.
__device__ __forceinline__ uint32_t combine_psq(int32_t acc1, int32_t acc2, const ModConst& c) {
    const uint32_t r2 = mod_s32(acc2, c.p, c.magic_p, c.off_p);
    const uint32_t r1 = mod_s32(acc1, c.m, c.magic_m, c.off_m);
    uint32_t v = r1 + c.p * r2;  // < 2 p^2
    return v >= c.m ? v - c.m : v;
}

// Fast epilogue combine for accumulators bounded by |acc| <= 2^31 - 2^17
// (guaranteed by the launcher's K chunking): ~11 integer instructions.
//   r2 = acc2 mod p;  result = (acc1 + p r2) mod p^2
// using the multiples c_p, c_m of p, p^2 to make both operands non-negative
// without signed fix-ups.
__device__ __forceinline__ uint32_t combine_psq_fast(int32_t acc1, int32_t acc2, uint32_t p,
                                                     uint32_t m, uint32_t magic_p,
                                                     uint32_t magic_m, uint32_t c_p,
                                                     uint32_t c_m) {
    const uint32_t r2 = mod_u32(static_cast<uint32_t>(acc2) + c_p, p, magic_p);
    const uint32_t u = static_cast<uint32_t>(acc1) + c_m + p * r2;
    return mod_u32(u, m, magic_m);
}

// Centred digit split of v in [0, p^2) (modmat.cpp:86-106):
// d0 = centre(v mod p), d1 = centre(((v - d0) / p) mod p).
__device__ __forceinline__ void digit_split(uint32_t v, const ModConst& c, int32_t& d0,
                                            int32_t& d1) {
    const int32_t p = static_cast<int32_t>(c.p);
    const int32_t half = (p - 1) / 2;
    int32_t a = static_cast<int32_t>(mod_u32(v, c.p, c.magic_p));
    if (a > half) a -= p;
    // (v - d0) is an exact multiple of p in [0, p^2]; Barrett quotient + fix.
    const uint32_t u = static_cast<uint32_t>(static_cast<int32_t>(v) - a);
    uint32_t hi = __umulhi(u, c.magic_p);
    if (u - hi * c.p >= c.p) ++hi;
    int32_t b = static_cast<int32_t>(hi >= c.p ? hi - c.p : hi);
    if (b > half) b -= p;
    d0 = a;
    d1 = b;
}

// Fast centred split of a 16-bit input x (any value < 2^16, reduced mod m
// first), ~12 integer instructions. floor(x / d) = umulhi(x, floor(2^32/d) + 1)
// is exact for x < 2^16 and 2 <= d < 2^16: the rounding error x*delta/2^32 <
// 2^-16 stays below 1/d, the smallest gap from frac(x/d) to 1.
// d0 = centre(v mod p); v - d0 = p * (q + carry) with q = floor(v / p) and
// carry = [v mod p > (p-1)/2], so d1 = centre((q + carry) mod p) where
// q + carry <= p (the value p maps to 0, which centring also yields).
__device__ __forceinline__ void digit_split_u16(uint32_t x, const ModConst& c, int32_t& d0, int32_t& d1) {
    const uint32_t v = x - c.m * __umulhi(x, c.magic_m + 1u);
    const int32_t p = static_cast<int32_t>(c.p);
    const int32_t half = (p - 1) / 2;
    if (c.e == 2) {
        const uint32_t q = __umulhi(v, c.magic_p + 1u);
        const int32_t r = static_cast<int32_t>(v - q * c.p);
        const bool up = r > half;
        d0 = up ? r - p : r;
        const int32_t q1 = static_cast<int32_t>(q) + (up ? 1 : 0);
        d1 = q1 > half ? q1 - p : q1;
    } else {
        const int32_t r = static_cast<int32_t>(v);
        d0 = r > half ? r - p : r;
        d1 = 0;
    }
}

// Odd-p variant of digit_split_u16 with the centring folded into the
// quotient: for odd p, centre(a) = ((a + h) mod p) - h with h = (p-1)/2, so
// q1 = floor((v + h) / p) and d0 = v - p q1 directly, and d1 = centre(q1)
// with q1 <= p. Inputs v < p^2 (already reduced). ~7 instructions.
__device__ __forceinline__ void digit_split_odd(uint32_t v, uint32_t p, uint32_t h, uint32_t magic_p1,
                                                int32_t& d0, int32_t& d1) {
    const uint32_t q1 = __umulhi(v + h, magic_p1);
    d0 = static_cast<int32_t>(v - q1 * p);
    d1 = static_cast<int32_t>(q1 > h ? q1 - p : q1);
}

}  // namespace irl
