// Probe: can the iris products (ternary masked codes, mask bits) run on the
// block-scaled FP4 tensor path (tcgen05.mma kind::mxf4, e2m1 operands, UE8M0
// scales all 1.0) exactly, and at what rate against kind::i8?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o fp4_probe profiles/fp4_probe.cu
//   ./fp4_probe
//
// One CTA per SM, 128 threads, cta_group::1, M = 128, N = 240 (TMEM: two
// accumulators of 240 columns plus scale-factor columns). Exactness: one
// 256-deep product of random {-1, 0, 1} x {-1, 0, 1} (and {0,1} x {0,1})
// against the host. Rate: the same SMEM tiles multiplied over and over.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2601_17561_b200/csrc/sm100_ptx.cuh"

namespace {

constexpr int kM = 128, kN = 240, kRowBytes = 128;  // one 128 B swizzle row per operand row
constexpr int kAcc2 = 256, kSfa = 240, kSfb = 248;   // TMEM columns

__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t byte) {  // SWIZZLE_128B K-major
    return row * 128u + ((((byte >> 4) ^ (row & 7u)) << 4) | (byte & 15u));
}

__device__ __forceinline__ void tmem_alloc1(uint32_t smem_dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_dst), "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc1(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, uint32_t v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %1, %1, %1};" ::"r"(taddr), "r"(v));
}
__device__ __forceinline__ void mma_mxf4(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc,
                                         uint32_t sfa, uint32_t sfb) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit1(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     irl::ptx::smem_u32(bar)));
}

// Block-scaled descriptor (CUTLASS InstrDescriptorBlockScaled): a/b format
// E2M1 = 1 (MXF4), scale format UE8M0, K-major, dense K = 64.
__host__ __device__ constexpr uint32_t idesc_mxf4(uint32_t m, uint32_t n) {
    return (1u << 7) | (1u << 10) | ((n >> 3) << 17) | (1u << 23) | ((m >> 4) << 24);
}

// kFp4: operands are packed e2m1 (2 per byte, low nibble first), 256 k per
// 128 B row; else int8, 128 k per row. planes: [2 planes][rows][128 B] for A
// (kM rows) and B (kN rows). mode 0: one pass, write accumulators; mode 1:
// iters passes, time them.
template <bool kFp4>
__global__ void __launch_bounds__(128) probe(const uint8_t* a_planes, const uint8_t* b_planes, float* out_f,
                                              int32_t* out_i, int iters, unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sa = smem;                        // 2 x 16 KB
    uint8_t* sb = smem + 2 * kM * kRowBytes;   // 2 x 30 KB
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const uint32_t tid = threadIdx.x, warp = tid / 32;
    for (uint32_t i = tid; i < 2u * kM * kRowBytes; i += blockDim.x) {
        const uint32_t p = i / (kM * kRowBytes), r = (i / kRowBytes) % kM, c = i % kRowBytes;
        sa[p * kM * kRowBytes + sw128(r, c)] = a_planes[i];
    }
    for (uint32_t i = tid; i < 2u * kN * kRowBytes; i += blockDim.x) {
        const uint32_t p = i / (kN * kRowBytes), r = (i / kRowBytes) % kN, c = i % kRowBytes;
        sb[p * kN * kRowBytes + sw128(r, c)] = b_planes[i];
    }
    asm volatile("fence.proxy.async.shared::cta;");
    if (warp == 0) tmem_alloc1(irl::ptx::smem_u32(&tbase), 512);
    if (tid == 0) {
        irl::ptx::mbar_init(&bar, 1);
        irl::ptx::fence_barrier_init();
    }
    irl::ptx::tc_fence_before();
    __syncthreads();
    irl::ptx::tc_fence_after();
    const uint32_t tm = tbase;
    if (kFp4) {  // scale factors: every byte 0x7F = 2^0
        const uint32_t lane_base = tm + ((warp * 32u) << 16);
        tmem_st4(lane_base + kSfa, 0x7F7F7F7Fu);
        tmem_st4(lane_base + kSfa + 4, 0x7F7F7F7Fu);
        tmem_st4(lane_base + kSfb, 0x7F7F7F7Fu);
        tmem_st4(lane_base + kSfb + 4, 0x7F7F7F7Fu);
        tmem_st4(lane_base + kAcc2 + kN, 0x7F7F7F7Fu);
        tmem_st4(lane_base + kAcc2 + kN + 4, 0x7F7F7F7Fu);
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    irl::ptx::tc_fence_before();
    __syncthreads();
    irl::ptx::tc_fence_after();
    const uint32_t idesc = kFp4 ? idesc_mxf4(kM, kN) : irl::ptx::idesc_i8(kM, kN);
    unsigned long long t0 = 0, t1 = 0;
    if (tid == 0) {
        const uint32_t a0 = irl::ptx::smem_u32(sa), a1 = a0 + kM * kRowBytes;
        const uint32_t b0 = irl::ptx::smem_u32(sb), b1 = b0 + kN * kRowBytes;
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // 4 x 32 B per 128 B row
                const uint32_t acc = (it > 0 || k > 0) ? 1u : 0u;
                const uint64_t da0 = irl::ptx::smem_desc_k_sw128(a0 + 32 * k);
                const uint64_t db0 = irl::ptx::smem_desc_k_sw128(b0 + 32 * k);
                const uint64_t da1 = irl::ptx::smem_desc_k_sw128(a1 + 32 * k);
                const uint64_t db1 = irl::ptx::smem_desc_k_sw128(b1 + 32 * k);
                if (kFp4) {
                    mma_mxf4(tm, da0, db0, idesc, acc, tm + kSfa, tm + kSfb);
                    mma_mxf4(tm + kAcc2, da1, db1, idesc, acc, tm + kSfa, tm + kSfb);
                } else {
                    mma_i8(tm, da0, db0, idesc, acc);
                    mma_i8(tm + kAcc2, da1, db1, idesc, acc);
                }
            }
        }
        commit1(&bar);
    }
    irl::ptx::mbar_wait(&bar, 0);
    irl::ptx::tc_fence_after();
    if (tid == 0) {
        t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    if (blockIdx.x == 0 && (out_f || out_i)) {
        const uint32_t row = warp * 32 + (tid & 31);
        for (int c = 0; c < kN; c += 16) {
            uint32_t r1[16], r2[16];
            irl::ptx::tmem_ld_32x32b_x16(tm + ((warp * 32u) << 16) + c, r1);
            irl::ptx::tmem_ld_32x32b_x16(tm + ((warp * 32u) << 16) + kAcc2 + c, r2);
            irl::ptx::tmem_ld_wait();
            for (int j = 0; j < 16; ++j) {
                if (kFp4) {
                    out_f[(0 * kN + c + j) * kM + row] = __uint_as_float(r1[j]);
                    out_f[(1 * kN + c + j) * kM + row] = __uint_as_float(r2[j]);
                } else {
                    out_i[(0 * kN + c + j) * kM + row] = static_cast<int32_t>(r1[j]);
                    out_i[(1 * kN + c + j) * kM + row] = static_cast<int32_t>(r2[j]);
                }
            }
        }
    }
    irl::ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc1(tm, 512);
}

uint8_t e2m1(int v) { return v == 0 ? 0x0 : (v > 0 ? 0x2 : 0xA); }  // 0, +1.0, -1.0

}  // namespace

int main() {
    // random ternary operands: plane 0 = masked codes {-1,0,1}, plane 1 = masks {0,1}
    const int kA = 2 * kM * kRowBytes, kB = 2 * kN * kRowBytes;
    srand(7);
    std::vector<int8_t> av(2 * kM * 256), bv(2 * kN * 256);  // fp4 view: 256 k per row
    for (int p = 0; p < 2; ++p) {
        for (int i = 0; i < kM * 256; ++i) av[p * kM * 256 + i] = p == 0 ? int8_t(rand() % 3 - 1) : int8_t(rand() % 2);
        for (int i = 0; i < kN * 256; ++i) bv[p * kN * 256 + i] = p == 0 ? int8_t(rand() % 3 - 1) : int8_t(rand() % 2);
    }
    std::vector<uint8_t> a4(kA), b4(kB), a8(kA), b8(kB);
    for (int p = 0; p < 2; ++p) {
        for (int r = 0; r < kM; ++r)
            for (int c = 0; c < kRowBytes; ++c) {
                const int8_t* v = &av[(p * kM + r) * 256 + 2 * c];
                a4[(p * kM + r) * kRowBytes + c] = uint8_t(e2m1(v[0]) | (e2m1(v[1]) << 4));
                a8[(p * kM + r) * kRowBytes + c] = uint8_t(av[(p * kM + r) * 256 + c]);  // first 128 k as int8
            }
        for (int r = 0; r < kN; ++r)
            for (int c = 0; c < kRowBytes; ++c) {
                const int8_t* v = &bv[(p * kN + r) * 256 + 2 * c];
                b4[(p * kN + r) * kRowBytes + c] = uint8_t(e2m1(v[0]) | (e2m1(v[1]) << 4));
                b8[(p * kN + r) * kRowBytes + c] = uint8_t(bv[(p * kN + r) * 256 + c]);
            }
    }
    uint8_t *da4, *db4, *da8, *db8;
    float* dof;
    int32_t* doi;
    unsigned long long* dcyc;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&da4, kA), cudaMalloc(&db4, kB), cudaMalloc(&da8, kA), cudaMalloc(&db8, kB);
    cudaMalloc(&dof, 2 * kM * kN * 4), cudaMalloc(&doi, 2 * kM * kN * 4), cudaMalloc(&dcyc, nsm * 8);
    cudaMemcpy(da4, a4.data(), kA, cudaMemcpyHostToDevice), cudaMemcpy(db4, b4.data(), kB, cudaMemcpyHostToDevice);
    cudaMemcpy(da8, a8.data(), kA, cudaMemcpyHostToDevice), cudaMemcpy(db8, b8.data(), kB, cudaMemcpyHostToDevice);
    const size_t smem = kA + kB + 1024;
    cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));

    // exactness: one pass (K = 256 fp4 / 128 int8)
    probe<true><<<1, 128, smem>>>(da4, db4, dof, nullptr, 1, dcyc);
    probe<false><<<1, 128, smem>>>(da8, db8, nullptr, doi, 1, dcyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        std::printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
        return 1;
    }
    std::vector<float> of(2 * kM * kN);
    std::vector<int32_t> oi(2 * kM * kN);
    cudaMemcpy(of.data(), dof, of.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(oi.data(), doi, oi.size() * 4, cudaMemcpyDeviceToHost);
    long bad4 = 0, bad8 = 0;
    for (int p = 0; p < 2; ++p)
        for (int n = 0; n < kN; ++n)
            for (int m = 0; m < kM; ++m) {
                long s4 = 0, s8 = 0;
                for (int k = 0; k < 256; ++k) s4 += av[(p * kM + m) * 256 + k] * bv[(p * kN + n) * 256 + k];
                for (int k = 0; k < 128; ++k) s8 += av[(p * kM + m) * 256 + k] * bv[(p * kN + n) * 256 + k];
                bad4 += of[(p * kN + n) * kM + m] != float(s4);
                bad8 += oi[(p * kN + n) * kM + m] != s8;
            }
    // rate: every SM multiplies its tiles `iters` times
    const int iters = 4096;
    double tops[2];
    for (int f = 0; f < 2; ++f) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0), cudaEventCreate(&e1);
        for (int w = 0; w < 2; ++w) {
            if (f) probe<true><<<nsm, 128, smem>>>(da4, db4, nullptr, nullptr, iters, dcyc);
            else probe<false><<<nsm, 128, smem>>>(da8, db8, nullptr, nullptr, iters, dcyc);
        }
        cudaEventRecord(e0);
        if (f) probe<true><<<nsm, 128, smem>>>(da4, db4, nullptr, nullptr, iters, dcyc);
        else probe<false><<<nsm, 128, smem>>>(da8, db8, nullptr, nullptr, iters, dcyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double k_per_pass = f ? 256.0 : 128.0;
        tops[f] = 2.0 * 2.0 * kM * kN * k_per_pass * iters * nsm / (ms * 1e-3) / 1e12;
    }
    e = cudaDeviceSynchronize();
    std::printf("{\"fp4_mismatches\": %ld, \"i8_mismatches\": %ld, \"checked\": %d, \"i8_tops\": %.1f, "
                "\"mxf4_tops\": %.1f, \"ratio\": %.3f, \"status\": \"%s\"}\n",
                bad4, bad8, 2 * kM * kN, tops[0], tops[1], tops[1] / tops[0], cudaGetErrorString(e));
    return 0;
}
