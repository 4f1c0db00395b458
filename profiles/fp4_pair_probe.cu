// Probe, CTA-pair form: tcgen05.mma.cta_group::2.kind::mxf4.block_scale (M = 256
// over two CTAs' TMEM, N = 240) against kind::i8 for the iris products, with
// unit UE8M0 scale factors written into both CTAs' TMEM. Exactness against
// the host and rate with SMEM-resident tiles, clusters of 2 on every SM pair.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o fp4_pair_probe profiles/fp4_pair_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2601_17561_b200/csrc/sm100_ptx.cuh"

namespace {

constexpr int kM = 256, kN = 240, kRowBytes = 128, kMc = kM / 2, kNc = kN / 2;
constexpr int kAcc2 = 256, kSfa = 240, kSfb = 248;

__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t byte) {
    return row * 128u + ((((byte >> 4) ^ (row & 7u)) << 4) | (byte & 15u));
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, uint32_t v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %1, %1, %1};" ::"r"(taddr), "r"(v));
}
__device__ __forceinline__ void mma_mxf4_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc,
                                              uint32_t sfa, uint32_t sfb) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}
__host__ __device__ constexpr uint32_t idesc_mxf4(uint32_t m, uint32_t n) {
    return (1u << 7) | (1u << 10) | ((n >> 3) << 17) | (1u << 23) | ((m >> 4) << 24);
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

template <bool kFp4>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128)
    probe(const uint8_t* a_planes, const uint8_t* b_planes, uint32_t* out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sa = smem;                       // 2 planes x 128 rows x 128 B
    uint8_t* sb = smem + 2 * kMc * kRowBytes; // 2 planes x 120 rows x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const uint32_t tid = threadIdx.x, warp = tid / 32, rank = irl::ptx::cluster_ctarank();
    for (uint32_t i = tid; i < 2u * kMc * kRowBytes; i += blockDim.x) {
        const uint32_t p = i / (kMc * kRowBytes), r = (i / kRowBytes) % kMc, c = i % kRowBytes;
        sa[p * kMc * kRowBytes + sw128(r, c)] = a_planes[(p * kM + rank * kMc + r) * kRowBytes + c];
    }
    for (uint32_t i = tid; i < 2u * kNc * kRowBytes; i += blockDim.x) {
        const uint32_t p = i / (kNc * kRowBytes), r = (i / kRowBytes) % kNc, c = i % kRowBytes;
        sb[p * kNc * kRowBytes + sw128(r, c)] = b_planes[(p * kN + rank * kNc + r) * kRowBytes + c];
    }
    asm volatile("fence.proxy.async.shared::cta;");
    if (warp == 0) irl::ptx::tmem_alloc_pair(irl::ptx::smem_u32(&tbase), 512);
    if (tid == 0) {
        irl::ptx::mbar_init(&bar, 1);
        irl::ptx::fence_barrier_init();
    }
    irl::ptx::tc_fence_before();
    __syncthreads();
    irl::ptx::tc_fence_after();
    const uint32_t tm = tbase;
    if (kFp4) {
        const uint32_t lb = tm + ((warp * 32u) << 16);
        for (uint32_t c = kSfa; c < 256; c += 4) tmem_st4(lb + c, 0x7F7F7F7Fu);
        for (uint32_t c = kAcc2 + kN; c < 512; c += 4) tmem_st4(lb + c, 0x7F7F7F7Fu);
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    irl::ptx::tc_fence_before();
    cluster_sync_all();
    irl::ptx::tc_fence_after();
    if (rank == 0 && tid == 0) {
        const uint32_t idesc = kFp4 ? idesc_mxf4(kM, kN) : irl::ptx::idesc_i8(kM, kN);
        const uint32_t a0 = irl::ptx::smem_u32(sa), a1 = a0 + kMc * kRowBytes;
        const uint32_t b0 = irl::ptx::smem_u32(sb), b1 = b0 + kNc * kRowBytes;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t acc = (it > 0 || k > 0) ? 1u : 0u;
                const uint64_t da0 = irl::ptx::smem_desc_k_sw128(a0 + 32 * k);
                const uint64_t db0 = irl::ptx::smem_desc_k_sw128(b0 + 32 * k);
                const uint64_t da1 = irl::ptx::smem_desc_k_sw128(a1 + 32 * k);
                const uint64_t db1 = irl::ptx::smem_desc_k_sw128(b1 + 32 * k);
                if (kFp4) {
                    mma_mxf4_pair(tm, da0, db0, idesc, acc, tm + kSfa, tm + kSfb);
                    mma_mxf4_pair(tm + kAcc2, da1, db1, idesc, acc, tm + kSfa, tm + kSfb);
                } else {
                    irl::ptx::mma_i8_pair(tm, da0, db0, idesc, acc);
                    irl::ptx::mma_i8_pair(tm + kAcc2, da1, db1, idesc, acc);
                }
            }
        }
        irl::ptx::mma_commit_pair(&bar, 0x3);
    }
    irl::ptx::mbar_wait(&bar, 0);
    irl::ptx::tc_fence_after();
    if (out && blockIdx.x < 2) {
        const uint32_t row = rank * kMc + warp * 32 + (tid & 31);
        for (int c = 0; c < kN; c += 16) {
            uint32_t r1[16], r2[16];
            irl::ptx::tmem_ld_32x32b_x16(tm + ((warp * 32u) << 16) + c, r1);
            irl::ptx::tmem_ld_32x32b_x16(tm + ((warp * 32u) << 16) + kAcc2 + c, r2);
            irl::ptx::tmem_ld_wait();
            for (int j = 0; j < 16; ++j) {
                out[(0 * kN + c + j) * kM + row] = r1[j];
                out[(1 * kN + c + j) * kM + row] = r2[j];
            }
        }
    }
    irl::ptx::tc_fence_before();
    cluster_sync_all();
    if (warp == 0) irl::ptx::tmem_dealloc_pair(tm, 512);
}

uint8_t e2m1(int v) { return v == 0 ? 0x0 : (v > 0 ? 0x2 : 0xA); }

}  // namespace

int main() {
    const int kA = 2 * kM * kRowBytes, kB = 2 * kN * kRowBytes;
    srand(11);
    std::vector<int8_t> av(2 * kM * 256), bv(2 * kN * 256);
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
                a8[(p * kM + r) * kRowBytes + c] = uint8_t(av[(p * kM + r) * 256 + c]);
            }
        for (int r = 0; r < kN; ++r)
            for (int c = 0; c < kRowBytes; ++c) {
                const int8_t* v = &bv[(p * kN + r) * 256 + 2 * c];
                b4[(p * kN + r) * kRowBytes + c] = uint8_t(e2m1(v[0]) | (e2m1(v[1]) << 4));
                b8[(p * kN + r) * kRowBytes + c] = uint8_t(bv[(p * kN + r) * 256 + c]);
            }
    }
    uint8_t *da4, *db4, *da8, *db8;
    uint32_t* dout;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&da4, kA), cudaMalloc(&db4, kB), cudaMalloc(&da8, kA), cudaMalloc(&db8, kB);
    cudaMalloc(&dout, 2 * kM * kN * 4);
    cudaMemcpy(da4, a4.data(), kA, cudaMemcpyHostToDevice), cudaMemcpy(db4, b4.data(), kB, cudaMemcpyHostToDevice);
    cudaMemcpy(da8, a8.data(), kA, cudaMemcpyHostToDevice), cudaMemcpy(db8, b8.data(), kB, cudaMemcpyHostToDevice);
    const size_t smem = 2 * kMc * kRowBytes + 2 * kNc * kRowBytes + 1024;
    cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    long bad[2] = {0, 0};
    std::vector<uint32_t> o(2 * kM * kN);
    for (int f = 0; f < 2; ++f) {
        if (f) probe<true><<<2, 128, smem>>>(da4, db4, dout, 1);
        else probe<false><<<2, 128, smem>>>(da8, db8, dout, 1);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            std::printf("{\"error\": \"%s\", \"fp4\": %d}\n", cudaGetErrorString(e), f);
            return 1;
        }
        cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
        const int kk = f ? 256 : 128;
        for (int p = 0; p < 2; ++p)
            for (int n = 0; n < kN; ++n)
                for (int m = 0; m < kM; ++m) {
                    long s = 0;
                    for (int k = 0; k < kk; ++k) s += av[(p * kM + m) * 256 + k] * bv[(p * kN + n) * 256 + k];
                    const uint32_t g = o[(p * kN + n) * kM + m];
                    float gf;
                    std::memcpy(&gf, &g, 4);
                    bad[f] += f ? (gf != float(s)) : (int32_t(g) != s);
                }
    }
    const int iters = 4096, grid = nsm / 2 * 2;
    double tops[2];
    for (int f = 0; f < 2; ++f) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0), cudaEventCreate(&e1);
        for (int w = 0; w < 3; ++w) {
            if (w == 2) cudaEventRecord(e0);
            if (f) probe<true><<<grid, 128, smem>>>(da4, db4, nullptr, iters);
            else probe<false><<<grid, 128, smem>>>(da8, db8, nullptr, iters);
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        tops[f] = 2.0 * 2.0 * kM * kN * (f ? 256.0 : 128.0) * iters * (grid / 2) / (ms * 1e-3) / 1e12;
    }
    std::printf("{\"pair_fp4_mismatches\": %ld, \"pair_i8_mismatches\": %ld, \"checked\": %d, \"pair_i8_tops\": %.1f, "
                "\"pair_mxf4_tops\": %.1f, \"ratio\": %.3f, \"status\": \"%s\"}\n",
                bad[1], bad[0], 2 * kM * kN, tops[0], tops[1], tops[1] / tops[0],
                cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
